"""The reference's OWN unit-test suite (/root/reference/pkg/tests/
test_poly.py + conftest.py, staged unmodified into oracle/_ref/ref_tests by
oracle.stage_reference_tests) run against the drop-in through the import
shim tests/ref_shim/f2xmul: what a reference user sees after switching the
import.  Every test must pass -- backend names, overrides, probes, counters
(t*t base products) and the reference's internal route names included."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "tests", "ref_shim")


def _staged():
    sys.path.insert(0, ROOT)
    import oracle

    return oracle.stage_reference_tests()


def test_shim_resolves_to_dropin():
    """CPU: the shim maps f2xmul.poly onto the package module (no device work
    beyond the shim's warm-up is needed to check the mapping, so only the
    module identity is checked here without importing the shim)."""
    src = open(os.path.join(SHIM, "f2xmul", "__init__.py")).read()
    assert "sys.modules[__name__ + \".poly\"] = poly" in src
    import paper_2201_10473_b200.poly as p

    for name in ("set_backend_override", "_machine_supports_wide_mul", "_int_mul_selfcheck",
                 "_convolution_mul_arrays", "_spread_mul_arrays", "backend_select"):
        assert hasattr(p, name), name


def test_backend_seam_matches_reference_priority(monkeypatch):
    """CPU: override > F2XMUL_BACKEND > probes, as poly.py:234-246."""
    import paper_2201_10473_b200.poly as p

    monkeypatch.delenv("F2XMUL_BACKEND", raising=False)
    assert p.backend_select() is p.BackendId.MULTILANE
    p.set_backend_override("portable")
    try:
        assert p.backend_select() is p.BackendId.PORTABLE
    finally:
        p.set_backend_override(None)
    monkeypatch.setenv("F2XMUL_BACKEND", "clmul")
    assert p.backend_select() is p.BackendId.CLMUL
    monkeypatch.setenv("F2XMUL_BACKEND", "bogus")
    with pytest.raises(ValueError):
        p.backend_select()
    monkeypatch.setenv("F2XMUL_BACKEND", "auto")
    monkeypatch.setattr(p, "_machine_supports_wide_mul", lambda: False)
    assert p.backend_select() is p.BackendId.CLMUL
    monkeypatch.setattr(p, "_int_mul_selfcheck", lambda: False)
    assert p.backend_select() is p.BackendId.PORTABLE
    with pytest.raises(ValueError):
        p.set_backend_override("nope")


@pytest.mark.gpu
def test_reference_unit_suite_on_dropin(cuda, tmp_path):
    staged = _staged()
    if staged is None:
        pytest.skip("reference tests not staged (build() stages them from /root/reference)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([SHIM, ROOT, staged, env.get("PYTHONPATH", "")])
    env.pop("F2XMUL_BACKEND", None)
    r = subprocess.run([sys.executable, "-m", "pytest", staged, "-q", "-p", "no:cacheprovider",
                        "-o", "addopts=", "--rootdir", str(tmp_path)],
                       cwd=str(tmp_path), env=env, capture_output=True, text=True, timeout=1800)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert " passed" in tail and "failed" not in tail, tail
