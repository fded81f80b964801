"""Constant-time SASS audit (tools/ct_sass_audit.py, SPEC.md:47,
141, 365): every kernel of the product library is free of data-dependent
branches and data-dependent addresses, and the audit is not vacuous -- the
deliberately leaky test fixture (F2X_LEAKY_LEAF=1: leaves skip all-zero a
words) is flagged in every node-kernel instantiation.  CPU only (cuobjdump on
the built libraries)."""

import os
import shutil
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

pytestmark = pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="needs cuobjdump")


@pytest.fixture(scope="module")
def libs():
    from paper_2201_10473_b200 import build as b

    return b.build(), b.build(leaky=True)


def test_product_library_has_no_secret_dependent_control_or_addressing(libs):
    import ct_sass_audit as audit

    res = audit.audit_lib(libs[0])
    assert len(res) >= 40, sorted(res)  # every kernel was parsed
    bad = {k: v for k, v in res.items() if v}
    assert not bad, bad


def test_leaky_fixture_is_flagged(libs):
    import ct_sass_audit as audit

    res = audit.audit_lib(libs[1])
    node = {k: v for k, v in res.items() if "k2_node_mul" in k}
    assert node and all(v for v in node.values()), {k: len(v) for k, v in node.items()}
    assert any("data-dependent branch" in line for v in node.values() for line in v)
    # the leak is confined to the leaves: the memory-side kernels stay clean
    assert not any(v for k, v in res.items() if "k2_node_mul" not in k)


def test_taint_rules_on_synthetic_sass():
    """Hand-written SASS: a branch on loaded data is flagged; a branch on a
    parameter, a predicated-complementary definition and a select on data
    are not."""
    import ct_sass_audit as audit

    def run(lines):
        text = "\n".join(f"        /*{16 * i:04x}*/                   {l} ;" for i, l in enumerate(lines))
        fn = audit.parse_functions("Function : f\n" + text)["f"]
        return audit.audit_function(fn)

    leak = ["LDC R2, c[0x0][0x380]", "LDG.E R4, desc[UR4][R2.64]", "ISETP.NE.AND P0, PT, R4, RZ, PT",
            "@P0 BRA 0x0060", "NOP", "EXIT"]
    assert any("branch" in v for v in run(leak))
    addr = ["LDC R2, c[0x0][0x380]", "LDG.E R4, desc[UR4][R2.64]", "LDS R6, [R4]", "EXIT"]
    assert any("address" in v for v in run(addr))
    ok = ["LDC R2, c[0x0][0x380]", "LDG.E R4, desc[UR4][R2.64]", "ISETP.NE.AND P0, PT, R2, RZ, PT",
          "SEL R6, R4, RZ, P0", "@P0 MOV R8, R2", "@!P0 MOV R8, RZ", "LDS R9, [R8]",
          "@P0 BRA 0x0090", "NOP", "EXIT"]
    assert run(ok) == []
