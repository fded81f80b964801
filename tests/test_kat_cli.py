"""Known-answer files and the CLI verify contract."""

import glob
import os
import subprocess
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
KATS = sorted(glob.glob(os.path.join(HERE, "golden", "kat_ring_n*.txt")))


def test_kat_files_exist_and_are_large_enough():
    assert len(KATS) >= 4
    total = sum(1 for f in KATS for ln in open(f) if ln.strip() and not ln.startswith("#"))
    assert total >= 50


@pytest.mark.parametrize("path", KATS)
def test_kat_vs_oracle(path):
    from oracle import c_mul_cyclic
    from paper_2201_10473_b200.cli import _read_kat
    from paper_2201_10473_b200.poly import from_hex

    ring, rows = _read_kat(path)
    A = np.stack([from_hex(r[0]).words for r in rows])
    B = np.stack([from_hex(r[1]).words for r in rows])
    C = np.stack([from_hex(r[2]).words for r in rows])
    assert np.array_equal(c_mul_cyclic(A, B, ring), C)


def test_cli_usage_errors():
    from paper_2201_10473_b200.cli import main

    assert main([]) == 1
    assert main(["verify", "/nonexistent/file.txt"]) == 1


def _run_cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2201_10473_b200.cli", *args], cwd=ROOT,
                          capture_output=True, text=True)


@pytest.mark.gpu
def test_cli_verify_gpu(tmp_path):
    for path in KATS:
        r = _run_cli("verify", path)
        assert r.returncode == 0, r.stdout + r.stderr
    # corrupt one output word -> exit 2
    lines = open(KATS[0]).read().splitlines()
    i = next(k for k, ln in enumerate(lines) if ln and not ln.startswith("#"))
    a, b, c = lines[i].split()
    c = c[:-1] + ("0" if c[-1] != "0" else "1")
    lines[i] = " ".join((a, b, c))
    bad = tmp_path / "bad.txt"
    bad.write_text("\n".join(lines) + "\n")
    assert _run_cli("verify", str(bad)).returncode == 2


@pytest.mark.gpu
def test_cli_mul_gpu(tmp_path):
    (tmp_path / "a").write_text("0000000000000001")
    (tmp_path / "b").write_text("0000000000000001")
    r = _run_cli("mul", str(tmp_path / "a"), str(tmp_path / "b"))
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == "0" * 16 + "0000000000000001"  # 1*1 = 1, 2t words
    r = _run_cli("mul", str(tmp_path / "a"), str(tmp_path / "b"), "--ring", "100")
    assert r.returncode == 0 and r.stdout.strip() == "0" * 16 + "0000000000000001"


@pytest.mark.gpu
def test_cli_bench_gpu():
    import json

    r = _run_cli("bench", "--sizes", "1000", "--batch", "64", "--datasets", "2", "--runs", "3",
                 "--format", "json")
    assert r.returncode == 0, r.stderr
    rows = json.loads(r.stdout)
    assert rows[0]["size_bits"] == 1000 and rows[0]["products_per_s"] > 0
