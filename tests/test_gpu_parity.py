"""GPU parity: the CUDA path (through the C ABI) vs the oracle and the golden
vectors produced by the real reference.  Bit-exact on every word."""

import numpy as np
import pytest

from conftest import int_clmul

pytestmark = pytest.mark.gpu


def _dev(x, cuda):
    """Device copy as int64 words (same bits; torch's uint64 kernels are thin)."""
    import torch

    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint64).view(np.int64)).to(cuda)


def _np(x):
    return x.cpu().numpy().view(np.uint64)


# ---------------------------------------------------------------- golden pins

def test_golden_full(golden, cuda):
    from paper_2201_10473_b200 import mul_full

    for t in golden["full_ts"]:
        A, B, C = golden[f"full_t{t}_A"], golden[f"full_t{t}_B"], golden[f"full_t{t}_C"]
        out = _np(mul_full(_dev(A, cuda), _dev(B, cuda)))
        assert np.array_equal(out, C), f"t={t}"


def test_golden_cyclic(golden, cuda):
    from paper_2201_10473_b200 import mul_cyclic

    for n in golden["cyc_ns"]:
        A, B, C = golden[f"cyc_n{n}_A"], golden[f"cyc_n{n}_B"], golden[f"cyc_n{n}_C"]
        out = _np(mul_cyclic(_dev(A, cuda), _dev(B, cuda), int(n)))
        assert np.array_equal(out, C), f"n={n}"


def test_golden_clmul_lanes(golden, cuda):
    from paper_2201_10473_b200 import clmul64_batch

    lo, hi = clmul64_batch(golden["clmul_a"], golden["clmul_b"])
    assert np.array_equal(lo, golden["clmul_lo"])
    assert np.array_equal(hi, golden["clmul_hi"])


# ------------------------------------------------- oracle at config sizes

@pytest.mark.parametrize("n,batch", [(12323, 256), (17669, 96), (35851, 64), (57637, 40)])
def test_cyclic_configs_vs_oracle(n, batch, cuda):
    from oracle import c_mul_cyclic
    from oracle.f2x_oracle import make_cyclic_inputs
    from paper_2201_10473_b200 import mul_cyclic

    A, B = make_cyclic_inputs(n, batch)
    out = _np(mul_cyclic(_dev(A, cuda), _dev(B, cuda), n))
    assert np.array_equal(out, c_mul_cyclic(A, B, n))


@pytest.mark.parametrize("t", [1, 2, 3, 16, 17, 33, 64, 100, 128, 256, 512, 1024])
def test_full_sizes_vs_oracle(t, cuda):
    from oracle import c_mul_full
    from oracle.f2x_oracle import make_full_inputs
    from paper_2201_10473_b200 import mul_full

    batch = 70 if t <= 256 else 33
    A, B = make_full_inputs(t, batch, words=True)
    out = _np(mul_full(_dev(A, cuda), _dev(B, cuda)))
    assert np.array_equal(out, c_mul_full(A, B))


@pytest.mark.parametrize("leaf", [16, 18, 23, 25, 29, 32, 35, 36, 40])
def test_forced_leaf_sizes(leaf, cuda):
    """Every leaf instantiation the planner can pick, on one ring size."""
    from oracle import c_mul_cyclic
    from oracle.f2x_oracle import make_cyclic_inputs
    from paper_2201_10473_b200 import mul_cyclic

    n = 17669
    A, B = make_cyclic_inputs(n, 33)
    out = _np(mul_cyclic(_dev(A, cuda), _dev(B, cuda), n, leaf=leaf))
    assert np.array_equal(out, c_mul_cyclic(A, B, n))


# ------------------------------------------------------------- edge cases

def test_ragged_batches(cuda):
    from oracle import c_mul_cyclic
    from oracle.f2x_oracle import make_cyclic_inputs
    from paper_2201_10473_b200 import mul_cyclic

    for batch in (1, 31, 32, 33, 65):
        A, B = make_cyclic_inputs(1000, batch)
        out = _np(mul_cyclic(_dev(A, cuda), _dev(B, cuda), 1000))
        assert np.array_equal(out, c_mul_cyclic(A, B, 1000)), batch


def test_empty_batch(cuda):
    import torch

    from paper_2201_10473_b200 import mul_cyclic, mul_full

    z = torch.zeros((0, 5), dtype=torch.int64, device=cuda)
    assert mul_full(z, z).shape == (0, 10)
    assert mul_cyclic(z, z, 300).shape == (0, 5)


def test_top_bits_rejected(cuda):
    from oracle.f2x_oracle import make_cyclic_inputs
    from paper_2201_10473_b200 import mul_cyclic

    n = 17669
    A, B = make_cyclic_inputs(n, 40)
    B[37, -1] |= np.uint64(1 << (n % 64))  # bit n set
    with pytest.raises(ValueError):
        mul_cyclic(_dev(A, cuda), _dev(B, cuda), n)
    A2, _ = make_cyclic_inputs(n, 40)
    A2[0, -1] |= np.uint64(1 << 63)
    with pytest.raises(ValueError):
        mul_cyclic(_dev(A2, cuda), _dev(A2, cuda), n)


def test_shape_errors(cuda):
    import torch

    from paper_2201_10473_b200 import mul_cyclic, mul_full

    a = torch.zeros((4, 3), dtype=torch.int64, device=cuda)
    b = torch.zeros((4, 2), dtype=torch.int64, device=cuda)
    with pytest.raises(ValueError):
        mul_full(a, b)
    with pytest.raises(ValueError):
        mul_cyclic(a, a, 1000)  # needs 16 words
    with pytest.raises(ValueError):
        mul_full(a.cpu(), a.cpu())


def test_ring_identities_all_presets(cuda):
    """A*1 = A and X^(N-1)*X = 1, at the HQC sizes."""
    from oracle.f2x_oracle import make_cyclic_inputs
    from paper_2201_10473_b200 import mul_cyclic

    for n in (17669, 35851, 57637):
        t = (n + 63) // 64
        A, _ = make_cyclic_inputs(n, 32)
        one = np.zeros_like(A)
        one[:, 0] = 1
        assert np.array_equal(_np(mul_cyclic(_dev(A, cuda), _dev(one, cuda), n)), A)
        xn1 = np.zeros((1, t), dtype=np.uint64)
        xn1[0, (n - 1) // 64] = np.uint64(1 << ((n - 1) % 64))
        x = np.zeros((1, t), dtype=np.uint64)
        x[0, 0] = 2
        r = _np(mul_cyclic(_dev(xn1, cuda), _dev(x, cuda), n))
        expect = np.zeros((1, t), dtype=np.uint64)
        expect[0, 0] = 1
        assert np.array_equal(r, expect)


# ------------------------------------- full-size properties (no oracle)

@pytest.mark.parametrize("n,batch", [(17669, 4096), (35851, 4096), (57637, 2048)])
def test_full_size_properties(n, batch, cuda):
    """At BASELINE sizes: commutativity, bilinearity and cyclic == fold(full),
    plus a 1-row-in-64 oracle subsample."""
    import torch

    from oracle import c_mul_cyclic
    from oracle.f2x_oracle import make_cyclic_inputs
    from paper_2201_10473_b200 import mul_cyclic, mul_full

    A, B = make_cyclic_inputs(n, batch)
    dA, dB = _dev(A, cuda), _dev(B, cuda)
    C = mul_cyclic(dA, dB, n)
    assert torch.equal(C, mul_cyclic(dB, dA, n))
    D = _dev(np.roll(B, 1, axis=0), cuda)
    lhs = mul_cyclic(dA, dB ^ D, n)
    rhs = mul_cyclic(dA, dB, n) ^ mul_cyclic(dA, D, n)
    assert torch.equal(lhs, rhs)
    # cyclic product equals the fold of the full product
    sub = slice(0, batch, 64)
    full = _np(mul_full(dA[sub].contiguous(), dB[sub].contiguous()))
    from oracle.f2x_oracle import fold_cyclic

    folded = np.stack([fold_cyclic(full[i], n) for i in range(full.shape[0])])
    Cn = _np(C)
    assert np.array_equal(Cn[sub], folded)
    assert np.array_equal(Cn[sub], c_mul_cyclic(A[sub], B[sub], n))


# ------------------------------------------------ reference-mirroring API

def test_scalar_api_known_answers(cuda):
    """The reference's own known answers (test_poly.py:134-143, 219-225)."""
    from paper_2201_10473_b200 import PolyWords, WideProduct, clmul64, schoolbook_mul

    assert clmul64(0x0, 0xDEADBEEF) == (0, 0)
    assert clmul64(0x1, 0xFEDCBA9876543210) == (0xFEDCBA9876543210, 0)
    assert clmul64(0x5, 0x3) == (0xF, 0)
    r = schoolbook_mul(PolyWords([1]), PolyWords([1 << 63]))
    assert isinstance(r, WideProduct) and r.word_len == 2 and r.to_int() == 1 << 63
    with pytest.raises(ValueError):
        schoolbook_mul(PolyWords([1]), PolyWords([1, 2]))
    with pytest.raises(ValueError):
        clmul64(1 << 64, 1)


def test_scalar_api_vs_bitwise(rng, cuda):
    from paper_2201_10473_b200 import PolyWords, clmul64, ring_mul, schoolbook_mul

    for _ in range(20):
        a, b = (int(x) for x in rng.integers(0, 1 << 64, 2, dtype=np.uint64))
        lo, hi = clmul64(a, b)
        assert lo | (hi << 64) == int_clmul(a, b)
    a = PolyWords(rng.integers(0, 1 << 64, 4, dtype=np.uint64))
    b = PolyWords(rng.integers(0, 1 << 64, 4, dtype=np.uint64))
    assert schoolbook_mul(a, b).to_int() == int_clmul(a.to_int(), b.to_int())
    n = 200
    ai = int(rng.integers(0, 1 << 63)) << 100 | 12345
    ai &= (1 << n) - 1
    bi = (1 << 199) | 77
    p = int_clmul(ai, bi)
    want = (p & ((1 << n) - 1)) ^ (p >> n)
    got = ring_mul(PolyWords.from_int(ai, 4), PolyWords.from_int(bi, 4), n)
    assert got.to_int() == want


def test_ring_weight75_dense_path(cuda):
    """A weight-75 sparse first operand goes through the same
    dense path and matches the oracle."""
    from oracle import c_mul_cyclic
    from oracle.f2x_oracle import make_cyclic_inputs
    from paper_2201_10473_b200 import sparse_to_dense

    import torch

    from paper_2201_10473_b200 import mul_cyclic

    n = 17669
    rng = np.random.default_rng(75)
    rows = [sparse_to_dense(rng.choice(n, 75, replace=False), n).words for _ in range(32)]
    A = np.stack(rows)
    _, B = make_cyclic_inputs(n, 32)
    out = mul_cyclic(_dev(A, cuda), _dev(B, cuda), n)
    assert np.array_equal(_np(out), c_mul_cyclic(A, B, n))


@pytest.mark.parametrize("kind,size,batch,chunks", [("cyclic", 17669, 300, 4), ("full", 64, 100, 3),
                                                     ("cyclic", 1000, 31, 2)])
def test_host_pipeline(kind, size, batch, chunks, cuda):
    """Pinned-host end-to-end path (chunked over streams) == oracle."""
    import torch

    from oracle import c_mul_cyclic, c_mul_full
    from oracle.f2x_oracle import make_cyclic_inputs, make_full_inputs
    from paper_2201_10473_b200.engine import HostPipeline

    if kind == "cyclic":
        A, B = make_cyclic_inputs(size, batch)
        want = c_mul_cyclic(A, B, size)
    else:
        A, B = make_full_inputs(size, batch, words=True)
        want = c_mul_full(A, B)
    hA = torch.from_numpy(A.view(np.int64)).pin_memory()
    hB = torch.from_numpy(B.view(np.int64)).pin_memory()
    hC = torch.empty((batch, want.shape[1]), dtype=torch.int64).pin_memory()
    pipe = HostPipeline(kind, size, batch, cuda, chunks=chunks, lanes=2)
    pipe.run(hA, hB, hC, lane=1)
    pipe.join()
    torch.cuda.synchronize()
    assert not pipe.rejected()
    assert np.array_equal(hC.numpy().view(np.uint64), want)


def test_host_pipeline_graph_replay(cuda):
    """The captured CUDA graph of the host path gives the oracle's answer on
    fresh data written into the same pinned buffers."""
    import torch

    from oracle import c_mul_cyclic
    from oracle.f2x_oracle import make_cyclic_inputs
    from paper_2201_10473_b200.engine import HostPipeline

    n, batch = 17669, 256
    A, B = make_cyclic_inputs(n, batch)
    hA = torch.from_numpy(A.view(np.int64).copy()).pin_memory()
    hB = torch.from_numpy(B.view(np.int64).copy()).pin_memory()
    hC = torch.empty_like(hA).pin_memory()
    pipe = HostPipeline("cyclic", n, batch, cuda, chunks=4)
    assert pipe.capture(hA, hB, hC), getattr(pipe, "capture_error", None)
    A2, B2 = np.roll(A, 3, axis=0), np.roll(B, 5, axis=0)
    hA.copy_(torch.from_numpy(A2.view(np.int64)))
    hB.copy_(torch.from_numpy(B2.view(np.int64)))
    pipe.run(hA, hB, hC)
    torch.cuda.synchronize()
    assert np.array_equal(hC.numpy().view(np.uint64), c_mul_cyclic(A2, B2, n))


_EL_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from oracle import c_mul_cyclic, c_mul_full
from oracle.f2x_oracle import make_cyclic_inputs, make_full_inputs
from paper_2201_10473_b200 import mul_cyclic, mul_full, plan
el = int(sys.argv[2])
dev = torch.device("cuda", 0)
d = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).to(dev)
for n, b in ((12323, 70), (17669, 64), (57637, 33)):
    assert plan("cyclic", b, n)["eval_levels"] == el
    A, B = make_cyclic_inputs(n, b)
    out = mul_cyclic(d(A), d(B), n).cpu().numpy().view(np.uint64)
    assert np.array_equal(out, c_mul_cyclic(A, B, n)), n
for t in (64, 256, 1024):
    A, B = make_full_inputs(t, 40, words=True)
    out = mul_full(d(A), d(B)).cpu().numpy().view(np.uint64)
    assert np.array_equal(out, c_mul_full(A, B)), t
print("ok")
"""


@pytest.mark.parametrize("el", [0, 1])
def test_eval_levels_override(el, cuda):
    """The slicing kernel's pre-evaluated global levels (default 2) are a pure
    schedule choice: 0 and 1 (F2X_EVAL_LEVELS, read once per process) give
    the same bits."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, F2X_EVAL_LEVELS=str(el), F2X_TOOM="0")  # Karatsuba-only plans
    r = subprocess.run([sys.executable, "-c", _EL_SCRIPT, root, str(el)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


_TOOM_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from oracle import c_mul_cyclic, c_mul_full
from oracle.f2x_oracle import make_cyclic_inputs, make_full_inputs
from paper_2201_10473_b200 import mul_cyclic, mul_full, plan
tl = int(sys.argv[2])
dev = torch.device("cuda", 0)
d = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).to(dev)
for n, b in ((1000, 7), (12323, 70), (17669, 64), (35851, 33), (57637, 40)):
    assert plan("cyclic", b, n)["toom_levels"] == tl
    A, B = make_cyclic_inputs(n, b)
    out = mul_cyclic(d(A), d(B), n).cpu().numpy().view(np.uint64)
    assert np.array_equal(out, c_mul_cyclic(A, B, n)), n
for t, b in ((16, 33), (64, 40), (277, 5), (1024, 40)):
    A, B = make_full_inputs(t, b, words=True)
    out = mul_full(d(A), d(B)).cpu().numpy().view(np.uint64)
    assert np.array_equal(out, c_mul_full(A, B)), t
print("ok")
"""


@pytest.mark.parametrize("tl,seq", [(0, None), (1, None), (2, None), (3, None), (2, 1), (3, 1), (2, 10 ** 9)])
def test_toom_levels_forced(tl, seq, cuda):
    """Toom-3 levels above the Karatsuba node problem (F2X_TOOM, read once per
    process): 0-3 levels give the oracle's bits for ring and full sizes,
    ragged batches included; both interpolation forms (F2X_TOOM_SEQ: one CTA
    per product for every level / the two-kernel form for every level)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, F2X_TOOM=str(tl))
    if seq is not None:
        env["F2X_TOOM_SEQ"] = str(seq)
    r = subprocess.run([sys.executable, "-c", _TOOM_SCRIPT, root, str(tl)], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


def test_workspace_budget_row_chunks(cuda):
    """A small scratch budget (F2X_WS_BUDGET, read at import) splits the batch
    into row chunks; results stay bit-exact."""
    import os
    import subprocess
    import sys

    script = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from oracle import c_mul_cyclic, c_mul_full
from oracle.f2x_oracle import make_cyclic_inputs, make_full_inputs
from paper_2201_10473_b200 import engine, mul_cyclic, mul_full
from paper_2201_10473_b200 import _lib
dev = torch.device("cuda", 0)
d = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).to(dev)
A, B = make_cyclic_inputs(17669, 1000)
assert len(engine._row_chunks(_lib.load(), _lib.KIND_CYCLIC, 1000, 17669, 0)[0]) > 3
assert np.array_equal(mul_cyclic(d(A), d(B), 17669).cpu().numpy().view(np.uint64), c_mul_cyclic(A, B, 17669))
A, B = make_full_inputs(64, 700, words=True)
assert np.array_equal(mul_full(d(A), d(B)).cpu().numpy().view(np.uint64), c_mul_full(A, B))
print("ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, F2X_WS_BUDGET=str(8 << 20))
    r = subprocess.run([sys.executable, "-c", script, root], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


@pytest.mark.parametrize("t", [2048, 4096, 8192])
def test_large_full_sizes_vs_oracle(t, cuda):
    """Beyond the d-sweep (131k-524k bits): Toom-3 plans with deep Karatsuba
    node problems stay bit-exact."""
    from oracle import c_mul_full
    from oracle.f2x_oracle import make_full_inputs
    from paper_2201_10473_b200 import mul_full

    A, B = make_full_inputs(t, 33, words=True)
    assert np.array_equal(_np(mul_full(_dev(A, cuda), _dev(B, cuda))), c_mul_full(A, B))


def test_integration_stub_runs(cuda):
    """The ctypes binding shown in INTEGRATION.md §2 (what a reference
    maintainer would add as f2xmul/gpu.py) runs as written against this
    build and gives the oracle's bits."""
    import os
    import re

    from oracle import c_mul_cyclic, c_mul_full
    from oracle.f2x_oracle import make_cyclic_inputs, make_full_inputs
    from paper_2201_10473_b200 import _lib

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    text = open(os.path.join(root, "INTEGRATION.md")).read()
    code = re.search(r"```python\n(# f2xmul/gpu.py.*?)```", text, re.S).group(1)
    code = code.replace("from .poly import PolyWords, WideProduct\n", "")
    code = code.replace('ctypes.CDLL("libf2x.so")', f'ctypes.CDLL("{_lib.LIB_PATH}")')
    ns: dict = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    A, B = make_full_inputs(64, 40, words=True)
    assert np.array_equal(ns["schoolbook_mul_batch"](A, B), c_mul_full(A, B))
    A, B = make_cyclic_inputs(17669, 40)
    assert np.array_equal(ns["ring_mul_batch"](A, B, 17669), c_mul_cyclic(A, B, 17669))


def test_captured_call_replays_exactly(cuda):
    """engine.CapturedCall (the call captured once as a CUDA graph) gives the
    oracle's bits on every replay, also after the inputs are rewritten in
    place, for a ring size, a Toom plan and a full product."""
    import torch

    from oracle import c_mul_cyclic, c_mul_full
    from oracle.f2x_oracle import make_cyclic_inputs, make_full_inputs
    from paper_2201_10473_b200.engine import CapturedCall

    for kind, size, batch in (("cyclic", 17669, 96), ("cyclic", 57637, 40), ("full", 64, 70)):
        if kind == "cyclic":
            A, B = make_cyclic_inputs(size, 2 * batch)
            ref = lambda a, b: c_mul_cyclic(a, b, size)  # noqa: E731
        else:
            A, B = make_full_inputs(size, 2 * batch, words=True)
            ref = c_mul_full
        dA, dB = _dev(A[:batch], cuda), _dev(B[:batch], cuda)
        out = torch.empty((batch, dA.shape[1] * (2 if kind == "full" else 1)),
                          dtype=torch.int64, device=cuda)
        cap = CapturedCall(kind, dA, dB, out, size)
        for _ in range(2):
            cap()
            assert np.array_equal(_np(out), ref(A[:batch], B[:batch])), (kind, size)
        dA.copy_(_dev(A[batch:], cuda))
        dB.copy_(_dev(B[batch:], cuda))
        cap()
        assert np.array_equal(_np(out), ref(A[batch:], B[batch:])), (kind, size)
        assert int(cap.err_flag.item()) == 0


@pytest.mark.parametrize("kind,size,batch", [("cyclic", 8000, 32768), ("cyclic", 4099, 40000),
                                             ("full", 100, 32800), ("full", 64, 65536)])
def test_k34_fused_last_pass_unslice(kind, size, batch, cuda):
    """Karatsuba-only plans with >= 1024 groups and a last pass of <= 3
    levels rebuild each group's root in shared memory and unslice it in the
    same kernel (k34_root_unslice; the ring's fold by shared-memory XOR):
    one launch fewer, bit-exact on the first/last rows and a stride
    (ragged batches included)."""
    from oracle import c_mul_cyclic, c_mul_full
    from oracle.f2x_oracle import make_cyclic_inputs, make_full_inputs
    from paper_2201_10473_b200 import mul_cyclic, mul_full, plan

    p = plan(kind, batch, size)
    assert p["toom_levels"] == 0 and p["groups"] >= 1024 and p["pass_levels"][p["num_passes"] - 1] <= 3
    assert p["launches"] == 2 + p["num_passes"], p
    rows = np.unique(np.r_[0:40, batch - 40:batch, 0:batch:997])
    if kind == "cyclic":
        A, B = make_cyclic_inputs(size, batch)
        out = _np(mul_cyclic(_dev(A, cuda), _dev(B, cuda), size))
        want = c_mul_cyclic(A[rows], B[rows], size)
    else:
        A, B = make_full_inputs(size, batch, words=True)
        out = _np(mul_full(_dev(A, cuda), _dev(B, cuda)))
        want = c_mul_full(A[rows], B[rows])
    assert np.array_equal(out[rows], want)


def test_release_workspaces_gpu(cuda):
    """The per-stream scratch cache refills after engine.release_workspaces
    and products stay exact."""
    from oracle import c_mul_cyclic
    from oracle.f2x_oracle import make_cyclic_inputs
    from paper_2201_10473_b200 import engine, mul_cyclic

    A, B = make_cyclic_inputs(17669, 64)
    want = c_mul_cyclic(A, B, 17669)
    assert np.array_equal(_np(mul_cyclic(_dev(A, cuda), _dev(B, cuda), 17669)), want)
    assert engine.release_workspaces(cuda.index) > 0 and not any(k[0] == cuda.index for k in engine._workspaces)
    assert np.array_equal(_np(mul_cyclic(_dev(A, cuda), _dev(B, cuda), 17669)), want)
    assert any(k[0] == cuda.index for k in engine._workspaces)
