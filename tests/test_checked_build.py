"""Memory-safety evidence without compute-sanitizer (closed on this pool:
profiles/r2/sanitizer/):

* global memory (memcheck/initcheck substitute): the C ABI is called with a
  workspace carved out of a larger buffer between two guard zones, the
  workspace itself filled with random garbage, and an output with guard rows
  around it.  The guards must come back untouched (no out-of-bounds write),
  and two different garbage fills must give the same, oracle-exact product
  (no read of scratch the call did not write first);
* shared memory (initcheck substitute): the checking fixture
  libf2x_checked.so (F2X_CHECKED=1: every kernel fills all of its shared
  memory with a per-CTA garbage pattern before starting) must stay
  bit-exact on the golden vectors, every config size, forced Toom levels
  (both interpolation forms) and full products."""

import ctypes
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GUARD = 1 << 20


def _call_guarded(kind, A, B, size, fill_seed):
    import torch

    from paper_2201_10473_b200 import _lib

    lib = _lib.load()
    batch, t = A.shape
    tout = t if kind == "cyclic" else 2 * t
    kid = _lib.KIND_CYCLIC if kind == "cyclic" else _lib.KIND_FULL
    need = int(lib.f2x_workspace_bytes(kid, batch, size, 0))
    assert need > 0
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(fill_seed)
    buf = torch.randint(0, 256, (GUARD + need + GUARD,), dtype=torch.uint8, device=dev, generator=g)
    guards = (buf[:GUARD].clone(), buf[GUARD + need:].clone())
    dA = torch.from_numpy(A.view(np.int64)).to(dev)
    dB = torch.from_numpy(B.view(np.int64)).to(dev)
    pad = 7  # guard rows around the output
    C = torch.full((batch + 2 * pad, tout), 0x5EED5EED5EED5EED, dtype=torch.int64, device=dev)
    out = C[pad:pad + batch]
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    ws = buf.data_ptr() + GUARD
    if kind == "cyclic":
        rc = lib.f2x_mul_cyclic(dA.data_ptr(), dB.data_ptr(), out.data_ptr(), batch, size, ws, need, 0,
                                flag.data_ptr(), stream)
    else:
        rc = lib.f2x_mul_full(dA.data_ptr(), dB.data_ptr(), out.data_ptr(), batch, size, ws, need, 0, stream)
    assert rc == 0, _lib.strerror(rc)
    torch.cuda.synchronize()
    assert torch.equal(buf[:GUARD], guards[0]) and torch.equal(buf[GUARD + need:], guards[1]), \
        "workspace guard zone overwritten"
    Cn = C.cpu().numpy()
    assert (Cn[:pad] == 0x5EED5EED5EED5EED).all() and (Cn[pad + batch:] == 0x5EED5EED5EED5EED).all(), \
        "output guard rows overwritten"
    assert int(flag.item()) == 0
    return Cn[pad:pad + batch].view(np.uint64)


@pytest.mark.parametrize("kind,size,batch", [
    ("cyclic", 12323, 64), ("cyclic", 17669, 40), ("cyclic", 35851, 33), ("cyclic", 57637, 40),
    ("cyclic", 1000, 7), ("full", 1, 65), ("full", 3, 9), ("full", 64, 33), ("full", 1024, 5),
    ("full", 4096, 3)])
def test_guard_zones_and_garbage_workspace(kind, size, batch, cuda):
    from oracle import c_mul_cyclic, c_mul_full
    from oracle.f2x_oracle import make_cyclic_inputs, make_full_inputs

    if kind == "cyclic":
        A, B = make_cyclic_inputs(size, batch)
        want = c_mul_cyclic(A, B, size)
    else:
        A, B = make_full_inputs(size, batch, words=True)
        want = c_mul_full(A, B)
    r1 = _call_guarded(kind, A, B, size, 1)
    r2 = _call_guarded(kind, A, B, size, 2)
    assert np.array_equal(r1, want)
    assert np.array_equal(r2, want)


_CHECKED_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2201_10473_b200 import _lib, mul_cyclic, mul_full, plan
from oracle import c_mul_cyclic, c_mul_full
from oracle.f2x_oracle import make_cyclic_inputs, make_full_inputs
assert _lib.LIB_PATH.endswith("libf2x_checked.so"), _lib.LIB_PATH
dev = torch.device("cuda", 0)
d = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).to(dev)
g = np.load(sys.argv[2])
for t in g["full_ts"]:
    A, B, C = g[f"full_t{t}_A"], g[f"full_t{t}_B"], g[f"full_t{t}_C"]
    assert np.array_equal(mul_full(d(A), d(B)).cpu().numpy().view(np.uint64), C), t
for n in g["cyc_ns"]:
    A, B, C = g[f"cyc_n{n}_A"], g[f"cyc_n{n}_B"], g[f"cyc_n{n}_C"]
    assert np.array_equal(mul_cyclic(d(A), d(B), int(n)).cpu().numpy().view(np.uint64), C), n
for n, b in ((12323, 256), (17669, 96), (35851, 64), (57637, 40)):
    A, B = make_cyclic_inputs(n, b)
    assert np.array_equal(mul_cyclic(d(A), d(B), n).cpu().numpy().view(np.uint64), c_mul_cyclic(A, B, n)), n
for t, b in ((16, 33), (128, 9), (512, 5), (1024, 3), (4096, 2)):
    A, B = make_full_inputs(t, b, words=True)
    assert np.array_equal(mul_full(d(A), d(B)).cpu().numpy().view(np.uint64), c_mul_full(A, B)), t
# >= 1024 groups: the fused last-pass + unslicing kernel (k34_root_unslice) when no Toom level is forced
rows = np.r_[0:40, 32728:32768]
A, B = make_full_inputs(64, 32768, words=True)
assert np.array_equal(mul_full(d(A), d(B)).cpu().numpy().view(np.uint64)[rows], c_mul_full(A[rows], B[rows]))
A, B = make_cyclic_inputs(8000, 32768)
assert np.array_equal(mul_cyclic(d(A), d(B), 8000).cpu().numpy().view(np.uint64)[rows],
                      c_mul_cyclic(A[rows], B[rows], 8000))
print("ok", plan("cyclic", 40, 57637)["toom_levels"])
"""


@pytest.mark.parametrize("env", [{}, {"F2X_TOOM": "1"}, {"F2X_TOOM": "2", "F2X_TOOM_SEQ": "1"},
                                 {"F2X_TOOM": "3", "F2X_TOOM_SEQ": "1"}, {"F2X_TOOM": "3"},
                                 # innermost level at x = X^8 (toom_eval_fused<TL, 8>, toom_interp_seq<.., 8>)
                                 {"F2X_TOOM": "2", "F2X_TOOM_SEQ": "1", "F2X_TOOM_WLAST": "8"},
                                 {"F2X_TOOM": "3", "F2X_TOOM_SEQ": "1", "F2X_TOOM_WLAST": "8"}])
def test_checked_build_shared_memory_poison(env, cuda):
    from conftest import GOLDEN
    from paper_2201_10473_b200 import build as b

    if not os.path.exists(b.LIB_CHECKED):
        pytest.skip("checked fixture not built (build.build(variant='checked'))")
    e = dict(os.environ, F2X_LIB_VARIANT="checked", **env)
    r = subprocess.run([sys.executable, "-c", _CHECKED_SCRIPT, ROOT, GOLDEN], env=e, capture_output=True,
                       text=True, timeout=1200)
    assert r.returncode == 0 and "ok" in r.stdout, (r.stdout + r.stderr)[-3000:]
