"""Per-call latency of the reference-style single-product API (development
aid): schoolbook_mul at t = 4 / 277 and ring_mul at n = 17669."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2201_10473_b200 import PolyWords, preset, ring_mul, schoolbook_mul

rng = np.random.default_rng(1)
for t in (4, 277):
    a, b = PolyWords(rng.integers(0, 1 << 64, t, dtype=np.uint64)), PolyWords(rng.integers(0, 1 << 64, t, dtype=np.uint64))
    schoolbook_mul(a, b)
    t0 = time.perf_counter()
    for _ in range(200):
        schoolbook_mul(a, b)
    print(f"schoolbook_mul t={t}: {(time.perf_counter() - t0) / 200 * 1e6:.1f} us/call")
p = preset("hqc-128")
A = PolyWords(rng.integers(0, 1 << 64, p.words, dtype=np.uint64) & np.uint64((1 << 64) - 1))
w = A.words.copy()
w[-1] &= np.uint64((1 << (p.N - 64 * (p.words - 1))) - 1)
A = PolyWords(w)
ring_mul(A, A, p)
t0 = time.perf_counter()
for _ in range(200):
    ring_mul(A, A, p)
print(f"ring_mul n={p.N}: {(time.perf_counter() - t0) / 200 * 1e6:.1f} us/call")

# the round-1 per-call path for comparison: pageable copies + eager launches
import torch  # noqa: E402

from paper_2201_10473_b200.engine import mul_cyclic, mul_full  # noqa: E402

dev = torch.device("cuda", 0)
for t in (4, 277):
    aw = rng.integers(0, 1 << 64, t, dtype=np.uint64)
    f = lambda: mul_full(torch.from_numpy(aw.view(np.int64).copy()).reshape(1, -1).to(dev),  # noqa: E731
                         torch.from_numpy(aw.view(np.int64).copy()).reshape(1, -1).to(dev)).cpu()
    f()
    t0 = time.perf_counter()
    for _ in range(200):
        f()
    print(f"eager per-call (round 1 path) t={t}: {(time.perf_counter() - t0) / 200 * 1e6:.1f} us/call")
f = lambda: mul_cyclic(torch.from_numpy(w.view(np.int64).copy()).reshape(1, -1).to(dev),  # noqa: E731
                       torch.from_numpy(w.view(np.int64).copy()).reshape(1, -1).to(dev), p.N).cpu()
f()
t0 = time.perf_counter()
for _ in range(200):
    f()
print(f"eager per-call (round 1 path) ring n={p.N}: {(time.perf_counter() - t0) / 200 * 1e6:.1f} us/call")
