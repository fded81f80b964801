"""Toom-3 plan parity + timing probe (development aid): F2X_TOOM=k python tools/toom_check.py"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import c_mul_cyclic, c_mul_full
from oracle.f2x_oracle import make_cyclic_inputs, make_full_inputs
from paper_2201_10473_b200 import mul_cyclic, mul_full, plan
dev = torch.device("cuda", 0)
d = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).to(dev)
for n, b in ((12323, 64), (17669, 96), (35851, 40), (57637, 33)):
    A, B = make_cyclic_inputs(n, b)
    out = mul_cyclic(d(A), d(B), n).cpu().numpy().view(np.uint64)
    ref = c_mul_cyclic(A, B, n)
    bad = np.nonzero((out != ref).any(axis=1))[0]
    p = plan("cyclic", b, n)
    print(f"n={n} TL={p['toom_levels']} M={p['toom_M']} LF={p['leaf_words']} K={p['levels']} bad rows {len(bad)}", flush=True)
for t in (64, 256, 1024):
    A, B = make_full_inputs(t, 40, words=True)
    out = mul_full(d(A), d(B)).cpu().numpy().view(np.uint64)
    bad = np.nonzero((out != c_mul_full(A, B)).any(axis=1))[0]
    print(f"full t={t} TL={plan('full', 40, t)['toom_levels']} bad rows {len(bad)}", flush=True)
