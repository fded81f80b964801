"""Randomised parity stress (development aid; the committed suite pins seeded
cases): random ring and full-product sizes at batches large enough for every
Toom depth / innermost point, a row subsample checked against the C oracle.
    python tools/stress_parity.py [cases] [seed]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import c_mul_cyclic, c_mul_full  # (checker only)
from oracle.f2x_oracle import make_cyclic_inputs, make_full_inputs
from paper_2201_10473_b200 import mul_cyclic, mul_full, plan

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 120
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
dev = torch.device("cuda", 0)
seen, bad = {}, 0
K34 = os.environ.get("STRESS_K34") == "1"  # many-group Karatsuba-only shapes (k34_root_unslice, k1_slice_groups)
for i in range(cases):
    cyc = i % 3 != 2
    if K34:
        batch = int(rng.integers(32768, 40000))
        if cyc:
            n = int(rng.integers(64, 9000))
            p = plan("cyclic", batch, n)
            A, B = make_cyclic_inputs(n, 4096)
        else:
            t = int(rng.integers(1, 139))
            p = plan("full", batch, t)
            A, B = make_full_inputs(t, 4096, words=True)
        reps = -(-batch // 4096)
        A, B = np.tile(A, (reps, 1))[:batch], np.tile(B, (reps, 1))[:batch]
        dA, dB = torch.from_numpy(A.view(np.int64)).to(dev), torch.from_numpy(B.view(np.int64)).to(dev)
        got = mul_cyclic(dA, dB, n) if cyc else mul_full(dA, dB)
    elif os.environ.get("STRESS_BIG") == "1":  # very large operands at small batches (deep global Karatsuba levels)
        cyc = False
        t = int(rng.integers(1400, 9000))
        batch = int(rng.choice([rng.integers(1, 8), rng.integers(8, 200)]))
        p = plan("full", batch, t)
        A, B = make_full_inputs(t, batch, words=True)
        got = mul_full(torch.from_numpy(A.view(np.int64)).to(dev), torch.from_numpy(B.view(np.int64)).to(dev))
    elif cyc:
        n = int(rng.integers(10240, 70000))
        batch = int(rng.choice([rng.integers(1, 64), rng.integers(600, 1500), rng.integers(2000, 4200)]))
        p = plan("cyclic", batch, n)
        A, B = make_cyclic_inputs(n, batch)
        got = mul_cyclic(torch.from_numpy(A.view(np.int64)).to(dev), torch.from_numpy(B.view(np.int64)).to(dev), n)
    else:
        t = int(rng.integers(160, 1400))
        batch = int(rng.choice([rng.integers(1, 48), rng.integers(600, 2200)]))
        p = plan("full", batch, t)
        A, B = make_full_inputs(t, batch, words=True)
        got = mul_full(torch.from_numpy(A.view(np.int64)).to(dev), torch.from_numpy(B.view(np.int64)).to(dev))
    if os.environ.get("STRESS_VERBOSE"):
        print(i, "cyclic" if cyc else "full", n if cyc else t, batch,
              {k: p[k] for k in ("toom_levels", "toom_w_last", "leaf_words", "levels", "toom_M")}, flush=True)
    got = got.cpu().numpy().view(np.uint64)
    rows = np.unique(np.r_[0:min(4, batch), max(0, batch - 4):batch, rng.integers(0, batch, 8)])
    want = c_mul_cyclic(A[rows], B[rows], n) if cyc else c_mul_full(A[rows], B[rows])
    ok = np.array_equal(got[rows], want)
    key = (p["toom_levels"], p["toom_w_last"])
    seen[key] = seen.get(key, 0) + 1
    if not ok:
        bad += 1
        print("MISMATCH", "cyclic" if cyc else "full", n if cyc else t, batch, p, flush=True)
print("cases", cases, "mismatches", bad, "plans (toom_levels, w_last):", dict(sorted(seen.items())))
sys.exit(1 if bad else 0)
