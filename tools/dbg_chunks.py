"""Chunked-schedule parity probe (development aid): F2X_CHUNKS=n python tools/dbg_chunks.py"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import c_mul_cyclic
from oracle.f2x_oracle import make_cyclic_inputs
from paper_2201_10473_b200 import mul_cyclic
dev = torch.device("cuda", 0)
for n, b in ((17669, 96), (17669, 4096), (12323, 256)):
    A, B = make_cyclic_inputs(n, b)
    out = mul_cyclic(torch.from_numpy(A.view(np.int64)).to(dev), torch.from_numpy(B.view(np.int64)).to(dev), n)
    torch.cuda.synchronize()
    o = out.cpu().numpy().view(np.uint64)
    ref = c_mul_cyclic(A, B, n)
    bad = np.nonzero((o != ref).any(axis=1))[0]
    print(n, b, "bad rows", len(bad), bad[:10], bad[-5:] if len(bad) else "")
