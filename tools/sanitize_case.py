"""Small cases for compute-sanitizer (one tool per gpurun call):
    compute-sanitizer --tool racecheck python tools/sanitize_case.py ring 12323 64
    F2X_TOOM=3 compute-sanitizer --tool memcheck python tools/sanitize_case.py ring 57637 40
Runs the engine once on seeded inputs and checks the result against the C
oracle (exit 1 on mismatch)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import c_mul_cyclic, c_mul_full
from oracle.f2x_oracle import make_cyclic_inputs, make_full_inputs
from paper_2201_10473_b200 import mul_cyclic, mul_full, plan

kind, size, batch = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
dev = torch.device("cuda", 0)
d = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).to(dev)  # noqa: E731
if kind == "ring":
    A, B = make_cyclic_inputs(size, batch)
    out = mul_cyclic(d(A), d(B), size).cpu().numpy().view(np.uint64)
    ok = np.array_equal(out, c_mul_cyclic(A, B, size))
    p = plan("cyclic", batch, size)
else:
    A, B = make_full_inputs(size, batch, words=True)
    out = mul_full(d(A), d(B)).cpu().numpy().view(np.uint64)
    ok = np.array_equal(out, c_mul_full(A, B))
    p = plan("full", batch, size)
torch.cuda.synchronize()
print(f"{kind} {size} x{batch}: toom_levels={p['toom_levels']} LF={p['leaf_words']} K={p['levels']} "
      f"launches={p['launches']} parity={'ok' if ok else 'MISMATCH'}", flush=True)
sys.exit(0 if ok else 1)
