"""Eager vs CUDA-graph replay of one device-resident ring-product call
(development aid): per-step CUDA events with an L2 flush before each step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle.f2x_oracle import make_cyclic_inputs
from paper_2201_10473_b200.engine import mul_cyclic

n, batch, K = int(sys.argv[1]) if len(sys.argv) > 1 else 17669, 4096, 200
dev = torch.device("cuda", 0)
A, B = make_cyclic_inputs(n, batch)
dA = torch.from_numpy(A.view(np.int64)).to(dev)
dB = torch.from_numpy(B.view(np.int64)).to(dev)
dC = torch.empty_like(dA)
flag = torch.zeros(1, dtype=torch.int32, device=dev)
flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)
step = lambda: mul_cyclic(dA, dB, n, out=dC, check=False, err_flag=flag)  # noqa: E731
for _ in range(5):
    step()
torch.cuda.synchronize()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    step()
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
torch.cuda.synchronize()


def timed(fn):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for i in range(K):
        flush.fill_(i)
        ev[i][0].record()
        fn()
        ev[i][1].record()
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) / K


for _ in range(2):
    print(f"n={n} eager {timed(step):.4f} ms  graph {timed(g.replay):.4f} ms", flush=True)
