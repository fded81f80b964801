"""e2e (pinned host buffers, copies inside the timed region) pipeline sweep at
n=17669 x 4096 (development aid): HostPipeline chunks x lanes, plus the
copy-only ceiling of the same per-batch transfers (no kernels) on this box."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle.f2x_oracle import make_cyclic_inputs
from paper_2201_10473_b200.engine import HostPipeline

dev = torch.device("cuda", 0)
n, batch, K = 17669, 4096, 100
A, B = make_cyclic_inputs(n, batch)
t = A.shape[1]


def timed(step, K):
    for _ in range(8):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        step()
    return e0, e1


def copy_only(lanes):
    hA = [torch.from_numpy(A.view(np.int64).copy()).pin_memory() for _ in range(lanes)]
    hB = [torch.from_numpy(B.view(np.int64).copy()).pin_memory() for _ in range(lanes)]
    hC = [torch.empty_like(hA[0]).pin_memory() for _ in range(lanes)]
    dA = [torch.empty_like(hA[0], device=dev) for _ in range(lanes)]
    dB = [torch.empty_like(hA[0], device=dev) for _ in range(lanes)]
    dC = [torch.zeros_like(hA[0], device=dev) for _ in range(lanes)]
    ss = [torch.cuda.Stream(dev) for _ in range(lanes)]
    i = [0]

    def step():
        j = i[0] % lanes
        with torch.cuda.stream(ss[j]):
            dA[j].copy_(hA[j], non_blocking=True)
            dB[j].copy_(hB[j], non_blocking=True)
            hC[j].copy_(dC[j], non_blocking=True)
        i[0] += 1

    e0, e1 = timed(step, K)
    for s in ss:
        torch.cuda.current_stream(dev).wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K


def pipeline(chunks, lanes):
    hA = [torch.from_numpy(A.view(np.int64).copy()).pin_memory() for _ in range(lanes)]
    hB = [torch.from_numpy(B.view(np.int64).copy()).pin_memory() for _ in range(lanes)]
    hC = [torch.empty_like(hA[0]).pin_memory() for _ in range(lanes)]
    pipe = HostPipeline("cyclic", n, batch, dev, chunks=chunks, streams=3, lanes=lanes)
    for j in range(lanes):
        pipe.capture(hA[j], hB[j], hC[j], lane=j)
    i = [0]

    def step():
        j = i[0] % lanes
        pipe.run(hA[j], hB[j], hC[j], lane=j)
        i[0] += 1

    e0, e1 = timed(step, K)
    pipe.join()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K


for lanes in (2, 4, 8):
    ms = copy_only(lanes)
    print(f"copy-only lanes={lanes}: {ms*1e3:.1f} us/batch  {batch/ms*1e3/1e6:.2f} M/s-equiv", flush=True)
for chunks, lanes in ((1, 4), (1, 6), (1, 8), (2, 4), (2, 6), (4, 4)):
    ms = pipeline(chunks, lanes)
    print(f"pipeline chunks={chunks} lanes={lanes}: {ms*1e3:.1f} us/batch  {batch/ms*1e3/1e6:.2f} M/s", flush=True)
