"""Per-kernel device time (CUPTI via torch.profiler) of full products for
d-sweep sizes given as bits (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import bench
from paper_2201_10473_b200 import mul_full

dev = torch.device("cuda", 0)
for d in [int(x) for x in sys.argv[1:]] or [1024, 4096]:
    t = d // 64
    batch = bench.DSWEEP_OPERAND_BYTES // (2 * 8 * t)
    dA = bench.device_words(torch, batch, t, 1, dev)
    dB = bench.device_words(torch, batch, t, 2, dev)
    dC = torch.empty((batch, 2 * t), dtype=torch.int64, device=dev)
    for _ in range(2):
        mul_full(dA, dB, out=dC)
    torch.cuda.synchronize()
    R = 5
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(R):
            mul_full(dA, dB, out=dC)
        torch.cuda.synchronize()
    tot = {}
    for e in prof.events():
        if e.device_type.name == "CUDA" and "f2x" in e.name:
            k = e.name.split("(")[0].replace("void ", "").replace("f2x::", "")[:28]
            tot[k] = tot.get(k, 0.0) + e.device_time / R
    print(f"d={d} batch={batch} total {sum(tot.values()):.1f} us: " +
          ", ".join(f"{k} {v:.1f}" for k, v in sorted(tot.items(), key=lambda kv: -kv[1])), flush=True)
    del dA, dB, dC
