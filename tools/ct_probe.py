"""Where does a fixed(sparse)-vs-random(dense) timing difference come from?
Per-kernel device times (CUPTI via torch.profiler) of the two classes,
interleaved, L2 flushed before every call (development aid for ct_check)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2201_10473_b200.ct_check import _dense_rows, _sparse_rows
from paper_2201_10473_b200.engine import mul_cyclic

n, batch, reps = 17669, 4096, int(sys.argv[1]) if len(sys.argv) > 1 else 300
seed = int(sys.argv[2], 0) if len(sys.argv) > 2 else 0xC9
rng = np.random.default_rng(seed)
dev = torch.device("cuda", 0)
B = torch.from_numpy(_dense_rows(n, batch, rng).view(np.int64)).to(dev)
fixed = _sparse_rows(n, 75, batch, rng)
cls_bufs = [[torch.from_numpy(fixed.view(np.int64).copy()).to(dev) for _ in range(4)],
            [torch.from_numpy(_dense_rows(n, batch, rng).view(np.int64)).to(dev) for _ in range(4)]]
flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)
out = torch.empty_like(B)
flag = torch.zeros(1, dtype=torch.int32, device=dev)
res = {}
for c in (0, 1, 0, 1):
    for i in range(3):
        mul_cyclic(cls_bufs[c][i % 4], B, n, out=out, check=False, err_flag=flag)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(reps):
            flush.fill_(i)
            mul_cyclic(cls_bufs[c][i % 4], B, n, out=out, check=False, err_flag=flag)
        torch.cuda.synchronize()
    tot = res.setdefault(c, {})
    for e in prof.events():
        if e.device_type.name == "CUDA" and "f2x" in e.name:
            k = e.name.split("(")[0].replace("void ", "")[:32]
            tot[k] = tot.get(k, 0.0) + e.device_time / reps / 2
for k in res[0]:
    print(f"{k:34s} sparse {res[0][k]:9.3f} us  dense {res[1][k]:9.3f} us  diff {res[0][k] - res[1][k]:+.3f}")
