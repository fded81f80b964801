"""Per-kernel device time of the live engine (torch.profiler / CUPTI) for
cyclic sizes given as n[:batch] (development aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
from oracle.f2x_oracle import make_cyclic_inputs
from paper_2201_10473_b200 import mul_cyclic

dev = torch.device("cuda", 0)
leaf = int(os.environ.get("LEAF", "0"))
for arg in sys.argv[1:] or ["17669"]:
    n, batch = (int(x) for x in (arg.split(":") + ["4096"])[:2])
    A, B = make_cyclic_inputs(n, min(batch, 4096))
    reps = batch // A.shape[0]
    dA = torch.from_numpy(np.tile(A, (reps, 1)).view(np.int64)).to(dev)
    dB = torch.from_numpy(np.tile(B, (reps, 1)).view(np.int64)).to(dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    for _ in range(3):
        mul_cyclic(dA, dB, n, check=False, err_flag=flag, leaf=leaf)
    torch.cuda.synchronize()
    R = 10
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(R):
            mul_cyclic(dA, dB, n, check=False, err_flag=flag, leaf=leaf)
        torch.cuda.synchronize()
    tot = {}
    for e in prof.events():
        if e.device_type.name == "CUDA":
            k = e.name.split("(")[0][:40]
            tot[k] = tot.get(k, 0.0) + e.device_time / R
    s = sum(tot.values())
    print(f"n={n} batch={batch} total {s:.1f} us/call: " +
          ", ".join(f"{k} {v:.1f}" for k, v in sorted(tot.items(), key=lambda kv: -kv[1])))
