"""n=57637 timing under the bench's protocol variants (development aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle.f2x_oracle import make_cyclic_inputs
from paper_2201_10473_b200.engine import mul_cyclic
dev = torch.device("cuda", 0)
n, batch = 57637, 16384
flag = torch.zeros(1, dtype=torch.int32, device=dev)
flush = torch.empty((256 << 20) // 4, dtype=torch.int32, device=dev)
for tiled in (False, True):
    if tiled:
        A, B = make_cyclic_inputs(n, 4096)
        A, B = np.tile(A, (4, 1)), np.tile(B, (4, 1))
    else:
        A, B = make_cyclic_inputs(n, batch)
    dA = torch.from_numpy(A.view(np.int64)).to(dev); dB = torch.from_numpy(B.view(np.int64)).to(dev)
    dC = torch.empty_like(dA)
    for _ in range(3):
        mul_cyclic(dA, dB, n, out=dC, check=False, err_flag=flag)
    torch.cuda.synchronize()
    for mode in ("flush+sync", "sync", "back-to-back"):
        ts = []
        if mode == "back-to-back":
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(5):
                mul_cyclic(dA, dB, n, out=dC, check=False, err_flag=flag)
            e1.record(); torch.cuda.synchronize(); ts = [e0.elapsed_time(e1) / 5]
        else:
            for i in range(5):
                if mode == "flush+sync":
                    flush.fill_(i)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); mul_cyclic(dA, dB, n, out=dC, check=False, err_flag=flag); e1.record()
                torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        print(f"tiled={tiled} {mode}: " + " ".join(f"{t:.3f}" for t in ts), flush=True)
