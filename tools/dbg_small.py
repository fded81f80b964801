import sys, os; sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2201_10473_b200 import mul_full, mul_cyclic
dev = torch.device("cuda", 0)
t = int(sys.argv[1])
A = torch.from_numpy(np.arange(3 * t, dtype=np.int64).reshape(3, t)).to(dev)
try:
    C = mul_full(A, A)
    torch.cuda.synchronize()
    print("t", t, "ok", C.cpu().numpy().view(np.uint64)[0][:4])
except Exception as e:
    print("t", t, "ERR", e)
