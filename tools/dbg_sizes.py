import sys, os; sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2201_10473_b200 import mul_full, mul_cyclic, plan
dev = torch.device("cuda", 0)
kind = sys.argv[1]
for s in map(int, sys.argv[2:]):
    p = plan("full" if kind == "full" else "cyclic", 3, s)
    t = p["t"]
    A = torch.from_numpy(np.arange(3 * t, dtype=np.int64).reshape(3, t) & 0xFFFF).to(dev)
    try:
        C = mul_full(A, A) if kind == "full" else mul_cyclic(A, A, s, check=False, err_flag=torch.zeros(1, dtype=torch.int32, device=dev))
        torch.cuda.synchronize()
        print(kind, s, "ok", {k: p[k] for k in ("leaf_words", "levels", "cta_levels", "global_levels", "pass_levels")}, flush=True)
    except Exception as e:
        print(kind, s, "ERR", str(e)[:200], {k: p[k] for k in ("leaf_words", "levels", "cta_levels", "global_levels", "pass_levels")}, flush=True)
        break
