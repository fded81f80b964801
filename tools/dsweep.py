"""Full-product d-sweep (BASELINE configs[4]): d in {1024..65536} bits, batch
= 2^26 / t rows (~1 GB of operands per GPU), default plan; device timing with
CUDA events (development aid / DESIGN table)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle.f2x_oracle import make_full_inputs
from paper_2201_10473_b200 import mul_full, plan

dev = torch.device("cuda", 0)
leaf = int(os.environ.get("LEAF", "0"))
for d in [int(x) for x in (sys.argv[1:] or ["1024", "4096", "8192", "16384", "32768", "65536"])]:
    t = d // 64
    batch = (1 << 26) // t
    A, B = make_full_inputs(t, min(batch, 8192), words=True)
    reps = batch // A.shape[0]
    dA = torch.from_numpy(np.tile(A, (reps, 1)).view(np.int64)).to(dev)
    dB = torch.from_numpy(np.tile(B, (reps, 1)).view(np.int64)).to(dev)
    out = torch.empty((dA.shape[0], 2 * t), dtype=torch.int64, device=dev)
    for _ in range(2):
        mul_full(dA, dB, out=out, leaf=leaf)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    R = 5
    e0.record()
    for _ in range(R):
        mul_full(dA, dB, out=out, leaf=leaf)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / R
    p = plan("full", dA.shape[0], t, leaf)
    W = 144 * t ** np.log2(3)
    v = dA.shape[0] / ms * 1e3
    print(json.dumps({"d": d, "t": t, "batch": int(dA.shape[0]), "ms": round(ms, 3), "products_per_s": round(v),
                      "frac_L64": round(v * W / (148 * 64 * 1.965e9), 3), "LF": p["leaf_words"], "K": p["levels"],
                      "toom": p["toom_levels"], "EL": p["eval_levels"]}), flush=True)
    del dA, dB, out
