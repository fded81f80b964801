"""Quick device timing of the engine per config (development aid)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle.f2x_oracle import make_cyclic_inputs, make_full_inputs
from paper_2201_10473_b200 import mul_cyclic, mul_full, plan
from paper_2201_10473_b200._lib import load
lib = load()

dev = torch.device("cuda", 0)
cfgs = [("cyc", 12323, 256), ("cyc", 17669, 4096), ("cyc", 35851, 4096), ("cyc", 57637, 16384),
        ("full", 16, 1 << 22), ("full", 64, 1 << 20), ("full", 256, 1 << 18), ("full", 1024, 1 << 16)]
if len(sys.argv) > 1:
    cfgs = [c for c in cfgs if str(c[1]) in sys.argv[1:]]
leaf = int(os.environ.get("LEAF", "0"))
for kind, size, batch in cfgs:
    print("cfg", kind, size, batch, flush=True)
    if kind == "cyc":
        A, B = make_cyclic_inputs(size, min(batch, 4096))
    else:
        A, B = make_full_inputs(size, min(batch, 4096), words=True)
    reps = batch // A.shape[0]
    dA = torch.from_numpy(np.tile(A, (reps, 1)).view(np.int64)).to(dev)
    dB = torch.from_numpy(np.tile(B, (reps, 1)).view(np.int64)).to(dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    f = (lambda: mul_cyclic(dA, dB, size, check=False, err_flag=flag, leaf=leaf)) if kind == "cyc" \
        else (lambda: mul_full(dA, dB, leaf=leaf))
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 10
    nv = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for a, b in nv:  # torch creates the cudaEvent_t lazily, on first record
        a.record(); b.record()
    e0.record()
    for i in range(iters):
        lib.f2x_set_node_events(nv[i][0].cuda_event, nv[i][1].cuda_event)
        f()
    e1.record()
    lib.f2x_set_node_events(None, None)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    node_ms = sum(a.elapsed_time(b) for a, b in nv) / iters
    p = plan("cyclic" if kind == "cyc" else "full", batch, size, leaf)
    t = p["t"]
    W = 144 * t ** np.log2(3) + (4 * t if kind == "cyc" else 0)
    pint = 148 * 64 * 1.965e9
    print(json.dumps({"kind": kind, "size": size, "batch": batch, "ms": round(ms, 4), "node_ms": round(node_ms, 4),
                      "prod_per_s": round(batch / ms * 1e3), "frac_L64": round(batch / ms * 1e3 * W / pint, 3),
                      "LF": p["leaf_words"], "K": p["levels"], "GL": p["global_levels"],
                      "passes": p["pass_levels"], "ctas": p["node_ctas"], "ws_MB": p["workspace_bytes"] >> 20}))
