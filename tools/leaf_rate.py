"""Leaf-LOP3 throughput of the node kernel alone and of the whole call, for
full-product sizes given as t:batch (development aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle.f2x_oracle import make_full_inputs
from paper_2201_10473_b200 import mul_full, plan
from paper_2201_10473_b200._lib import load
lib = load()
dev = torch.device("cuda", 0)
for t, batch in [(int(a.split(":")[0]), int(a.split(":")[1])) for a in sys.argv[1:]]:
    A, B = make_full_inputs(t, batch, words=True)
    dA = torch.from_numpy(A.view(np.int64)).to(dev); dB = torch.from_numpy(B.view(np.int64)).to(dev)
    for _ in range(3): mul_full(dA, dB)
    torch.cuda.synchronize()
    R = 10
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(R)]
    nv = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(R)]
    for a, b in nv:  # torch creates the cudaEvent_t lazily, on first record
        a.record(); b.record()
    for i in range(R):
        lib.f2x_set_node_events(nv[i][0].cuda_event, nv[i][1].cuda_event)
        ev[i][0].record(); mul_full(dA, dB); ev[i][1].record()
    lib.f2x_set_node_events(None, None)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / R
    nms = sum(a.elapsed_time(b) for a, b in nv) / R
    p = plan("full", batch, t)
    leaf = p["leaf_ops_per_product"] * batch
    print(f"t={t} LF={p['leaf_words']} K={p['levels']} GL={p['global_levels']} ms={ms:.3f} node={nms:.3f} "
          f"leaf rate node {leaf / nms / 1e9 / 18.56:.3f}  whole {leaf / ms / 1e9 / 18.56:.3f} of peak")
