"""Experiment: one batched call split into S row chunks on S forked streams,
all captured in ONE CUDA graph, vs the whole batch on one stream.  The
chunks' memory-bound passes (slicing, interpolation, unslicing) can then
overlap another chunk's ALU-bound node kernel, and kernel tails overlap.

usage: python tools/split_streams.py 17669:4096 35851:4096 57637:16384 [--splits 1,2,3,4]
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import c_mul_cyclic  # noqa: E402  (checker only)
from oracle.f2x_oracle import make_cyclic_inputs  # noqa: E402
from paper_2201_10473_b200 import _lib  # noqa: E402
from paper_2201_10473_b200.engine import _row_chunks, mul_cyclic  # noqa: E402


def build_graph(A, B, C, n, S, flag):
    dev = A.device
    batch = A.shape[0]
    groups = -(-batch // 32)
    per = -(-groups // S) * 32
    ranges = [(lo, min(lo + per, batch)) for lo in range(0, batch, per)]
    lib = _lib.load()
    streams = [torch.cuda.Stream(dev) for _ in ranges]
    wss = [torch.empty(max(_row_chunks(lib, _lib.KIND_CYCLIC, hi - lo, n, 0)[1], 256), dtype=torch.uint8,
                       device=dev) for lo, hi in ranges]

    def body():
        cur = torch.cuda.current_stream(dev)
        for s, (lo, hi), ws in zip(streams, ranges, wss):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                mul_cyclic(A[lo:hi], B[lo:hi], n, out=C[lo:hi], check=False, err_flag=flag, workspace=ws)
        for s in streams:
            cur.wait_stream(s)

    body()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        body()
    torch.cuda.synchronize()
    return g, len(ranges)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfgs", nargs="+")
    ap.add_argument("--splits", default="1,2,3,4")
    ap.add_argument("--reps", type=int, default=30)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for cfg in a.cfgs:
        n, batch = (int(x) for x in cfg.split(":"))
        Ah, Bh = make_cyclic_inputs(n, batch)
        A = torch.from_numpy(Ah.view(np.int64)).to(dev)
        B = torch.from_numpy(Bh.view(np.int64)).to(dev)
        want_rows = np.r_[0:32, batch - 32:batch]
        want = c_mul_cyclic(Ah[want_rows], Bh[want_rows], n)
        for S in (int(x) for x in a.splits.split(",")):
            C = torch.zeros_like(A)
            flag = torch.zeros(1, dtype=torch.int32, device=dev)
            g, used = build_graph(A, B, C, n, S, flag)
            ts = []
            for r in range(a.reps + 3):
                flush.random_(0, 255) if r == 0 else flush.fill_(r & 0xFF)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                if r >= 3:
                    ts.append(e0.elapsed_time(e1))
            got = C.cpu().numpy().view(np.uint64)[want_rows]
            ok = bool(np.array_equal(got, want)) and int(flag.item()) == 0
            ts = np.array(ts)
            print(f"n={n} batch={batch} splits={used}: median {np.median(ts)*1e3:.1f} us  "
                  f"min {ts.min()*1e3:.1f} us  ok={ok}", flush=True)
            del g, C


if __name__ == "__main__":
    main()
