"""Benchmark: batched constant-time GF(2)[X] ring products on B200.

Contract (one JSON line on rank 0):
  python bench.py --gpus N --steps K --warmup W [--impl reference]
  N>1: torchrun --nproc-per-node N ... bench.py --gpus N ...

Workload (BASELINE.json configs[1]): hqc-128 ring multiplication
A*B mod X^17669 - 1, t = 277 uint64 words per operand, 4096 products per GPU
per step (weak scaling: rank r owns rows [4096 r, 4096 (r+1)) of one seeded
global batch; shards are independent -- no collective on the data path).
A step = one call of the engine on a device-resident batch; inputs are seeded
synthetic operands with i.i.d. uniform bits (SURVEY.md §8(d) generator) --
no public dataset is involved.  L2 is flushed (256 MiB write) before every
timed step; flushes are outside the per-step CUDA events.

--impl reference times the reference's CPU path (the oracle port of
schoolbook_mul's default route, poly.py:517-561, plus the SPEC fold) on the
host cores; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cyclic GF(2)[X] products/sec at n=17669/35851/57637; % of int-ALU roofline"
UNIT = "products/s"
N_RING = 17669
BATCH_PER_GPU = 4096
L2_FLUSH_BYTES = 256 << 20
EXTRA_CONFIGS = ((35851, 4096), (57637, 16384))


def w_alg(t: int, cyclic: bool = True) -> float:
    """W = 144 t^log2(3) (+ 4t for the fold) int32 lane-ops."""
    return 144.0 * t ** math.log2(3) + (4.0 * t if cyclic else 0.0)


def shard_rows(rank: int, world: int, per_gpu: int) -> slice:
    """Rank r owns rows [per_gpu*r, per_gpu*(r+1)) of the seeded global batch
    (weak scaling; independent products, no data-path collective)."""
    if not 0 <= rank < world:
        raise ValueError("rank outside [0, world)")
    return slice(rank * per_gpu, (rank + 1) * per_gpu)


def committed_ncu(pl) -> dict | None:
    """Pipe utilisation / DRAM figures of the node kernel from the latest
    committed ncu --set full capture for this workload."""
    import csv
    import glob

    out = None
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "k2_node_mul_raw.csv"))):
        try:
            rows = list(csv.reader(open(f)))
            d = dict(zip(rows[0], rows[2]))
            dur_s = float(d["gpu__time_duration.sum"]) * 1e-6
            dram = (float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"])) * 1e6
            out = {
                "source": os.path.relpath(f, ROOT),
                "pipe_alu_pct": float(d["sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"]),
                "pipe_fma_pct": float(d["sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"]),
                "issue_active_pct": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
                "dram_GBps": round(dram / dur_s / 1e9, 1),
                "duration_us": float(d["gpu__time_duration.sum"]),
            }
        except Exception:
            continue
    return out if pl.get("leaf_words") == 35 else None


def committed_traffic(pl) -> dict | None:
    """DRAM bytes per node-kernel launch from the latest committed ncu --set
    full capture (profiles/r*/k2_traffic.json) for this workload, else None."""
    import glob

    best = None
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "k2_traffic.json"))):
        try:
            d = json.load(open(f))
        except Exception:
            continue
        if d.get("workload") == "n=17669 x4096" and pl.get("leaf_words") == 35:
            # algorithmic: both (pre-evaluated) bitsliced operands read once + every
            # node product written once
            el = pl.get("eval_levels", 0)
            ns = 3 ** el * (pl["leaf_stride"] << (pl["levels"] - el))
            ss = pl["leaf_stride"] << pl["cta_levels"]
            words = 3 ** pl["global_levels"] * 2 * ss
            alg = 4 * pl["groups"] * (2 * ns + words)
            best = {"dram_bytes_per_launch": d["dram_bytes_per_launch"], "source": d["source"],
                    "algorithmic_bytes_per_launch": alg,
                    "note": "DRAM < algorithmic: L2 (126 MB) absorbs most node-product writes"}
    return best


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------ CPU baseline

def _ref_rows(args):
    n, lo, hi = args
    import numpy as np

    from oracle.f2x_oracle import fold_cyclic, make_cyclic_inputs, mul_full_row

    A, B = make_cyclic_inputs(n, hi)
    t0 = time.perf_counter()
    for r in range(lo, hi):
        fold_cyclic(mul_full_row(A[r], B[r]), n)
    return hi - lo, time.perf_counter() - t0


def cpu_reference(n: int, rows_per_core: int = 48, pool=None, c_port: bool = True) -> dict:
    """Reference CPU path on all host cores: the oracle's restatement of
    schoolbook_mul's default (bit-spread big-int) route + SPEC fold, one
    product per row (the reference has no batched API), processes because
    the big-int route holds the GIL.  Also times the C port (word
    convolution, poly.py:493-514) for context."""
    import concurrent.futures as cf

    import numpy as np

    cores = len(os.sched_getaffinity(0))
    sample = cores * rows_per_core
    chunks = [(n, i * rows_per_core, (i + 1) * rows_per_core) for i in range(cores)]
    t0 = time.perf_counter()
    if pool is not None:
        res = list(pool.map(_ref_rows, chunks))
    else:
        with cf.ProcessPoolExecutor(max_workers=cores) as ex:
            res = list(ex.map(_ref_rows, chunks))
    wall = time.perf_counter() - t0
    done = sum(r[0] for r in res)
    # steady-state rate: rows / max per-worker compute time (excludes pool startup)
    busy = max(r[1] for r in res)
    value = done / busy
    out = {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
           "sample": f"{done} rows of the n={n} ring workload ({rows_per_core}/core), "
                     f"oracle port of schoolbook_mul default route (spread + CPython int) + SPEC fold",
           "wall_s": round(wall, 2)}
    if not c_port:
        return out
    try:
        from oracle import c_mul_cyclic
        from oracle.f2x_oracle import make_cyclic_inputs

        A, B = make_cyclic_inputs(n, cores * 64)
        t1 = time.perf_counter()
        c_mul_cyclic(A, B, n, threads=cores)
        out["c_port_value"] = round(A.shape[0] / (time.perf_counter() - t1), 1)
    except Exception as e:  # context only
        out["c_port_error"] = str(e)[:100]
    return out


# ------------------------------------------------------------ clocks

class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], 0
        self._stop = threading.Event()
        self._th = None
        self.ok = False

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.ok = True
            self._th = threading.Thread(target=self._run, daemon=True)
            self._th.start()
        except Exception:
            self.ok = False
        return self

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self._th:
            self._th.join()

    def summary(self) -> dict:
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        nv = self._nv
        names = []
        table = {
            "gpu_idle": getattr(nv, "nvmlClocksEventReasonGpuIdle", 0x1),
            "applications_clocks_setting": 0x2,
            "sw_power_cap": 0x4,
            "hw_slowdown": 0x8,
            "sync_boost": 0x10,
            "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80,
            "display_clock_setting": 0x100,
        }
        for k, bit in table.items():
            if self.reasons & bit:
                names.append(k)
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(s)}


# ------------------------------------------------------------ GPU arm

def int_alu_peak(torch, lib, dev) -> dict:
    """Live integer-ALU peak: LOP3 (c ^ a&b) microbenchmark over the whole chip."""
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    blocks, iters = sms * 8, 4096
    out = torch.empty(blocks * 256, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    for _ in range(2):
        lib.f2x_bench_lop3(out.data_ptr(), blocks, 256, stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rc = lib.f2x_bench_lop3(out.data_ptr(), blocks, iters, stream)
    e1.record()
    torch.cuda.synchronize()
    if rc:
        raise RuntimeError(f"lop3 microbenchmark failed ({rc})")
    sec = e0.elapsed_time(e1) / 1e3
    ops = blocks * 256 * iters * 128
    return {"ops_per_s": ops / sec, "sms": sms, "sec": sec}


def gpu_arm(args) -> None:
    import numpy as np
    import torch

    rank, world, local = dist_env()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    from oracle.f2x_oracle import make_cyclic_inputs
    from paper_2201_10473_b200 import _lib
    from paper_2201_10473_b200.engine import mul_cyclic, plan

    lib = _lib.load()
    n, bpg = args.n, args.batch
    t = (n + 63) // 64
    # one seeded global batch; this rank's contiguous shard
    A_all, B_all = make_cyclic_inputs(n, bpg * world)
    A = A_all[shard_rows(rank, world, bpg)]
    B = B_all[shard_rows(rank, world, bpg)]
    dA = torch.from_numpy(np.ascontiguousarray(A).view(np.int64)).to(dev)
    dB = torch.from_numpy(np.ascontiguousarray(B).view(np.int64)).to(dev)
    dC = torch.empty_like(dA)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    pl = plan("cyclic", bpg, n, args.leaf)

    def step():
        mul_cyclic(dA, dB, n, out=dC, leaf=args.leaf, check=False, err_flag=flag)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    peak = int_alu_peak(torch, lib, dev)

    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    nev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for a, b in nev:  # torch creates the cudaEvent_t lazily, on first record
        a.record()
        b.record()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(K):
            flush.fill_(i)
            lib.f2x_set_node_events(nev[i][0].cuda_event, nev[i][1].cuda_event)
            ev[i][0].record()
            step()
            ev[i][1].record()
        lib.f2x_set_node_events(None, None)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    step_ms = sum(a.elapsed_time(b) for a, b in ev)
    node_ms = sum(a.elapsed_time(b) for a, b in nev)
    if int(flag.item()) != 0:
        raise RuntimeError("top-bit check fired on seeded inputs")

    # parity spot check of the timed output against the C oracle (not timed)
    from oracle import c_mul_cyclic

    sub = slice(0, bpg, max(1, bpg // 64))
    assert np.array_equal(dC.cpu().numpy().view(np.uint64)[sub], c_mul_cyclic(A[sub], B[sub], n)), \
        "timed output differs from the oracle"

    # ---- e2e: host pinned buffers, H2D + compute + D2H inside the timed region
    from paper_2201_10473_b200.engine import HostPipeline

    # several host batches in flight (one pinned buffer set and pipeline lane
    # each) so batch j's H2D/D2H run under batch j-1's kernels; measured on
    # the box (n=17669 x 4096): 1 chunk x 4 lanes 10.6 M/s, 2 x 2 9.7 M/s,
    # 1 x 2 8.5 M/s (a whole-batch launch keeps the node grid at 23 waves)
    LANES = max(1, args.e2e_lanes)
    hAs = [torch.from_numpy(np.ascontiguousarray(A).view(np.int64).copy()).pin_memory()
           for _ in range(LANES)]
    hBs = [torch.from_numpy(np.ascontiguousarray(B).view(np.int64).copy()).pin_memory()
           for _ in range(LANES)]
    hCs = [torch.empty_like(hAs[0]).pin_memory() for _ in range(LANES)]
    pipe = HostPipeline("cyclic", n, bpg, dev, chunks=args.e2e_chunks, streams=3, leaf=args.leaf,
                        lanes=LANES)
    graphed = all(pipe.capture(hAs[i], hBs[i], hCs[i], lane=i) for i in range(LANES)) \
        if not args.no_graph else False
    e2e_i = [0]

    def e2e_step():
        i = e2e_i[0] % LANES
        pipe.run(hAs[i], hBs[i], hCs[i], lane=i)
        e2e_i[0] += 1

    for _ in range(max(2 * LANES, args.warmup)):
        e2e_step()
    pipe.join()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    KE = max(3, K // 2)
    e0.record()
    for _ in range(KE):
        e2e_step()
    pipe.join()
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / KE
    if pipe.rejected():
        raise RuntimeError("top-bit check fired on seeded inputs (e2e)")
    for hC in hCs:
        assert np.array_equal(hC.numpy().view(np.uint64)[sub], c_mul_cyclic(A[sub], B[sub], n)), \
            "e2e output differs from the oracle"

    # max over ranks
    stats = torch.tensor([step_ms, node_ms, e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(stats, op=torch.distributed.ReduceOp.MAX)
    step_ms, node_ms, e2e_ms = stats.tolist()
    ms_per_step = step_ms / K
    value = bpg * world / (ms_per_step / 1e3)

    per_cfg = {}
    if rank == 0 and world == 1 and not args.quick:
        per_cfg = extra_configs(torch, np, dev, args, peak)

    if rank == 0:
        W = w_alg(t)
        node_s = node_ms / K / 1e3
        achieved = bpg * W / node_s / 1e12
        pk = peak["ops_per_s"] / 1e12
        cl = clk.summary()
        nominal = peak["sms"] * 64 * (cl["sm_max_mhz"] or 1965) * 1e6 / 1e12
        line = {
            "metric": METRIC,
            "value": round(value, 1),
            "unit": UNIT,
            "n_gpus": world,
            "steps": K,
            "warmup": args.warmup,
            "ms_per_step": round(ms_per_step, 5),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "u32 (GF(2) bitsliced, int-ALU)",
            "data": "synthetic: seeded uniform-bit operands (SURVEY §8(d) generator), top bits >= n zeroed",
            "config": {
                "workload": f"hqc-128 ring mul mod X^{n}-1, {bpg} products/GPU/step (configs[1])",
                "n": n, "t_words": t, "batch_per_gpu": bpg, "global_batch": bpg * world,
                "parallelism": f"independent batch shards x{world}, no collectives",
                "l2": "flushed before each timed step (256 MiB write, outside events)",
                "plan": {k: pl[k] for k in ("N", "leaf_words", "levels", "cta_levels",
                                             "global_levels", "pass_levels", "node_ctas")},
            },
            "roofline": {
                "bound": "int_alu",
                "kernel": "k2_node_mul",
                "achieved": round(achieved, 3),
                "peak": round(pk, 3),
                "unit": "T int32-lane-op/s",
                "frac": round(achieved / pk, 4),
                # dram__bytes_read + write per node-kernel launch (committed ncu --set full
                # capture of this workload), details in traffic_detail
                "traffic": (lambda tr: round(tr["dram_bytes_per_launch"]) if tr else None)(committed_traffic(pl)),
                "traffic_detail": committed_traffic(pl),
                "work_per_product": round(W, 1),
                "work_model": "W_alg = 144 t^log2(3) + 4t (SURVEY §8(d)), t=ceil(n/64)",
                "peak_source": "live LOP3 microbenchmark (c^(a&b), 8 chains/thread, 8 CTAs/SM) this run",
                "peak_nominal_L64": round(nominal, 3),
                "frac_of_nominal_L64": round(achieved / nominal, 4),
                "node_ms_per_step": round(node_ms / K, 5),
                "step_frac_in_node_kernel": round(node_ms / step_ms, 4),
                "whole_step_frac": round(bpg * W / (ms_per_step / 1e3) / 1e12 / pk, 4),
            },
            "e2e": {
                "value": round(bpg * world / (e2e_ms / 1e3), 1),
                "unit": UNIT,
                "h2d_bytes_per_step": int(2 * bpg * t * 8),
                "d2h_bytes_per_step": int(bpg * t * 8),
                "ms_per_step": round(e2e_ms, 5),
                "path": f"pinned host A,B -> H2D -> mul_cyclic (C ABI) -> D2H; engine.HostPipeline, "
                        f"{args.e2e_chunks} row chunk(s) per batch"
                        + (", each batch replayed as one CUDA graph" if graphed else ", eager launches")
                        + f"; {LANES} host batches in flight (one pinned buffer set per lane), so a "
                        "batch's copies overlap the previous batches' kernels; pipeline fill and "
                        "drain inside the timed region",
            },
            "plan_work": {
                "leaf_lop3_per_product": round(pl["leaf_ops_per_product"], 1),
                "karatsuba_xor_ops_per_product": round(pl["karatsuba_ops_per_product"], 1),
                "base_mul_64x64_equiv_per_product": round(pl["leaf_ops_per_product"] / 128.0, 1),
                "note": "analytic counts of the executed plan; W_alg charges 144 t^log2(3)",
            },
            "ncu_node_kernel": committed_ncu(pl),
            "gpu_launches": int(K * pl["launches"]),
            "clocks": cl,
        }
        if per_cfg:
            line["per_config"] = per_cfg
        if world == 1 and not args.no_cpu:
            line["cpu_baseline"] = cpu_reference(n)
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def extra_configs(torch, np, dev, args, peak) -> dict:
    """n=35851 x4096 and n=57637 x16384 (the metric's other sizes), device timing."""
    from oracle.f2x_oracle import make_cyclic_inputs
    from paper_2201_10473_b200.engine import mul_cyclic

    out = {}
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    for n, batch in EXTRA_CONFIGS:
        A, B = make_cyclic_inputs(n, batch)
        dA = torch.from_numpy(A.view(np.int64)).to(dev)
        dB = torch.from_numpy(B.view(np.int64)).to(dev)
        dC = torch.empty_like(dA)
        for _ in range(3):
            mul_cyclic(dA, dB, n, out=dC, check=False, err_flag=flag)
        torch.cuda.synchronize()
        reps = 5
        tot = 0.0
        for i in range(reps):
            flush.fill_(i)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            mul_cyclic(dA, dB, n, out=dC, check=False, err_flag=flag)
            e1.record()
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
            if os.environ.get("F2X_BENCH_DEBUG"):
                print(f"extra n={n} rep {i}: {e0.elapsed_time(e1):.3f} ms", file=sys.stderr)
        ms = tot / reps
        t = (n + 63) // 64
        v = batch / (ms / 1e3)
        from paper_2201_10473_b200.engine import plan as eng_plan

        p = eng_plan("cyclic", batch, n)
        out[f"n{n}"] = {"batch": batch, "ms_per_call": round(ms, 4), "value": round(v, 1),
                        "whole_call_frac_int_alu": round(v * w_alg(t) / peak["ops_per_s"], 4),
                        "plan": {"toom_levels": p["toom_levels"], "toom_M": p["toom_M"],
                                 "leaf_words": p["leaf_words"], "levels": p["levels"],
                                 "global_levels": p["global_levels"]}}
        del dA, dB, dC
    return out


def reference_arm(args) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import concurrent.futures as cf

    n = args.n
    vals = []
    cb = None
    # one worker pool for the whole run (pool start-up is not part of a step)
    with cf.ProcessPoolExecutor(max_workers=len(os.sched_getaffinity(0))) as pool:
        for i in range(args.warmup + args.steps):
            last = i == args.warmup + args.steps - 1
            cb = cpu_reference(n, rows_per_core=8 if i < args.warmup else 16, pool=pool, c_port=last)
            if i >= args.warmup:
                vals.append(cb["value"])
    value = sum(vals) / len(vals)
    cb["value"] = value
    line = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": UNIT,
        "impl": "reference",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u64 (GF(2), CPython int)",
        "data": "synthetic: seeded uniform-bit operands (SURVEY §8(d) generator)",
        "config": {"workload": f"hqc-128 ring mul mod X^{n}-1 (configs[1]); each step a bounded "
                               f"sample of rows on all host cores", "n": n, "t_words": (n + 63) // 64},
        "cpu_baseline": cb,
        "e2e": {"value": round(value, 2), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--n", type=int, default=N_RING)
    ap.add_argument("--batch", type=int, default=BATCH_PER_GPU)
    ap.add_argument("--leaf", type=int, default=0)
    ap.add_argument("--e2e-chunks", type=int, default=1,
                    help="row chunks per host batch in the e2e pipeline")
    ap.add_argument("--no-graph", action="store_true", help="eager e2e launches (no CUDA graph)")
    ap.add_argument("--e2e-lanes", type=int, default=4,
                    help="host batches in flight in the e2e pipeline (one pinned buffer set each)")
    ap.add_argument("--quick", action="store_true", help="skip the extra-config lines")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "engine":
        args.warmup = 3
    if args.impl == "reference":
        reference_arm(args)
    else:
        gpu_arm(args)


if __name__ == "__main__":
    main()
