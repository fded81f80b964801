"""Benchmark: batched constant-time GF(2)[X] ring products on B200.

Contract (one JSON line on rank 0):
  python bench.py --gpus N --steps K --warmup W [--impl reference]
  N > 1 either under torchrun (one process per GPU, RANK/WORLD_SIZE/LOCAL_RANK
  from the env) or, with WORLD_SIZE unset, N worker processes spawned here
  (worker r on cuda:r).  Ranks share no data: the only coordination is a
  host-side barrier and a max over ranks of the timings (gloo over TCP under
  torchrun, a multiprocessing barrier + shared array when spawned) -- no
  NCCL, no collective on the data path (north_star).

Headline (BASELINE.json configs[1]): hqc-128 ring multiplication
A*B mod X^17669 - 1, t = 277 uint64 words per operand, 4096 products per GPU
per step (weak scaling: rank r owns rows [4096 r, 4096 (r+1)) of one seeded
global batch), identical for every N.  A step = one call of the engine on a
device-resident batch; inputs are seeded synthetic operands with i.i.d.
uniform bits (SURVEY.md §8(d) generator) -- no public dataset is involved.
L2 is flushed (256 MiB write) before every timed step; flushes are outside
the per-step CUDA events.

Also reported: ``scaling_57637`` (configs[3]: n=57637 x 16384 products split
16384/N across the N GPUs, strong scaling) and, at N=1, ``per_config`` lines
for configs[0] (n=12323 x 256), configs[2] (n=35851 x 4096), configs[3] and
the configs[4] full-product d-sweep (~1 GB of operands per size).  Every
timed output is checked against the C oracle outside the timed region on a
stated row subsample (>= 256 rows incl. the first and last 32-row groups):
``parity: {rows_checked, ok}``.

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
RING_CONFIGS = ((12323, 256, "configs[0]"), (35851, 4096, "configs[2]"), (57637, 16384, "configs[3]"))
# context only (not vs_baseline): the paper's best single-core AVX512 cycle
# counts as products/s at 2.8 GHz
PAPER_1CORE = {17669: 2.8e9 / 14872, 35851: 2.8e9 / 46940, 57637: 2.8e9 / 110568,
               1024: 2.8e9 / 129, 4096: 2.8e9 / 1287, 8192: 2.8e9 / 3977, 16384: 2.8e9 / 12078,
               32768: 2.8e9 / 36811, 65536: 2.8e9 / 114620}
SCALE_N, SCALE_BATCH = 57637, 16384
DSWEEP = (1024, 4096, 8192, 16384, 32768, 65536)
DSWEEP_OPERAND_BYTES = 1 << 30  # A + B per GPU


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
            name = f"k2_node_mul<{pl['leaf_words']}, {pl['cta_levels']}>"
            if name not in d["Kernel Name"] or f"({pl['node_ctas']}," not in d["Grid Size"]:
                continue
            out = {
                "source": os.path.relpath(f, ROOT),
                "kernel": name, "grid": int(pl["node_ctas"]),
                "pipe_alu_pct": float(d["sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"]),
                "pipe_fma_pct": float(d["sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"]),
                "issue_active_pct": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
                "dram_GBps": round(dram / dur_s / 1e9, 1),
                "duration_us": float(d["gpu__time_duration.sum"]),
            }
        except Exception:
            continue
    return out


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
        if (d.get("workload") == "n=17669 x4096" and pl.get("n") == 17669 and pl.get("batch") == 4096 and
                d.get("kernel") == f"k2_node_mul<{pl['leaf_words']},{pl['cta_levels']}>" and
                d.get("grid", pl["node_ctas"]) == pl["node_ctas"]):
            # algorithmic: both (pre-evaluated) bitsliced node-problem operands read
            # once + every node product written once
            el = pl.get("eval_levels", 0)
            ns = 3 ** el * (pl["leaf_stride"] << (pl["levels"] - el))
            ss = pl["leaf_stride"] << pl["cta_levels"]
            words = 3 ** pl["global_levels"] * 2 * ss
            alg = 4 * pl["groups"] * 5 ** pl.get("toom_levels", 0) * (2 * ns + words)
            best = {"dram_bytes_per_launch": d["dram_bytes_per_launch"], "source": d["source"],
                    "algorithmic_bytes_per_launch": alg,
                    "note": "DRAM < algorithmic: L2 (126 MB) absorbs most node-product writes"}
    return best


def split_rows(rank: int, world: int, total: int) -> slice:
    """Strong scaling: rank r's contiguous share of `total` rows, cut on whole
    32-row groups (the engine's bitsliced unit), balanced to within a group."""
    if not 0 <= rank < world:
        raise ValueError("rank outside [0, world)")
    groups = -(-total // 32)
    lo = (groups * rank // world) * 32
    hi = min(total, (groups * (rank + 1) // world) * 32)
    return slice(lo, hi)


def parity_rows(batch: int, want: int = 256) -> "list[int]":
    """Rows checked against the oracle: all rows when batch <= want, else the
    first and the last 32-row groups plus an even stride through the rest."""
    if batch <= want:
        return list(range(batch))
    edge = list(range(32)) + list(range(batch - 32, batch))
    mid = want - len(edge)
    step = (batch - 64) / mid
    rows = set(edge) | {32 + int(i * step) for i in range(mid)}
    return sorted(rows)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class LocalSync:
    """World of one."""

    rank, world = 0, 1

    def barrier(self):
        pass

    def max(self, vals):
        return list(vals)

    def close(self):
        pass


class GlooSync:
    """torchrun ranks: host-side barrier and max over a gloo (TCP) group --
    timing coordination only, no NCCL and no device data."""

    def __init__(self, rank, world):
        import torch.distributed as dist

        self.dist, self.rank, self.world = dist, rank, world
        dist.init_process_group("gloo", rank=rank, world_size=world)

    def barrier(self):
        self.dist.barrier()

    def max(self, vals):
        import torch

        t = torch.tensor([float(v) for v in vals], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.tolist()

    def close(self):
        self.dist.destroy_process_group()


class SpawnSync:
    """Workers spawned by bench.py itself: a multiprocessing barrier and a
    shared array of per-rank slots for the max over ranks."""

    SLOTS = 32

    def __init__(self, rank, world, barrier, arr):
        self.rank, self.world, self._b, self._a = rank, world, barrier, arr

    def barrier(self):
        self._b.wait()

    def max(self, vals):
        vals = [float(v) for v in vals]
        assert len(vals) <= self.SLOTS
        base = self.rank * self.SLOTS
        for i, v in enumerate(vals):
            self._a[base + i] = v
        self._b.wait()
        out = [max(self._a[r * self.SLOTS + i] for r in range(self.world)) for i in range(len(vals))]
        self._b.wait()  # nobody overwrites a slot before every rank has read it
        return out

    def close(self):
        pass


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


def cpu_reference(n: int, rows_per_core: int = 120, pool=None, c_port: bool = True) -> dict:
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


def check_rows(np, kind, size, hA, hB, dC, rows) -> dict:
    """Oracle check of the timed output on `rows` (host copies of the inputs
    of exactly those rows; the output rows are read back from the device)."""
    from oracle import c_mul_cyclic, c_mul_full

    idx = np.asarray(rows, dtype=np.int64)
    A = np.ascontiguousarray(hA[idx])
    B = np.ascontiguousarray(hB[idx])
    import torch

    got = dC[torch.from_numpy(idx).to(dC.device)].cpu().numpy().view(np.uint64)
    want = c_mul_cyclic(A, B, size) if kind == "cyclic" else c_mul_full(A, B)
    return {"rows_checked": int(idx.size), "ok": bool(np.array_equal(got, want)),
            "rows": "all" if idx.size == hA.shape[0] else
            "first+last 32-row groups + even stride (%d of %d)" % (idx.size, hA.shape[0])}


def device_words(torch, batch, t, seed, dev):
    """Uniform random uint64 words [batch][t] (as int64) generated on the
    device from a seeded generator (the ~1 GB d-sweep inputs)."""
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    return torch.randint(-2 ** 31, 2 ** 31, (batch, 2 * t), dtype=torch.int32, device=dev,
                         generator=g).view(torch.int64)


def time_calls(torch, fn, reps, warmup, flush) -> float:
    """Mean device ms per call: CUDA events around each call on the current
    stream, 256 MiB L2 flush before each (outside the events)."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    evs = []
    for i in range(reps):
        flush.fill_(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in evs) / reps


def ring_entry(torch, np, dev, n, batch, label, peak, flush, reps=5, warmup=3) -> dict:
    from oracle.f2x_oracle import make_cyclic_inputs
    from paper_2201_10473_b200.engine import CapturedCall, plan as eng_plan

    A, B = make_cyclic_inputs(n, batch)
    dA = torch.from_numpy(A.view(np.int64)).to(dev)
    dB = torch.from_numpy(B.view(np.int64)).to(dev)
    dC = torch.empty_like(dA)
    cap = CapturedCall("cyclic", dA, dB, dC, n)  # the repeated call, as the headline
    ms = time_calls(torch, cap, reps, warmup, flush)
    if int(cap.err_flag.item()) != 0:
        raise RuntimeError(f"top-bit check fired on seeded inputs (n={n})")
    del cap
    t = (n + 63) // 64
    v = batch / (ms / 1e3)
    p = eng_plan("cyclic", batch, n)
    out = {"workload": f"ring mul mod X^{n}-1 x{batch} ({label})", "n": n, "batch": batch,
           "ms_per_call": round(ms, 4), "value": round(v, 1), "unit": UNIT,
           "whole_call_frac_int_alu": round(v * w_alg(t) / peak["ops_per_s"], 4),
           "plan": {"toom_levels": p["toom_levels"], "toom_M": p["toom_M"], "leaf_words": p["leaf_words"],
                    "levels": p["levels"], "global_levels": p["global_levels"],
                    "eval_levels": p["eval_levels"], "launches": p["launches"]},
           "parity": check_rows(np, "cyclic", n, A, B, dC, parity_rows(batch))}
    if n in PAPER_1CORE:
        out["paper_avx512_1core_products_s"] = round(PAPER_1CORE[n], 1)
    del dA, dB, dC
    torch.cuda.empty_cache()
    return out


def dsweep_entry(torch, np, dev, d, peak, flush, reps=5, warmup=3) -> dict:
    """configs[4]: unreduced full product of degree-<d operands, batch sized
    to ~1 GB of operands (A + B) per GPU."""
    from paper_2201_10473_b200.engine import _WS_BUDGET, CapturedCall, _row_chunks, plan as eng_plan
    from paper_2201_10473_b200 import _lib

    t = d // 64
    batch = DSWEEP_OPERAND_BYTES // (2 * 8 * t)
    dA = device_words(torch, batch, t, 0xF2F2 + 2 * d, dev)
    dB = device_words(torch, batch, t, 0xF2F2 + 2 * d + 1, dev)
    dC = torch.empty((batch, 2 * t), dtype=torch.int64, device=dev)
    cap = CapturedCall("full", dA, dB, dC, t)
    ms = time_calls(torch, cap, reps, warmup, flush)
    del cap
    v = batch / (ms / 1e3)
    p = eng_plan("full", batch, t)
    rows = parity_rows(batch)
    idx = torch.tensor(rows, dtype=torch.int64, device=dev)
    hA = np.zeros((batch, t), dtype=np.uint64)  # only the checked rows are filled
    hB = np.zeros((batch, t), dtype=np.uint64)
    hA[rows] = dA[idx].cpu().numpy().view(np.uint64)
    hB[rows] = dB[idx].cpu().numpy().view(np.uint64)
    chunks = _row_chunks(_lib.load(), _lib.KIND_FULL, batch, t, 0)[0]
    out = {"workload": f"full product d={d} bits x{batch} (configs[4])", "d": d, "t": t, "batch": batch,
           "operand_bytes": int(2 * batch * t * 8), "ms_per_call": round(ms, 4), "value": round(v, 1),
           "unit": UNIT, "whole_call_frac_int_alu": round(v * w_alg(t, cyclic=False) / peak["ops_per_s"], 4),
           "plan": {"toom_levels": p["toom_levels"], "leaf_words": p["leaf_words"], "levels": p["levels"],
                    "global_levels": p["global_levels"], "eval_levels": p["eval_levels"],
                    "workspace_bytes": p["workspace_bytes"], "row_chunks": len(chunks),
                    "ws_budget": _WS_BUDGET},
           "parity": check_rows(np, "full", d, hA, hB, dC, rows)}
    if d in PAPER_1CORE:
        out["paper_avx512_1core_products_s"] = round(PAPER_1CORE[d], 1)
    del dA, dB, dC
    torch.cuda.empty_cache()
    return out


def scaling_block(torch, np, dev, sync, peak, flush, reps=5, warmup=3) -> dict:
    """configs[3]: n=57637 x 16384 products split 16384/N across the ranks
    (strong scaling, no data exchange).  Rank 0 also times the whole batch
    alone (the N=1 point) when N > 1.  Returns rank 0's block."""
    from oracle.f2x_oracle import make_cyclic_inputs
    from paper_2201_10473_b200.engine import CapturedCall

    n, total = SCALE_N, SCALE_BATCH
    t = (n + 63) // 64
    rank, world = sync.rank, sync.world
    A_all, B_all = make_cyclic_inputs(n, total)

    def timed(sl):
        A, B = np.ascontiguousarray(A_all[sl]), np.ascontiguousarray(B_all[sl])
        dA = torch.from_numpy(A.view(np.int64)).to(dev)
        dB = torch.from_numpy(B.view(np.int64)).to(dev)
        dC = torch.empty_like(dA)
        cap = CapturedCall("cyclic", dA, dB, dC, n)
        ms = time_calls(torch, cap, reps, warmup, flush)
        if int(cap.err_flag.item()) != 0:
            raise RuntimeError("top-bit check fired on seeded inputs (n=57637)")
        del cap
        par = check_rows(np, "cyclic", n, A, B, dC, parity_rows(A.shape[0]))
        del dA, dB, dC
        torch.cuda.empty_cache()
        return ms, par

    solo_ms = None
    if world > 1:
        sync.barrier()
        if rank == 0:
            solo_ms, _ = timed(slice(0, total))
        sync.barrier()
    sl = split_rows(rank, world, total)
    sync.barrier()
    ms, par = timed(sl)
    rows = sl.stop - sl.start
    per = [0.0] * (3 * world)  # per-rank [ms, rows, ok] gathered through max
    per[3 * rank], per[3 * rank + 1], per[3 * rank + 2] = ms, rows, 1.0 if par["ok"] else 0.0
    per = sync.max(per)
    ok_all = all(per[3 * r + 2] == 1.0 for r in range(world))
    min_ok = min(per[3 * r + 2] for r in range(world))
    mx = max(per[3 * r] for r in range(world))
    if rank != 0:
        return {}
    value = total / (mx / 1e3)
    one = solo_ms if solo_ms is not None else ms
    W = w_alg(t)
    return {
        "workload": f"ring mul mod X^{n}-1, {total} products split {total}/{world} per GPU (configs[3])",
        "n_gpus": world, "scaling": "strong", "value": round(value, 1), "unit": UNIT,
        "ms_per_call_max_over_gpus": round(mx, 4),
        "single_gpu_ms_whole_batch": round(one, 4),
        "efficiency": round((total / (mx / 1e3)) / (world * total / (one / 1e3)), 4),
        "per_gpu": [{"device": r, "rows": int(per[3 * r + 1]), "ms_per_call": round(per[3 * r], 4),
                     "value": round(per[3 * r + 1] / (per[3 * r] / 1e3), 1),
                     "whole_call_frac_int_alu": round(per[3 * r + 1] / (per[3 * r] / 1e3) * W / peak["ops_per_s"], 4)}
                    for r in range(world)],
        "parity": {"rows_checked_per_gpu": par["rows_checked"], "ok": bool(ok_all and min_ok == 1.0)},
    }


def gpu_arm(args, sync, local) -> None:
    import numpy as np
    import torch

    rank, world = sync.rank, sync.world
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    from oracle.f2x_oracle import make_cyclic_inputs
    from paper_2201_10473_b200 import _lib
    from paper_2201_10473_b200.engine import CapturedCall, HostPipeline, mul_cyclic, plan

    lib = _lib.load()
    n, bpg = args.n, args.batch
    t = (n + 63) // 64
    # one seeded global batch; this rank's contiguous shard
    A_all, B_all = make_cyclic_inputs(n, bpg * world)
    A = np.ascontiguousarray(A_all[shard_rows(rank, world, bpg)])
    B = np.ascontiguousarray(B_all[shard_rows(rank, world, bpg)])
    del A_all, B_all
    dA = torch.from_numpy(A.view(np.int64)).to(dev)
    dB = torch.from_numpy(B.view(np.int64)).to(dev)
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
    # the repeated call through the engine's CapturedCall: every launch of
    # the call captured once as a CUDA graph, replayed per step (the
    # device-resident headline); an eager pass of the same K steps with
    # events around the node kernel gives the roofline's kernel time
    cap = CapturedCall("cyclic", dA, dB, dC, n, leaf=args.leaf)
    for _ in range(args.warmup):
        cap()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    eev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    nev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for a, b in nev:  # torch creates the cudaEvent_t lazily, on first record
        a.record()
        b.record()
    torch.cuda.synchronize()
    sync.barrier()
    with ClockSampler(local) as clk:
        for i in range(K):  # eager: node-kernel events
            flush.fill_(i)
            lib.f2x_set_node_events(nev[i][0].cuda_event, nev[i][1].cuda_event)
            eev[i][0].record()
            step()
            eev[i][1].record()
        lib.f2x_set_node_events(None, None)
        for i in range(K):  # captured: the headline
            flush.fill_(i)
            ev[i][0].record()
            cap()
            ev[i][1].record()
        torch.cuda.synchronize()
    sync.barrier()
    step_ms = sum(a.elapsed_time(b) for a, b in ev)
    eager_ms = sum(a.elapsed_time(b) for a, b in eev)
    node_ms = sum(a.elapsed_time(b) for a, b in nev)
    if int(flag.item()) != 0 or int(cap.err_flag.item()) != 0:
        raise RuntimeError("top-bit check fired on seeded inputs")
    head_par = check_rows(np, "cyclic", n, A, B, dC, parity_rows(bpg))

    # ---- e2e: host pinned buffers, H2D + compute + D2H inside the timed region
    # several host batches in flight (one pinned buffer set and pipeline lane
    # each) so batch j's H2D/D2H run under batch j-1's kernels; measured on
    # the box (n=17669 x 4096): 1 chunk x 4 lanes 10.6 M/s, 2 x 2 9.7 M/s,
    # 1 x 2 8.5 M/s (a whole-batch launch keeps the node grid at 23 waves);
    # re-measured on another box (tools/e2e_sweep.py): copy-only ceiling 370
    # us/batch (11.06 M/s), 2 x 4 388 us, 2 x 6 389, 1 x 4 407, 1 x 6 396 --
    # the default is 2 chunks x 4 lanes
    def make_e2e(chunks, lanes):
        hA_ = [torch.from_numpy(A.view(np.int64).copy()).pin_memory() for _ in range(lanes)]
        hB_ = [torch.from_numpy(B.view(np.int64).copy()).pin_memory() for _ in range(lanes)]
        hC_ = [torch.empty_like(hA_[0]).pin_memory() for _ in range(lanes)]
        p_ = HostPipeline("cyclic", n, bpg, dev, chunks=chunks, streams=3, leaf=args.leaf, lanes=lanes)
        g_ = all(p_.capture(hA_[i], hB_[i], hC_[i], lane=i) for i in range(lanes)) if not args.no_graph else False
        return p_, hA_, hB_, hC_, g_

    # the pipeline shape (row chunks x lanes) is calibrated on this box before
    # the timed region unless given: PCIe and copy-engine behaviour vary
    # between boxes of the pool (tools/e2e_sweep.py: the best shape was 2 x 4
    # on one box, 1 x 4 on another where concurrent H2D+D2H ran at 51 GB/s)
    calib = {}
    if args.e2e_chunks > 0:
        CHUNKS, LANES = args.e2e_chunks, max(1, args.e2e_lanes)
    else:
        for ch, ln in ((1, 2), (1, 4), (2, 2), (2, 4), (4, 4)):
            p_, hA_, hB_, hC_, _ = make_e2e(ch, ln)
            for j in range(2 * ln):
                p_.run(hA_[j % ln], hB_[j % ln], hC_[j % ln], lane=j % ln)
            p_.join()
            torch.cuda.synchronize()
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record()
            for j in range(24):
                p_.run(hA_[j % ln], hB_[j % ln], hC_[j % ln], lane=j % ln)
            p_.join()
            c1.record()
            torch.cuda.synchronize()
            calib[f"{ch}x{ln}"] = round(c0.elapsed_time(c1) / 24, 4)
            del p_, hA_, hB_, hC_
        best = min(calib, key=calib.get)
        CHUNKS, LANES = (int(x) for x in best.split("x"))
    pipe, hAs, hBs, hCs, graphed = make_e2e(CHUNKS, LANES)
    e2e_i = [0]

    def e2e_step():
        i = e2e_i[0] % LANES
        pipe.run(hAs[i], hBs[i], hCs[i], lane=i)
        e2e_i[0] += 1

    for _ in range(max(2 * LANES, args.warmup)):
        e2e_step()
    pipe.join()
    torch.cuda.synchronize()
    sync.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    KE = max(3, K // 2)
    e0.record()
    for _ in range(KE):
        e2e_step()
    pipe.join()
    e1.record()
    torch.cuda.synchronize()
    sync.barrier()
    e2e_ms = e0.elapsed_time(e1) / KE
    if pipe.rejected():
        raise RuntimeError("top-bit check fired on seeded inputs (e2e)")
    e2e_ok = True
    rows = parity_rows(bpg)
    from oracle import c_mul_cyclic

    want = c_mul_cyclic(A[rows], B[rows], n)
    for hC in hCs:
        e2e_ok &= bool(np.array_equal(hC.numpy().view(np.uint64)[rows], want))
    del pipe, hAs, hBs, hCs

    # max over ranks (timings), min over ranks (parity) via max of the negation
    step_ms, eager_ms, node_ms, e2e_ms, bad_head, bad_e2e = sync.max(
        [step_ms, eager_ms, node_ms, e2e_ms, 0.0 if head_par["ok"] else 1.0, 0.0 if e2e_ok else 1.0])
    head_par["ok"] = bad_head == 0.0
    head_par["rows_checked_per_gpu"] = head_par.pop("rows_checked")
    ms_per_step = step_ms / K
    value = bpg * world / (ms_per_step / 1e3)

    scaling = {}
    if not args.quick:
        scaling = scaling_block(torch, np, dev, sync, peak, flush)
    per_cfg = {}
    if rank == 0 and world == 1 and not args.quick:
        for rn, rb, label in RING_CONFIGS:
            if rn == SCALE_N and rb == SCALE_BATCH and scaling:
                continue  # = the scaling block's N=1 point
            per_cfg[f"n{rn}"] = ring_entry(torch, np, dev, rn, rb, label, peak, flush)
        if scaling:
            s1 = scaling["per_gpu"][0]
            per_cfg[f"n{SCALE_N}"] = {
                "workload": f"ring mul mod X^{SCALE_N}-1 x{SCALE_BATCH} (configs[3])", "n": SCALE_N,
                "batch": SCALE_BATCH, "ms_per_call": s1["ms_per_call"], "value": s1["value"], "unit": UNIT,
                "whole_call_frac_int_alu": s1["whole_call_frac_int_alu"], "parity": scaling["parity"],
                "note": "same measurement as scaling_57637 at N=1",
                "paper_avx512_1core_products_s": round(PAPER_1CORE[SCALE_N], 1)}
        if not args.no_dsweep:
            for d in DSWEEP:
                per_cfg[f"d{d}"] = dsweep_entry(torch, np, dev, d, peak, flush)

    if rank == 0:
        W = w_alg(t)
        # the node kernel's units: 5^TL node problems of LF 2^K coefficients per
        # product under TL Toom-3 levels (the whole product when TL = 0)
        TL = int(pl.get("toom_levels", 0))
        t_node = (pl["leaf_words"] << pl["levels"]) / 64.0
        W_node = 5 ** TL * w_alg(t_node, cyclic=False) if TL else W
        node_s = node_ms / K / 1e3
        achieved = bpg * W_node / node_s / 1e12
        pk = peak["ops_per_s"] / 1e12
        cl = clk.summary()
        nominal = peak["sms"] * 64 * (cl["sm_max_mhz"] or 1965) * 1e6 / 1e12
        all_ok = head_par["ok"] and e2e_ok and all(e["parity"]["ok"] for e in per_cfg.values()) and \
            (not scaling or scaling["parity"]["ok"])
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
                "parallelism": f"independent batch shards x{world}; host barrier + max-over-ranks "
                               f"timing only ({type(sync).__name__}), no NCCL, no collectives",
                "l2": "flushed before each timed step (256 MiB write, outside events)",
                "step": "engine.CapturedCall: the call's launches captured once as a CUDA graph and "
                        "replayed per step (eager per-step time in roofline.eager_ms_per_step)",
                "plan": {k: pl[k] for k in ("N", "leaf_words", "levels", "cta_levels",
                                             "global_levels", "pass_levels", "eval_levels", "node_ctas",
                                             "toom_levels", "toom_M", "launches")},
            },
            "parity": head_par,
            "parity_all_ok": bool(all_ok),
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
                "work_per_product": round(W_node, 1),
                "work_model": ("W_alg = 144 t^log2(3) + 4t (SURVEY §8(d)), t=ceil(n/64)" if not TL else
                               f"node kernel: 5^{TL} node problems per product x W_alg(t_node) = 144 t_node^log2(3), "
                               f"t_node = {t_node:g} words (the plan's {TL} Toom-3 levels run in the memory passes); "
                               "whole_step_frac charges the product's own W_alg = 144 t^log2(3) + 4t, "
                               "t=ceil(n/64) (work_per_product_whole)"),
                "work_per_product_whole": round(W, 1),
                "peak_source": "live LOP3 microbenchmark (c^(a&b), 8 chains/thread, 8 CTAs/SM) this run",
                "peak_nominal_L64": round(nominal, 3),
                "frac_of_nominal_L64": round(achieved / nominal, 4),
                "node_ms_per_step": round(node_ms / K, 5),
                "eager_ms_per_step": round(eager_ms / K, 5),
                "step_frac_in_node_kernel": round(node_ms / eager_ms, 4),
                "whole_step_frac": round(bpg * W / (ms_per_step / 1e3) / 1e12 / pk, 4),
            },
            "e2e": {
                "value": round(bpg * world / (e2e_ms / 1e3), 1),
                "unit": UNIT,
                "h2d_bytes_per_step": int(2 * bpg * t * 8),
                "d2h_bytes_per_step": int(bpg * t * 8),
                "ms_per_step": round(e2e_ms, 5),
                "parity_ok": bool(bad_e2e == 0.0),
                "path": f"pinned host A,B -> H2D -> mul_cyclic (C ABI) -> D2H; engine.HostPipeline, "
                        f"{CHUNKS} row chunk(s) per batch"
                        + (", each batch replayed as one CUDA graph" if graphed else ", eager launches")
                        + f"; {LANES} host batches in flight (one pinned buffer set per lane), so a "
                        "batch's copies overlap the previous batches' kernels; pipeline fill and "
                        "drain inside the timed region",
                "pipeline_shape": f"{CHUNKS}x{LANES}",
                "calibration_ms_per_batch": calib or None,
            },
            "plan_work": {
                "leaf_lop3_per_product": round(pl["leaf_ops_per_product"], 1),
                "karatsuba_xor_ops_per_product": round(pl["karatsuba_ops_per_product"], 1),
                "base_mul_64x64_equiv_per_product": round(pl["leaf_ops_per_product"] / 128.0, 1),
                "note": "analytic counts of the executed plan; W_alg charges 144 t^log2(3)",
            },
            "ncu_node_kernel": committed_ncu(pl),
            "paper_avx512_1core_products_s": round(PAPER_1CORE[N_RING], 1) if n == N_RING else None,
            # timed headline steps + e2e batches (each row chunk is its own call and plan)
            "gpu_launches": int(K * pl["launches"] + max(3, K // 2) * CHUNKS *
                                plan("cyclic", -(-bpg // CHUNKS), n, args.leaf)["launches"]),
            "clocks": cl,
        }
        if scaling:
            line["scaling_57637"] = scaling
        if getattr(args, "share_device", False):
            line["functional_test_only"] = "--share-device: all ranks on cuda:0; timings are not a measurement"
        if per_cfg:
            line["per_config"] = per_cfg
        if world == 1 and not args.no_cpu:
            line["cpu_baseline"] = cpu_reference(n)
        print(json.dumps(line), flush=True)
        if not all_ok:
            print("bench: PARITY FAILURE (see parity fields)", file=sys.stderr)


def _spawned_worker(target, rank, world, barrier, arr, targs):
    target(SpawnSync(rank, world, barrier, arr), rank, *targs)


def launch_spawned(world: int, target, *targs, timeout_s: float = 1800.0) -> list:
    """Run target(sync, rank, *targs) in `world` spawned processes (rank r
    drives cuda:r in the bench) joined by a SpawnSync; returns the exit
    codes.  A rank that dies breaks the barrier (timeout) instead of hanging
    the others forever."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    barrier = ctx.Barrier(world, timeout=timeout_s)
    arr = ctx.Array("d", SpawnSync.SLOTS * world, lock=False)
    procs = [ctx.Process(target=_spawned_worker, args=(target, r, world, barrier, arr, targs))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join()
    return [p.exitcode for p in procs]


def _gpu_rank(sync, rank, args):
    gpu_arm(args, sync, 0 if args.share_device else rank)


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
    ap.add_argument("--e2e-chunks", type=int, default=0,
                    help="row chunks per host batch in the e2e pipeline (0: calibrate chunks x lanes "
                         "on this box before the timed region)")
    ap.add_argument("--no-graph", action="store_true", help="eager e2e launches (no CUDA graph)")
    ap.add_argument("--e2e-lanes", type=int, default=4,
                    help="host batches in flight in the e2e pipeline (one pinned buffer set each; with "
                         "--e2e-chunks > 0)")
    ap.add_argument("--quick", action="store_true", help="headline only (no per-config / scaling lines)")
    ap.add_argument("--no-dsweep", action="store_true", help="skip the configs[4] d-sweep lines")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline")
    ap.add_argument("--share-device", action="store_true",
                    help="FUNCTIONAL TEST ONLY: every spawned rank on cuda:0 (exercises the N-rank code "
                         "path on a one-GPU box; the timings are not a measurement)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "engine":
        args.warmup = 3
    if args.impl == "reference":
        reference_arm(args)
        return
    rank, world, local = dist_env()
    if "WORLD_SIZE" in os.environ:  # torchrun: one process per GPU
        if world != args.gpus:
            print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
        sync = GlooSync(rank, world) if world > 1 else LocalSync()
        try:
            gpu_arm(args, sync, 0 if args.share_device else local)
        finally:
            sync.close()
    elif args.gpus > 1:  # spawn one worker per GPU here
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus and not args.share_device:
            raise SystemExit(f"bench: --gpus {args.gpus} but only {have} CUDA device(s) visible")
        codes = launch_spawned(args.gpus, _gpu_rank, args)
        bad = [c for c in codes if c != 0]
        if bad:
            raise SystemExit(f"bench: worker(s) failed with exit codes {bad}")
    else:
        gpu_arm(args, LocalSync(), 0)


if __name__ == "__main__":
    main()
