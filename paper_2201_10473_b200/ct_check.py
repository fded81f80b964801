"""Statistical constant-time check (SPEC ``ct_check``).

Fixed-vs-random timing test: a weight-w sparse first operand (the HQC secret
shape) against a dense random first operand, interleaved
trials, Welch's t statistic on the per-call times; |t| < 4.5 passes; fewer
than 10^4 trials ("pre: trials >= 10^4") is "inconclusive".  On
the GPU every call is timed with CUDA events around one ring-product call of
a batch of 4096 (the configs[1] batch; every row of the fixed class has a
weight-w first operand).  At batch 32 (one bitsliced group) the call is
launch-latency bound and even the leaky fixture below passed (measured), so
the test had no detection power there; at 4096 the leaves dominate.
Controls:

* ``control=True``: dense fixed vs dense random -- must pass;
* the deliberately leaky GPU build (``F2X_LIB_VARIANT=leaky``, the
  ``F2X_LEAKY_LEAF`` fixture: leaves skip all-zero a words) -- must FAIL;
* ``leaky_mul``: a CPU sparse convolution that only visits the set bits of
  A -- must FAIL (``ct_check_leaky``).

``masked=True`` times ``engine.mul_cyclic_masked`` (A*B = (A^R)*B ^ R*B
with fresh random R): the engine has no data-dependent branch or address,
but a ~0.1 % physical timing effect of sparse operands (switching power /
clock management) shows up for some seeds; masking removes it.
"""

from __future__ import annotations

import math
import time

import numpy as np

THRESHOLD = 4.5
MIN_TRIALS = 10_000


def welch_t(x, y) -> float:
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    vx, vy = x.var(ddof=1) / x.size, y.var(ddof=1) / y.size
    if vx + vy == 0:
        return 0.0
    return float((x.mean() - y.mean()) / math.sqrt(vx + vy))


def _sparse_rows(n: int, weight: int, rows: int, rng) -> np.ndarray:
    from .ring import sparse_to_dense

    return np.stack([sparse_to_dense(rng.choice(n, weight, replace=False), n).words
                     for _ in range(rows)])


def _dense_rows(n: int, rows: int, rng) -> np.ndarray:
    t = (n + 63) // 64
    A = rng.integers(0, 1 << 64, size=(rows, t), dtype=np.uint64)
    r = n - 64 * (t - 1)
    if r < 64:
        A[:, -1] &= np.uint64((1 << r) - 1)
    return A


def ct_check(n: int = 17669, weight: int = 75, trials: int = MIN_TRIALS, seed: int = 0xC7,
             batch: int = 4096, control: bool = False, masked: bool = False) -> dict:
    """GPU fixed-vs-random(dense) timing test of ``mul_cyclic``: the fixed
    first operand is weight-``weight`` sparse, or dense with ``control``.
    ``trials`` calls per class."""
    import torch

    from .engine import mul_cyclic, mul_cyclic_masked

    if masked:
        gen = torch.Generator(device=torch.device("cuda", torch.cuda.current_device()))
        gen.manual_seed(seed)
        mul_cyclic = lambda A, B, n, out, check, err_flag: mul_cyclic_masked(  # noqa: E731
            A, B, n, out=out, generator=gen, check=check, err_flag=err_flag)

    rng = np.random.default_rng(seed)
    dev = torch.device("cuda", torch.cuda.current_device())
    B = torch.from_numpy(_dense_rows(n, batch, rng).view(np.int64)).to(dev)
    fixed = _dense_rows(n, batch, rng) if control else _sparse_rows(n, weight, batch, rng)
    # both classes cycle through the same number of distinct device buffers
    # (the fixed class: 8 copies of the fixed operand) and L2 is flushed
    # before every call, so the classes differ ONLY in the operand bits --
    # a single re-used fixed buffer would stay L2-resident and time faster
    NBUF = 8
    fixed_bufs = [torch.from_numpy(fixed.view(np.int64).copy()).to(dev) for _ in range(NBUF)]
    pool = [torch.from_numpy(_dense_rows(n, batch, rng).view(np.int64)).to(dev) for _ in range(NBUF)]
    flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)  # 256 MiB > L2
    out = torch.empty_like(B)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    for i in range(10):
        mul_cyclic(fixed_bufs[i % NBUF], B, n, out=out, check=False, err_flag=flag)
        mul_cyclic(pool[i % NBUF], B, n, out=out, check=False, err_flag=flag)
    torch.cuda.synchronize()
    t_fix, t_rnd = [], []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    order = rng.permutation(np.repeat([0, 1], trials))  # exactly `trials` per class, interleaved
    seen = [0, 0]
    for cls in order:
        A = (fixed_bufs if cls == 0 else pool)[seen[cls] % NBUF]
        seen[cls] += 1
        flush.fill_(int(seen[0] + seen[1]))
        e0.record()
        mul_cyclic(A, B, n, out=out, check=False, err_flag=flag)
        e1.record()
        e1.synchronize()
        (t_fix if cls == 0 else t_rnd).append(e0.elapsed_time(e1))
    t = welch_t(t_fix, t_rnd)
    verdict = "pass" if abs(t) < THRESHOLD else "fail"
    if min(len(t_fix), len(t_rnd)) < MIN_TRIALS and verdict == "pass":
        verdict = "inconclusive"  # too few trials to call it constant time
    return {"n": n, "weight": None if control else weight, "control": control, "masked": masked,
            "trials": [len(t_fix), len(t_rnd)],
            "mean_ms": [float(np.mean(t_fix)), float(np.mean(t_rnd))], "t": t, "verdict": verdict}


def leaky_mul(a: int, b: int, n: int) -> int:
    """Deliberately leaky ring product: loops over the set bits of a only."""
    r = 0
    mask = (1 << n) - 1
    while a:
        low = a & -a
        i = low.bit_length() - 1
        r ^= ((b << i) | (b >> (n - i))) & mask if i else b
        a ^= low
    return r


def ct_check_leaky(n: int = 2000, weight: int = 20, trials: int = 300, seed: int = 0xC8) -> dict:
    """Positive control on the CPU: the leaky multiplier must FAIL."""
    rng = np.random.default_rng(seed)
    b = int.from_bytes(rng.bytes((n + 7) // 8), "little") & ((1 << n) - 1)
    sparse = sum(1 << int(i) for i in rng.choice(n, weight, replace=False))
    t_fix, t_rnd = [], []
    for cls in rng.integers(0, 2, size=2 * trials):
        a = sparse if cls == 0 else int.from_bytes(rng.bytes((n + 7) // 8), "little") & ((1 << n) - 1)
        t0 = time.perf_counter()
        leaky_mul(a, b, n)
        (t_fix if cls == 0 else t_rnd).append(time.perf_counter() - t0)
    t = welch_t(t_fix, t_rnd)
    return {"n": n, "weight": weight, "t": t, "verdict": "pass" if abs(t) < THRESHOLD else "fail"}


if __name__ == "__main__":
    import json
    import sys

    if "--control" in sys.argv:
        print(json.dumps(ct_check(control=True)))
    else:
        print(json.dumps(ct_check()))
    if "--cpu-leaky" in sys.argv:
        print(json.dumps(ct_check_leaky()))
