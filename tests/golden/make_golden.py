"""Generate golden vectors by running the REAL reference (f2xmul.poly).

Run in the build container, where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nbcache \
        python tests/golden/make_golden.py

The reference cannot travel to the GPU box, so its outputs are committed here
as small .npz fixtures.  Full products come straight from
``f2xmul.poly.schoolbook_mul`` (poly.py:547-561, default route: spread for
t > 48, convolution otherwise) and ``clmul64_batch`` (poly.py:451-480).
Cyclic products are ``schoolbook_mul`` followed by the SPEC fold
 -- the reference ships no ring module, so the fold is
restated here (and pinned against the rotation-sum definition at small n in
tests/test_oracle.py).
"""

from __future__ import annotations

import os
import sys

import numpy as np

import f2xmul.poly as poly  # the reference package

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.f2x_oracle import make_cyclic_inputs  # noqa: E402  (seeded generator only)

SEED = 0xF2F2  # conftest.py:46


def ref_full(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    return poly.schoolbook_mul(poly.PolyWords(a), poly.PolyWords(b)).words.copy()


def ref_cyclic(a: np.ndarray, b: np.ndarray, n: int) -> np.ndarray:
    p = poly.schoolbook_mul(poly.PolyWords(a), poly.PolyWords(b)).to_int()
    r = (p & ((1 << n) - 1)) ^ (p >> n)
    t = (n + 63) // 64
    return np.frombuffer(r.to_bytes(8 * t, "little"), dtype=np.uint64).copy()


def main() -> None:
    out = {}
    rng = np.random.default_rng(SEED)

    # clmul64 lanes, both reference backends (poly.py:451-480)
    a = rng.integers(0, 1 << 64, 4096, dtype=np.uint64)
    b = rng.integers(0, 1 << 64, 4096, dtype=np.uint64)
    edge = np.array([0, 1, 5, (1 << 64) - 1, 1 << 63, 0xDEADBEEFCAFEF00D], dtype=np.uint64)
    a = np.concatenate([edge, edge[::-1], a])
    b = np.concatenate([edge[::-1], edge, b])
    lo, hi = poly.clmul64_batch(a, b, backend="portable")
    lo2, hi2 = poly.clmul64_batch(a, b, backend="multilane")
    assert np.array_equal(lo, lo2) and np.array_equal(hi, hi2)
    out["clmul_a"], out["clmul_b"], out["clmul_lo"], out["clmul_hi"] = a, b, lo, hi

    # full products through the reference's public entry point
    full_ts = [1, 2, 3, 4, 5, 7, 8, 15, 16, 17, 31, 32, 33, 48, 49, 64, 100, 128,
               193, 256, 277, 512, 561, 901, 1024]
    for t in full_ts:
        pairs = 3 if t <= 256 else 2
        A = rng.integers(0, 1 << 64, (pairs, t), dtype=np.uint64)
        B = rng.integers(0, 1 << 64, (pairs, t), dtype=np.uint64)
        if t >= 4:  # sparse / extreme rows
            A[0, :] = 0
            A[0, t - 1] = 1 << 63
            B[0, :] = np.uint64((1 << 64) - 1)
        C = np.stack([ref_full(A[i], B[i]) for i in range(pairs)])
        out[f"full_t{t}_A"], out[f"full_t{t}_B"], out[f"full_t{t}_C"] = A, B, C
    out["full_ts"] = np.array(full_ts, dtype=np.int64)

    # cyclic products: the bench generator's rows at the config sizes plus
    # small/edge n (word-aligned, one-bit top word, ...)
    cyc_ns = [1, 2, 63, 64, 65, 127, 128, 129, 1000, 4097, 12323, 17669, 35851, 57637]
    for n in cyc_ns:
        pairs = 4 if n >= 12323 else 6
        A, B = make_cyclic_inputs(n, pairs)
        t = A.shape[1]
        if t >= 2:
            # X^(n-1) * X = 1 and A * 1 = A
            A[0, :] = 0
            A[0, (n - 1) // 64] = np.uint64(1 << ((n - 1) % 64))
            B[0, :] = 0
            B[0, 0] = 2
            B[1, :] = 0
            B[1, 0] = 1
        C = np.stack([ref_cyclic(A[i], B[i], n) for i in range(pairs)])
        out[f"cyc_n{n}_A"], out[f"cyc_n{n}_B"], out[f"cyc_n{n}_C"] = A, B, C
    out["cyc_ns"] = np.array(cyc_ns, dtype=np.int64)

    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes; reference _HAS_GMPY2 =",
          poly._HAS_GMPY2, "backend =", poly.backend_select())


if __name__ == "__main__":
    main()
