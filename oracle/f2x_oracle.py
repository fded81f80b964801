"""CPU ORACLE — test infrastructure only, never the product path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module, and only as the checker or
as the timed CPU baseline.  The GPU engine (``paper_2201_10473_b200``) never
imports it and has no CPU fallback.

This is a numpy / Python-int restatement of the reference's dense F2[X]
multiply path (``f2xmul.poly`` in /root/reference/pkg/src/f2xmul/poly.py) plus
the cyclic fold that the reference's SPEC defines but does not ship
(SPEC.md:345-353, 367-370).  Parity is PINNED: ``tests/test_oracle.py`` checks
this module against golden vectors produced by importing the real reference
(``tests/golden/make_golden.py``) and against the reference's own
known-answer tests (test_poly.py:134-143, 219-225).

Layout contract (poly.py:4-8): a polynomial is a little-endian array of uint64
words; bit i of word j is the coefficient of X^(64 j + i).  Batched operands
are row-major ``uint64[batch][t]``.
"""

from __future__ import annotations

import numpy as np

__all__ = [
    "clmul64_shift_xor",
    "clmul64_int_mul",
    "clmul64_lanes",
    "mul_convolution",
    "mul_spread",
    "mul_full_row",
    "mul_full",
    "fold_cyclic",
    "mul_cyclic",
    "cyclic_words",
    "make_full_inputs",
    "make_cyclic_inputs",
    "to_hex",
    "from_hex",
]

_MASK64 = (1 << 64) - 1


# ---------------------------------------------------------------- base case

def clmul64_shift_xor(a: int, b: int) -> int:
    """Fixed 64-step masked shift-and-XOR, 128-bit result (poly.py:261-266)."""
    p = 0
    for k in range(64):
        p ^= (a << k) & -((b >> k) & 1)
    return p


_C0, _C1, _C2, _C3 = (0x1111111111111111, 0x2222222222222222,
                      0x4444444444444444, 0x8888888888888888)


def _k32(x: int, y: int) -> int:
    """32x32 carry-less product from integer multiplies over 4-bit-spaced bit
    classes; column sums stay < 16 so each kept bit is the column parity
    (poly.py:275-291)."""
    xs = (x & _C0, x & _C1, x & _C2, x & _C3)
    ys = (y & _C0, y & _C1, y & _C2, y & _C3)
    out = 0
    masks = (_C0, _C1, _C2, _C3)
    for r in range(4):
        z = 0
        for i in range(4):
            z ^= xs[i] * ys[(r - i) % 4]
        out |= z & masks[r]
    return out


def clmul64_int_mul(a: int, b: int) -> int:
    """One Karatsuba step over 32-bit halves of ``_k32`` (poly.py:294-302)."""
    al, ah = a & 0xFFFFFFFF, a >> 32
    bl, bh = b & 0xFFFFFFFF, b >> 32
    pll = _k32(al, bl)
    phh = _k32(ah, bh)
    pm = _k32(al ^ ah, bl ^ bh) ^ pll ^ phh
    return pll ^ (pm << 32) ^ (phh << 64)


_U = {k: np.uint64(k) for k in range(65)}
_NM = [np.uint64(m) for m in (_C0, _C1, _C2, _C3)]


def _k32_lanes(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Lane-wise ``_k32`` on uint64 arrays holding 32-bit values
    (poly.py:422-435).  Products of two 32-bit values fit in 64 bits."""
    xs = [x & m for m in _NM]
    ys = [y & m for m in _NM]
    out = np.zeros_like(x)
    for r in range(4):
        z = np.zeros_like(x)
        for i in range(4):
            z ^= xs[i] * ys[(r - i) % 4]
        out |= z & _NM[r]
    return out


def clmul64_lanes(a: np.ndarray, b: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Lane-wise 64x64->128 carry-less product, (lo, hi) (poly.py:438-448)."""
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    if a.shape != b.shape:
        raise ValueError("lane arrays must have equal shapes")
    l32 = np.uint64(0xFFFFFFFF)
    al, ah = a & l32, a >> _U[32]
    bl, bh = b & l32, b >> _U[32]
    pll = _k32_lanes(al, bl)
    phh = _k32_lanes(ah, bh)
    pm = _k32_lanes(al ^ ah, bl ^ bh) ^ pll ^ phh
    lo = pll ^ (pm << _U[32])
    hi = phh ^ (pm >> _U[32])
    return lo, hi


# ------------------------------------------------------------- full product

def mul_convolution(aw: np.ndarray, bw: np.ndarray) -> np.ndarray:
    """Word-level schoolbook: t^2 lane products, skewed XOR-reduction of the
    lo words at i+j and hi words at i+j+1 (poly.py:493-514)."""
    aw = np.asarray(aw, dtype=np.uint64)
    bw = np.asarray(bw, dtype=np.uint64)
    t = aw.shape[0]
    lo, hi = clmul64_lanes(np.repeat(aw, t), np.tile(bw, t))
    lo = lo.reshape(t, t)
    hi = hi.reshape(t, t)
    out = np.zeros(2 * t, dtype=np.uint64)
    for i in range(t):
        out[i:i + t] ^= lo[i]
        out[i + 1:i + t + 1] ^= hi[i]
    return out


def mul_spread(aw: np.ndarray, bw: np.ndarray) -> np.ndarray:
    """Bit-spread evaluation route (the reference's default for t > 48,
    poly.py:517-544): every coefficient becomes a k-byte column of one big
    integer, one integer multiply, bit 0 of each column is the F2 coefficient.
    k = 2 while 64t < 2^16, else 3 (poly.py:533); limit 64t < 2^24."""
    aw = np.ascontiguousarray(aw, dtype=np.uint64)
    bw = np.ascontiguousarray(bw, dtype=np.uint64)
    t = aw.shape[0]
    if 64 * t >= 1 << 24:
        raise ValueError("operand too large for the spread evaluation route")
    k = 2 if 64 * t < (1 << 16) else 3

    def spread(w: np.ndarray) -> int:
        bits = np.unpackbits(w.view(np.uint8), bitorder="little")
        cols = np.zeros((bits.shape[0], k), dtype=np.uint8)
        cols[:, 0] = bits
        return int.from_bytes(cols.tobytes(), "little")

    p = spread(aw) * spread(bw)
    raw = np.frombuffer(p.to_bytes(128 * t * k, "little"), dtype=np.uint8)[::k]
    packed = np.packbits(raw & 1, bitorder="little")
    return np.frombuffer(packed.tobytes(), dtype=np.uint64).copy()


SPREAD_CUTOFF_WORDS = 48  # poly.py:490


def mul_full_row(aw: np.ndarray, bw: np.ndarray) -> np.ndarray:
    """``schoolbook_mul`` value for one pair with the reference's route choice
    (poly.py:547-561): equal lengths required, 2t-word product."""
    aw = np.asarray(aw, dtype=np.uint64)
    bw = np.asarray(bw, dtype=np.uint64)
    if aw.ndim != 1 or aw.shape != bw.shape or aw.shape[0] < 1:
        raise ValueError("schoolbook needs two equal-length 1-D operands, t >= 1")
    if aw.shape[0] > SPREAD_CUTOFF_WORDS:
        return mul_spread(aw, bw)
    return mul_convolution(aw, bw)


def mul_full(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Row-wise full products: uint64[batch][t] x2 -> uint64[batch][2t]."""
    A = np.asarray(A, dtype=np.uint64)
    B = np.asarray(B, dtype=np.uint64)
    if A.ndim != 2 or A.shape != B.shape:
        raise ValueError("A and B must be equal-shape uint64[batch][t]")
    out = np.zeros((A.shape[0], 2 * A.shape[1]), dtype=np.uint64)
    for r in range(A.shape[0]):
        out[r] = mul_full_row(A[r], B[r])
    return out


# ----------------------------------------------------------- cyclic product

def cyclic_words(n: int) -> int:
    return (n + 63) // 64


def _to_int(w: np.ndarray) -> int:
    return int.from_bytes(np.ascontiguousarray(w, dtype=np.uint64).tobytes(), "little")


def _from_int(v: int, words: int) -> np.ndarray:
    return np.frombuffer(v.to_bytes(8 * words, "little"), dtype=np.uint64).copy()


def fold_cyclic(P: np.ndarray, n: int) -> np.ndarray:
    """One fold mod X^n - 1: R = (P mod X^n) xor (P div X^n).
    deg P <= 2n-2 so one fold suffices; output has ceil(n/64) words with the
    bits >= n zero."""
    n = int(n)
    v = _to_int(P)
    r = (v & ((1 << n) - 1)) ^ (v >> n)
    if r >> n:
        raise ValueError("product degree exceeds 2n-2; inputs were not reduced")
    return _from_int(r, cyclic_words(n))


def _check_top_bits(W: np.ndarray, n: int) -> None:
    t = cyclic_words(n)
    if W.shape[-1] != t:
        raise ValueError(f"ring operands need {t} words for n={n}, got {W.shape[-1]}")
    r = n - 64 * (t - 1)
    if r < 64 and np.any(W[..., t - 1] >> _U[r]):
        # reject, never mask
        raise ValueError("operand has bits set at or above n")


def mul_cyclic(A: np.ndarray, B: np.ndarray, n: int) -> np.ndarray:
    """Row-wise ring products mod X^n - 1 through the reference's full product
    and the SPEC fold."""
    n = int(n)
    A = np.asarray(A, dtype=np.uint64)
    B = np.asarray(B, dtype=np.uint64)
    if A.ndim != 2 or A.shape != B.shape:
        raise ValueError("A and B must be equal-shape uint64[batch][t]")
    _check_top_bits(A, n)
    _check_top_bits(B, n)
    out = np.zeros_like(A)
    for r in range(A.shape[0]):
        out[r] = fold_cyclic(mul_full_row(A[r], B[r]), n)
    return out


# ------------------------------------------------------------ seeded inputs

def make_full_inputs(d_or_t: int, batch: int, *, words: bool = False,
                     seed_base: int = 0xF2F2) -> tuple[np.ndarray, np.ndarray]:
    """rng = default_rng([0xF2F2, d]); A then B drawn with
    ``integers(0, 1<<64, (batch, t), dtype=uint64)`` (conftest.py:40-41, 46).
    ``d_or_t`` is the bit size d unless ``words`` is set."""
    t = d_or_t if words else d_or_t // 64
    key = 64 * t if words else d_or_t
    rng = np.random.default_rng([seed_base, key])
    A = rng.integers(0, 1 << 64, size=(batch, t), dtype=np.uint64)
    B = rng.integers(0, 1 << 64, size=(batch, t), dtype=np.uint64)
    return A, B


def make_cyclic_inputs(n: int, batch: int, *, seed_base: int = 0xF2F2
                       ) -> tuple[np.ndarray, np.ndarray]:
    """Same generator keyed on n, top word masked to n - 64(t-1) bits."""
    t = cyclic_words(n)
    rng = np.random.default_rng([seed_base, n])
    A = rng.integers(0, 1 << 64, size=(batch, t), dtype=np.uint64)
    B = rng.integers(0, 1 << 64, size=(batch, t), dtype=np.uint64)
    r = n - 64 * (t - 1)
    if r < 64:
        m = np.uint64((1 << r) - 1)
        A[:, t - 1] &= m
        B[:, t - 1] &= m
    return A, B


# -------------------------------------------------------------- hex format

def to_hex(words: np.ndarray) -> str:
    """Lowercase hex, most-significant word first, 16 digits/word (poly.py:569-571)."""
    return "".join(f"{int(w):016x}" for w in np.asarray(words)[::-1])


def from_hex(s: str) -> np.ndarray:
    """Exact inverse of ``to_hex`` (poly.py:574-584)."""
    s = s.strip()
    if not s or len(s) % 16:
        raise ValueError("hex length must be a positive multiple of 16")
    try:
        vals = [int(s[i:i + 16], 16) for i in range(0, len(s), 16)]
    except ValueError:
        raise ValueError(f"invalid hex polynomial: {s[:32]}...") from None
    if s != "".join(f"{v:016x}" for v in vals):
        raise ValueError("hex polynomials must be lowercase, fixed width")
    return np.array(vals[::-1], dtype=np.uint64)
