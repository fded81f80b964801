"""Executable numpy model of the engine's Toom-3 levels (test infrastructure).

Bitsliced like the kernels: an operand is a uint32 array indexed by
coefficient, bit p = coefficient of product p of a 32-product group, so the
model checks 32 products at once.  Follows the paper's Toom-3 over GF(2)[X]
(Appendix D) with evaluation points
{0, 1, x, x+1, inf}, x = X^w, and the interpolation in the grouped-numerator
form of SURVEY.md Appendix A.2 (every division exact):

  c0 = C(0);  c4 = C(inf)
  c3 = [C(0) + C(1) + C(x) + C(x+1)] / (x^2 + x)
  c2 = [C(1) + x C(x) + (x+1) C(x+1)] / (x^2 + x) + (x^2 + x + 1) C(inf)
  c1 = C(0) + C(1) + [C(0) + (x+1) C(x) + x C(x+1)] / (x^2 + x) + (x^2 + x) C(inf)

In the bitsliced layout x = X^w is an index shift: dividing by x drops w
coefficients and dividing by x + 1 = 1 + X^w is a prefix XOR with stride w,
q[k] = u[k] ^ q[k - w].  It is NOT an oracle (it is checked against one).
"""

from __future__ import annotations

import numpy as np


def slice32(W: np.ndarray, ncoef: int) -> np.ndarray:
    """uint64[rows<=32][t] packed -> uint32[ncoef] bitsliced (zero padded)."""
    rows, t = W.shape
    out = np.zeros(ncoef, dtype=np.uint32)
    for p in range(rows):
        bits = np.unpackbits(W[p].astype("<u8").view(np.uint8), bitorder="little")
        k = min(len(bits), ncoef)
        out[:k] |= bits[:k].astype(np.uint32) << np.uint32(p)
    return out


def unslice32(c: np.ndarray, rows: int, words: int) -> np.ndarray:
    """uint32[ncoef] bitsliced -> uint64[rows][words] packed."""
    out = np.zeros((rows, words), dtype=np.uint64)
    n = min(len(c), 64 * words)
    for p in range(rows):
        bits = ((c[:n] >> np.uint32(p)) & np.uint32(1)).astype(np.uint8)
        bits = np.concatenate([bits, np.zeros(64 * words - n, dtype=np.uint8)])
        out[p] = np.packbits(bits, bitorder="little").view("<u8")
    return out


def bs_mul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Bitsliced schoolbook: c[i+j] ^= a[i] & b[j]; length len(a)+len(b)."""
    c = np.zeros(len(a) + len(b), dtype=np.uint32)
    for i in range(len(a)):
        c[i:i + len(b)] ^= a[i] & b
    return c


def shift(u: np.ndarray, s: int, n: int) -> np.ndarray:
    """(X^s * u) truncated/padded to n coefficients (s may be negative: / X^-s)."""
    out = np.zeros(n, dtype=np.uint32)
    if s >= 0:
        m = max(0, min(len(u), n - s))
        out[s:s + m] = u[:m]
    else:
        m = max(0, min(len(u) + s, n))
        out[:m] = u[-s:-s + m]
    return out


def toom_eval(a: np.ndarray, M: int, w: int, S: int) -> list[np.ndarray]:
    """Operand of 3M coefficients -> its values at 0, 1, x, x+1, inf (x = X^w),
    each zero-padded to S >= M + 2w coefficients."""
    a0, a1, a2 = (shift(a[i * M:(i + 1) * M], 0, S) for i in range(3))
    x1, x2 = shift(a1, w, S), shift(a2, 2 * w, S)
    p1 = a0 ^ a1 ^ a2
    return [a0, p1, a0 ^ x1 ^ x2, p1 ^ x1 ^ x2, a2]


def div_x2_plus_x(n: np.ndarray, w: int) -> np.ndarray:
    """Exact n / (X^2w + X^w): drop w coefficients, then the prefix XOR of
    stride w.  Asserts exactness (the low w coefficients and the carry out of
    the top w)."""
    assert not n[:w].any(), "numerator not divisible by x"
    u = n[w:].copy()
    q = u.copy()
    for k in range(w, len(q)):
        q[k] ^= q[k - w]
    assert not q[len(q) - w:].any(), "numerator not divisible by x + 1"
    return q


def toom_interp(C: list[np.ndarray], M: int, w: int) -> np.ndarray:
    """Products at 0, 1, x, x+1, inf -> the 6M-coefficient product."""
    L = 2 * M                         # c_i have 2M - 1 coefficients
    n = max(len(c) for c in C) + 2 * w
    C0, C1, Cx, Cx1, Ci = (shift(c, 0, n) for c in C)
    X = lambda v, s: shift(v, s, n)   # noqa: E731  multiply by X^s
    c3 = div_x2_plus_x(C0 ^ C1 ^ Cx ^ Cx1, w)
    c2 = div_x2_plus_x(C1 ^ X(Cx, w) ^ Cx1 ^ X(Cx1, w), w) ^ (Ci ^ X(Ci, w) ^ X(Ci, 2 * w))[:n - w]
    c1 = (C0 ^ C1)[:n - w] ^ div_x2_plus_x(C0 ^ Cx ^ X(Cx, w) ^ X(Cx1, w), w) ^ (X(Ci, w) ^ X(Ci, 2 * w))[:n - w]
    for c in (c1, c2, c3):
        assert not c[L:].any()
    c1, c2, c3 = c1[:L], c2[:L], c3[:L]
    R = np.zeros(6 * M, dtype=np.uint32)
    for i, ci in enumerate((C0[:L], c1, c2, c3, Ci[:L])):
        R[i * M:i * M + L] ^= ci
    return R


def toom_mul(a: np.ndarray, b: np.ndarray, levels: list[tuple[int, int, int]]) -> np.ndarray:
    """Product of two operands of 3*M0 coefficients through len(levels) Toom-3
    levels (M, w, S) per level, schoolbook below."""
    if not levels:
        return bs_mul(a, b)
    (M, w, S), rest = levels[0], levels[1:]
    A, B = toom_eval(a, M, w, S), toom_eval(b, M, w, S)
    return toom_interp([toom_mul(x, y, rest) for x, y in zip(A, B)], M, w)
