"""Executable numpy model of the GPU algorithm (test infrastructure).

Mirrors the index arithmetic of paper_2201_10473_b200/csrc kernels one to one
so that the plan / layout logic can be checked on a CPU box against the
oracle.  It is NOT an oracle (it is checked against one) and never runs on the
product path.

Stages:
  k1  packed uint64[batch][t] -> bitsliced, chunked uint32[G][Ns]
  k2  per (group, path): XOR-load of the path's operand segments, in-CTA
      breadth-first Karatsuba (appended-mid layout), leaf schoolbook, in-place
      interpolation -> node product
  k3  global interpolation passes (elementwise over the quarter index)
  k4  fold mod X^n-1 (cyclic) + transpose back to packed uint64
"""

from __future__ import annotations

import os

import numpy as np


def pow3(k: int) -> int:
    return 3 ** k


def transpose32(x: np.ndarray) -> np.ndarray:
    """x: uint32[32, ...] -> y with bit p of y[i] = bit i of x[p]."""
    x = x.astype(np.uint32).copy()
    j, m = 16, np.uint32(0x0000FFFF)
    while j:
        for k in range(32):
            if k & j == 0:
                t = ((x[k] >> np.uint32(j)) ^ x[k + j]) & m
                x[k + j] ^= t
                x[k] ^= (t << np.uint32(j)).astype(np.uint32)
        j //= 2
        if j:
            m = m ^ np.uint32((int(m) << j) & 0xFFFFFFFF)
    return x


class Plan:
    def __init__(self, LF: int, K: int, KC: int, *, kind: str, t: int, n: int, batch: int):
        self.LF, self.K, self.KC = LF, K, KC
        self.GL = K - KC
        q = (LF + 3) // 4
        self.LFS = 4 * (q if q % 2 else q + 1)  # odd number of quads per chunk
        self.N = LF << K            # logical coefficients per operand
        self.Ns = self.LFS << K     # storage words per operand per group
        self.S = LF << KC
        self.Ss = self.LFS << KC
        self.kind, self.t, self.n, self.batch = kind, t, n, batch
        self.G = (batch + 31) // 32
        assert self.N >= 64 * t

    def idx(self, k):
        return (k // self.LF) * self.LFS + k % self.LF


def k1(plan: Plan, X: np.ndarray) -> np.ndarray:
    G, t = plan.G, plan.t
    out = np.zeros((G, plan.Ns), dtype=np.uint32)
    Xp = np.zeros((G * 32, t), dtype=np.uint64)
    Xp[: X.shape[0]] = X
    lo = (Xp & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    hi = (Xp >> np.uint64(32)).astype(np.uint32)
    for g in range(G):
        for u in range((plan.N + 63) // 64):
            if u < t:
                ylo = transpose32(lo[32 * g: 32 * g + 32, u])
                yhi = transpose32(hi[32 * g: 32 * g + 32, u])
                words = np.concatenate([ylo, yhi])
            else:
                words = np.zeros(64, dtype=np.uint32)
            for i in range(64):
                k = 64 * u + i
                if k < plan.N:
                    out[g, plan.idx(k)] = words[i]
    return out


def leaf_positions(plan: Plan):
    """P_j(nu) in words for j = 0..KC; R_j = LFS * 2^(KC-j) * 3^j."""
    KC, LFS = plan.KC, plan.LFS
    P = [[0]]
    for j in range(1, KC + 1):
        hq = LFS << (KC - j)          # half of a level-(j-1) node
        R = LFS * (2 ** (KC - j + 1)) * pow3(j - 1)
        cur = []
        for nu in range(pow3(j)):
            par, d = divmod(nu, 3)
            p = P[j - 1][par]
            cur.append(p if d == 0 else p + hq if d == 1 else R + par * hq)
        P.append(cur)
    return P


def path_segments(plan: Plan, path: int):
    """Chunk offsets of the segments XORed into the path's operand."""
    GL, K = plan.GL, plan.K
    digits = []
    for _ in range(GL):
        path, d = divmod(path, 3)
        digits.append(d)
    digits = digits[::-1]  # most significant = top level
    base, mids = 0, []
    for j, d in enumerate(digits, start=1):
        hc = 1 << (K - j)
        if d == 1:
            base += hc
        elif d == 2:
            mids.append(hc)
    offs = []
    for mask in range(1 << len(mids)):
        o = base + sum(m for b, m in enumerate(mids) if mask >> b & 1)
        offs.append(o)
    return offs


def k2(plan: Plan, Abs: np.ndarray, Bbs: np.ndarray) -> np.ndarray:
    LF, LFS, KC, GL, Ss = plan.LF, plan.LFS, plan.KC, plan.GL, plan.Ss
    R = LFS * pow3(KC)  # region words
    P = leaf_positions(plan)
    out = np.zeros((plan.G, pow3(GL), 2 * Ss), dtype=np.uint32)
    for g in range(plan.G):
        for path in range(pow3(GL)):
            As = np.zeros(R, dtype=np.uint32)
            Bs = np.zeros(R, dtype=np.uint32)
            for o in path_segments(plan, path):
                As[:Ss] ^= Abs[g, o * LFS: o * LFS + Ss]
                Bs[:Ss] ^= Bbs[g, o * LFS: o * LFS + Ss]
            # eval
            for j in range(KC):
                h = LFS << (KC - j - 1)
                Rj = LFS * (2 ** (KC - j)) * pow3(j)
                for it in range(pow3(j) * h):
                    nu, u = divmod(it, h)
                    s = P[j][nu]
                    As[Rj + it] = As[s + u] ^ As[s + h + u]
                    Bs[Rj + it] = Bs[s + u] ^ Bs[s + h + u]
            # leaves
            for leaf in range(pow3(KC)):
                p = P[KC][leaf]
                a = As[p: p + LF].astype(np.uint32)
                b = Bs[p: p + LF].astype(np.uint32)
                c = np.zeros(2 * LF, dtype=np.uint32)
                for i in range(LF):
                    c[i: i + LF] ^= a[i] & b
                As[p: p + LFS] = 0
                Bs[p: p + LFS] = 0
                As[p: p + LF] = c[:LF]
                Bs[p: p + LF] = c[LF:]
            # interp
            for j in range(KC - 1, -1, -1):
                h = LFS << (KC - j - 1)
                Rj = LFS * (2 ** (KC - j)) * pow3(j)
                for it in range(pow3(j) * h):
                    nu, u = divmod(it, h)
                    s = P[j][nu]
                    L0, H0 = As[s + u], Bs[s + u]
                    L1, H1 = As[s + h + u], Bs[s + h + u]
                    Ml, Mh = As[Rj + it], Bs[Rj + it]
                    T = H0 ^ L1
                    As[s + h + u] = T ^ L0 ^ Ml
                    Bs[s + u] = T ^ H1 ^ Mh
            out[g, path, :Ss] = As[:Ss]
            out[g, path, Ss:] = Bs[:Ss]
    return out


def k3_pass(plan: Plan, Pin: np.ndarray, d_hi: int, glp: int) -> np.ndarray:
    d_lo = d_hi - glp
    S_hi = plan.Ns >> d_hi
    qw = S_hi // 2
    G = plan.G

    def rec(D, desc, g, w):
        if D == 0:
            return [Pin[g, desc, q * qw + w] for q in range(4)]
        out = rec(D - 1, desc * 3 + 0, g, w) + rec(D - 1, desc * 3 + 1, g, w)
        m = rec(D - 1, desc * 3 + 2, g, w)
        Lc = 2 << D
        half = Lc // 2
        for i in range(half):
            T = out[half + i] ^ out[Lc + i]
            out[half + i] = T ^ out[i] ^ m[i]
            out[Lc + i] = T ^ out[Lc + half + i] ^ m[half + i]
        return out

    Pout = np.zeros((G, pow3(d_lo), 2 * (plan.Ns >> d_lo)), dtype=np.uint32)
    for g in range(G):
        for nu in range(pow3(d_lo)):
            for w in range(qw):
                v = rec(glp, nu, g, w)
                for m_, val in enumerate(v):
                    Pout[g, nu, m_ * qw + w] = val
    return Pout


def k4(plan: Plan, C: np.ndarray) -> np.ndarray:
    """C: uint32[G][2Ns] root product (chunked)."""
    t, n, batch = plan.t, plan.n, plan.batch
    tout = 2 * t if plan.kind == "full" else t
    out = np.zeros((batch, tout), dtype=np.uint64)
    for g in range(plan.G):
        for u in range(tout):
            words = np.zeros(64, dtype=np.uint32)
            for i in range(64):
                k = 64 * u + i
                if plan.kind == "full":
                    words[i] = C[g, plan.idx(k)]
                elif k < n:
                    words[i] = C[g, plan.idx(k)] ^ C[g, plan.idx(k + n)]
            lo = transpose32(words[:32])
            hi = transpose32(words[32:])
            for p in range(32):
                if 32 * g + p < batch:
                    out[32 * g + p, u] = np.uint64(lo[p]) | (np.uint64(hi[p]) << np.uint64(32))
    return out


def split_passes(GL: int, maxp: int = 4):
    passes = []
    rem = GL
    while rem > 0:
        p = min(maxp, rem)
        passes.append(p)
        rem -= p
    return passes  # bottom first


def run(plan: Plan, A: np.ndarray, B: np.ndarray) -> np.ndarray:
    Abs = k1(plan, A)
    Bbs = k1(plan, B)
    P = k2(plan, Abs, Bbs)
    d = plan.GL
    for glp in split_passes(plan.GL):
        P = k3_pass(plan, P, d, glp)
        d -= glp
    return k4(plan, P[:, 0, :])


# ---------------------------------------------------------------------------
# v2 node schedule (mirrors the current kernel): eval levels 0..KC-2 in merged
# pairs (4 loads -> 5 stores per quarter index), the bottom eval level fused
# into the leaves (a mid leaf XORs its parent's two chunks while loading),
# interpolation in merged pairs from the bottom, in place.

def eval_pair(As, Bs, P, LFS, KC, j):
    """Levels j and j+1 at once for every level-j node (needs j+1 <= KC-1)."""
    q = LFS << (KC - j - 2)                     # quarter of a level-j node
    Rj = LFS * (2 ** (KC - j)) * pow3(j)
    Rj1 = LFS * (2 ** (KC - j - 1)) * pow3(j + 1)
    for nu in range(pow3(j)):
        p = P[j][nu]
        for X in (As, Bs):
            x0 = X[p: p + q].copy(); x1 = X[p + q: p + 2 * q].copy()
            x2 = X[p + 2 * q: p + 3 * q].copy(); x3 = X[p + 3 * q: p + 4 * q].copy()
            m0, m1 = x0 ^ x2, x1 ^ x3
            X[Rj + nu * 2 * q: Rj + nu * 2 * q + q] = m0
            X[Rj + nu * 2 * q + q: Rj + nu * 2 * q + 2 * q] = m1
            X[Rj1 + (3 * nu) * q: Rj1 + (3 * nu + 1) * q] = x0 ^ x1
            X[Rj1 + (3 * nu + 1) * q: Rj1 + (3 * nu + 2) * q] = x2 ^ x3
            X[Rj1 + (3 * nu + 2) * q: Rj1 + (3 * nu + 3) * q] = m0 ^ m1


def eval_single(As, Bs, P, LFS, KC, j):
    h = LFS << (KC - j - 1)
    Rj = LFS * (2 ** (KC - j)) * pow3(j)
    for nu in range(pow3(j)):
        s = P[j][nu]
        for X in (As, Bs):
            X[Rj + nu * h: Rj + (nu + 1) * h] = X[s: s + h] ^ X[s + h: s + 2 * h]


def interp_single(As, Bs, P, LFS, KC, j):
    h = LFS << (KC - j - 1)
    Rj = LFS * (2 ** (KC - j)) * pow3(j)
    for nu in range(pow3(j)):
        s = P[j][nu]
        L0, H0 = As[s: s + h].copy(), Bs[s: s + h].copy()
        L1, H1 = As[s + h: s + 2 * h].copy(), Bs[s + h: s + 2 * h].copy()
        Ml, Mh = As[Rj + nu * h: Rj + (nu + 1) * h].copy(), Bs[Rj + nu * h: Rj + (nu + 1) * h].copy()
        T = H0 ^ L1
        As[s + h: s + 2 * h] = T ^ L0 ^ Ml
        Bs[s: s + h] = T ^ H1 ^ Mh


def interp_pair(As, Bs, P, LFS, KC, j):
    """Levels j+1 and j at once for every level-j node (j+1 <= KC-1), per
    quarter index w: 18 reads (grandchildren halves), 6 writes, in place."""
    q = LFS << (KC - j - 2)
    for nu in range(pow3(j)):
        kids = [3 * nu, 3 * nu + 1, 3 * nu + 2]
        Qs = []
        for kappa in kids:
            pk = P[j + 1][kappa]
            g0, g1, g2 = P[j + 2][3 * kappa], P[j + 2][3 * kappa + 1], P[j + 2][3 * kappa + 2]
            L0, H0 = As[g0: g0 + q].copy(), Bs[g0: g0 + q].copy()
            L1, H1 = As[g1: g1 + q].copy(), Bs[g1: g1 + q].copy()
            Ml, Mh = As[g2: g2 + q].copy(), Bs[g2: g2 + q].copy()
            T = H0 ^ L1
            Qs.append((L0, T ^ L0 ^ Ml, T ^ H1 ^ Mh, H1, pk))
        (c0q0, c0q1, c0q2, c0q3, p0), (c1q0, c1q1, c1q2, c1q3, p1), (c2q0, c2q1, c2q2, c2q3, _) = Qs
        T0 = c0q2 ^ c1q0
        T1 = c0q3 ^ c1q1
        As[p0 + q: p0 + 2 * q] = c0q1
        As[p1: p1 + q] = T0 ^ c0q0 ^ c2q0
        As[p1 + q: p1 + 2 * q] = T1 ^ c0q1 ^ c2q1
        Bs[p0: p0 + q] = T0 ^ c1q2 ^ c2q2
        Bs[p0 + q: p0 + 2 * q] = T1 ^ c1q3 ^ c2q3
        Bs[p1: p1 + q] = c1q2


def mid_perm(KC: int):
    """The kernels' mid-leaf assignment (gen_instances.py MID_PERM, KC = 5):
    chunk Rm + i holds the mid leaf of level-(KC-1) node perm[i]."""
    if KC != 5:
        return list(range(pow3(KC - 1))) if KC >= 1 else []
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "gen", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "paper_2201_10473_b200", "csrc", "gen_instances.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    return list(gen.MID_PERM)


def k2_v2(plan: Plan, Abs: np.ndarray, Bbs: np.ndarray) -> np.ndarray:
    LF, LFS, KC, GL, Ss = plan.LF, plan.LFS, plan.KC, plan.GL, plan.Ss
    R = LFS * pow3(KC)
    P = leaf_positions(plan)
    sigma = mid_perm(KC)
    if KC >= 1:  # mid leaf of node kappa is stored at chunk Rm + sigma^-1(kappa)
        Rm_w = R - pow3(KC - 1) * LFS
        for i, kappa in enumerate(sigma):
            P[KC][3 * kappa + 2] = Rm_w + i * LFS
    out = np.zeros((plan.G, pow3(GL), 2 * Ss), dtype=np.uint32)
    for g in range(plan.G):
        for path in range(pow3(GL)):
            As = np.zeros(R, dtype=np.uint32)
            Bs = np.zeros(R, dtype=np.uint32)
            for o in path_segments(plan, path):
                As[:Ss] ^= Abs[g, o * LFS: o * LFS + Ss]
                Bs[:Ss] ^= Bbs[g, o * LFS: o * LFS + Ss]
            n_ev = KC - 1                       # levels evaluated in smem
            j = 0
            while j + 1 < n_ev:
                eval_pair(As, Bs, P, LFS, KC, j)
                j += 2
            if j < n_ev:
                eval_single(As, Bs, P, LFS, KC, j)
            # leaves, one per chunk; a mid leaf (chunk >= R_{KC-1}) XORs its
            # parent's two chunks (bottom eval level fused)
            Rm = (R // LFS) - pow3(KC - 1) if KC >= 1 else R // LFS
            prods = {}
            for ch in range(R // LFS):
                if KC >= 1 and ch >= Rm:
                    pp = P[KC - 1][sigma[ch - Rm]]
                    a = As[pp: pp + LF] ^ As[pp + LFS: pp + LFS + LF]
                    b = Bs[pp: pp + LF] ^ Bs[pp + LFS: pp + LFS + LF]
                else:
                    a = As[ch * LFS: ch * LFS + LF].copy()
                    b = Bs[ch * LFS: ch * LFS + LF].copy()
                c = np.zeros(2 * LF, dtype=np.uint32)
                for i in range(LF):
                    c[i: i + LF] ^= a[i] & b
                prods[ch] = c
            for ch, c in prods.items():   # written after all reads (barrier)
                As[ch * LFS: (ch + 1) * LFS] = 0
                Bs[ch * LFS: (ch + 1) * LFS] = 0
                As[ch * LFS: ch * LFS + LF] = c[:LF]
                Bs[ch * LFS: ch * LFS + LF] = c[LF:]
            j = KC - 2
            while j >= 0:
                interp_pair(As, Bs, P, LFS, KC, j)
                j -= 2
            if j == -1:
                interp_single(As, Bs, P, LFS, KC, 0)
            out[g, path, :Ss] = As[:Ss]
            out[g, path, Ss:] = Bs[:Ss]
    return out


def run_v2(plan: Plan, A: np.ndarray, B: np.ndarray) -> np.ndarray:
    P = k2_v2(plan, k1(plan, A), k1(plan, B))
    d = plan.GL
    for glp in split_passes(plan.GL):
        P = k3_pass(plan, P, d, glp)
        d -= glp
    return k4(plan, P[:, 0, :])


def k1_eval(plan: Plan, X: np.ndarray, el: int) -> np.ndarray:
    """k1_slice_eval: the top ``el`` global levels pre-evaluated -> 3^el
    sub-operands per group (digits lo, hi, mid; top level most significant)."""
    Xs = k1(plan, X)                                   # [G][Ns]
    subs = [Xs]
    for _ in range(el):
        nxt = []
        for s in subs:
            h = s.shape[1] // 2
            lo, hi = s[:, :h], s[:, h:]
            nxt += [lo, hi, lo ^ hi]
        subs = nxt
    return np.stack(subs, axis=1).reshape(plan.G * pow3(el), -1)


def run_v3(plan: Plan, A: np.ndarray, B: np.ndarray, el: int) -> np.ndarray:
    """run_v2 with the slicing kernel's pre-evaluation of ``el`` levels: the
    node kernel sees 3^el x the groups with K - el levels; node numbering,
    interpolation and unslicing are unchanged."""
    import copy

    sub = copy.copy(plan)
    sub.K, sub.GL, sub.Ns, sub.G = plan.K - el, plan.GL - el, plan.Ns >> el, plan.G * pow3(el)
    P = k2_v2(sub, k1_eval(plan, A, el), k1_eval(plan, B, el))
    P = P.reshape(plan.G, pow3(plan.GL), -1)
    d = plan.GL
    for glp in split_passes(plan.GL):
        P = k3_pass(plan, P, d, glp)
        d -= glp
    return k4(plan, P[:, 0, :])
