// Device code of the bitsliced GF(2)[X] engine (sm_100a).
//
// Data layout: products are processed in GROUPS of 32;
// a group's operand is BITSLICED -- uint32 word k holds coefficient k of the
// 32 products (bit p = product 32g+p).  Coefficients are stored in CHUNKS of
// LF (the leaf size) at a stride of LFS = 4*Q words, Q = ceil(LF/4) rounded
// up to an ODD number of 16-byte quads: every Karatsuba half, leaf and
// quarter is a whole number of quads, and 8 threads touching quad q of 8
// consecutive chunks hit 8 different bank groups (Q odd => Q*t mod 8
// distinct), so the leaf loads/stores are bank-conflict free.
//
// A bitsliced AND+XOR (one LOP3) performs 32 coefficient products, i.e. a
// 32x32 leaf costs exactly the 64*64/32 = 128 lane-ops per 64x64 block that
// the W_alg roofline charges; the Karatsuba additions are
// plain word XORs with no bit shifting, and the fold mod X^n-1 is pure index
// arithmetic.  No branch or address depends on operand bits.
#pragma once

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "f2x_postab.cuh"

namespace f2x {

__host__ __device__ constexpr int pow3c(int k) { return k <= 0 ? 1 : 3 * pow3c(k - 1); }

// Programmatic dependent launch (F2X_PDL=1: every kernel of a call is launched
// with programmatic stream serialisation, see launch_pdl): a kernel lets its
// successor's CTAs launch once all of its own CTAs are running, and waits for
// its predecessor's completion (and memory) before touching anything, so
// launch latency and wave tails overlap across the call's kernels.  Both
// instructions are no-ops for a normal launch.
__device__ __forceinline__ void pdl_prologue() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" :::);
}

// F2X_PDL=1 launches with the programmatic serialisation attribute.  Off by
// default: measured 1-2 % slower per call (n=17669 0.3375 -> 0.3412 ms,
// n=35851 0.964 -> 0.972 ms) -- the successor's early-resident CTAs only
// wait, while holding registers and shared memory during the predecessor's
// tail.
inline bool pdl_enabled() {
    static const bool v = [] {
        const char *e = getenv("F2X_PDL");
        return e && e[0] == '1';
    }();
    return v;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// chunk stride in words for leaf size LF (see the layout note above)
__host__ __device__ constexpr int leaf_stride_words(int LF) {
    return 4 * ((((LF + 3) / 4) % 2) ? (LF + 3) / 4 : (LF + 3) / 4 + 1);
}

__device__ __forceinline__ uint4 operator^(uint4 a, uint4 b) {
    return make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w);
}
__device__ __forceinline__ uint4 xor3(uint4 a, uint4 b, uint4 c) {
    return make_uint4(a.x ^ b.x ^ c.x, a.y ^ b.y ^ c.y, a.z ^ b.z ^ c.z, a.w ^ b.w ^ c.w);
}

// ------------------------------------------------------------ 32x32 transpose
// After transpose32(x): bit p of x[i] == old bit i of x[p].  Five butterfly
// stages of masked swaps (block transpose), 16 pairs each.
template <int J>
struct TMask;
template <> struct TMask<16> { static constexpr uint32_t v = 0x0000FFFFu; };
template <> struct TMask<8> { static constexpr uint32_t v = 0x00FF00FFu; };
template <> struct TMask<4> { static constexpr uint32_t v = 0x0F0F0F0Fu; };
template <> struct TMask<2> { static constexpr uint32_t v = 0x33333333u; };
template <> struct TMask<1> { static constexpr uint32_t v = 0x55555555u; };

template <int J>
__device__ __forceinline__ void tstage(uint32_t (&x)[32]) {
    constexpr uint32_t m = TMask<J>::v;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        if ((k & J) == 0) {
            const uint32_t s = ((x[k] >> J) ^ x[k + J]) & m;
            x[k + J] ^= s;
            x[k] ^= s << J;
        }
    }
}

// the 16- and 8-bit stages move whole bytes: one PRMT per output word
// (selectors checked against the shift/mask form in tests/test_model_and_plan.py)
template <int J, unsigned SX, unsigned SY>
__device__ __forceinline__ void tstage_prmt(uint32_t (&x)[32]) {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        if ((k & J) == 0) {
            const uint32_t a = x[k], c = x[k + J];
            x[k] = __byte_perm(a, c, SX);
            x[k + J] = __byte_perm(a, c, SY);
        }
    }
}

__device__ __forceinline__ void transpose32(uint32_t (&x)[32]) {
    tstage_prmt<16, 0x5410u, 0x7632u>(x);
    tstage_prmt<8, 0x6240u, 0x7351u>(x);
    tstage<4>(x);
    tstage<2>(x);
    tstage<1>(x);
}

// ----------------------------------------------------------- node kernel (K2)
// Node positions of the in-CTA Karatsuba layout, in chunks, for KC = 0..5:
// entry (3^j - 1)/2 + nu = pos_j(nu); the children of nu sit at lo = pos,
// hi = pos + half, mid = R_j + nu*half (appended).  Generated by
// gen_instances.py (f2x_postab.cuh, kPosChunks); identical to
// tests/model_bitsliced.py.
struct K2Params {
    const uint32_t *Abs;  // [G][Ns] bitsliced, chunked
    const uint32_t *Bbs;
    uint32_t *Pout;       // [G][3^GL][2 Ss]
    int64_t Ns;           // storage words per operand per group
    int K;                // total Karatsuba levels
    int GL;               // global levels (paths = 3^GL)
    int paths;
    long long *prof;      // optional per-CTA phase clocks (F2X_PHASE_PROF), [blocks][8]
    int combine;          // fuse mode: 0 node products; 1 clusters of 3 siblings write their
                          // PARENT product (Pout = [G][3^(GL-1)][4 Ss]); 2 node products, then
                          // the last sibling overwrites its triple's slots with the parent
                          // (stride 6 Ss)
    unsigned *cnt;        // fuse mode 2: per-parent arrival counters (zeroed before the launch)
};

template <int LF, int KC>
struct K2Cfg {
    static constexpr int LFS = leaf_stride_words(LF);
    static constexpr int Q = LFS / 4;                 // quads per chunk
    static constexpr int NLEAF = pow3c(KC);
    static constexpr int NT = NLEAF <= 32 ? 32 : ((NLEAF + 31) / 32) * 32;
    static constexpr int SQ = Q << KC;                // node operand, quads
    static constexpr int RQ = Q * NLEAF;              // region after KC levels
    static constexpr int NPOS = (pow3c(KC + 1) - 1) / 2;
    static constexpr size_t SMEM = size_t(2) * RQ * 16;
    static constexpr int REGS = 2 * LF + 14;  // two-pass leaf: b + half of c
    // LF <= 26: 64 registers and 28-word chunks (54 KB) -> 4 CTAs/SM
    static constexpr int MINB_REG = REGS <= 66 ? 4 : (REGS <= 90 ? 3 : 2);
    // 228 KB per SM; 1 KB reserved + ~1 KB of static tables per CTA
    static constexpr int MINB_SMEM = int((228u * 1024u) / (SMEM + 2048u));
    static constexpr int MINB = MINB_REG < MINB_SMEM ? MINB_REG : MINB_SMEM;
};

// ------------------------------------------------------------------
// Node phases.  NTH = threads executing the phase, t = index among them,
// Bar = barrier functor (the CTA barrier).

// Path digits -> (base chunk offset, bitmask of mid half-sizes); every
// thread computes them, so segment offsets need no shared table.
__device__ __forceinline__ void path_base_mids(const K2Params &p, int path, uint32_t &base,
                                               uint32_t &mids) {
    base = 0;
    mids = 0;
    int rem = path;
    for (int j = p.GL; j >= 1; --j) {
        const int d = rem % 3;
        rem /= 3;
        const uint32_t hc = 1u << (p.K - j);
        base += d == 1 ? hc : 0u;
        mids |= d == 2 ? hc : 0u;
    }
}

// node operand = XOR of the path's 2^popc(mids) segments, enumerated with
// the subset walk sub -> (sub - mids) & mids; all of a thread's items advance
// together, 2 segments per step (ITEMS x 2 x 2 16-byte loads in flight).
template <int LF, int KC, int NTH>
__device__ __forceinline__ void node_load_direct(const K2Params &p, int64_t g, uint32_t base,
                                                 uint32_t mids, uint4 *As, uint4 *Bs, int t) {
    using C = K2Cfg<LF, KC>;
    constexpr int ITEMS = (C::SQ + NTH - 1) / NTH;
    const uint4 *Ag = reinterpret_cast<const uint4 *>(p.Abs) + g * (p.Ns / 4);
    const uint4 *Bg = reinterpret_cast<const uint4 *>(p.Bbs) + g * (p.Ns / 4);
    uint4 a[ITEMS], b[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) a[i] = b[i] = make_uint4(0, 0, 0, 0);
    const bool two = mids != 0;  // segment count is a power of two
    uint32_t sub = 0;
#pragma unroll 1
    do {
        const uint32_t o0 = (base + sub) * C::Q;
        sub = (sub - mids) & mids;
        const uint32_t o1 = (base + sub) * C::Q;
        if (two) sub = (sub - mids) & mids;
        uint4 xa[ITEMS][2], xb[ITEMS][2];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int u = t + i * NTH;
            if (C::SQ % NTH == 0 || u < C::SQ) {
                xa[i][0] = __ldg(Ag + o0 + u);
                xb[i][0] = __ldg(Bg + o0 + u);
                if (two) {
                    xa[i][1] = __ldg(Ag + o1 + u);
                    xb[i][1] = __ldg(Bg + o1 + u);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int u = t + i * NTH;
            if (C::SQ % NTH == 0 || u < C::SQ) {
                a[i] = a[i] ^ xa[i][0];
                b[i] = b[i] ^ xb[i][0];
                if (two) {
                    a[i] = a[i] ^ xa[i][1];
                    b[i] = b[i] ^ xb[i][1];
                }
            }
        }
    } while (sub != 0);
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const int u = t + i * NTH;
        if (C::SQ % NTH == 0 || u < C::SQ) {
            As[u] = a[i];
            Bs[u] = b[i];
        }
    }
}

// Operand load fused with the first evaluation pair (levels 0 and 1; KC >= 3):
// item (operand, w) gathers the root operand's four quarter quads at w from
// the path's segments, stores them, and writes the level-0 mid (2 quads) and
// the three level-1 mids (3 quads) straight from registers -- one barrier and
// the pair's shared-memory reads fewer than load + eval_pair<0>.
template <int LF, int KC, int NTH>
__device__ __forceinline__ void node_load_eval0(const K2Params &p, int64_t g, uint32_t base, uint32_t mids,
                                                uint4 *As, uint4 *Bs, int t) {
    using C = K2Cfg<LF, KC>;
    constexpr int q = C::Q << (KC - 2);                 // root quarter, quads
    constexpr int SQ = C::SQ;                           // = 4 q
    constexpr int Rj1 = C::Q * (1 << (KC - 1)) * 3;     // level-1 mids (eval_pair<0>)
    constexpr int ITEMS = (2 * q + NTH - 1) / NTH;
    uint4 x[ITEMS][4];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k) x[i][k] = make_uint4(0, 0, 0, 0);
    const bool two = mids != 0;
    uint32_t sub = 0;
#pragma unroll 1
    do {
        const uint32_t o0 = (base + sub) * C::Q;
        sub = (sub - mids) & mids;
        const uint32_t o1 = (base + sub) * C::Q;
        if (two) sub = (sub - mids) & mids;
        uint4 y[ITEMS][4][2];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int it = t + i * NTH;
            if ((2 * q) % NTH == 0 || it < 2 * q) {
                const int op = it >= q, w = it - op * q;
                const uint4 *G = reinterpret_cast<const uint4 *>(op ? p.Bbs : p.Abs) + g * (p.Ns / 4) + w;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    y[i][k][0] = __ldg(G + o0 + k * q);
                    if (two) y[i][k][1] = __ldg(G + o1 + k * q);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int it = t + i * NTH;
            if ((2 * q) % NTH == 0 || it < 2 * q) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    x[i][k] = x[i][k] ^ y[i][k][0];
                    if (two) x[i][k] = x[i][k] ^ y[i][k][1];
                }
            }
        }
    } while (sub != 0);
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const int it = t + i * NTH;
        if ((2 * q) % NTH == 0 || it < 2 * q) {
            const int op = it >= q, w = it - op * q;
            uint4 *X = op ? Bs : As;
            const uint4 m0 = x[i][0] ^ x[i][2], m1 = x[i][1] ^ x[i][3];
#pragma unroll
            for (int k = 0; k < 4; ++k) X[w + k * q] = x[i][k];
            X[SQ + w] = m0;
            X[SQ + q + w] = m1;
            X[Rj1 + w] = x[i][0] ^ x[i][1];
            X[Rj1 + q + w] = x[i][2] ^ x[i][3];
            X[Rj1 + 2 * q + w] = m0 ^ m1;
        }
    }
}

// One Karatsuba level.  ITER = ceil(items/NTH) is a compile-time constant and// One Karatsuba level.  ITER = ceil(items/NTH) is a compile-time constant and
// items are processed in unrolled batches of UNR: all shared-memory loads of
// a batch are issued before its first XOR (one smem round trip per batch
// instead of one per item) while the register footprint stays bounded.
// Items are (node nu, quad u) pairs, u fastest.
template <int LF, int KC, int J, int NTH, bool EVAL>
__device__ __forceinline__ void node_level(uint4 *As, uint4 *Bs, const uint16_t *pos, int t) {
    using C = K2Cfg<LF, KC>;
    constexpr int sh = KC - J - 1;
    constexpr int hq = C::Q << sh;
    constexpr int Rq = C::Q * (1 << (KC - J)) * pow3c(J);
    constexpr int items = pow3c(J) * hq;
    constexpr int ITER = (items + NTH - 1) / NTH;
    constexpr int UNR = 2;
    const uint16_t *P = pos + (pow3c(J) - 1) / 2;
    (void)ITER;
#pragma unroll 1
    for (int base = t; base < items; base += UNR * NTH) {
        int sv[UNR];
        bool ok[UNR];
#pragma unroll
        for (int r = 0; r < UNR; ++r) {
            const int it = base + r * NTH;
            ok[r] = it < items;
            const int nu = (it >> sh) / C::Q;
            sv[r] = ok[r] ? int(P[nu]) + (it - nu * hq) : 0;
        }
        if constexpr (EVAL) {
            uint4 x0[UNR], x1[UNR], y0[UNR], y1[UNR];
#pragma unroll
            for (int r = 0; r < UNR; ++r) {
                if (ok[r]) {
                    x0[r] = As[sv[r]];
                    x1[r] = As[sv[r] + hq];
                    y0[r] = Bs[sv[r]];
                    y1[r] = Bs[sv[r] + hq];
                }
            }
#pragma unroll
            for (int r = 0; r < UNR; ++r) {
                const int it = base + r * NTH;
                if (ok[r]) {
                    As[Rq + it] = x0[r] ^ x1[r];
                    Bs[Rq + it] = y0[r] ^ y1[r];
                }
            }
        } else {
            uint4 L0[UNR], H0[UNR], L1[UNR], H1[UNR], Ml[UNR], Mh[UNR];
#pragma unroll
            for (int r = 0; r < UNR; ++r) {
                const int it = base + r * NTH;
                if (ok[r]) {
                    L0[r] = As[sv[r]];
                    H0[r] = Bs[sv[r]];
                    L1[r] = As[sv[r] + hq];
                    H1[r] = Bs[sv[r] + hq];
                    Ml[r] = As[Rq + it];
                    Mh[r] = Bs[Rq + it];
                }
            }
#pragma unroll
            for (int r = 0; r < UNR; ++r) {
                if (ok[r]) {
                    const uint4 T = H0[r] ^ L1[r];
                    As[sv[r] + hq] = xor3(T, L0[r], Ml[r]);
                    Bs[sv[r]] = xor3(T, H1[r], Mh[r]);
                }
            }
        }
    }
}

// Item -> (node nu, quad w) for a phase over NODES nodes of q quads each: the// Item -> (node nu, quad w) for a phase over NODES nodes of q quads each: the
// first q & ~7 quads of every node are taken 8 at a time (an 8-thread shared
// memory phase then touches 8 consecutive quads of ONE node: conflict-free),
// the remaining q % 8 quads of all nodes come last.
template <int NODES, int q>
__device__ __forceinline__ void item_node_quad(int it, int &nu, int &w) {
    constexpr int qa = q & ~7, qt = q - qa;
    constexpr int qa1 = qa > 0 ? qa : 1, qt1 = qt > 0 ? qt : 1;  // (no division by zero)
    if (qa > 0 && it < NODES * qa) {
        nu = it / qa1;
        w = it - nu * qa;
    } else {
        const int r = it - NODES * qa;
        nu = qt > 0 ? r / qt1 : 0;
        w = qa + r - nu * qt;
    }
}

// Eval levels J and J+1 at once for every level-J node (J+1 <= KC-1): per
// quarter index, 4 loads -> 5 stores (the level-J mid, and the mids of the
// lo, hi and mid children).  Half the shared-memory traffic of two single
// levels and one barrier instead of two.
template <int LF, int KC, int J, int NTH>
__device__ __forceinline__ void eval_pair(uint4 *As, uint4 *Bs, const uint16_t *pos, int t) {
    using C = K2Cfg<LF, KC>;
    constexpr int sh = KC - J - 2;
    constexpr int q = C::Q << sh;  // quarter of a level-J node, quads
    constexpr int Rj = C::Q * (1 << (KC - J)) * pow3c(J);
    constexpr int Rj1 = C::Q * (1 << (KC - J - 1)) * pow3c(J + 1);
    constexpr int items = pow3c(J) * q;
    const uint16_t *P = pos + (pow3c(J) - 1) / 2;
#pragma unroll 1
    for (int it = t; it < items; it += NTH) {
        int nu, w;
        item_node_quad<pow3c(J), q>(it, nu, w);
        const int p = P[nu] + w;
        const uint4 a0 = As[p], a1 = As[p + q], a2 = As[p + 2 * q], a3 = As[p + 3 * q];
        const uint4 b0 = Bs[p], b1 = Bs[p + q], b2 = Bs[p + 2 * q], b3 = Bs[p + 3 * q];
        const int m = Rj + nu * 2 * q + w;
        const int c = Rj1 + 3 * nu * q + w;
        const uint4 am0 = a0 ^ a2, am1 = a1 ^ a3, bm0 = b0 ^ b2, bm1 = b1 ^ b3;
        As[m] = am0;
        As[m + q] = am1;
        Bs[m] = bm0;
        Bs[m + q] = bm1;
        As[c] = a0 ^ a1;
        As[c + q] = a2 ^ a3;
        As[c + 2 * q] = am0 ^ am1;
        Bs[c] = b0 ^ b1;
        Bs[c + q] = b2 ^ b3;
        Bs[c + 2 * q] = bm0 ^ bm1;
    }
}

// Interp levels J+1 and J at once for every level-J node (J+1 <= KC-1), in
// place: per quarter index w, the 9 grandchildren's product halves (18
// reads) give the 3 children's products (4 quarters each, in registers) and
// then the node's; 6 writes.  Each thread touches only index w of its node,
// so no two threads race.
template <int LF, int KC, int J, int NTH>
__device__ __forceinline__ void interp_pair(uint4 *As, uint4 *Bs, const uint16_t *pos, const uint8_t *minv,
                                            int t) {
    using C = K2Cfg<LF, KC>;
    constexpr int sh = KC - J - 2;
    constexpr int q = C::Q << sh;
    constexpr int items = pow3c(J) * q;
    constexpr int RJ = C::Q * (1 << (KC - J)) * pow3c(J);            // level-(J+1) mids
    constexpr int RJ1 = C::Q * (1 << (KC - J - 1)) * pow3c(J + 1);   // level-(J+2) mids
    const uint16_t *P = pos + (pow3c(J) - 1) / 2;
#pragma unroll 1
    for (int it = t; it < items; it += NTH) {
        int nu, w;
        item_node_quad<pow3c(J), q>(it, nu, w);
        // every position follows from the node's: children lo = p, hi = p+2q,
        // mid = RJ + 2q nu; grandchildren of child k: lo = p_k, hi = p_k+q,
        // mid = RJ1 + q (3nu + c)
        const int p = P[nu] + w;
        const int pc[3] = {p, p + 2 * q, RJ + 2 * q * nu + w};
        uint4 Q0[3], Q1[3], Q2[3], Q3[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            // level-KC mid leaves are stored permuted (kMidPerm, KC = 5)
            const int m = (KC == 5 && J == KC - 2) ? int(minv[3 * nu + c]) : 3 * nu + c;
            const int g0 = pc[c], g1 = pc[c] + q, g2 = RJ1 + q * m + w;
            const uint4 L0 = As[g0], H0 = Bs[g0], L1 = As[g1], H1 = Bs[g1];
            const uint4 Ml = As[g2], Mh = Bs[g2];
            const uint4 T = H0 ^ L1;
            Q0[c] = L0;
            Q1[c] = xor3(T, L0, Ml);
            Q2[c] = xor3(T, H1, Mh);
            Q3[c] = H1;
        }
        const int p0 = pc[0], p1 = pc[1];
        const uint4 T0 = Q2[0] ^ Q0[1], T1 = Q3[0] ^ Q1[1];
        As[p0 + q] = Q1[0];
        As[p1] = xor3(T0, Q0[0], Q0[2]);
        As[p1 + q] = xor3(T1, Q1[0], Q1[2]);
        Bs[p0] = xor3(T0, Q2[1], Q2[2]);
        Bs[p0 + q] = xor3(T1, Q3[1], Q3[2]);
        Bs[p1] = Q2[1];
    }
}

// F2X_FUSED_BOTTOM_EVAL = 1: the bottom evaluation level is fused into the
// mid leaves (they XOR their parent's chunks while loading); 0: it is a
// separate level done by all threads and the leaves touch only their own
// chunk (single leaf code path, no barriers inside the leaf phase).
#ifndef F2X_PROF_BUILD
#define F2X_PROF_BUILD 0
#endif

#ifndef F2X_FUSED_LOAD_EVAL
#define F2X_FUSED_LOAD_EVAL 1
#endif


#ifndef F2X_FUSED_STORE
#define F2X_FUSED_STORE 1
#endif

#ifndef F2X_FUSED_BOTTOM_EVAL
#define F2X_FUSED_BOTTOM_EVAL 1
#endif
__host__ __device__ constexpr int kEvalLevels(int KC) { return F2X_FUSED_BOTTOM_EVAL ? KC - 1 : KC; }
template <int LF, int KC, int NTH, int J, class Bar>
__device__ __forceinline__ void node_eval_from(uint4 *As, uint4 *Bs, const uint16_t *pos, int t, Bar bar) {
    constexpr int NE = kEvalLevels(KC);  // levels 0..NE-1 evaluated here
    if constexpr (J + 1 < NE) {
        eval_pair<LF, KC, J, NTH>(As, Bs, pos, t);
        bar();
        node_eval_from<LF, KC, NTH, J + 2>(As, Bs, pos, t, bar);
    } else if constexpr (J < NE) {
        node_level<LF, KC, J, NTH, true>(As, Bs, pos, t);
        bar();
    }
}
template <int LF, int KC, int NTH, int J, class Bar>
__device__ __forceinline__ void node_interp_from(uint4 *As, uint4 *Bs, const uint16_t *pos, const uint8_t *minv,
                                                 int t, Bar bar) {
    if constexpr (J >= 0) {
        interp_pair<LF, KC, J, NTH>(As, Bs, pos, minv, t);
        bar();
        node_interp_from<LF, KC, NTH, J - 2>(As, Bs, pos, minv, t, bar);
    } else if constexpr (J == -1) {
        node_level<LF, KC, 0, NTH, false>(As, Bs, pos, t);
        bar();
    }
}

// Top interpolation level fused with the node-product store (KC odd, node
// products to HBM): item it of the root reads the six quads of its children
// and writes the four product quads straight to global memory -- no shared
// memory write-back, no barrier, no separate store pass.
template <int LF, int KC, int NTH>
__device__ __forceinline__ void node_level0_store(const K2Params &p, int64_t node, const uint4 *As,
                                                  const uint4 *Bs, int t) {
    using C = K2Cfg<LF, KC>;
    constexpr int SQ = C::SQ, hq = SQ / 2;
    uint4 *out = reinterpret_cast<uint4 *>(p.Pout) + node * (2 * SQ);
    constexpr int UNR = 2;
#pragma unroll 1
    for (int base = t; base < hq; base += UNR * NTH) {
        uint4 L0[UNR], H0[UNR], L1[UNR], H1[UNR], Ml[UNR], Mh[UNR];
#pragma unroll
        for (int r = 0; r < UNR; ++r) {
            const int it = base + r * NTH;
            if (it < hq) {
                L0[r] = As[it];
                H0[r] = Bs[it];
                L1[r] = As[it + hq];
                H1[r] = Bs[it + hq];
                Ml[r] = As[SQ + it];
                Mh[r] = Bs[SQ + it];
            }
        }
#pragma unroll
        for (int r = 0; r < UNR; ++r) {
            const int it = base + r * NTH;
            if (it < hq) {
                const uint4 T = H0[r] ^ L1[r];
                out[it] = L0[r];
                out[hq + it] = xor3(T, L0[r], Ml[r]);
                out[SQ + it] = xor3(T, H1[r], Mh[r]);
                out[SQ + hq + it] = H1[r];
            }
        }
    }
}

// interp levels KC-1..1 in pairs, then the fused top level + store (KC odd)
template <int LF, int KC, int NTH, int J, class Bar>
__device__ __forceinline__ void node_interp_store_from(const K2Params &p, int64_t node, uint4 *As, uint4 *Bs,
                                                       const uint16_t *pos, const uint8_t *minv, int t, Bar bar) {
    if constexpr (J >= 0) {
        interp_pair<LF, KC, J, NTH>(As, Bs, pos, minv, t);
        bar();
        node_interp_store_from<LF, KC, NTH, J - 2>(p, node, As, Bs, pos, minv, t, bar);
    } else {
        static_assert(J == -1, "fused store needs an odd KC");
        node_level0_store<LF, KC, NTH>(p, node, As, Bs, t);
    }
}

// eval: levels 0..KC-2 in merged pairs (+ a single level when the count is odd)
template <int LF, int KC, int NTH, class Bar>
__device__ __forceinline__ void node_eval(uint4 *As, uint4 *Bs, const uint16_t *pos, int t, Bar bar) {
    node_eval_from<LF, KC, NTH, 0>(As, Bs, pos, t, bar);
}

// interp: levels KC-1..0 in merged pairs from the bottom (+ level 0 alone
// when KC is odd), elementwise in place
template <int LF, int KC, int NTH, class Bar>
__device__ __forceinline__ void node_interp(uint4 *As, uint4 *Bs, const uint16_t *pos, const uint8_t *minv, int t,
                                            Bar bar) {
    node_interp_from<LF, KC, NTH, KC - 2>(As, Bs, pos, minv, t, bar);
}

// store node product: lo half from A region, hi half from B region
template <int LF, int KC, int NTH>
__device__ __forceinline__ void node_store(const K2Params &p, int64_t node, const uint4 *As,
                                           const uint4 *Bs, int t) {
    using C = K2Cfg<LF, KC>;
    uint4 *out = reinterpret_cast<uint4 *>(p.Pout) + node * (2 * C::SQ);
    for (int u = t; u < C::SQ; u += NTH) {
        out[u] = As[u];
        out[C::SQ + u] = Bs[u];
    }
}

// Cluster combine (K2Params::combine): the 3 CTAs of a cluster hold the
// products L, H, M of the lo, hi and mid children of one parent (cluster rank
// = path digit; consecutive node indices are siblings at the deepest global
// level).  Parent product quarters (Ss storage words each):
//   P0 = L.lo, P1 = L.hi ^ L.lo ^ H.lo ^ M.lo, P2 = L.hi ^ H.lo ^ H.hi ^ M.hi, P3 = H.hi
// (the k3_interp formula).  CTA r builds quarter index w in [r SQ/3, (r+1) SQ/3)
// of all four quarters from the six quads at w, read over distributed shared
// memory, and stores them: the node products never go to HBM and the
// interpolation passes start one level higher.
template <int LF, int KC, int NTH>
__device__ __forceinline__ void node_combine_store(const K2Params &p, int64_t node, uint4 *As, uint4 *Bs, int t) {
    namespace cg = cooperative_groups;
    using C = K2Cfg<LF, KC>;
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();  // all three children's products are complete
    const uint4 *Al = cl.map_shared_rank(As, 0), *Bl = cl.map_shared_rank(Bs, 0);
    const uint4 *Ah = cl.map_shared_rank(As, 1), *Bh = cl.map_shared_rank(Bs, 1);
    const uint4 *Am = cl.map_shared_rank(As, 2), *Bm = cl.map_shared_rank(Bs, 2);
    const int r = int(cl.block_rank());
    constexpr int SQ = C::SQ;
    const int w0 = (r * SQ) / 3, w1 = ((r + 1) * SQ) / 3;
    uint4 *out = reinterpret_cast<uint4 *>(p.Pout) + (node / 3) * (4 * SQ);
    for (int w = w0 + t; w < w1; w += NTH) {
        const uint4 llo = Al[w], lhi = Bl[w], hlo = Ah[w], hhi = Bh[w], mlo = Am[w], mhi = Bm[w];
        const uint4 T = lhi ^ hlo;
        out[w] = llo;
        out[SQ + w] = xor3(T, llo, mlo);
        out[2 * SQ + w] = xor3(T, hhi, mhi);
        out[3 * SQ + w] = hhi;
    }
    cl.sync();  // siblings may still be reading this CTA's shared memory
}

// Last-arrival combine (K2Params::combine == 2): every node CTA stores its
// product as usual; the third sibling of a parent to finish (per-parent
// atomic counter) builds the parent product from its own product (shared
// memory) and the two siblings' products (L2-resident, read with ld.cg) and
// writes it IN PLACE over the triple's first 4 Ss words: quarter index w of
// the parent reads exactly the six quads at w of L, H, M and writes the four
// quads at w of the parent, which are the L.lo/L.hi/H.lo/H.hi slots it just
// read.  No cluster co-scheduling; the memory work overlaps the co-resident
// CTAs' leaves; one interpolation level less.
template <int LF, int KC, int NTH>
__device__ __forceinline__ void node_combine_last(const K2Params &p, int64_t node, const uint4 *As,
                                                  const uint4 *Bs, int t, int *s_flag) {
    using C = K2Cfg<LF, KC>;
    constexpr int SQ = C::SQ;
    __threadfence();  // this thread's product stores, before the arrival count
    __syncthreads();
    const int64_t par = node / 3;
    if (t == 0) {
        __threadfence();
        *s_flag = atomicAdd(p.cnt + par, 1u) == 2u;
    }
    __syncthreads();
    if (!*s_flag) return;
    __threadfence();
    const int me = int(node - par * 3);
    uint4 *base = reinterpret_cast<uint4 *>(p.Pout) + par * (3 * 2 * SQ);
    const uint4 *g[3] = {base, base + 2 * SQ, base + 4 * SQ};
    for (int w = t; w < SQ; w += NTH) {
        uint4 lo[3], hi[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (c == me) {
                lo[c] = As[w];
                hi[c] = Bs[w];
            } else {
                lo[c] = __ldcg(g[c] + w);
                hi[c] = __ldcg(g[c] + SQ + w);
            }
        }
        const uint4 T = hi[0] ^ lo[1];
        base[w] = lo[0];
        base[SQ + w] = xor3(T, lo[0], lo[2]);
        base[2 * SQ + w] = xor3(T, hi[1], hi[2]);
        base[3 * SQ + w] = hi[1];
    }
    if (t == 0) p.cnt[par] = 0u;  // (the counters are also zeroed before every launch)
}

struct SyncAll {
    __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
// A mid leaf reads its parent's lo and hi chunks; odd threads read the hi
// chunk first (see node_leaves), so an 8-thread phase hits
// 4 even and 4 odd chunk positions (bank-conflict-free with kMidPerm).
template <int LF, int Q, bool MID>
__device__ __forceinline__ void leaf_load_b(const uint4 *Bs, int src, int src2, bool mid, uint32_t (&b)[LF]) {
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        uint4 v = Bs[src + q];
        if (MID && mid) v = v ^ Bs[src2 + q];
        const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int r = 0; r < 4; ++r)
            if (4 * q + r < LF) b[4 * q + r] = vv[r];
    }
}

// hi half of the product -> B chunk `own`; then lo half left in c
template <int LF, int Q, bool MID>
__device__ __forceinline__ void leaf_passes(const uint4 *As, uint4 *Bs, int src, int src2, int own, bool mid,
                                            const uint32_t (&b)[LF], uint32_t (&c)[LF]) {
    // hi half: c[LF + k], k in [0, LF-1)
#pragma unroll
    for (int k = 0; k < LF; ++k) c[k] = 0u;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        uint4 v = As[src + q];
        if (MID && mid) v = v ^ As[src2 + q];
        const uint32_t av[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int i = 4 * q + r;
#pragma unroll
            for (int j = 0; j < LF; ++j)
                if (i < LF && i + j >= LF) c[i + j - LF] ^= av[r] & b[j];
        }
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        uint32_t o[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) o[r] = 4 * q + r < LF ? c[4 * q + r] : 0u;
        Bs[own + q] = make_uint4(o[0], o[1], o[2], o[3]);
    }
    // lo half: c[k], k in [0, LF)
#pragma unroll
    for (int k = 0; k < LF; ++k) c[k] = 0u;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        uint4 v = As[src + q];
        if (MID && mid) v = v ^ As[src2 + q];
        const uint32_t av[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int i = 4 * q + r;
#pragma unroll
            for (int j = 0; j < LF; ++j)
                if (i + j < LF) c[i + j] ^= av[r] & b[j];
        }
    }
}

// F2X_LEAF_LOOP = 1: compact leaf, one code path for mid and non-mid threads.
// The a rows are streamed ONCE, top quad first, against b in registers;
// w[k] is a sliding window of product words c[4q + k] (k < LF + 3) while
// quad q (rows 4q..4q+3) is processed.  After quad q, c[4q + LF - 1 ..] are
// final: hi-half words go straight to the thread's own B chunk as whole
// aligned quads (the hi word 4q+3 is held one iteration in `kept`), then
// the window shifts by 4 (LF - 1 register moves).  The loop body is
// 4*LF LOP3 instead of LF^2 unrolled (the two unrolled leaf variants are
// ~42 KB of code; the node kernel's top stall was no_instruction).  The lo
// half c[0..LF-1] ends in lo[] (stored by the caller after the barrier).
// Used up to LF = 33: at LF >= 34 the window + b + loop state exceed the 80
// registers of 3 CTAs/SM and the loop spills (measured: LF = 35 node kernel
// 0.2987 -> 0.3258 ms at n=17669), so those sizes keep the unrolled leaf.
#ifndef F2X_LEAF_LOOP
#define F2X_LEAF_LOOP 1
#endif
__host__ __device__ constexpr bool kLeafLoop(int LF) { return F2X_LEAF_LOOP && LF <= 33; }
template <int LF, int Q>
__device__ __forceinline__ uint4 leaf_a_quad(const uint4 *As, int src, int src2, int q, bool warp_mid, bool mid) {
    uint4 v = As[src + q];
    if (warp_mid) {
        uint4 x = make_uint4(0, 0, 0, 0);
        if (mid) x = As[src2 + q];
        v = v ^ x;
    }
    return v;
}

template <int LF, int Q>
__device__ __forceinline__ void leaf_loop(const uint4 *As, uint4 *Bs, int src, int src2, int own, bool warp_mid,
                                          bool mid, const uint32_t (&b)[LF], uint32_t (&lo)[LF]) {
    constexpr int QA = (LF + 3) / 4;      // quads holding real rows
    constexpr int RT = LF - 4 * (QA - 1);  // rows in the top quad (1..4)
    static_assert(QA >= 2, "leaf loop needs LF >= 5");
    uint32_t *Bw = reinterpret_cast<uint32_t *>(Bs + own);
    uint32_t w[LF + 3];
    // pad quads of the hi half
#pragma unroll
    for (int q = QA; q < Q; ++q) Bs[own + q] = make_uint4(0, 0, 0, 0);
    // top quad: rows 4(QA-1) .. LF-1, window base 4(QA-1)
    {
#pragma unroll
        for (int k = 0; k < LF + 3; ++k) w[k] = 0u;  // folded into the first AND
        const uint4 v = leaf_a_quad<LF, Q>(As, src, src2, QA - 1, warp_mid, mid);
        const uint32_t av[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int r = RT - 1; r >= 0; --r)
#pragma unroll
            for (int j = 0; j < LF; ++j) w[r + j] ^= av[r] & b[j];
        // final: w[LF .. LF+RT-2] = hi words 4(QA-1) .. LF-2 (quad QA-1);
        // w[LF-1] = hi word 4(QA-1)-1 is stored by the next quad
        uint32_t o[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) o[r] = r < RT - 1 ? w[LF + r] : 0u;
        Bs[own + QA - 1] = make_uint4(o[0], o[1], o[2], o[3]);
    }
    // quads QA-2 .. 0, rows 3, 2, 1, 0 of each: w[LF+2-s] is final after
    // row 3-s, so the hi words leave as soon as they are done (window peak
    // LF instead of LF+3 live words)
    const uint4 *ap = As + src + (QA - 2);
    const int dmid = src2 - src;
    uint32_t *bp = Bw + 4 * (QA - 2);
#pragma unroll 1
    for (; bp >= Bw; bp -= 4, --ap) {
        bp[3] = w[LF - 1];  // hi word 4q+3, final since the previous quad
#pragma unroll
        for (int k = LF - 2; k >= 0; --k) w[k + 4] = w[k];
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = 0u;
        uint4 v = *ap;
        if (warp_mid) {
            uint4 x = make_uint4(0, 0, 0, 0);
            if (mid) x = ap[dmid];
            v = v ^ x;
        }
        const uint32_t av[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int r = 3; r >= 0; --r) {
#pragma unroll
            for (int j = 0; j < LF; ++j) w[r + j] ^= av[r] & b[j];
            if (r > 0) bp[r - 1] = w[LF + r - 1];
        }
    }
#pragma unroll
    for (int k = 0; k < LF; ++k) lo[k] = w[k];
}

// Single-copy form of leaf_passes for the unrolled leaf (F2X_LEAF_ONE): the
// mid XOR loads sit behind warp-uniform branches instead of a second
// instantiation of the whole leaf.
template <int LF, int Q>
__device__ __forceinline__ uint4 leaf_ld(const uint4 *As, int src, int src2, int q, bool warp_mid, bool mid) {
    uint4 v = As[src + q];
    if (warp_mid) {
        uint4 x = make_uint4(0, 0, 0, 0);
        if (mid) x = As[src2 + q];
        v = v ^ x;
    }
    return v;
}
template <int LF, int Q>
__device__ __forceinline__ void leaf_passes_one(const uint4 *As, uint4 *Bs, int src, int src2, int own,
                                                bool warp_mid, bool mid, const uint32_t (&b)[LF],
                                                uint32_t (&c)[LF]) {
#pragma unroll
    for (int k = 0; k < LF; ++k) c[k] = 0u;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const uint4 v = leaf_ld<LF, Q>(As, src, src2, q, warp_mid, mid);
        const uint32_t av[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int i = 4 * q + r;
#pragma unroll
            for (int j = 0; j < LF; ++j)
                if (i < LF && i + j >= LF) c[i + j - LF] ^= av[r] & b[j];
        }
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        uint32_t o[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) o[r] = 4 * q + r < LF ? c[4 * q + r] : 0u;
        Bs[own + q] = make_uint4(o[0], o[1], o[2], o[3]);
    }
#pragma unroll
    for (int k = 0; k < LF; ++k) c[k] = 0u;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const uint4 v = leaf_ld<LF, Q>(As, src, src2, q, warp_mid, mid);
        const uint32_t av[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int i = 4 * q + r;
#pragma unroll
            for (int j = 0; j < LF; ++j)
                if (i + j < LF) c[i + j] ^= av[r] & b[j];
        }
    }
}
#ifndef F2X_LEAF_ONE
#define F2X_LEAF_ONE 1
#endif

template <int LF, int KC, class Bar>
__device__ __forceinline__ void node_leaves(uint4 *As, uint4 *Bs, const uint16_t *pos, const uint8_t *mperm,
                                            int t, Bar bar) {
    using C = K2Cfg<LF, KC>;
    constexpr int Q = C::Q;
    if constexpr (!F2X_FUSED_BOTTOM_EVAL) {
        // every leaf's operands are in its own chunk pair: no barriers needed
        (void)pos;
        (void)mperm;
        (void)bar;
        if (t < C::NLEAF) {
            const int own = t * Q;
            uint32_t b[LF], c[LF];
            leaf_load_b<LF, Q, false>(Bs, own, own, false, b);
            leaf_passes<LF, Q, false>(As, Bs, own, own, own, false, b, c);
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                uint32_t o[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) o[r] = 4 * q + r < LF ? c[4 * q + r] : 0u;
                As[own + q] = make_uint4(o[0], o[1], o[2], o[3]);
            }
        }
        return;
    }
    constexpr int RM = C::NLEAF - pow3c(KC - 1);  // first mid-leaf chunk
    const bool active = t < C::NLEAF;
    const bool mid = active && t >= RM;
    // warp-uniform: only warps that hold mid leaves run the XOR-loading code
    const bool warp_mid = ((t | 31) >= RM) && ((t & ~31) < C::NLEAF);
    const int own = t * Q;
    // thread RM+i computes the mid leaf of level-(KC-1) node kMidPerm[i] (KC =
    // 5; bank-conflict-reducing order) and keeps its own chunk for the product
    const int par = mid ? int(pos[(pow3c(KC - 1) - 1) / 2 + (KC == 5 ? int(mperm[t - RM]) : t - RM)]) : own;
    const int src = par + ((mid && (t & 1)) ? Q : 0);  // odd threads: hi chunk first
    const int src2 = par + ((t & 1) ? 0 : Q);
    uint32_t b[LF];
    if (active) {
        if (warp_mid) leaf_load_b<LF, Q, true>(Bs, src, src2, mid, b);
        else leaf_load_b<LF, Q, false>(Bs, src, src2, mid, b);
    }
    bar();  // all b operands loaded: B chunks may be overwritten
    uint32_t c[LF];
    if (active) {
        if constexpr (kLeafLoop(LF)) {
            leaf_loop<LF, Q>(As, Bs, src, src2, own, warp_mid, mid, b, c);
        } else {
            if constexpr (F2X_LEAF_ONE) {
                leaf_passes_one<LF, Q>(As, Bs, src, src2, own, warp_mid, mid, b, c);
            } else {
                if (warp_mid) leaf_passes<LF, Q, true>(As, Bs, src, src2, own, mid, b, c);
                else leaf_passes<LF, Q, false>(As, Bs, src, src2, own, mid, b, c);
            }
        }
    }
    bar();  // every thread finished streaming a: A chunks may be overwritten
    if (active) {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            uint32_t o[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) o[r] = 4 * q + r < LF ? c[4 * q + r] : 0u;
            As[own + q] = make_uint4(o[0], o[1], o[2], o[3]);
        }
    }
}

// Node kernel (default form): one CTA = one (group, global path) node of
// S = LF*2^KC coefficients (3 CTAs/SM at the hot sizes; CTAs start whenever
// a slot frees up, so co-resident CTAs stay out of phase and one CTA's leaf
// phase overlaps another's tree phases).  All threads run every phase:
//   load -> eval (levels 0..KC-2) -> 3^KC register leaves -> interp -> store.
// (A persistent grid-stride variant lock-steps the co-resident CTAs and
// makes the compiler hoist every level's index math out of the node loop --
// spills -- so it is not used.)
template <int LF, int KC>
__global__ void __launch_bounds__(K2Cfg<LF, KC>::NT, K2Cfg<LF, KC>::MINB)
k2_node_mul(const K2Params p, int64_t nodes) {
    using C = K2Cfg<LF, KC>;
    extern __shared__ uint4 smem[];
    uint4 *As = smem;
    uint4 *Bs = smem + C::RQ;
    __shared__ uint16_t pos[C::NPOS];  // node positions (quads), level-major
    __shared__ uint8_t mtab[KC == 5 ? 2 * 81 : 1];  // mid-leaf permutation + inverse (KC = 5)

    pdl_prologue();
    const int tid = threadIdx.x;
    const int64_t node = blockIdx.x;
    (void)nodes;
#if F2X_PROF_BUILD
    // phase clocks (F2X_PHASE_PROF at run time; compiled in only with
    // -DF2X_PROF_BUILD=1: the pointer and clock would otherwise hold 4
    // registers through the leaf)
    long long *prof = p.prof ? p.prof + node * 8 : nullptr;
    long long tc = prof ? clock64() : 0;
    auto mark = [&](int i) {
        if (prof && tid == 0) {
            const long long c2 = clock64();
            prof[i] = c2 - tc;
            tc = c2;
        }
    };
#else
    constexpr long long *prof = nullptr;
    auto mark = [](int) {};
#endif
    const int64_t g = node / p.paths;
    const int path = int(node - g * p.paths);
    // position table entries: two cached global loads per thread, issued
    // first so their latency overlaps the operand loads (an arithmetic
    // rebuild costs ~15% of the kernel's instructions)
    constexpr int PER = (C::NPOS + C::NT - 1) / C::NT;
    uint32_t pv[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = tid + i * C::NT;
        pv[i] = e < C::NPOS ? __ldg(&kPosChunks[KC][e]) : 0u;
    }
    const uint32_t mt = (KC == 5 && tid < 2 * 81) ? __ldg(&kMidPerm[0][0] + tid) : 0u;
    uint32_t base, mids;
    path_base_mids(p, path, base, mids);
    mark(0);
    constexpr bool kFuseEval0 = F2X_FUSED_LOAD_EVAL && kEvalLevels(KC) >= 2;
    if constexpr (kFuseEval0) node_load_eval0<LF, KC, C::NT>(p, g, base, mids, As, Bs, tid);
    else node_load_direct<LF, KC, C::NT>(p, g, base, mids, As, Bs, tid);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = tid + i * C::NT;
        if (e < C::NPOS) pos[e] = uint16_t(pv[i] * C::Q);
    }
    if (KC == 5 && tid < 2 * 81) mtab[tid] = uint8_t(mt);
    __syncthreads();
    mark(1);
    if constexpr (kFuseEval0) {
        node_eval_from<LF, KC, C::NT, 2>(As, Bs, pos, tid, SyncAll{});
    } else {
        node_eval<LF, KC, C::NT>(As, Bs, pos, tid, SyncAll{});
    }
    mark(2);
    node_leaves<LF, KC>(As, Bs, pos, mtab, tid, SyncAll{});
    __syncthreads();
    mark(3);
    if constexpr (KC % 2 == 1 && F2X_FUSED_STORE) {
        if (p.combine == 0) {  // top level fused with the store (the common case)
            node_interp_store_from<LF, KC, C::NT, KC - 2>(p, node, As, Bs, pos, mtab + (KC == 5 ? 81 : 0), tid,
                                                          SyncAll{});
            mark(4);
            mark(5);
#if F2X_PROF_BUILD
            if (prof) {
                __syncthreads();
                if (tid == 0) prof[7] = -1;
            }
#endif
            return;
        }
    }
    node_interp<LF, KC, C::NT>(As, Bs, pos, mtab + (KC == 5 ? 81 : 0), tid, SyncAll{});
    mark(4);
    if (p.combine == 1) {
        node_combine_store<LF, KC, C::NT>(p, node, As, Bs, tid);
    } else {
        node_store<LF, KC, C::NT>(p, node, As, Bs, tid);
        if (p.combine == 2) {
            __shared__ int s_last;
            node_combine_last<LF, KC, C::NT>(p, node, As, Bs, tid, &s_last);
        }
    }
#if F2X_PROF_BUILD
    if (prof) {
        __syncthreads();
        mark(5);
        if (tid == 0) prof[7] = -1;
    }
#else
    (void)prof;
#endif
}

template <int LF, int KC>
int launch_k2(const K2Params &p, int64_t blocks, cudaStream_t stream) {
    using C = K2Cfg<LF, KC>;
    // F2X_SMEM_PAD (bytes) inflates the dynamic shared memory to force lower
    // occupancy -- occupancy / phase-overlap experiments only.
    static const int pad = [] {
        const char *v = getenv("F2X_SMEM_PAD");
        return v ? atoi(v) : 0;
    }();
    static std::atomic<uint32_t> configured_dev_mask{0};  // devices configured (idempotent set)
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 31 && !(configured_dev_mask.load() & (1u << dev))) {
        cudaError_t e = cudaFuncSetAttribute(k2_node_mul<LF, KC>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(C::SMEM) + pad);
        if (e != cudaSuccess) return -1000 - int(e);
        configured_dev_mask.fetch_or(1u << dev);
    }
    // one node per CTA (see k2_node_mul); clusters of 3 siblings when combining
    cudaError_t e;
    if (p.combine == 1) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(blocks));
        cfg.blockDim = dim3(C::NT);
        cfg.dynamicSmemBytes = C::SMEM + pad;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 3;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, k2_node_mul<LF, KC>, p, blocks);
        if (e == cudaSuccess) e = cudaGetLastError();
    } else {
        e = launch_pdl(k2_node_mul<LF, KC>, dim3(unsigned(blocks)), dim3(C::NT), C::SMEM + pad, stream, p,
                       blocks);
        if (e == cudaSuccess) e = cudaGetLastError();
    }
    return e == cudaSuccess ? 0 : -1000 - int(e);
}

struct K2Entry {
    int LF, KC, threads;
    size_t smem;
    int (*launch)(const K2Params &, int64_t, cudaStream_t);
};

}  // namespace f2x
