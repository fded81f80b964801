// Host side of the engine: planner, the C ABI of include/f2x.h, and the
// memory-side kernels around the node kernel (f2x_kernels.cuh):
//   K1 k1_slice / k1_slice_eval<EL>
//                    packed uint64[batch][t] -> bitsliced chunked groups, the
//                    top EL global Karatsuba levels pre-evaluated
//                    (+ constant-time top-bit check for ring operands)
//   toom_eval_level  Toom-3 evaluation, one level (large operands only)
//   K2 k2_node_mul   per (group, Karatsuba path) node product  [hot kernel]
//   K3 k3_interp<D>  global Karatsuba interpolation, D levels per pass
//   toom_interp_*    Toom-3 interpolation, one level (exact divisions)
//   K4 k4_unslice    fold mod X^n-1 (cyclic) + transpose back to uint64 rows
// Reference interfaces replaced: schoolbook_mul (poly.py:547-561),
// clmul64_batch (poly.py:451-480), SPEC ring_mul.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/f2x.h"
#include "f2x_kernels.cuh"

namespace f2x {

extern const K2Entry k2_part0[];
extern const int k2_part0_n;
extern const K2Entry k2_part1[];
extern const int k2_part1_n;
extern const K2Entry k2_part2[];
extern const int k2_part2_n;
extern const K2Entry k2_part3[];
extern const int k2_part3_n;

static const K2Entry *find_k2(int LF, int KC) {
    const K2Entry *parts[4] = {k2_part0, k2_part1, k2_part2, k2_part3};
    const int ns[4] = {k2_part0_n, k2_part1_n, k2_part2_n, k2_part3_n};
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < ns[i]; ++j)
            if (parts[i][j].LF == LF && parts[i][j].KC == KC) return &parts[i][j];
    return nullptr;
}

static constexpr int kMaxKC = 5;
static constexpr int kMaxGL = 8;
static constexpr int kMaxPassLevels = 4;
static constexpr int kThreads = 128;
static constexpr int kMaxToom = 3;      // Toom-3 levels above the node problem
static constexpr int kToomW = 16;       // x = X^w (coefficients)
// Planner cost constants, in units of one leaf LOP3 per 32-product group
// (3.8e-5 ns on B200), from a least-squares fit of 130 measured calls (ring
// sizes 8000..57637 bits x 256..16384 rows x 0..3 Toom levels, DESIGN §7b
// "planner regret"): mean regret of the picks 0.1 %, worst 2.5 %.
static constexpr double kPassWordCost = 21.5;        // per word of the global Karatsuba passes / slicing output
static constexpr double kToomWordCost = 10.5;        // per word the Toom passes move, plans of >= 2 levels
static constexpr double kToomWordCostSingle = 21.0;  // same for one-level plans (one product per group and level: latency-bound)
static constexpr double kToomLevelLatency = 2.63e8;  // per Toom level and CALL (~10 us: two more launches that cannot fill the GPU at small batches)
// Toom is considered from 160 words (n=10000: 0 / 1 / 2 levels tie; d=8192
// 11996 / 14350 / 12530 us); below 512 words it used to be off (round 1/2:
// the passes were slower) -- n=17669 x 4096 now takes two levels (323.7 ->
// 310.9 us), n=20000 x 4096 456 -> 358, while n=17669 x 2048 stays at 0.
static constexpr int kToomMinWords = 160;
// The innermost Toom level may evaluate at x = X^8 instead of X^16: the node
// problem then holds M_TL + 16 instead of + 32 coefficients, which at some
// sizes is one leaf word less (n=57637: LF 35 -> 34); its interpolation scans
// twice the segments per block (measured +8..13 %), charged below.
static constexpr int kToomWSmall = 8;
static constexpr double kToomSmallWInterpPenalty = 1.25;  // (1.2 .. 1.3 give the measured-best picks: d=32768 stays at w = 16)

static inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

#define F2X_LAUNCH(kern, grid, block, smem, stream, ...)                             \
    do {                                                                             \
        kern<<<dim3(grid), dim3(block), size_t(smem), stream>>>(__VA_ARGS__);        \
        const cudaError_t le_ = cudaGetLastError();                                  \
        if (le_ != cudaSuccess) return F2X_ECUDA - int(le_);                         \
    } while (0)

static inline int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }
static inline int64_t ipow5(int k) {
    int64_t r = 1;
    while (k-- > 0) r *= 5;
    return r;
}
static inline int64_t ipow3(int k) {
    int64_t r = 1;
    while (k-- > 0) r *= 3;
    return r;
}

// ------------------------------------------------------------------- K1/K4
// Both memory-side kernels work on a TILE of 64 operand words (4096
// coefficients) of one group with 128 threads: thread i owns half-word i
// (32 coefficients) of the tile and does one 32x32 bit transpose in
// registers; the chunked bitsliced side goes through a shared stage and is
// read/written as a contiguous run of storage words by all 128 threads
// (coalesced, pads included), walked incrementally (StorageWalk).
constexpr int kTileWords = 64;                 // uint64 operand words per tile
constexpr int kTileCoeffs = 64 * kTileWords;   // 4096
constexpr int kTileThreads = 2 * kTileWords;   // one 32x32 transpose each

__device__ __forceinline__ void chunk_split(int k, int LF, int &c, int &r) {
    c = k / LF;
    r = k - c * LF;
}

// half-word stage index with one pad word per 32 (conflict-free transposes)
__device__ __forceinline__ int stg(int k) { return k + (k >> 5); }

// K1 load phase: 32 rows (rows < 32 only in a ragged last group; 0 for words
// u >= t) x one 32-bit half-word column of operand word u (adjacent threads =
// adjacent halves: coalesced), the ring's constant-time top-bit check on the
// last word (an OR-reduction into *d_err), the 32x32 transpose.
// Every branch is on public shape values (batch, t, n, thread index).
__device__ __forceinline__ void k1_column(const uint32_t *X, int64_t g, int t, int u, int half, int rows,
                                          int ncyc, uint32_t *d_err, uint32_t (&x)[32]) {
    const uint32_t *px = X + ((g * 32) * t + u) * 2 + half;
    const int64_t rs = 2 * int64_t(t);
#pragma unroll
    for (int pr = 0; pr < 32; ++pr) {
        x[pr] = pr < rows ? __ldg(px) : 0u;
        px += rs;
    }
    if (ncyc > 0 && u == t - 1) {
        const int sh = ncyc - 64 * u - 32 * half;  // bits of this half-word below n
        uint32_t bad = 0;
        if (sh < 32) {
            const uint32_t himask = sh <= 0 ? ~0u : ~0u << sh;
#pragma unroll
            for (int pr = 0; pr < 32; ++pr) bad |= x[pr] & himask;
        }
        if (d_err != nullptr) atomicOr(d_err, uint32_t(bad != 0));
    }
    transpose32(x);
}

// Walk storage words sw = s0 + tid, s0 + tid + 128, ... < s1 of the chunked
// layout, tracking r = sw mod LFS and the coefficient index kk = chunk*LF + r
// (relative to kbase) incrementally: one divmod per thread, then adds.
template <int STEP>
struct StorageWalkN {
    int r, kk, dr, dkk, LF, LFS;
    __device__ __forceinline__ StorageWalkN(int sw, int kbase, int LF_, int LFS_) : LF(LF_), LFS(LFS_) {
        const int c = sw / LFS;
        r = sw - c * LFS;
        kk = c * LF + r - kbase;
        const int dc = STEP / LFS;
        dr = STEP - dc * LFS;
        dkk = dc * LF + dr;
    }
    __device__ __forceinline__ bool data() const { return r < LF; }
    __device__ __forceinline__ void next() {
        r += dr;
        kk += dkk;
        if (r >= LFS) {
            r -= LFS;
            kk += LF - LFS;
        }
    }
};
using StorageWalk = StorageWalkN<kTileThreads>;

__global__ void __launch_bounds__(kTileThreads)
k1_slice(const uint64_t *__restrict__ A, const uint64_t *__restrict__ B, uint32_t *__restrict__ Abs,
         uint32_t *__restrict__ Bbs, int64_t batch, int t, int N, int LF, int LFS, int64_t Ns,
         int ncyc, uint32_t *d_err, int tiles) {
    __shared__ uint32_t stage[kTileCoeffs + kTileCoeffs / 32];
    check_poison(stage, sizeof(stage));
    check_poison_sync();
    const int tid = threadIdx.x;
    const int64_t g = blockIdx.x / tiles;
    const int tile = int(blockIdx.x - g * tiles);
    const int u = tile * kTileWords + (tid >> 1);  // operand word of this half-word
    const int half = tid & 1;
    const uint32_t *X = reinterpret_cast<const uint32_t *>(blockIdx.y ? B : A);
    uint32_t *out = (blockIdx.y ? Bbs : Abs) + g * Ns;

    uint32_t x[32];
    const int rows = u < t ? int(batch - g * 32 < 32 ? batch - g * 32 : 32) : 0;
    k1_column(X, g, t, u, half, rows, ncyc, d_err, x);
#pragma unroll
    for (int i = 0; i < 32; ++i) stage[stg(32 * tid + i)] = x[i];
    __syncthreads();
    // store the contiguous storage range of coefficients [k0, k1)
    const int k0 = tile * kTileCoeffs, k1 = min(k0 + kTileCoeffs, N);
    if (k0 >= k1) return;
    if (LF == LFS && (Ns & 3) == 0 && (k1 & 3) == 0) {
        // plain layout (Toom plans' slice): storage = coefficients, whole
        // 16-byte quads (the tile starts on a quad; N and Ns are quads)
        uint4 *o = reinterpret_cast<uint4 *>(out + k0);
        for (int q = tid; q < ((k1 - k0) >> 2); q += kTileThreads) {
            const int k = 4 * q;
            o[q] = make_uint4(stage[stg(k)], stage[stg(k + 1)], stage[stg(k + 2)], stage[stg(k + 3)]);
        }
        return;
    }
    int c, r;
    chunk_split(k0, LF, c, r);
    const int s0 = c * LFS + r;
    chunk_split(k1, LF, c, r);
    const int s1 = c * LFS + r;  // k1 on a chunk boundary => previous chunk's pads included
    StorageWalk w(s0 + tid, k0, LF, LFS);
#pragma unroll 4
    for (int sw = s0 + tid; sw < s1; sw += kTileThreads) {
        out[sw] = w.data() ? stage[stg(w.kk)] : 0u;
        w.next();
    }
}

// K1 for operands of at most one tile (N <= 4096 coefficients, W =
// ceil(N/64) words): a CTA of 128 threads slices GPC = 64 / W whole groups at once
// (thread = (group, half-word column); one tile per group left 75 % of the
// threads idle at d=1024), and since a group's storage range is its whole
// operand -- [0, Ns), whole 16-byte quads -- it is written as storage quads.
template <int Q>  // storage quads per chunk (LFS / 4)
__global__ void __launch_bounds__(kTileThreads)
k1_slice_groups(const uint64_t *__restrict__ A, const uint64_t *__restrict__ B, uint32_t *__restrict__ Abs,
                uint32_t *__restrict__ Bbs, int64_t batch, int t, int N, int LF, int LFS, int64_t Ns, int ncyc,
                uint32_t *d_err, int64_t G) {
    __shared__ uint32_t stage[kTileCoeffs + kTileCoeffs / 32];
    check_poison(stage, sizeof(stage));
    check_poison_sync();
    const int tid = threadIdx.x;
    const int W = (N + 63) >> 6, GPC = kTileWords / W, STG = 64 * W + 2 * W;
    const int gi = tid / (2 * W), h = tid - gi * (2 * W);
    const int64_t g = int64_t(blockIdx.x) * GPC + gi;
    const uint32_t *X = reinterpret_cast<const uint32_t *>(blockIdx.y ? B : A);
    if (gi < GPC && g < G) {
        const int u = h >> 1, half = h & 1;
        uint32_t x[32];
        const int rows = u < t ? int(batch - g * 32 < 32 ? batch - g * 32 : 32) : 0;
        k1_column(X, g, t, u, half, rows, ncyc, d_err, x);
#pragma unroll
        for (int i = 0; i < 32; ++i) stage[gi * STG + stg(32 * h + i)] = x[i];
    }
    __syncthreads();
    // storage quads of the CTA's groups, chunk c = q / Q at compile time;
    // (group, quad) advanced incrementally (no division in the loop)
    const int qpg = int(Ns >> 2);
    const int64_t g0 = int64_t(blockIdx.x) * GPC;
    const int ng = int(G - g0 < GPC ? G - g0 : GPC);
    uint4 *o = reinterpret_cast<uint4 *>((blockIdx.y ? Bbs : Abs) + g0 * Ns);
    int gg = tid / qpg, q = tid - gg * qpg;
    for (int x = tid; x < ng * qpg; x += kTileThreads) {
        const int c = q / Q, r0 = (q - c * Q) * 4, kb = c * LF + r0;
        const uint32_t *S = stage + gg * STG;
        uint32_t v[4];
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) v[rr] = r0 + rr < LF ? S[stg(kb + rr)] : 0u;
        o[x] = make_uint4(v[0], v[1], v[2], v[3]);
        q += kTileThreads;
        while (q >= qpg) {
            q -= qpg;
            ++gg;
        }
    }
}

// K1 with the top EL global Karatsuba levels pre-evaluated (EL = 1, 2): the
// CTA transposes the same tile of each of the 2^EL parts of the operand
// (part j = coefficients [j N/2^EL, (j+1) N/2^EL)) into 2^EL stages, then
// writes the 3^EL evaluated sub-operands (per level: lo, hi, lo^hi; top level
// most significant -- the node numbering of the node kernel is unchanged; it
// runs on 3^EL x the groups with K-EL levels and loads 2^EL x fewer segments
// per mid path).  A tile is TW operand words of each part covering WHOLE
// chunks (64 TW a multiple of LF: TW = LF, or the whole part), so its storage
// range is a run of whole 16-byte quads: the second phase writes storage
// quads (one 16-byte store per sub-operand and quad) and no two CTAs share a
// quad.  Thread x < 2^EL 2 TW owns half-word column x of the tile (one 32x32
// bit transpose); all threads walk the quads.
template <int EL, int Q>  // Q: storage quads per chunk (LFS / 4)
__global__ void __launch_bounds__(8 * 40, 4)  // <= 4 parts x 2 x 40 words; 4 CTAs/SM: one wave at n=17669
k1_slice_eval(const uint64_t *__restrict__ A, const uint64_t *__restrict__ B, uint32_t *__restrict__ Ea,
              uint32_t *__restrict__ Eb, int64_t batch, int t, int N, int LF, int LFS, int64_t NsE,
              int ncyc, uint32_t *d_err, int tiles, int TW) {
    constexpr int NP = 1 << EL;               // parts
    constexpr int NO = EL == 1 ? 3 : 9;       // evaluated sub-operands
    const int STG = 64 * TW + 2 * TW;         // stage words per part (1 pad per 32)
    extern __shared__ uint32_t stage[];       // [NP][STG]
    check_poison(stage, unsigned(NP * STG * 4));
    check_poison_sync();
    const int x = threadIdx.x, nthr = blockDim.x;
    const int64_t g = blockIdx.x / tiles;
    const int tile = int(blockIdx.x - g * tiles);
    const int NE = N >> EL;                   // coefficients per part (multiple of 64)
    const uint32_t *X = reinterpret_cast<const uint32_t *>(blockIdx.y ? B : A);
    const int rows = int(batch - g * 32 < 32 ? batch - g * 32 : 32);
    if (x < NP * 2 * TW) {
        const int j = x / (2 * TW), h = x - j * (2 * TW);  // part, half-word column in the tile
        const int half = h & 1;
        const int ul = tile * TW + (h >> 1);  // word within the part
        const int u = j * (NE / 64) + ul;     // operand word
        uint32_t xv[32];
        k1_column(X, g, t, u, half, u < t ? rows : 0, ncyc, d_err, xv);
#pragma unroll
        for (int i = 0; i < 32; ++i) stage[j * STG + stg(32 * h + i)] = xv[i];
    }
    __syncthreads();
    const int nc = (64 * TW) / LF;  // whole chunks per tile
    constexpr int qpc = Q;
    const int nq = nc * qpc;
    uint32_t *out = (blockIdx.y ? Eb : Ea) + g * (NO * NsE) + int64_t(tile) * nc * LFS;
    for (int q = x; q < nq; q += nthr) {
        const int c = q / qpc, r0 = (q - c * qpc) * 4;
        const int kb = c * LF + r0;  // tile-local coefficient of the quad's first word
        uint32_t v[NP][4];
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
            const bool data = r0 + rr < LF;
#pragma unroll
            for (int jj = 0; jj < NP; ++jj) v[jj][rr] = data ? stage[jj * STG + stg(kb + rr)] : 0u;
        }
        uint4 *o = reinterpret_cast<uint4 *>(out) + q;
        const int64_t s4 = NsE >> 2;  // sub-operand stride in quads
        if constexpr (EL == 1) {
            const uint4 lo = make_uint4(v[0][0], v[0][1], v[0][2], v[0][3]);
            const uint4 hi = make_uint4(v[1][0], v[1][1], v[1][2], v[1][3]);
            o[0] = lo;
            o[s4] = hi;
            o[2 * s4] = lo ^ hi;
        } else {
            uint4 p[4];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) p[jj] = make_uint4(v[jj][0], v[jj][1], v[jj][2], v[jj][3]);
            const uint4 h[3][2] = {{p[0], p[1]}, {p[2], p[3]}, {p[0] ^ p[2], p[1] ^ p[3]}};
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                o[(3 * d) * s4] = h[d][0];
                o[(3 * d + 1) * s4] = h[d][1];
                o[(3 * d + 2) * s4] = h[d][0] ^ h[d][1];
            }
        }
    }
}

// --------------------------------------------------------------- Toom-3
// ---------------------------------------------------------- fused Toom eval
// All TL Toom-3 evaluation levels in ONE pass (instead of TL launches with
// HBM round trips of the intermediate levels): a CTA owns one (group,
// operand, tile of Tc node-problem chunks = T coefficients) and produces that
// tile of all 5^TL node-problem operands.  Evaluation is local: a
// level-(l+1) coefficient k reads level-l coefficients k, M+k, 2M+k, M+k-w,
// 2M+k-2w (M = M_{l+1}), so a level-(l+1) window of length L needs three
// level-l windows ("pieces") of length L + 2w.  Piece pi at level l has
// digits (p_{l+1} .. p_TL), most significant first, and starts at
// sigma_l(pi) = p_{l+1} M_{l+1} + sigma_{l+1}(rest) - 2w (sigma_TL = tile
// start k0).  The planner makes every M_l, the level-0 row and k0 multiples
// of 4 coefficients, so every piece is 16-byte aligned in HBM and in shared
// memory and every mask boundary (k = 0, M, M+w, M+2w) falls on a quad:
//   * the 3^TL level-0 pieces are staged by bulk async copies
//     (cp.async.bulk, completion on an mbarrier, no register staging);
//   * the intermediate levels are built in shared memory depth first, one
//     16-byte quad (4 coefficients) per thread-item, masks per quad;
//   * the last level is written as chunked storage quads (16-byte stores).
struct ToomEvalGeo {
    int M[4];       // M[1..TL]: part sizes (multiples of 4)
    int N0;         // level-0 operand coefficients (3 M_1, plain)
    int LF, LFS;    // node-problem chunk layout
    int chunks;     // node-problem chunks (2^K)
    int Tc;         // chunks per tile (Tc LF multiple of 4)
    int64_t G;      // groups
    int64_t Ns;     // storage words per node-problem operand
};

constexpr int kEvalFusedThreads = 256;
constexpr int kEvalFusedMaxT = 288;  // coefficients per tile (Tc LF <= 288)

__host__ __device__ constexpr int efpow3(int k) { return k <= 0 ? 1 : 3 * efpow3(k - 1); }
// piece slot words at level l (pieces of T + 2w (TL - l) coefficients)
__host__ __device__ constexpr int efslot(int TL, int l) { return kEvalFusedMaxT + 2 * kToomW * (TL - l); }

// shared-memory words: L0 (3^TL pieces), then for TL = 3 one e1's L1 (9
// pieces) and all five e2's L2 (15 pieces), for TL = 2 all five e1's L1
__host__ __device__ constexpr int eval_fused_smem_words(int TL) {
    return efpow3(TL) * efslot(TL, 0) +
           (TL == 3 ? 9 * efslot(3, 1) + 15 * efslot(3, 2) : TL == 2 ? 15 * efslot(2, 1) : 0);
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return uint32_t(__cvta_generic_to_shared(p));
}

// Evaluation of quad jq (coefficients 4jq..4jq+3 of the next-level piece,
// first coordinate k) from the three level-l pieces: E = -1 all five points,
// else only point E (0, 1, x, x+1, inf).  Quads at local j+2w, j+w, j.
template <int E>
__device__ __forceinline__ void eval_quad(const uint4 *P0, const uint4 *P1, const uint4 *P2, int jq, int k, int M,
                                          uint4 (&y)[E < 0 ? 5 : 1]) {
    constexpr int wq = kToomW / 4;
    const bool ka = unsigned(k) < unsigned(M), k1 = unsigned(k - kToomW) < unsigned(M),
               k2 = unsigned(k - 2 * kToomW) < unsigned(M);
    const uint4 z = make_uint4(0, 0, 0, 0);
    const bool use_a0 = E < 0 || E <= 3, use_a1 = E < 0 || E == 1 || E == 3,
               use_a2 = E < 0 || E == 1 || E == 3 || E == 4, use_s = E < 0 || E == 2 || E == 3;
    const uint4 a0 = (use_a0 && ka) ? P0[jq + 2 * wq] : z;
    const uint4 a1 = (use_a1 && ka) ? P1[jq + 2 * wq] : z;
    const uint4 a2 = (use_a2 && ka) ? P2[jq + 2 * wq] : z;
    const uint4 s1 = (use_s && k1) ? P1[jq + wq] : z;
    const uint4 s2 = (use_s && k2) ? P2[jq] : z;
    if constexpr (E < 0) {
        const uint4 p1 = xor3(a0, a1, a2), xs = s1 ^ s2;
        y[0] = a0;
        y[1] = p1;
        y[2] = a0 ^ xs;
        y[3] = p1 ^ xs;
        y[4] = a2;
    } else if constexpr (E == 0) {
        y[0] = a0;
    } else if constexpr (E == 1) {
        y[0] = xor3(a0, a1, a2);
    } else if constexpr (E == 2) {
        y[0] = xor3(a0, s1, s2);
    } else if constexpr (E == 3) {
        y[0] = xor3(a0, a1, a2) ^ (s1 ^ s2);
    } else {
        y[0] = a2;
    }
}

// Level-1 pieces (9 of them) of evaluation point E from the 27 level-0
// pieces (TL = 3), with the point E a runtime (CTA-uniform) value: one code
// copy for all five points, so the point loop below stays a loop without an
// indirect-branch dispatch (tools/ct_sass_audit.py) and without the spills
// of a written-out sequence.  Unused terms load nothing and are zero.
__device__ __forceinline__ void eval_l1_point_rt(int E, const uint32_t *L0, uint32_t *L1, const ToomEvalGeo &geo,
                                                 int k0, int nq1, int tid) {
    constexpr int w = kToomW, wq = kToomW / 4, Z0 = efslot(3, 0), Z1 = efslot(3, 1);
    const int M2 = geo.M[2], M3 = geo.M[3], M1 = geo.M[1];
    const bool use_a0 = E <= 3, use_a1 = E == 1 || E == 3, use_a2 = E == 1 || E == 3 || E == 4,
               use_s = E == 2 || E == 3;
    const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int pi1 = 0; pi1 < 9; ++pi1) {
        const int p2 = pi1 / 3, p3 = pi1 - 3 * p2;
        const int sig1 = p2 * M2 + p3 * M3 + k0 - 4 * w;
        const uint4 *P0 = reinterpret_cast<const uint4 *>(L0 + pi1 * Z0);
        const uint4 *P1 = reinterpret_cast<const uint4 *>(L0 + (9 + pi1) * Z0);
        const uint4 *P2 = reinterpret_cast<const uint4 *>(L0 + (18 + pi1) * Z0);
        uint4 *D = reinterpret_cast<uint4 *>(L1 + pi1 * Z1);
        for (int jq = tid; jq < nq1; jq += kEvalFusedThreads) {
            const int k = sig1 + 4 * jq;
            const bool ka = unsigned(k) < unsigned(M1), k1 = unsigned(k - w) < unsigned(M1),
                       k2 = unsigned(k - 2 * w) < unsigned(M1);
            const uint4 a0 = (use_a0 && ka) ? P0[jq + 2 * wq] : z;
            const uint4 a1 = (use_a1 && ka) ? P1[jq + 2 * wq] : z;
            const uint4 a2 = (use_a2 && ka) ? P2[jq + 2 * wq] : z;
            const uint4 s1 = (use_s && k1) ? P1[jq + wq] : z;
            const uint4 s2 = (use_s && k2) ? P2[jq] : z;
            D[jq] = xor3(a0, a1, a2) ^ (s1 ^ s2);
        }
    }
}

// all five points of nq quads of `np` pieces at once: piece p of the output
// (of every point e) from input pieces (0, p), (1, p), (2, p) (stride np);
// output piece (e, p) at D + (e np + p) Zd
__device__ __forceinline__ void eval_level5(const uint32_t *S, int Zs, uint32_t *D, int Zd, int np, int nq,
                                            const int *sig, int M, int tid) {
#pragma unroll
    for (int p = 0; p < 3; ++p) {
        const uint4 *P0 = reinterpret_cast<const uint4 *>(S + p * Zs);
        const uint4 *P1 = reinterpret_cast<const uint4 *>(S + (np + p) * Zs);
        const uint4 *P2 = reinterpret_cast<const uint4 *>(S + (2 * np + p) * Zs);
        for (int jq = tid; jq < nq; jq += kEvalFusedThreads) {
            uint4 y[5];
            eval_quad<-1>(P0, P1, P2, jq, sig[p] + 4 * jq, M, y);
#pragma unroll
            for (int e = 0; e < 5; ++e) reinterpret_cast<uint4 *>(D + (e * np + p) * Zd)[jq] = y[e];
        }
    }
}

template <int TL, int WL = kToomW>  // WL: the innermost level's point x = X^WL
__global__ void __launch_bounds__(kEvalFusedThreads, 3)
toom_eval_fused(const uint32_t *__restrict__ X0, uint32_t *__restrict__ Ya, uint32_t *__restrict__ Yb,
                const ToomEvalGeo geo, int64_t x0_words) {
    constexpr int w = kToomW;
    constexpr int wl = WL;  // the final level's point (its window still starts 2w before the tile)
    constexpr int NP0 = efpow3(TL), Z0 = efslot(TL, 0);
    extern __shared__ __align__(16) uint32_t efs[];
    __shared__ __align__(8) uint64_t mbar;
    check_poison(efs, unsigned(eval_fused_smem_words(TL) * 4));
    check_poison_sync();
    const int tid = threadIdx.x;
    const int tiles = (geo.chunks + geo.Tc - 1) / geo.Tc;
    const int64_t g = blockIdx.x / tiles;
    const int tile = int(blockIdx.x - g * tiles);
    const int op = blockIdx.y;
    const int LF = geo.LF, LFS = geo.LFS;
    const int c0 = tile * geo.Tc;
    const int tc = min(geo.Tc, geo.chunks - c0);  // chunks in this tile
    const int T = (tc * LF + 3) & ~3;             // coefficients (whole quads)
    const int k0 = c0 * LF;                       // multiple of 4 (planner)
    uint32_t *L0 = efs;

    // ---- stage the level-0 pieces: one bulk copy per piece (lanes of warp 0)
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid < 32) {
        uint32_t bytes = 0, dst = 0;
        int64_t src = 0;
        if (tid < NP0) {
            int sig = k0, rem = tid;  // sigma_0 of piece tid, digits p_TL first
#pragma unroll
            for (int l = TL; l >= 1; --l) {
                const int p = rem % 3;
                rem /= 3;
                sig = p * geo.M[l] + sig - 2 * w;
            }
            const int64_t A = (int64_t(op) * geo.G + g) * geo.N0 + sig;  // 16-byte aligned word index
            const int64_t E = A + T + 2 * w * TL;
            const int64_t a0c = A < 0 ? 0 : A, ec = E > x0_words ? x0_words : E;
            if (ec > a0c) {  // (words outside the operand are never read unmasked)
                bytes = uint32_t(ec - a0c) * 4u;
                src = a0c;
                dst = smem_u32(L0 + tid * Z0 + (a0c - A));
            }
        }
        const uint32_t total = __reduce_add_sync(0xffffffffu, bytes);
        if (tid == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar)),
                         "r"(total)
                         : "memory");
        __syncwarp();
        if (bytes)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                "l"(X0 + src), "r"(bytes), "r"(smem_u32(&mbar))
                : "memory");
    }
    // final level, per-thread work fixed for the whole CTA: item slots it =
    // tid + 256 u < 5 nq -> (point e, storage quad qi of the tile); a quad
    // holds the consecutive coefficients j0 .. j0+3 of one chunk (data mask
    // dm: pads are zero); precomputed once, no division in the loops
    const int nq = (tc * LFS) >> 2;
    // 5 nq <= 2 x 256: nq = Tc LFS / 4 <= 88 (Tc = 8 up to LF = 36, else 4; LFS <= 44)
    constexpr int FS = 2;
    int fe[FS], fs0[FS], fj0[FS];
    uint32_t fdm[FS];
#pragma unroll
    for (int u = 0; u < FS; ++u) {
        const int it = tid + u * kEvalFusedThreads;
        const int e = it / nq, qi = it - e * nq;
        const int s0 = qi * 4, c = s0 / LFS, r0 = s0 - c * LFS;
        fe[u] = it < 5 * nq ? e : -1;
        fs0[u] = s0;
        fj0[u] = c * LF + r0;
        fdm[u] = (LF - r0 >= 4) ? 0xFu : ((1u << max(LF - r0, 0)) - 1u);
    }
    const int Mt = geo.M[TL];
    // interior tile: every mask of the last level is true (no per-word checks)
    const bool interior = k0 >= 2 * w && k0 + tc * LF <= Mt;
    {
        uint32_t done = 0;
        while (!done)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(smem_u32(&mbar))
                : "memory");
    }
    uint32_t *out = (op ? Yb : Ya) + int64_t(c0) * LFS;
    const int64_t Ns = geo.Ns;
    // final level: the 5 points of every slot's quad from the three pieces of
    // the level-(TL-1) window of point e (P + e 3 Zp) (items 5 item5 + e')
    auto final_level = [&](const uint32_t *P, int Zp, int64_t item5) {
#pragma unroll
        for (int u = 0; u < FS; ++u) {
            if (fe[u] < 0) continue;
            const uint32_t *P0 = P + fe[u] * 3 * Zp, *P1 = P0 + Zp, *P2 = P1 + Zp;
            uint32_t v[5][4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int j = fj0[u] + r, k = k0 + j;
                const bool data = (fdm[u] >> r) & 1u;
                const bool ka = data && (interior || unsigned(k) < unsigned(Mt));
                const bool k1 = data && (interior || unsigned(k - wl) < unsigned(Mt));
                const bool k2 = data && (interior || unsigned(k - 2 * wl) < unsigned(Mt));
                const uint32_t a0 = ka ? P0[j + 2 * w] : 0u, a1 = ka ? P1[j + 2 * w] : 0u,
                               a2 = ka ? P2[j + 2 * w] : 0u;
                const uint32_t s1 = k1 ? P1[j + 2 * w - wl] : 0u, s2 = k2 ? P2[j + 2 * w - 2 * wl] : 0u;
                const uint32_t p1 = a0 ^ a1 ^ a2, xs = s1 ^ s2;
                v[0][r] = a0;
                v[1][r] = p1;
                v[2][r] = a0 ^ xs;
                v[3][r] = p1 ^ xs;
                v[4][r] = a2;
            }
            uint32_t *o = out + ((item5 * 5 + fe[u]) * 5) * Ns + fs0[u];
#pragma unroll
            for (int e = 0; e < 5; ++e)
                *reinterpret_cast<uint4 *>(o + e * Ns) = make_uint4(v[e][0], v[e][1], v[e][2], v[e][3]);
        }
    };
    if constexpr (TL == 1) {
        // TL = 1 has no outer evaluation point: every thread walks the quads
        for (int qi = tid; qi < nq; qi += kEvalFusedThreads) {
            const int s0 = qi * 4, c = s0 / LFS, r0 = s0 - c * LFS;
            uint32_t v[5][4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int j = c * LF + r0 + r, k = k0 + j;
                const bool data = r0 + r < LF;
                const bool ka = data && unsigned(k) < unsigned(Mt), k1 = data && unsigned(k - wl) < unsigned(Mt),
                           k2 = data && unsigned(k - 2 * wl) < unsigned(Mt);
                const uint32_t a0 = ka ? L0[j + 2 * w] : 0u, a1 = ka ? L0[Z0 + j + 2 * w] : 0u,
                               a2 = ka ? L0[2 * Z0 + j + 2 * w] : 0u;
                const uint32_t s1 = k1 ? L0[Z0 + j + 2 * w - wl] : 0u, s2 = k2 ? L0[2 * Z0 + j + 2 * w - 2 * wl] : 0u;
                const uint32_t p1 = a0 ^ a1 ^ a2, xs = s1 ^ s2;
                v[0][r] = a0;
                v[1][r] = p1;
                v[2][r] = a0 ^ xs;
                v[3][r] = p1 ^ xs;
                v[4][r] = a2;
            }
#pragma unroll
            for (int e = 0; e < 5; ++e)
                *reinterpret_cast<uint4 *>(out + (g * 5 + e) * Ns + s0) = make_uint4(v[e][0], v[e][1], v[e][2], v[e][3]);
        }
    } else if constexpr (TL == 2) {
        constexpr int Z1 = efslot(2, 1);
        uint32_t *L1 = L0 + NP0 * Z0;  // [e1][p2]
        int sig[3];
#pragma unroll
        for (int p = 0; p < 3; ++p) sig[p] = p * geo.M[2] + k0 - 2 * w;
        eval_level5(L0, Z0, L1, Z1, 3, (T + 2 * w) >> 2, sig, geo.M[1], tid);
        __syncthreads();
        final_level(L1, Z1, g);
    } else {
        static_assert(TL == 3, "1..3 Toom levels");
        constexpr int Z1 = efslot(3, 1), Z2 = efslot(3, 2);
        uint32_t *L1 = L0 + NP0 * Z0;  // [p2 p3] (9 pieces) of one e1
        uint32_t *L2 = L1 + 9 * Z1;    // [e2][p3] (15 pieces)
        const int nq1 = (T + 4 * w) >> 2, nq2 = (T + 2 * w) >> 2;
        int sig2[3];
#pragma unroll
        for (int p = 0; p < 3; ++p) sig2[p] = p * geo.M[3] + k0 - 2 * w;
        const int M2 = geo.M[2];
        // phases: L1(0) | L2(0) | final(0) + L1(1) | L2(1) | ... | final(4):
        // the next point's level-1 pass writes only L1, which the final level
        // does not read, so it shares the final level's phase (11 phases
        // instead of 15 for the same barriers)
        eval_l1_point_rt(0, L0, L1, geo, k0, nq1, tid);
        __syncthreads();
#pragma unroll 1
        for (int e1 = 0; e1 < 5; ++e1) {
            eval_level5(L1, Z1, L2, Z2, 3, nq2, sig2, M2, tid);
            __syncthreads();
            final_level(L2, Z2, g * 5 + e1);
            if (e1 < 4) {
                eval_l1_point_rt(e1 + 1, L0, L1, geo, k0, nq1, tid);
                __syncthreads();
            }
        }
    }
}

// One Toom-3 interpolation level, from the 5 products C_e of every output
// item i (items 5i+e, Lin coefficients in the (LFi, LFSi) layout, stride inS)
// to R = c0 + c1 y + c2 y^2 + c3 y^3 + c4 y^4, y = X^M (6M coefficients,
// plain, stride outS).  Grouped numerators: after
// the exact division by x, each numerator u_j is a 4-term XOR of inputs and
// the exact division by x + 1 = 1 + X^w is a prefix XOR along the w chains
// k = r (mod w):
//   c3 = scan(u3),                            u3[k] = (C0+C1+Cx+Cx1)[k+w]
//   c2 = scan(u2) + (1 + x + x^2) Cinf,       u2[k] = C1[k+w] + Cx[k] + Cx1[k+w] + Cx1[k]
//   c1 = C0 + C1 + scan(u1) + (x + x^2) Cinf, u1[k] = C0[k+w] + Cx[k+w] + Cx[k] + Cx1[k]
// Two kernels: (A) per block of kToomBlk coefficients, u1..u3 and their
// block-local chain scans (written to Q) plus each chain's block total;
// (B) per block of outputs, the carries (XOR of earlier blocks' totals) and
// the assembly of R from two c_j terms per coefficient.
constexpr int kToomBlk = 2048;   // coefficients per block (multiple of w)
constexpr int kToomScanT = 256;  // threads of the scan kernel
// staging index: 16 pad words per 128, so the two half-warps of a row scan
// (rows 8 apart = 128 words) hit different banks
__device__ __forceinline__ int tstg(int h) { return h + 16 * (h >> 7); }
__host__ __device__ constexpr int toom_stg_stride(int blk) {
    return (blk + 3 * kToomW) + 16 * (((blk + 3 * kToomW) >> 7) + 1);
}
constexpr int kToomStgStride = toom_stg_stride(kToomBlk);

struct ToomIn {
    const uint32_t *C;  // item base (5 products)
    int64_t inS;
    int LFi, LFSi, Lin;
    float invLF;
    __device__ __forceinline__ uint32_t rd(int e, int k) const {
        if (k < 0 || k >= Lin) return 0u;
        if (LFi == LFSi) return __ldg(C + e * inS + k);
        // exact: k < 2^24, LF <= 64 (fraction >= 0.5/LF from an integer)
        const int c = __float2int_rz((float(k) + 0.5f) * invLF);
        return __ldg(C + e * inS + int64_t(c) * LFSi + (k - c * LFi));
    }
};

// Kernel A: block b of item i.  The block's inputs (5 products over
// [k0 - 2w, k0 + B + w)) are staged in shared memory once; u1..u3 are scanned
// along their chains inside the block; Q receives c0, c1..c3 without the
// carry from earlier blocks, and c4 (5 x 2M words per item); Tot receives
// each chain's block total.
__global__ void __launch_bounds__(kToomScanT)
toom_interp_scan(const uint32_t *__restrict__ Cin, uint32_t *__restrict__ Q, uint32_t *__restrict__ Tot, int M,
                 int w, int LFi, int LFSi, int64_t inS, int Lin, int nb) {
    extern __shared__ uint32_t tsm[];
    const int H = kToomBlk + 3 * w;          // staged span per input
    constexpr int HP = kToomStgStride;        // padded stride per input (see tstg)
    uint32_t *Stg = tsm;                      // [5][H], index k - (k0 - 2w)
    check_poison(tsm, unsigned(5 * HP * 4));
    check_poison_sync();
    const int64_t item = blockIdx.x / nb;
    const int b = int(blockIdx.x - item * nb);
    const int L = 2 * M, k0 = b * kToomBlk, kb = k0 - 2 * w;
    const ToomIn in{Cin + item * 5 * inS, inS, LFi, LFSi, Lin, 1.0f / float(LFi)};
    // staging: all of a thread's loads (5 inputs x ceil(H/256)) are issued
    // before the first shared-memory store -- one memory round trip per CTA
    {
        constexpr int T = kToomScanT, NI = (kToomBlk + 3 * kToomW + T - 1) / T;
        const bool plain = LFi == LFSi;
        uint32_t v[5][NI];
#pragma unroll
        for (int e = 0; e < 5; ++e) {
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const int h = int(threadIdx.x) + i * T, k = kb + h;
                uint32_t x = 0;
                if (h < H && k >= 0 && k < Lin) {
                    int64_t off = k;
                    if (!plain) {
                        const int c = __float2int_rz((float(k) + 0.5f) * in.invLF);
                        off = int64_t(c) * LFSi + (k - c * LFi);
                    }
                    x = __ldg(in.C + e * inS + off);
                }
                v[e][i] = x;
            }
        }
#pragma unroll
        for (int e = 0; e < 5; ++e) {
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const int h = int(threadIdx.x) + i * T;
                if (h < H) Stg[e * HP + tstg(h)] = v[e][i];
            }
        }
    }
    __syncthreads();
    auto S = [&](int e, int k) -> uint32_t { return Stg[e * HP + tstg(k - kb)]; };
    // the block as ROWS x w: thread (column r, segment sg) keeps SEGR rows of
    // u1..u3 and their running prefix in registers; segment carries go
    // through shared memory
    constexpr int W = kToomW, ROWS = kToomBlk / W, NSEG = kToomScanT / W, SEGR = ROWS / NSEG;
    __shared__ uint32_t stot[3][NSEG][W];
    check_poison(stot, sizeof(stot));
    check_poison_sync();
    const int r = int(threadIdx.x) % W, sg = int(threadIdx.x) / W;
    const int kr = k0 + sg * SEGR * W + r;  // first coefficient of this thread
    uint32_t v1[SEGR], v2[SEGR], v3[SEGR];
    {
        uint32_t a1 = 0, a2 = 0, a3 = 0;
        uint32_t cx = S(2, kr), cx1 = S(3, kr);
#pragma unroll
        for (int i = 0; i < SEGR; ++i) {
            const int k = kr + i * W;
            const uint32_t c0w = S(0, k + W), c1w = S(1, k + W), cxw = S(2, k + W), cx1w = S(3, k + W);
            a1 ^= c0w ^ cxw ^ cx ^ cx1;
            a2 ^= c1w ^ cx ^ cx1w ^ cx1;
            a3 ^= c0w ^ c1w ^ cxw ^ cx1w;
            v1[i] = a1;
            v2[i] = a2;
            v3[i] = a3;
            cx = cxw;
            cx1 = cx1w;
        }
        stot[0][sg][r] = a1;
        stot[1][sg][r] = a2;
        stot[2][sg][r] = a3;
    }
    __syncthreads();
    uint32_t g1 = 0, g2 = 0, g3 = 0;  // carry from the block's earlier segments
    for (int s2 = 0; s2 < sg; ++s2) {
        g1 ^= stot[0][s2][r];
        g2 ^= stot[1][s2][r];
        g3 ^= stot[2][s2][r];
    }
    uint32_t *q = Q + item * 5 * int64_t(L);
    {
        uint32_t c4m2 = S(4, kr - 2 * W), c4m1 = S(4, kr - W);
#pragma unroll
        for (int i = 0; i < SEGR; ++i) {
            const int k = kr + i * W;
            const uint32_t c0 = S(0, k), c4 = S(4, k), c4w = c4m1 ^ c4m2;
            if (k < L) {
                q[k] = c0;
                q[L + k] = v1[i] ^ g1 ^ c0 ^ S(1, k) ^ c4w;  // c1 (no block carry)
                q[2 * L + k] = v2[i] ^ g2 ^ c4 ^ c4w;       // c2 (no block carry)
                q[3 * L + k] = v3[i] ^ g3;                  // c3 (no block carry)
                q[4 * L + k] = c4;
            }
            c4m2 = c4m1;
            c4m1 = c4;
        }
    }
    if (sg == NSEG - 1) {  // block totals per chain (the last segment's inclusive values)
        uint32_t *tt = Tot + (item * nb + b) * 3 * W;
        tt[r] = v1[SEGR - 1] ^ g1;
        tt[W + r] = v2[SEGR - 1] ^ g2;
        tt[2 * W + r] = v3[SEGR - 1] ^ g3;
    }
}

// Resident-root form (RES, the innermost Toom level of a plan whose last
// global Karatsuba pass is a single level, n=57637): the CTA first builds its
// five node-problem roots in shared memory straight from their three path
// products each (the k3_interp<1> recombination, per storage quad w of a
// path product: root octant m = 0..7 from the quarters lo_q, hi_q, mid_q at
// w), then walks the blocks reading the roots in place -- no staging and no
// root round trip through HBM (k3_interp<1> wrote and this level re-read
// 2.3 GB per n=57637 call).  Path product c (0 lo, 1 hi, 2 mid) of node
// problem np is at P + (3 np + c) inS, chunked (LF, LFS), quarters of qw
// storage words; root octants have oc = (qw / LFS) LF coefficients.
struct KRootIn {
    const uint32_t *P;
    int64_t inS;
    int qw, oc, LF, LFS;
    int hp;  // resident root stride in shared memory, words
};
// words per resident root: slots h = k + 2w for k in [-2w, nb blk + w) in the
// tstg layout, plus a spare slot past the walk's span (branch-free stores)
__host__ __device__ constexpr int kres_words(int nb, int blk) {
    return (nb * blk + 3 * kToomW) + 16 * (((nb * blk + 3 * kToomW) >> 7) + 1);
}

// Single-kernel variant: one CTA per item walks its blocks in order, so the
// chain carries flow from block to block in shared memory and the c_j go
// straight into R (first contribution to a coefficient written, the second
// added by an L2 XOR reduction): no c_j round trip through HBM, one launch.
// NT = 512 (with BLK = 4096) for levels with at most one product per SM.
template <int BLK, bool RES, int NT = kToomScanT, int W = kToomW>
__global__ void __launch_bounds__(NT, RES ? 2 : (NT > 256 ? 1 : 3))
toom_interp_seq(const uint32_t *__restrict__ Cin, uint32_t *__restrict__ R, int M, int LFi, int LFSi, int64_t inS,
                int Lin, int64_t outS, const KRootIn kr) {
    extern __shared__ uint32_t tsm[];
    constexpr int ROWS = BLK / W, NSEG = NT / W, SEGR = ROWS / NSEG;
    constexpr int H = BLK + 3 * W;  // (W <= kToomW: the strides below are sized for kToomW)
    const int HP = RES ? kr.hp : toom_stg_stride(BLK);  // padded stride per input (see tstg)
    uint32_t *Stg = tsm;  // [5][HP]
    __shared__ uint32_t stot[3][NSEG][W];
    __shared__ uint32_t bcar[3][W];  // carry into the current block, per chain
    check_poison(tsm, unsigned(5 * HP * 4));
    check_poison(stot, sizeof(stot));
    check_poison(bcar, sizeof(bcar));
    check_poison_sync();
    const int64_t item = blockIdx.x;
    const int L = 2 * M, nb = (L + BLK - 1) / BLK;
    if constexpr (RES) {
        // roots -> Stg[e HP + tstg(k + 2w)], k in [-2w, nb BLK + w); zero outside [0, Lin)
        const int span = nb * BLK + 3 * W;  // resident slots h = k + 2w the block walk reads
        for (int h = int(threadIdx.x); h < span; h += NT) {
            const int k = h - 2 * W;
            if (k < 0 || k >= Lin) {
#pragma unroll
                for (int e = 0; e < 5; ++e) Stg[e * HP + tstg(h)] = 0u;
            }
        }
        const int q4 = kr.qw >> 2, qsz = kr.LFS >> 2;  // quads per quarter / per chunk
        const uint4 *P4 = reinterpret_cast<const uint4 *>(kr.P + item * 15 * kr.inS);
        const int64_t cs = kr.inS >> 2;  // path-product stride, quads
#pragma unroll 1  // (2-3 items in flight per thread measured 4-16 % slower)
        for (int x = int(threadIdx.x); x < 5 * q4; x += NT) {
            const int e = x / q4, wq = x - e * q4;
            const uint4 *lo = P4 + (3 * e) * cs + wq, *hi = lo + cs, *mid = hi + cs;
            uint4 l[4], hh[4], m[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                l[q] = __ldg(lo + q * q4);
                hh[q] = __ldg(hi + q * q4);
                m[q] = __ldg(mid + q * q4);
            }
            uint4 o[8];
#pragma unroll
            for (int i = 0; i < 2; ++i) {  // k3_rec<1>
                const uint4 T = l[2 + i] ^ hh[i];
                o[i] = l[i];
                o[2 + i] = xor3(T, l[i], m[i]);
                o[4 + i] = xor3(T, hh[2 + i], m[2 + i]);
                o[6 + i] = hh[2 + i];
            }
            const int c = wq / qsz, r0 = 4 * (wq - c * qsz);  // chunk, first word in it
            const int kq = c * kr.LF + r0 + 2 * W;             // resident index of octant 0's first word
            const int base = e * HP, dump = base + HP - 1;  // (a spare slot past the walk's span)
            const int nw = min(4, kr.LF - r0);             // data words in this storage quad
#pragma unroll
            for (int mo = 0; mo < 8; ++mo) {
                const uint32_t vv[4] = {o[mo].x, o[mo].y, o[mo].z, o[mo].w};
                // one tstg per quad: the four words are consecutive slots unless
                // they cross a 128-word pad boundary (then +16 from there on);
                // a chunk's pad word goes to the spare slot (no branches)
                const int h0 = kq + mo * kr.oc;
                const int t0 = base + tstg(h0), cross = 128 - (h0 & 127);
#pragma unroll
                for (int j = 0; j < 4; ++j) Stg[j < nw ? t0 + j + (j >= cross ? 16 : 0) : dump] = vv[j];
            }
        }
        __syncthreads();
    }
    const ToomIn in{Cin + item * 5 * inS, inS, LFi, LFSi, Lin, 1.0f / float(LFi)};
    uint32_t *Rg = R + item * outS;
    const bool plain = LFi == LFSi;
    // quad staging: plain inputs whose item/row offsets and length are whole
    // quads (block starts are multiples of 4: BLK and 2w are)
    const bool vec = plain && (inS % 4) == 0 && (Lin % 4) == 0 &&
                     (reinterpret_cast<uintptr_t>(Cin) & 15) == 0;
    const int r = int(threadIdx.x) % W, sg = int(threadIdx.x) / W;
    if (threadIdx.x < 3 * W) bcar[threadIdx.x / W][threadIdx.x % W] = 0u;
#pragma unroll 1
    for (int b = 0; b < nb; ++b) {
        const int k0 = b * BLK, kb = k0 - 2 * W;
        if constexpr (RES) {
            __syncthreads();  // previous block's readers of stot / bcar are done
        } else if (vec) {  // plain, 16-byte aligned inputs: quads, all in flight per half
            constexpr int T = NT, H4 = H / 4, NQ = (5 * H4 + T - 1) / T, NH = (NQ + 1) / 2;
            __syncthreads();  // previous block's readers of Stg / stot are done
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                uint4 q4[NH];
#pragma unroll
                for (int i = 0; i < NH; ++i) {
                    const int x = int(threadIdx.x) + (half * NH + i) * T;
                    const int e = x / H4, hq = x - e * H4, k = kb + 4 * hq;
                    uint4 v = make_uint4(0, 0, 0, 0);
                    if (x < 5 * H4 && k >= 0 && k < Lin)  // Lin % 4 == 0: whole quads
                        v = __ldg(reinterpret_cast<const uint4 *>(in.C + e * inS + k));
                    q4[i] = v;
                }
#pragma unroll
                for (int i = 0; i < NH; ++i) {
                    const int x = int(threadIdx.x) + (half * NH + i) * T;
                    const int e = x / H4, hq = x - e * H4;
                    if (x < 5 * H4) *reinterpret_cast<uint4 *>(Stg + e * HP + tstg(4 * hq)) = q4[i];
                }
            }
        } else         {  // staging: every load of the block in flight at once
            constexpr int T = NT, NI = (H + T - 1) / T;
            uint32_t v[5][NI];
            // storage offset of coefficient k = kb + tid + i T, walked
            // incrementally (one chunk split per block instead of one per
            // word; the per-word split was the kernel's top cost)
            int off[NI];
            bool ok[NI];
            {
                const int k0w = kb + int(threadIdx.x);
                const int kk = k0w < 0 ? 0 : k0w;  // (negative k only in block 0, masked below)
                int c = plain ? 0 : kk / LFi, rr = plain ? kk : kk - c * LFi;
                const int dc = plain ? 0 : T / LFi, dr = plain ? T : T - dc * LFi;
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                    const int h = int(threadIdx.x) + i * T, k = kb + h;
                    ok[i] = h < H && k >= 0 && k < Lin;
                    off[i] = plain ? k : c * LFSi + rr;
                    if (k0w < 0 && k + T >= 0 && k < 0) {  // the walk starts at the first k >= 0
                        const int kn = k + T;
                        c = plain ? 0 : kn / LFi;
                        rr = plain ? kn : kn - c * LFi;
                    } else if (k >= 0) {
                        rr += dr;
                        c += dc;
                        if (!plain && rr >= LFi) {
                            rr -= LFi;
                            ++c;
                        }
                    }
                }
            }
            const uint32_t *Ce = in.C;
#pragma unroll
            for (int e = 0; e < 5; ++e) {
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                    // unconditional load from a clamped in-row offset, value masked:
                    // no predicated address arithmetic (tools/ct_sass_audit.py)
                    const uint32_t x = __ldg(Ce + (ok[i] ? off[i] : 0));
                    v[e][i] = ok[i] ? x : 0u;
                }
                Ce += inS;
            }
            __syncthreads();  // previous block's readers of Stg / stot are done
#pragma unroll
            for (int e = 0; e < 5; ++e) {
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                    const int h = int(threadIdx.x) + i * T;
                    if (h < H) Stg[e * HP + tstg(h)] = v[e][i];
                }
            }
        }
        if constexpr (!RES) __syncthreads();
        auto S = [&](int e, int k) -> uint32_t { return Stg[e * HP + tstg(RES ? k + 2 * W : k - kb)]; };
        const int kr0 = k0 + sg * SEGR * W + r;
        uint32_t v1[SEGR], v2[SEGR], v3[SEGR];
        {
            uint32_t a1 = 0, a2 = 0, a3 = 0;
            uint32_t cx = S(2, kr0), cx1 = S(3, kr0);
#pragma unroll
            for (int i = 0; i < SEGR; ++i) {
                const int k = kr0 + i * W;
                const uint32_t c0w = S(0, k + W), c1w = S(1, k + W), cxw = S(2, k + W), cx1w = S(3, k + W);
                a1 ^= c0w ^ cxw ^ cx ^ cx1;
                a2 ^= c1w ^ cx ^ cx1w ^ cx1;
                a3 ^= c0w ^ c1w ^ cxw ^ cx1w;
                v1[i] = a1;
                v2[i] = a2;
                v3[i] = a3;
                cx = cxw;
                cx1 = cx1w;
            }
            stot[0][sg][r] = a1;
            stot[1][sg][r] = a2;
            stot[2][sg][r] = a3;
        }
        __syncthreads();
        uint32_t g1 = bcar[0][r], g2 = bcar[1][r], g3 = bcar[2][r];
        for (int s2 = 0; s2 < sg; ++s2) {
            g1 ^= stot[0][s2][r];
            g2 ^= stot[1][s2][r];
            g3 ^= stot[2][s2][r];
        }
        // c_0..c_4 of each row once: first contributions to R[k + jM] (k < M,
        // or j = 4) are plain stores; c_0..c_3 of rows with k >= M are kept
        // in registers for the read-modify-write after the barrier
        uint32_t keep[SEGR][4];
        {
            uint32_t c4m2 = S(4, kr0 - 2 * W), c4m1 = S(4, kr0 - W);
#pragma unroll
            for (int i = 0; i < SEGR; ++i) {
                const int k = kr0 + i * W;
                const uint32_t c0 = S(0, k), c4 = S(4, k), c4w = c4m1 ^ c4m2;
                const uint32_t cj[5] = {c0, v1[i] ^ g1 ^ c0 ^ S(1, k) ^ c4w, v2[i] ^ g2 ^ c4 ^ c4w, v3[i] ^ g3, c4};
                if (k < L) {
                    if (k < M) {
#pragma unroll
                        for (int j = 0; j < 5; ++j) Rg[k + j * M] = cj[j];
                    } else {
                        Rg[k + 4 * M] = c4;
                    }
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) keep[i][j] = cj[j];
                c4m2 = c4m1;
                c4m1 = c4;
            }
        }
        // a second contribution's first one comes from coefficient k - M: from
        // this block only when M < BLK (then a barrier orders the two)
        if (M < BLK) __syncthreads();
        // ... second contributions XOR onto them (written by this CTA, earlier
        // or before the barrier above) as fire-and-forget L2 reductions
        // (red.global.xor: no load round trip; XOR commutes, and a barrier
        // orders every first contribution before them)
#pragma unroll
        for (int i = 0; i < SEGR; ++i) {
            const int k = kr0 + i * W;
            if (k < L && k >= M) {
#pragma unroll
                for (int j = 0; j < 4; ++j) atomicXor(Rg + k + j * M, keep[i][j]);
            }
        }
        if (sg == NSEG - 1) {  // carry into the next block: this block's chain totals
            bcar[0][r] = v1[SEGR - 1] ^ g1;
            bcar[1][r] = v2[SEGR - 1] ^ g2;
            bcar[2][r] = v3[SEGR - 1] ^ g3;
        }
    }
}

// Kernel B: output block ob of item i.  R[k] = c_a[k - aM] + c_{a-1}[k - (a-1)M]
// (a = k / M), the c_1..c_3 terms plus their chain carries (XOR of the earlier
// blocks' totals).
__global__ void __launch_bounds__(256)
toom_interp_assemble(const uint32_t *__restrict__ Q, const uint32_t *__restrict__ Tot, uint32_t *__restrict__ R,
                     int M, int w, int nb, int nbo, int64_t outS) {
    extern __shared__ uint32_t carry[];  // [nb][3][w]
    check_poison(carry, unsigned(nb * 3 * w * 4));
    check_poison_sync();
    const int64_t item = blockIdx.x / nbo;
    const int ob = int(blockIdx.x - item * nbo);
    const int L = 2 * M;
    const uint32_t *tot = Tot + item * nb * 3 * w;
    // chain carries = exclusive prefix (over blocks) of the block totals: all
    // totals loaded by all threads at once (coalesced, independent), then a
    // short in-shared-memory scan per chain
    for (int x = threadIdx.x; x < nb * 3 * w; x += blockDim.x) carry[x] = __ldg(tot + x);
    __syncthreads();
    for (int c = threadIdx.x; c < 3 * w; c += blockDim.x) {
        uint32_t acc = 0;
        for (int b = 0; b < nb; ++b) {
            const uint32_t v = carry[b * 3 * w + c];
            carry[b * 3 * w + c] = acc;
            acc ^= v;
        }
    }
    __syncthreads();
    const uint32_t *q = Q + item * 5 * int64_t(L);
    auto cj = [&](int j, int k) -> uint32_t {
        uint32_t v = __ldg(q + j * int64_t(L) + k);
        if (j >= 1 && j <= 3) v ^= carry[(k / kToomBlk) * 3 * w + (j - 1) * w + (k & (w - 1))];
        return v;
    };
    uint32_t *out = R + item * outS;
    const int kbeg = ob * kToomBlk, kend = min(kbeg + kToomBlk, 6 * M);
    constexpr int NI = kToomBlk / 256;  // outputs per thread, all loads in flight
    const int a0 = kbeg / M;
    if (a0 == (kend - 1) / M) {
        // the whole block lies in [aM, (a+1)M): two fixed streams
        // R[kk] = c_a[kk - aM] + c_{a-1}[kk - (a-1)M]
        const int a = a0;
        const bool ha = a <= 4, hb = a >= 1;
        const uint32_t *pa = q + (ha ? a : 0) * int64_t(L) - int64_t(a) * M;
        const uint32_t *pb = q + (hb ? a - 1 : 0) * int64_t(L) - int64_t(a - 1) * M;
        const uint32_t *ca = carry + (a - 1) * w, *cb = carry + (a - 2) * w;  // per-block stride 3w
        const bool cra = a >= 1 && a <= 3, crb = a - 1 >= 1 && a - 1 <= 3;
        uint32_t v[NI];
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const int kk = kbeg + int(threadIdx.x) + i * 256;
            uint32_t x = 0;
            if (kk < kend) {
                if (ha) {
                    const int k = kk - a * M;
                    x ^= __ldg(pa + kk);
                    if (cra) x ^= ca[(k / kToomBlk) * 3 * w + (k & (w - 1))];
                }
                if (hb) {
                    const int k = kk - (a - 1) * M;
                    x ^= __ldg(pb + kk);
                    if (crb) x ^= cb[(k / kToomBlk) * 3 * w + (k & (w - 1))];
                }
            }
            v[i] = x;
        }
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const int kk = kbeg + int(threadIdx.x) + i * 256;
            if (kk < kend) out[kk] = v[i];
        }
        return;
    }
    uint32_t v[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
        const int kk = kbeg + int(threadIdx.x) + i * 256;
        const int a = (kk >= M) + (kk >= 2 * M) + (kk >= 3 * M) + (kk >= 4 * M) + (kk >= 5 * M);
        uint32_t x = 0;
        if (kk < kend) {
            if (a <= 4) x ^= cj(a, kk - a * M);
            if (a >= 1) x ^= cj(a - 1, kk - (a - 1) * M);
        }
        v[i] = x;
    }
#pragma unroll
    for (int i = 0; i < NI; ++i) {
        const int kk = kbeg + int(threadIdx.x) + i * 256;
        if (kk < kend) out[kk] = v[i];
    }
}

// ------------------------------------------------------------------- K3
// Global Karatsuba interpolation, D levels in one pass.  Node products are
// split into 4 quarters; a node's quarter index w only touches its
// children's quarter index w, so each thread owns one w of one top node and
// rebuilds the D-level subtree in registers.
template <int D>
__device__ __forceinline__ void k3_rec(uint32_t *out, const uint32_t *__restrict__ Pin,
                                       int64_t inStride, int64_t desc, int qw, int w) {
    if constexpr (D == 0) {
        const uint32_t *src = Pin + desc * inStride + w;
#pragma unroll
        for (int q = 0; q < 4; ++q) out[q] = __ldg(src + int64_t(q) * qw);
    } else {
        constexpr int Lc = 2 << D;  // child vector length
        constexpr int half = Lc / 2;
        k3_rec<D - 1>(out, Pin, inStride, desc * 3 + 0, qw, w);
        k3_rec<D - 1>(out + Lc, Pin, inStride, desc * 3 + 1, qw, w);
        uint32_t m[Lc];
        k3_rec<D - 1>(m, Pin, inStride, desc * 3 + 2, qw, w);
#pragma unroll
        for (int i = 0; i < half; ++i) {
            const uint32_t T = out[half + i] ^ out[Lc + i];
            out[half + i] = T ^ out[i] ^ m[i];
            out[Lc + i] = T ^ out[Lc + half + i] ^ m[half + i];
        }
    }
}

// plainLF > 0 (the last pass of a Toom plan): the output root is written
// PLAIN -- chunk pads dropped, coefficient c LF + r at word c LF + r -- so
// the Toom interpolation stages it with 16-byte loads; qw is a multiple of
// LFS there, so all of a thread's words share one chunk residue r.
template <int D>
__global__ void __launch_bounds__(kThreads)
k3_interp(const uint32_t *__restrict__ Pin, uint32_t *__restrict__ Pout, int64_t items, int qw,
          int64_t inStride, int64_t outStride, int plainLF, int LFS) {
    // blocks walk the nodes in REVERSE order: the node kernel wrote them in
    // forward order, so the most recently written (still L2-resident)
    // products are consumed first instead of being evicted by the rest
    const int64_t nblk = (items + blockDim.x - 1) / blockDim.x;
    const int64_t item = (nblk - 1 - int64_t(blockIdx.x)) * blockDim.x + threadIdx.x;
    if (item >= items) return;
    const int64_t node = item / qw;
    const int w = int(item - node * qw);
    uint32_t v[4 << D];
    k3_rec<D>(v, Pin, inStride, node, qw, w);  // leaves: node*3^D + local
    if (plainLF > 0) {
        const int c0 = w / LFS, r = w - c0 * LFS, qc = qw / LFS;
        if (r >= plainLF) return;  // a chunk pad: not stored in the plain root
        uint32_t *dst = Pout + node * outStride + int64_t(c0) * plainLF + r;
#pragma unroll
        for (int m = 0; m < (4 << D); ++m) dst[int64_t(m) * qc * plainLF] = v[m];
        return;
    }
    uint32_t *dst = Pout + node * outStride + w;
#pragma unroll
    for (int m = 0; m < (4 << D); ++m) dst[int64_t(m) * qw] = v[m];
}

// K4: the tile's 64 TW coefficients of the root product are gathered (and,
// for the ring, folded: c[k] ^= c[k+n]; k >= n zero) into the
// stage, then thread i transposes half-word i back to 32 rows and stores its
// 32-bit halves (adjacent threads = adjacent halves of a row: coalesced).
// QD > 0: chunked root (LF <= 40 data words per chunk, QD = ceil(LF / 4) data
// quads, chunk stride LFS): gather items are (chunk, data quad) pairs, quad
// fastest (coalesced 16-byte loads), mapped with compile-time divisions.
// QD = 0: plain root (coefficient k at word k; Toom plans): items are quads.
// (Round 2: the per-quad runtime division, the per-word range/pad tests and
// an always-run zero-fill loop made the old form issue-bound: 1648 warp
// instructions per tile at d=1024, 81 % issue, 57 % of HBM.)
template <int TW, int QD>
__global__ void __launch_bounds__(2 * TW)
k4_unslice(const uint32_t *__restrict__ Croot, uint64_t *__restrict__ out, int64_t batch, int tout,
           int LF, int LFS, int64_t rootStride, int ncyc, int tiles) {
    constexpr int TC = 64 * TW, TT = 2 * TW;  // coefficients, threads per tile
    __shared__ uint32_t stage[TC + TC / 32];
    check_poison(stage, sizeof(stage));
    check_poison_sync();
    const int tid = threadIdx.x;
    const int64_t g = blockIdx.x / tiles;
    const int tile = int(blockIdx.x - g * tiles);
    const uint32_t *Cg = Croot + g * rootStride;
    const int k0 = tile * TC, kend = min(k0 + TC, 64 * tout);
    const int kvalid = ncyc > 0 ? min(kend, ncyc) : kend;
    // positions no gather writes (k >= n of the ring, or past the output) are zero
    for (int k = max(kvalid, k0) + tid; k < k0 + TC; k += TT) stage[stg(k - k0)] = 0u;
    // gather root coefficients [ka, kb) into stage index k - ka (XOR when folding)
    auto gather = [&](int ka, int kb, bool fold) {
        const uint4 *C4 = reinterpret_cast<const uint4 *>(Cg);
        const int span = kb - ka;
        if constexpr (QD > 0) {
            const int c0 = ka / LF, items = ((kb - 1) / LF - c0 + 1) * QD, qs = LFS >> 2;
            constexpr int NI = (TC / (4 * QD - 3) + 2) * QD / TT + 1;  // items per thread (LF >= 4 QD - 3)
            uint4 v[NI];
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const int it = tid + i * TT, cc = it / QD, iq = it - cc * QD;
                v[i] = it < items ? __ldg(C4 + (c0 + cc) * qs + iq) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const int it = tid + i * TT, cc = it / QD, iq = it - cc * QD;
                const int kq = (c0 + cc) * LF + 4 * iq - ka;  // stage index of the quad's first word
                const uint32_t vv[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int kk = kq + j;
                    if (it < items && 4 * iq + j < LF && unsigned(kk) < unsigned(span)) {
                        if (fold) stage[stg(kk)] ^= vv[j];
                        else stage[stg(kk)] = vv[j];
                    }
                }
            }
        } else {
            const int q0 = ka >> 2, items = ((kb + 3) >> 2) - q0;  // root rows are whole quads
            constexpr int NI = (TC / 4 + 1 + TT - 1) / TT;
            uint4 v[NI];
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const int it = tid + i * TT;
                v[i] = it < items ? __ldg(C4 + q0 + it) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const int it = tid + i * TT, kq = 4 * (q0 + it) - ka;
                const uint32_t vv[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int kk = kq + j;
                    if (it < items && unsigned(kk) < unsigned(span)) {
                        if (fold) stage[stg(kk)] ^= vv[j];
                        else stage[stg(kk)] = vv[j];
                    }
                }
            }
        }
    };
    if (k0 < kvalid) gather(k0, kvalid, false);
    __syncthreads();
    if (ncyc > 0 && k0 < kvalid) {  // fold: coefficients [k0+n, kvalid+n)
        gather(k0 + ncyc, kvalid + ncyc, true);
        __syncthreads();
    }
    uint32_t x[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = stage[stg(32 * tid + i)];
    transpose32(x);
    const int u = tile * TW + (tid >> 1);
    if (u < tout) {
        const int rows = int(batch - g * 32 < 32 ? batch - g * 32 : 32);
        uint32_t *po = reinterpret_cast<uint32_t *>(out) + ((g * 32) * tout + u) * 2 + (tid & 1);
        const int64_t rs = 2 * int64_t(tout);
        if (rows == 32) {
#pragma unroll
            for (int pr = 0; pr < 32; ++pr) po[pr * rs] = x[pr];
        } else {
#pragma unroll
            for (int pr = 0; pr < 32; ++pr)
                if (pr < rows) po[pr * rs] = x[pr];
        }
    }
}

// K3 (last pass) + K4 in one CTA per group (Karatsuba-only plans with many
// groups, the configs[4] d-sweep): the group's root is rebuilt by the last
// global interpolation pass (k3_rec<D> per quarter index w, all 4 2^D root
// slabs of that w) straight into a shared stage in coefficient order (the
// K4 stage layout; the ring's fold XORs coefficient k >= n onto k - n), then
// every thread transposes half-word columns back to rows as in K4.  The root
// never goes through HBM (d=4096: 1.2 GB written and re-read per call).
constexpr int kK34Threads = 256;
template <int D>
__global__ void __launch_bounds__(kK34Threads, D <= 2 ? 4 : 2)  // D <= 3 (see k34_fused)
k34_root_unslice(const uint32_t *__restrict__ Pin, uint64_t *__restrict__ out, int64_t batch, int tout, int qw,
                 int64_t inStride, int LF, int LFS, int ncyc) {
    extern __shared__ uint32_t stage[];  // [stg(64 tout)]
    const int KS = 64 * tout;            // output coefficients
    check_poison(stage, unsigned(stg(KS) * 4));
    check_poison_sync();
    const int tid = threadIdx.x;
    const int64_t g = blockIdx.x;
    if (ncyc > 0) {  // the fold accumulates: zero first
        for (int k = tid; k < KS; k += kK34Threads) stage[stg(k)] = 0u;
        __syncthreads();
    }
    const int qc = qw / LFS;  // chunks per root slab
#pragma unroll 1
    for (int w = tid; w < qw; w += kK34Threads) {
        uint32_t v[4 << D];
        k3_rec<D>(v, Pin, inStride, g, qw, w);
        const int cw = w / LFS, r = w - cw * LFS;
        if (r < LF) {
#pragma unroll
            for (int m = 0; m < (4 << D); ++m) {
                const int k = (m * qc + cw) * LF + r;  // root coefficient
                if (ncyc > 0) {
                    if (k < 2 * ncyc) atomicXor(&stage[stg(k < ncyc ? k : k - ncyc)], v[m]);
                } else if (k < KS) {
                    stage[stg(k)] = v[m];
                }
            }
        }
    }
    __syncthreads();
    const int rows = int(batch - g * 32 < 32 ? batch - g * 32 : 32);
#pragma unroll 1
    for (int h = tid; h < 2 * tout; h += kK34Threads) {
        uint32_t x[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) x[i] = stage[stg(32 * h + i)];
        transpose32(x);
        uint32_t *po = reinterpret_cast<uint32_t *>(out) + (g * 32) * 2 * int64_t(tout) + h;
        const int64_t rs = 2 * int64_t(tout);
#pragma unroll
        for (int pr = 0; pr < 32; ++pr)
            if (pr < rows) po[pr * rs] = x[pr];
    }
}

// ---------------------------------------------------------------- planner

struct Layout {
    int64_t Ns, Ss;
    int64_t off_abs, off_bbs, off_p0, off_p1, total;
    int el;                          // pre-evaluated top global levels (K1b)
    int tl = 0;                      // Toom-3 levels
    int wl = 16;                     // w of the innermost Toom level (x = X^wl)
    int64_t G2 = 0;                  // node-problem groups (G 5^tl)
    int64_t M[kMaxToom + 1] = {};    // Toom part sizes, level 1..tl
    int64_t off_x0 = 0;              // Toom plans: plain bitsliced slice (both operands)
    int64_t off_r[kMaxToom + 1] = {};  // Toom interpolation outputs, level l
    int64_t off_q[kMaxToom + 1] = {};  // level-l c_0..c_4 before carries (5 x 2M per item)
    int64_t off_tot[kMaxToom + 1] = {};  // level-l chain totals per block
};

// Top global levels pre-evaluated by the slicing kernel (k1_slice_eval):
// 2 where the parts are whole operand words; F2X_EVAL_LEVELS=0/1/2 overrides
// (experiments).
static int eval_levels_for(int GL, int64_t N) {
    static const int v = [] {  // thread-safe one-time read
        const char *e = getenv("F2X_EVAL_LEVELS");
        return (e && e[0] >= '0' && e[0] <= '2') ? e[0] - '0' : -1;
    }();
    // default 2: measured +1.3% (n=17669), +2.6% (35851), +1.8% (57637)
    int el = v >= 0 ? v : 2;
    if (el > GL) el = GL;
    while (el > 0 && (N >> el) % 64 != 0) --el;  // parts must be whole operand words
    return el;
}

// Leaf size LF and Karatsuba depth K for a node problem of >= Smin
// coefficients: minimises 3^K (LF^2 + 48 LF) (leaf LOP3 + the per-leaf
// tree overhead, ~48 LOP3-equivalents per leaf word measured on B200).
static bool best_leaf(int64_t Smin, int leaf_hint, int &bestLF, int &bestK, double &best) {
    bestLF = 0;
    const int maxK = kMaxKC + kMaxGL;
    for (int K = 1; K <= maxK; ++K) {
        int64_t LF = ceil_div(Smin, int64_t(1) << K);
        if (K >= kMaxKC) {
            if (LF < 16) LF = 16;
            if (LF > 40) continue;
        } else {
            LF = LF <= 16 ? 16 : (LF <= 32 ? 32 : 0);
            if (!LF) continue;
        }
        if (leaf_hint) {
            if (LF > leaf_hint) continue;
            LF = leaf_hint;
        }
        const int KC = std::min(K, kMaxKC);
        if (!find_k2(int(LF), KC)) continue;
        // LF >= 37 has 11-quad chunks: 85 KB of shared memory, 2 CTAs/SM (~15 % slower)
        const double cost = double(ipow3(K)) * double(LF * LF + 48 * LF) * (LF >= 37 ? 1.15 : 1.0);
        if (!bestLF || cost < best) {
            best = cost;
            bestLF = int(LF);
            bestK = K;
        }
        if (leaf_hint) break;  // smallest K that fits the forced leaf
    }
    return bestLF != 0;
}

// Toom-3 top levels (TL): level l splits an operand of 3 M_l coefficients
// into thirds and evaluates at 0, 1, x, x+1, inf (x = X^w): 5 operands of
// S_l >= M_l + 2w coefficients; S_l = 3 M_{l+1} below another Toom level,
// the node size LF 2^K at the last.  Sizes for Nmin coefficients:
static void toom_sizes(int64_t Nmin, int TL, int wl, int64_t *M, int64_t &Smin_last) {
    // multiples of 4 coefficients: every Toom piece is a whole 16-byte quad
    // (toom_eval_fused); costs <= 3 coefficients of padding per level
    M[1] = (ceil_div(Nmin, 3) + 3) & ~int64_t(3);
    for (int l = 1; l < TL; ++l) M[l + 1] = (ceil_div(M[l] + 2 * kToomW, 3) + 3) & ~int64_t(3);
    Smin_last = M[TL] + 2 * wl;  // the innermost level evaluates at x = X^wl (kToomW or kToomWSmall)
}

// Toom interpolation: levels with >= this many products use the one-CTA-per-
// product kernel (F2X_TOOM_SEQ overrides; measured: 512 products sequential
// (n=57637 level 1: 263 vs 389 us); 128 products: two-kernel in round 1, the
// sequential form once the node-problem roots became plain (16-byte staging):
// n=35851 level 1 39 vs 59 us)
// F2X_TOOM_BLK=2048 pins the sequential interpolation to 2048-coefficient
// blocks (experiments)
static int toom_blk_choice() {
    static const int v = [] {
        const char *e = getenv("F2X_TOOM_BLK");
        return e ? atoi(e) : 0;
    }();
    return v;
}

static int64_t toom_seq_min() {
    static const int64_t v = [] {
        const char *e = getenv("F2X_TOOM_SEQ");
        return e ? int64_t(atoll(e)) : int64_t(96);
    }();
    return v;
}

// One CTA per product (toom_interp_seq) when a level has enough products to
// fill the GPU; otherwise the two-kernel form, whose assembly kernel keeps
// the chain carries of all nb = ceil(2M/2048) blocks in shared memory
// (nb x 3w words): above the 48 KB default it also falls back to the
// sequential form (t > ~12K words with few products).
static bool toom_use_seq(int64_t items, int64_t M) {
    const int64_t nb = ceil_div(2 * M, kToomBlk);
    return items >= toom_seq_min() || nb * 3 * kToomW * 4 > 48 * 1024;
}

// Block size of a one-CTA-per-product interpolation level: 2304-coefficient
// blocks (9 rows per scan segment) cost ~10 % more per coefficient than 2048
// (8 rows), so they are taken only when they stage clearly fewer
// coefficients: n=57637 level 3 (2M = 4300: 2 blocks instead of 3, 704 ->
// 592 us); levels 1-2 measured 4-10 % slower with 2304
static int toom_seq_blk(int64_t M) {
    const int64_t nb2048 = ceil_div(2 * M, 2048), nb2304 = ceil_div(2 * M, 2304);
    return double(nb2304) * 2304 * 1.1 < double(nb2048) * 2048 && toom_blk_choice() != 2048 ? 2304 : 2048;
}

// Resident-root interpolation (toom_interp_seq<BLK, true>): the last global
// pass, when it is a single Karatsuba level into the node-problem root, is
// folded into the innermost Toom level if that level runs one CTA per
// product and its five roots fit in shared memory (2 CTAs/SM).
// F2X_KROOT=0 keeps the separate k3_interp<1> pass (A/B).
static constexpr int kResSmemMax = 110 * 1024;
static constexpr int64_t kWideSeqMaxItems = 148;  // 512-thread form: at most one product per SM
static bool kroot_enabled() {
    static const bool v = [] {
        const char *e = getenv("F2X_KROOT");
        return !(e && e[0] == '0');
    }();
    return v;
}
static int kroot_hp(int64_t M) {  // resident root stride (words)
    const int blk = toom_seq_blk(M);
    return kres_words(int(ceil_div(2 * M, blk)), blk);
}
// Last global pass + K4 fused (k34_root_unslice): Karatsuba-only plans with
// enough groups to fill the GPU with one CTA per group and a root stage that
// fits shared memory.  F2X_K34=0 keeps the separate passes (A/B).
// Measured (d-sweep, µs): D = 2 (d=4096) k3 571 + K4 369 -> 768; D = 3
// (d=8192) 762 + 368 -> 1050; D = 4 (d=16384, 135 KB stage, 1 CTA/SM) 1064 +
// 369 -> 1955 -- so only up to three levels and two CTAs per SM.
static constexpr int64_t kK34MinGroups = 1024;
static constexpr int kK34SmemMax = 72 * 1024;
static bool k34_enabled() {
    static const bool v = [] {
        const char *e = getenv("F2X_K34");
        return !(e && e[0] == '0');
    }();
    return v;
}
static bool k34_fused(int TL, int np, const int32_t *pass_levels, int64_t G, int tout) {
    const int64_t ks = 64 * int64_t(tout);
    return k34_enabled() && TL == 0 && np > 0 && pass_levels[np - 1] <= 3 && G >= kK34MinGroups &&
           (ks + ks / 32) * 4 <= kK34SmemMax;
}
// `root` = coefficients of the node problem (LF 2^K): its product (2 root
// words, staged whole at slots k + 2w) must fit the resident span of
// nb blk + 3w slots -- a node problem padded well past M + 2w does not
// (n=54718: M = 2044, root 2112: 4224 > 4096 + 16), and keeps the separate pass.
static bool kroot_fused(int TL, int np, const int32_t *pass_levels, int64_t G, int64_t M_TL, int64_t root) {
    if (!(kroot_enabled() && TL > 0 && np > 0 && pass_levels[np - 1] == 1)) return false;
    const int blk = toom_seq_blk(M_TL);
    const int64_t nb = ceil_div(2 * M_TL, blk);
    return toom_use_seq(G * ipow5(TL - 1), M_TL) && int64_t(5) * kroot_hp(M_TL) * 4 <= kResSmemMax &&
           2 * root <= nb * blk + kToomWSmall;
}

// F2X_TOOM=0..3 forces the number of Toom-3 levels (tests / experiments)
static int toom_override() {
    static const int v = [] {
        const char *e = getenv("F2X_TOOM");
        return (e && e[0] >= '0' && e[0] <= '3') ? e[0] - '0' : -1;
    }();
    return v;
}

// F2X_TOOM_LEAF=LF forces the node-problem leaf of Toom plans (experiments;
// a leaf_hint argument forces the leaf AND disables Toom)
static int toom_leaf_override() {
    static const int v = [] {
        const char *e = getenv("F2X_TOOM_LEAF");
        return e ? atoi(e) : 0;
    }();
    return v;
}

// Words moved per node-problem group by the memory passes around the node
// kernel of a (TL, LF, K) plan: the pre-evaluated operand slices written by
// k1_slice_eval (Karatsuba-only plans) and every global interpolation pass
// (children read + parent written; a last pass folded into the resident-root
// Toom interpolation or into k34_root_unslice costs only the children's extra
// words over the parent's).
static double karatsuba_pass_words(int kind, int t, int TL, int LF, int K, int64_t G, const int64_t *M) {
    const int KC = std::min(K, kMaxKC), GL = K - KC;
    const int64_t LFS = leaf_stride_words(LF), Ns = LFS << K, Ss = LFS << KC;
    double w = 0;
    if (TL == 0) {
        const int el = eval_levels_for(GL, int64_t(LF) << K);
        w += 2.0 * double(ipow3(el)) * double(Ns >> el);
    }
    int32_t pass_levels[kMaxGL] = {0};
    int rem = GL, np = 0;
    while (rem > 0) {
        const int p = std::min(kMaxPassLevels, rem);
        pass_levels[np++] = p;
        rem -= p;
    }
    const bool folded = np > 0 && (kroot_fused(TL, np, pass_levels, G, M[TL], int64_t(LF) << K) ||
                                   k34_fused(TL, np, pass_levels, G, kind == F2X_KIND_FULL ? 2 * t : t));
    rem = GL;
    int64_t S = 2 * Ss;  // words of one product at the current level
    for (int i = 0; i < np; ++i) {
        w += double(ipow3(rem)) * double(S);
        rem -= pass_levels[i];
        S <<= pass_levels[i];
        // a folded pass writes no parent, and its consumer reads the children
        // instead of the parent it is already charged for
        w += (folded && i == np - 1 ? -1.0 : 1.0) * double(ipow3(rem)) * double(S);
    }
    return w;
}

static bool toom_considered(int t) { return t >= kToomMinWords; }

static int toom_wlast_override() {  // F2X_TOOM_WLAST=8|16 forces the innermost level's w (experiments / tests)
    static const int v = [] {
        const char *e = getenv("F2X_TOOM_WLAST");
        const int x = e ? atoi(e) : 0;
        return (x == kToomW || x == kToomWSmall) ? x : 0;
    }();
    return v;
}

static bool plan_candidate_w(int kind, int t, int TL, int wl, int leaf_hint, int64_t G, int &LF, int &K,
                             int64_t *M, double &c) {
    const int64_t Nmin = int64_t(64) * t;
    int64_t Smin = Nmin;
    if (TL > 0) toom_sizes(Nmin, TL, wl, M, Smin);
    if (!best_leaf(Smin, TL > 0 && toom_leaf_override() ? toom_leaf_override() : leaf_hint, LF, K, c)) return false;
    // the small point needs the one-CTA-per-product interpolation at the innermost level
    if (TL > 0 && wl != kToomW && !toom_use_seq(G * ipow5(TL - 1), M[TL])) return false;
    c += kPassWordCost * karatsuba_pass_words(kind, t, TL, LF, K, G, M);
    c *= double(ipow5(TL));
    if (TL > 0) c += kPassWordCost * 2.0 * 3.0 * double(M[1]);  // plain bitsliced slice (k1_slice)
    // Toom passes: HBM-bound per word moved, plus a per-call latency per level
    for (int l = 1; l <= TL; ++l) {
        const double Sl = l < TL ? 3.0 * double(M[l + 1]) : double(int64_t(LF) << K);
        const double ev = 2.0 * double(ipow5(l - 1)) * 3.0 * double(M[l]) + 2.0 * double(ipow5(l)) * Sl;
        double ip = 3.0 * double(ipow5(l)) * 2.0 * Sl + 1.5 * double(ipow5(l - 1)) * 6.0 * double(M[l]);
        if (l == TL && wl != kToomW) ip *= kToomSmallWInterpPenalty;
        c += (TL == 1 ? kToomWordCostSingle : kToomWordCost) * (ev + ip);
    }
    c += kToomLevelLatency * double(TL) / double(G);
    return true;
}

// Modelled cost per 32-product group of the best (LF, K, innermost w) under TL
// Toom-3 levels (cost units: ~one leaf LOP3 per group): node kernel
// (best_leaf), the global Karatsuba passes and slicing output, the Toom
// passes, and the call's share of the per-level launch latency (so the depth
// depends on the batch: small batches stay Karatsuba-only).
static bool plan_candidate(int kind, int t, int TL, int leaf_hint, int64_t G, int &LF, int &K, int64_t *M,
                           double &c, int &wl) {
    bool any = false;
    const int forced = toom_wlast_override();
    for (int w : {kToomWSmall, kToomW}) {
        if (TL == 0 && w != kToomW) continue;
        if (TL > 0 && forced && w != forced && !(w == kToomW && forced == kToomWSmall)) continue;
        if (TL > 0 && forced == kToomWSmall && w == kToomW && any) continue;  // (kToomW only as the fallback)
        int lf, k;
        int64_t m[kMaxToom + 1] = {0};
        double cc;
        if (!plan_candidate_w(kind, t, TL, w, leaf_hint, G, lf, k, m, cc)) continue;
        if (!any || cc < c) {
            any = true;
            c = cc;
            LF = lf;
            K = k;
            wl = w;
            std::memcpy(M, m, sizeof(m));
        }
    }
    return any;
}

static int plan_impl(int kind, int64_t batch, int t_or_n, int leaf_hint, f2x_plan *pl,
                     Layout *lay) {
    if (!pl || batch < 1 || t_or_n < 1) return F2X_EINVAL;
    std::memset(pl, 0, sizeof(*pl));
    int t, n;
    if (kind == F2X_KIND_FULL) {
        t = t_or_n;
        if (t > (1 << 20)) return F2X_ERANGE;
        n = 64 * t;
    } else if (kind == F2X_KIND_CYCLIC) {
        n = t_or_n;
        t = (n + 63) / 64;
    } else {
        return F2X_EINVAL;
    }
    const int64_t Nmin = int64_t(64) * t;
    // candidates: 0..kMaxToom Toom-3 levels on top of the Karatsuba node problem
    int bestTL = -1, bestLF = 0, bestK = 0, bestWl = kToomW;
    double best = 0;
    int64_t bestM[kMaxToom + 1] = {0};
    const int forced = leaf_hint ? 0 : toom_override();
    const int64_t Gp = ceil_div(batch, 32);
    for (int TL = 0; TL <= kMaxToom; ++TL) {
        if (forced >= 0 && TL != forced) continue;
        if (TL > 0 && (leaf_hint || (forced < 0 && !toom_considered(t)))) continue;
        int64_t M[kMaxToom + 1] = {0};
        int LF, K, wl = kToomW;
        double c;
        if (!plan_candidate(kind, t, TL, leaf_hint, Gp, LF, K, M, c, wl)) continue;
        if (bestTL < 0 || c < best) {
            best = c;
            bestTL = TL;
            bestLF = LF;
            bestK = K;
            bestWl = wl;
            std::memcpy(bestM, M, sizeof(M));
        }
    }
    if (bestTL < 0) return F2X_ERANGE;
    const int TL = bestTL, LF = bestLF, K = bestK, KC = std::min(K, kMaxKC), GL = K - KC;
    const K2Entry *e = find_k2(LF, KC);
    const int LFS = leaf_stride_words(LF);
    const int64_t G = ceil_div(batch, 32);
    const int64_t G2 = G * ipow5(TL);  // node-problem groups

    pl->kind = kind;
    pl->t = t;
    pl->n = n;
    pl->N = TL ? int32_t(3 * bestM[1]) : (LF << K);
    pl->batch = batch;
    pl->groups = G;
    pl->leaf_words = LF;
    pl->leaf_stride = LFS;
    pl->levels = K;
    pl->cta_levels = KC;
    pl->global_levels = GL;
    int rem = GL, np = 0;
    while (rem > 0) {
        const int p = std::min(kMaxPassLevels, rem);
        pl->pass_levels[np++] = p;
        rem -= p;
    }
    pl->num_passes = np;
    pl->launches = 3 + np + 2 * TL - (kroot_fused(TL, np, pl->pass_levels, G, bestM[TL], int64_t(LF) << K) ? 1 : 0) -
                   (k34_fused(TL, np, pl->pass_levels, G, kind == F2X_KIND_FULL ? 2 * t : t) ? 1 : 0);
    pl->cta_threads = e->threads;
    pl->node_ctas = G2 * ipow3(GL);
    pl->node_smem_bytes = int64_t(e->smem);
    pl->toom_levels = TL;
    pl->toom_w = TL ? kToomW : 0;
    pl->toom_w_last = TL ? bestWl : 0;
    for (int l = 1; l <= TL; ++l) pl->toom_M[l - 1] = int32_t(bestM[l]);
    // analytic operation counts per product (bitsliced: 1 LOP3 = 32 products)
    pl->leaf_ops_per_product = double(ipow5(TL)) * double(ipow3(K)) * LF * LF / 32.0;
    {
        // eval: each level-j node writes one mid of h_j words per operand;
        // interp: 3 XOR-ops per half word.  Summed over all K levels.
        double ev = 0, ip = 0;
        for (int j = 0; j < K; ++j) {
            const double hj = double(int64_t(LF) << (K - j - 1));
            ev += 2.0 * double(ipow3(j)) * hj;
            ip += 3.0 * double(ipow3(j)) * hj;
        }
        pl->karatsuba_ops_per_product = double(ipow5(TL)) * (ev + ip) / 32.0;
    }
    Layout L;
    L.tl = TL;
    L.wl = TL ? bestWl : kToomW;
    L.G2 = G2;
    for (int l = 0; l <= kMaxToom; ++l) L.M[l] = bestM[l];
    L.Ns = int64_t(LFS) << K;
    L.Ss = int64_t(LFS) << KC;
    L.el = TL ? 0 : eval_levels_for(GL, int64_t(LF) << K);
    int64_t off = 0;
    if (TL > 0) {  // plain bitsliced operands (the fused evaluation's input)
        L.off_x0 = off;
        off = align256(off + 2 * G * 3 * L.M[1] * 4);
    }
    const int64_t opw = G2 * ipow3(L.el) * (L.Ns >> L.el);  // node-problem operand words
    L.off_abs = off;
    L.off_bbs = align256(L.off_abs + opw * 4);
    L.off_p0 = align256(L.off_bbs + opw * 4);
    const int64_t p0 = G2 * ipow3(GL) * 2 * L.Ss * 4;  // node products
    L.off_p1 = align256(L.off_p0 + p0);
    // the last pass is folded into a later kernel (resident-root Toom
    // interpolation or k34_root_unslice): it writes nothing to the ping-pong
    // buffers
    const int tout_pl = kind == F2X_KIND_FULL ? 2 * t : t;
    const int np_exec = np - ((kroot_fused(TL, np, pl->pass_levels, G, bestM[TL], int64_t(LF) << K) ||
                               k34_fused(TL, np, pl->pass_levels, G, tout_pl)) ? 1 : 0);
    int64_t p1 = 0;
    if (np_exec >= 1) {  // first pass output (the largest one written to P1)
        const int d1 = GL - pl->pass_levels[0];
        p1 = G2 * ipow3(d1) * 2 * (L.Ns >> d1) * 4;
    }
    off = align256(L.off_p1 + p1);
    for (int l = TL; l >= 1; --l) {  // Toom interpolation: [block scans, totals,] outputs
        const int64_t items = G * ipow5(l - 1);
        L.off_q[l] = L.off_tot[l] = off;
        if (!toom_use_seq(items, L.M[l])) {  // two-kernel form: c_j and chain totals in HBM
            off = align256(off + items * 5 * 2 * L.M[l] * 4);
            L.off_tot[l] = off;
            off = align256(off + items * ceil_div(2 * L.M[l], kToomBlk) * 3 * kToomW * 4);
        }
        L.off_r[l] = off;
        off = align256(off + items * 6 * L.M[l] * 4);
    }
    L.total = off;
    {  // every pass output must fit the ping-pong buffer it is written to
        int d = GL;
        for (int i = 0; i < np_exec; ++i) {
            const int dlo = d - pl->pass_levels[i];
            const int64_t outb = G2 * ipow3(dlo) * 2 * (L.Ns >> dlo) * 4;
            if (outb > ((i & 1) ? p0 : p1)) return F2X_ERANGE;
            d = dlo;
        }
    }
    pl->workspace_bytes = L.total;
    pl->eval_levels = L.el;
    if (lay) *lay = L;
    return F2X_OK;
}

template <int D>
static int launch_k3(const uint32_t *Pin, uint32_t *Pout, int64_t items, int qw, int64_t inS,
                     int64_t outS, int plainLF, int LFS, cudaStream_t s) {
    k3_interp<D><<<unsigned(ceil_div(items, kThreads)), kThreads, 0, s>>>(Pin, Pout, items, qw, inS, outS,
                                                                          plainLF, LFS);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : F2X_ECUDA - int(e);
}

// Optional per-thread events recorded around the node kernel (bench.py uses
// them to time the dominant kernel live on the launching stream).
static thread_local cudaEvent_t g_node_ev[2] = {nullptr, nullptr};

// Integer-ALU peak microbenchmark: 8 independent chains per thread of the
// leaf's exact instruction, d = c ^ (a & b) (LOP3 LUT 0x6A), 16 distinct
// operands so nothing folds.  lane-ops = blocks*threads*iters*128.
__global__ void __launch_bounds__(256) lop3_peak(uint32_t *out, int iters, uint32_t seed) {
    uint32_t acc[8], x[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = seed * (i + 1) + threadIdx.x;
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = (seed + 0x9E3779B9u * k) ^ (blockIdx.x << 5);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
                asm volatile("lop3.b32 %0, %1, %2, %0, 0x6A;" : "+r"(acc[i]) : "r"(x[k]), "r"(x[(k + i + 1) & 15]));
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r ^= acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// F2X_DEBUG_SYNC=1: synchronise after every launch and report the failing
// stage (development aid; never set in benchmarks).
static int debug_sync(cudaStream_t s, int stage) {
    static const bool enabled = [] {
        const char *v = getenv("F2X_DEBUG_SYNC");
        return v && v[0] == '1';
    }();
    if (!enabled) return 0;
    cudaError_t e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "f2x: stage %d failed: %s\n", stage, cudaGetErrorString(e));
        return F2X_ECUDA - int(e);
    }
    return 0;
}

// Makes the device of a (non-legacy) stream current for the duration of a
// call when it differs from the caller's current device.
struct DeviceGuard {
    int prev = -1;
    int to_stream(cudaStream_t s) {
        // (not while the stream is being captured into a graph: the query
        // would invalidate the capture; a captured call replays on the
        // graph's device anyway)
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return 0;
        int sdev = -1, cdev = -1;
        if (cudaStreamGetDevice(s, &sdev) != cudaSuccess || cudaGetDevice(&cdev) != cudaSuccess) return 0;
        if (sdev == cdev) return 0;
        const cudaError_t e = cudaSetDevice(sdev);
        if (e != cudaSuccess) return F2X_ECUDA - int(e);
        prev = cdev;
        return 0;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

static int run(int kind, const uint64_t *A, const uint64_t *B, uint64_t *C, int64_t batch,
               int t_or_n, void *ws, size_t ws_bytes, int leaf_hint, uint32_t *d_err,
               cudaStream_t stream) {
    if (!A || !B || !C || !ws) return F2X_EINVAL;
    int rc0 = 0;
    // rows are read and written as 32-bit half-words: any uint64-aligned row
    // view works (e.g. A[1:] of an odd-t batch); the workspace holds 16-byte
    // quads
    if (((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) |
          reinterpret_cast<uintptr_t>(C)) & 7) || (reinterpret_cast<uintptr_t>(ws) & 15))
        return F2X_EINVAL;
    // launch on the stream's device; the caller's current device is restored
    DeviceGuard dg;
    if (stream != nullptr && (rc0 = dg.to_stream(stream))) return rc0;
    f2x_plan pl;
    Layout L;
    int rc = plan_impl(kind, batch, t_or_n, leaf_hint, &pl, &L);
    if (rc) return rc;
    if (int64_t(ws_bytes) < L.total) return F2X_ENOSPC;
    char *w = static_cast<char *>(ws);
    uint32_t *Abs = reinterpret_cast<uint32_t *>(w + L.off_abs);
    uint32_t *Bbs = reinterpret_cast<uint32_t *>(w + L.off_bbs);
    uint32_t *P0 = reinterpret_cast<uint32_t *>(w + L.off_p0);
    uint32_t *P1 = reinterpret_cast<uint32_t *>(w + L.off_p1);
    const int64_t G = pl.groups;
    const int ncyc = kind == F2X_KIND_CYCLIC ? pl.n : 0;

    // K1 (with the top L.el global levels pre-evaluated when L.el > 0;
    // Toom plans slice to a plain operand of N = 3 M_1 coefficients)
    if (L.tl > 0) {
        const int tiles = int(ceil_div(pl.N, kTileCoeffs));
        dim3 grid(unsigned(G * tiles), 2);
        uint32_t *X0a = reinterpret_cast<uint32_t *>(w + L.off_x0);
        F2X_LAUNCH(k1_slice, grid, kTileThreads, 0, stream, A, B, X0a, X0a + G * int64_t(pl.N), batch, pl.t, pl.N,
                                                    pl.N, pl.N, int64_t(pl.N), ncyc, d_err, tiles);
        if ((rc = debug_sync(stream, 1))) return rc;
        ToomEvalGeo geo{};
        for (int l = 1; l <= L.tl; ++l) geo.M[l] = int(L.M[l]);
        geo.N0 = pl.N;
        geo.LF = pl.leaf_words;
        geo.LFS = pl.leaf_stride;
        geo.chunks = 1 << pl.levels;
        // Tc LF must be a multiple of 4 (quad-aligned tiles)
        geo.Tc = 8 * pl.leaf_words <= kEvalFusedMaxT ? 8 : 4;
        geo.G = G;
        geo.Ns = L.Ns;
        const int etiles = int(ceil_div(geo.chunks, geo.Tc));
        const size_t sm = size_t(eval_fused_smem_words(L.tl)) * 4;
        static std::atomic<uint32_t> ef_dev_mask{0};
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 31 && !(ef_dev_mask.load() & (1u << dev))) {
            cudaError_t ae = cudaSuccess;
#define F2X_EF_ATTR(TLV)                                                                                      \
    if (ae == cudaSuccess)                                                                                    \
        ae = cudaFuncSetAttribute(toom_eval_fused<TLV, kToomW>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                                  int(eval_fused_smem_words(TLV) * 4));                                       \
    if (ae == cudaSuccess)                                                                                    \
        ae = cudaFuncSetAttribute(toom_eval_fused<TLV, kToomWSmall>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                  int(eval_fused_smem_words(TLV) * 4));
            F2X_EF_ATTR(1)
            F2X_EF_ATTR(2)
            F2X_EF_ATTR(3)
#undef F2X_EF_ATTR
            if (ae != cudaSuccess) return F2X_ECUDA - int(ae);
            ef_dev_mask.fetch_or(1u << dev);
        }
        const dim3 egrid(unsigned(etiles * G), 2);
        const int64_t x0w = 2 * G * int64_t(pl.N);
#define F2X_EF_LAUNCH(TLV)                                                                                    \
    do {                                                                                                      \
        if (L.wl == kToomWSmall)                                                                              \
            F2X_LAUNCH((toom_eval_fused<TLV, kToomWSmall>), egrid, kEvalFusedThreads, sm, stream, X0a, Abs, Bbs, geo, \
                       x0w);                                                                                  \
        else                                                                                                  \
            F2X_LAUNCH((toom_eval_fused<TLV, kToomW>), egrid, kEvalFusedThreads, sm, stream, X0a, Abs, Bbs, geo, x0w); \
    } while (0)
        switch (L.tl) {
            case 1: F2X_EF_LAUNCH(1); break;
            case 2: F2X_EF_LAUNCH(2); break;
            default: F2X_EF_LAUNCH(3); break;
        }
        if ((rc = debug_sync(stream, 2))) return rc;
    } else if (L.el == 0 && pl.N <= kTileCoeffs) {
        // one tile per group: several groups per CTA, storage quads
        const int gpc = kTileWords / int(ceil_div(pl.N, 64));
        dim3 grid(unsigned(ceil_div(G, gpc)), 2);
#define F2X_K1G(Q) F2X_LAUNCH(k1_slice_groups<Q>, grid, kTileThreads, 0, stream, A, B, Abs, Bbs, batch, pl.t, \
                               pl.N, pl.leaf_words, pl.leaf_stride, L.Ns, ncyc, d_err, G)
        switch (pl.leaf_stride / 4) {  // storage quads per chunk (odd: 5, 7, 9, 11)
            case 5: F2X_K1G(5); break;
            case 7: F2X_K1G(7); break;
            case 9: F2X_K1G(9); break;
            case 11: F2X_K1G(11); break;
            default: return F2X_ERANGE;
        }
#undef F2X_K1G
    } else if (L.el == 0) {
        const int tiles = int(ceil_div(pl.N, kTileCoeffs));
        dim3 grid(unsigned(G * tiles), 2);
        F2X_LAUNCH(k1_slice, grid, kTileThreads, 0, stream, A, B, Abs, Bbs, batch, pl.t, pl.N,
                                                    pl.leaf_words, pl.leaf_stride, L.Ns, ncyc,
                                                    d_err, tiles);
    } else {
        // tiles of whole chunks: TW = LF words per part (64 chunks) when the
        // part holds >= 64 chunks, else the whole part
        const int pw = (pl.N >> L.el) / 64;
        const int levels_left = pl.levels - L.el;
        const int TW = levels_left >= 6 ? pl.leaf_words : pw;
        const int tiles = pw / TW;
        const int nthr = int(ceil_div((1 << L.el) * 2 * TW, 32) * 32);
        if (nthr > 8 * 40) return F2X_ERANGE;  // (launch bounds: TW <= LF <= 40)
        dim3 grid(unsigned(G * tiles), 2);
        const size_t sm = size_t(1 << L.el) * (64 * TW + 2 * TW) * 4;
        const size_t sm_max = size_t(1 << L.el) * (64 * kTileWords + 2 * kTileWords) * 4;
        const int Qc = pl.leaf_stride / 4;  // storage quads per chunk (odd: 5, 7, 9, 11)
        const int qi = Qc == 5 ? 0 : Qc == 7 ? 1 : Qc == 9 ? 2 : Qc == 11 ? 3 : -1;
        if (qi < 0) return F2X_ERANGE;
        static std::atomic<uint32_t> attr_dev_mask[3][4];  // per (EL, Q): devices configured
        int dev = 0;
        cudaGetDevice(&dev);
#define F2X_K1E(EL, Q)                                                                                       \
    do {                                                                                                     \
        if (dev < 31 && !(attr_dev_mask[EL][qi].load() & (1u << dev))) {                                     \
            const cudaError_t ae = cudaFuncSetAttribute(k1_slice_eval<EL, Q>,                                \
                                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm_max)); \
            if (ae != cudaSuccess) return F2X_ECUDA - int(ae);                                               \
            attr_dev_mask[EL][qi].fetch_or(1u << dev);                                                       \
        }                                                                                                    \
        F2X_LAUNCH((k1_slice_eval<EL, Q>), grid, nthr, sm, stream, A, B, Abs, Bbs, batch, pl.t, pl.N,        \
                   pl.leaf_words, pl.leaf_stride, L.Ns >> EL, ncyc, d_err, tiles, TW);                       \
    } while (0)
        if (L.el == 1) {
            switch (Qc) {
                case 5: F2X_K1E(1, 5); break;
                case 7: F2X_K1E(1, 7); break;
                case 9: F2X_K1E(1, 9); break;
                default: F2X_K1E(1, 11); break;
            }
        } else {
            switch (Qc) {
                case 5: F2X_K1E(2, 5); break;
                case 7: F2X_K1E(2, 7); break;
                case 9: F2X_K1E(2, 9); break;
                default: F2X_K1E(2, 11); break;
            }
        }
#undef F2X_K1E
    }
    if ((rc = debug_sync(stream, 1))) return rc;
    // K2
    const K2Entry *e = find_k2(pl.leaf_words, pl.cta_levels);
    K2Params kp;
    kp.Abs = Abs;
    kp.Bbs = Bbs;
    kp.Pout = P0;
    kp.Ns = L.Ns >> L.el;
    kp.K = pl.levels - L.el;
    kp.GL = pl.global_levels - L.el;
    kp.paths = int(ipow3(pl.global_levels - L.el));
    if (g_node_ev[0]) cudaEventRecord(g_node_ev[0], stream);
    rc = e->launch(kp, pl.node_ctas, stream);
    if (rc) return rc;
    if (g_node_ev[1]) cudaEventRecord(g_node_ev[1], stream);
    // K3 passes
    uint32_t *cur = P0, *nxt = P1;
    int d = pl.global_levels;
    const int64_t in_stride0 = 2 * (L.Ns >> d);  // node products
    // last pass folded into the innermost Toom interpolation (resident roots)
    const bool kroot = kroot_fused(L.tl, pl.num_passes, pl.pass_levels, G, L.M[L.tl], int64_t(pl.leaf_words) << pl.levels);
    KRootIn kr{};
    const int tout = kind == F2X_KIND_FULL ? 2 * pl.t : pl.t;
    const bool k34 = k34_fused(L.tl, pl.num_passes, pl.pass_levels, G, tout);
    int k34D = 0, k34qw = 0;
    int64_t k34inS = 0;
    for (int i = 0; i < pl.num_passes; ++i) {
        const int D = pl.pass_levels[i];
        if (k34 && i == pl.num_passes - 1) {  // last pass: done by k34_root_unslice (K4 below)
            const int64_t Shi = L.Ns >> d;
            k34D = D;
            k34qw = int(Shi / 2);
            k34inS = i == 0 ? in_stride0 : 2 * Shi;
            d -= D;
            break;
        }
        if (kroot && i == pl.num_passes - 1) {  // D = 1 into the root
            const int64_t Shi = L.Ns >> d;
            kr.P = cur;
            kr.inS = i == 0 ? in_stride0 : 2 * Shi;
            kr.qw = int(Shi / 2);
            kr.oc = kr.qw / pl.leaf_stride * pl.leaf_words;
            kr.LF = pl.leaf_words;
            kr.LFS = pl.leaf_stride;
            kr.hp = kroot_hp(L.M[L.tl]);
            d -= D;
            break;
        }
        const int dlo = d - D;
        const int64_t Shi = L.Ns >> d, Slo = L.Ns >> dlo;
        const int qw = int(Shi / 2);
        const int64_t items = L.G2 * ipow3(dlo) * qw;
        const int64_t inS = i == 0 ? in_stride0 : 2 * Shi;
        // the last pass of a Toom plan writes the node-problem root plain
        // (2 LF 2^K words per root) for the interpolation's 16-byte staging
        const bool plain_root = L.tl > 0 && i == pl.num_passes - 1 && dlo == 0;
        const int pLF = plain_root ? pl.leaf_words : 0;
        const int64_t outS = plain_root ? 2 * (int64_t(pl.leaf_words) << pl.levels) : 2 * Slo;
        switch (D) {
            case 1: rc = launch_k3<1>(cur, nxt, items, qw, inS, outS, pLF, pl.leaf_stride, stream); break;
            case 2: rc = launch_k3<2>(cur, nxt, items, qw, inS, outS, pLF, pl.leaf_stride, stream); break;
            case 3: rc = launch_k3<3>(cur, nxt, items, qw, inS, outS, pLF, pl.leaf_stride, stream); break;
            case 4: rc = launch_k3<4>(cur, nxt, items, qw, inS, outS, pLF, pl.leaf_stride, stream); break;
            default: return F2X_ERANGE;
        }
        if (rc) return rc;
        if ((rc = debug_sync(stream, 3))) return rc;
        std::swap(cur, nxt);
        d = dlo;
    }
    // Toom interpolation levels, innermost first: level tl reads the node
    // problem's chunked root products, the others the plain 6 M_{l+1}
    // products of the level below
    const uint32_t *root = cur;
    int rootLF = pl.leaf_words, rootLFS = pl.leaf_stride;
    int64_t rootS = pl.num_passes == 0 ? in_stride0 : 2 * L.Ns;
    if (L.tl > 0 && pl.num_passes > 0 && !kroot) {  // plain root (last K3 pass above)
        rootS = 2 * (int64_t(pl.leaf_words) << pl.levels);
        rootLF = rootLFS = int(rootS);
    }
    for (int l = L.tl; l >= 1; --l) {
        uint32_t *out = reinterpret_cast<uint32_t *>(w + L.off_r[l]);
        uint32_t *Q = reinterpret_cast<uint32_t *>(w + L.off_q[l]);
        uint32_t *Tot = reinterpret_cast<uint32_t *>(w + L.off_tot[l]);
        const int M = int(L.M[l]);
        const int64_t items = G * ipow5(l - 1), outS = 6 * int64_t(M);
        const int Lin = l == L.tl ? (2 * pl.leaf_words) << pl.levels : int(6 * L.M[l + 1]);
        const int nb = int(ceil_div(2 * M, kToomBlk)), nbo = int(ceil_div(6 * M, kToomBlk));
        const size_t sms = size_t(5) * kToomStgStride * 4;
        // one CTA per item (carries in shared memory) when there are enough
        // items to fill the GPU, else the two-kernel form
        const bool seq = toom_use_seq(items, M);
        static std::atomic<uint32_t> attr_dev_mask{0};  // devices configured (idempotent set)
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 31 && !(attr_dev_mask.load() & (1u << dev))) {
            cudaError_t ae = cudaFuncSetAttribute(toom_interp_scan, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  int(sms));
#define F2X_SEQ_ATTR(BLK, RES, NT, BYTES)                                                                      \
    if (ae == cudaSuccess)                                                                                    \
        ae = cudaFuncSetAttribute(toom_interp_seq<BLK, RES, NT, kToomW>,                                      \
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(BYTES));                   \
    if (ae == cudaSuccess)                                                                                    \
        ae = cudaFuncSetAttribute(toom_interp_seq<BLK, RES, NT, kToomWSmall>,                                 \
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(BYTES));
            F2X_SEQ_ATTR(2048, false, kToomScanT, 5 * toom_stg_stride(2048) * 4)
            F2X_SEQ_ATTR(2304, false, kToomScanT, 5 * toom_stg_stride(2304) * 4)
            F2X_SEQ_ATTR(4096, false, 512, 5 * toom_stg_stride(4096) * 4)
            F2X_SEQ_ATTR(2048, true, kToomScanT, kResSmemMax)
            F2X_SEQ_ATTR(2304, true, kToomScanT, kResSmemMax)
#undef F2X_SEQ_ATTR
            if (ae != cudaSuccess) return F2X_ECUDA - int(ae);
            attr_dev_mask.fetch_or(1u << dev);
        }
        if (seq) {
            const bool res = kroot && l == L.tl;  // roots built in shared memory from the path products
            const size_t smr = res ? size_t(5) * kr.hp * 4 : 0;
            // the innermost level's point may be x = X^8 (planner: only with this one-CTA-per-product form)
            const bool small_w = l == L.tl && L.wl == kToomWSmall;
#define F2X_SEQ_LAUNCH(BLK, RES, NT, BYTES)                                                                   \
    do {                                                                                                      \
        if (small_w)                                                                                          \
            F2X_LAUNCH((toom_interp_seq<BLK, RES, NT, kToomWSmall>), unsigned(items), NT, BYTES, stream, root, out, \
                       M, rootLF, rootLFS, rootS, Lin, outS, kr);                                             \
        else                                                                                                  \
            F2X_LAUNCH((toom_interp_seq<BLK, RES, NT, kToomW>), unsigned(items), NT, BYTES, stream, root, out, M,   \
                       rootLF, rootLFS, rootS, Lin, outS, kr);                                                \
    } while (0)
            if (!res && items <= kWideSeqMaxItems && 2 * M > 4096) {
                // at most one product per SM: 512 threads walk 4096-coefficient
                // blocks (half the sequential block steps of the 256-thread form)
                F2X_SEQ_LAUNCH(4096, false, 512, 5 * toom_stg_stride(4096) * 4);
            } else if (toom_seq_blk(M) == 2304) {
                if (res) F2X_SEQ_LAUNCH(2304, true, kToomScanT, smr);
                else F2X_SEQ_LAUNCH(2304, false, kToomScanT, 5 * toom_stg_stride(2304) * 4);
            } else {
                if (res) F2X_SEQ_LAUNCH(2048, true, kToomScanT, smr);
                else F2X_SEQ_LAUNCH(2048, false, kToomScanT, 5 * toom_stg_stride(2048) * 4);
            }
#undef F2X_SEQ_LAUNCH
            if ((rc = debug_sync(stream, 5))) return rc;
        } else {
            F2X_LAUNCH(toom_interp_scan, unsigned(items * nb), kToomScanT, sms, stream, root, Q, Tot, M, kToomW, rootLF,
                                                                                rootLFS, rootS, Lin, nb);
            if ((rc = debug_sync(stream, 5))) return rc;
            const size_t sm = size_t(nb) * 3 * kToomW * 4;
            F2X_LAUNCH(toom_interp_assemble, unsigned(items * nbo), 256, sm, stream, Q, Tot, out, M, kToomW, nb, nbo,
                                                                             outS);
            if ((rc = debug_sync(stream, 5))) return rc;
        }
        root = out;
        rootLF = rootLFS = int(outS);
        rootS = outS;
    }
    // K4
    if (k34) {
        const size_t sm = size_t(64 * tout + 2 * tout) * 4;
        static std::atomic<uint32_t> k34_dev_mask{0};
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 31 && !(k34_dev_mask.load() & (1u << dev))) {
            cudaError_t ae = cudaSuccess;
            ae = cudaFuncSetAttribute(k34_root_unslice<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kK34SmemMax);
            if (ae == cudaSuccess)
                ae = cudaFuncSetAttribute(k34_root_unslice<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kK34SmemMax);
            if (ae == cudaSuccess)
                ae = cudaFuncSetAttribute(k34_root_unslice<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, kK34SmemMax);
            if (ae != cudaSuccess) return F2X_ECUDA - int(ae);
            k34_dev_mask.fetch_or(1u << dev);
        }
        switch (k34D) {
            case 1: F2X_LAUNCH(k34_root_unslice<1>, unsigned(G), kK34Threads, sm, stream, cur, C, batch, tout, k34qw, k34inS, pl.leaf_words, pl.leaf_stride, ncyc); break;
            case 2: F2X_LAUNCH(k34_root_unslice<2>, unsigned(G), kK34Threads, sm, stream, cur, C, batch, tout, k34qw, k34inS, pl.leaf_words, pl.leaf_stride, ncyc); break;
            case 3: F2X_LAUNCH(k34_root_unslice<3>, unsigned(G), kK34Threads, sm, stream, cur, C, batch, tout, k34qw, k34inS, pl.leaf_words, pl.leaf_stride, ncyc); break;
            default: return F2X_ERANGE;
        }
    } else {
        // 32-word tiles: twice the CTAs of the slicing tiles (the grid is
        // under one wave at 64 words)
        constexpr int TW4 = 32;
        const int tiles = int(ceil_div(tout, TW4));
        const unsigned grid = unsigned(G * tiles);
#define F2X_K4(QD) F2X_LAUNCH((k4_unslice<TW4, QD>), grid, 2 * TW4, 0, stream, root, C, batch, tout, rootLF, \
                               rootLFS, rootS, ncyc, tiles)
        if (rootLF == rootLFS) {
            F2X_K4(0);  // plain root
        } else {
            switch ((rootLF + 3) / 4) {  // data quads per chunk (LF 16..40)
                case 4: F2X_K4(4); break;
                case 5: F2X_K4(5); break;
                case 6: F2X_K4(6); break;
                case 7: F2X_K4(7); break;
                case 8: F2X_K4(8); break;
                case 9: F2X_K4(9); break;
                case 10: F2X_K4(10); break;
                default: return F2X_ERANGE;
            }
        }
#undef F2X_K4
    }
    if ((rc = debug_sync(stream, 4))) return rc;
    const cudaError_t ce = cudaGetLastError();
    return ce == cudaSuccess ? F2X_OK : F2X_ECUDA - int(ce);
}

}  // namespace f2x

// ------------------------------------------------------------------ C ABI
extern "C" {

int f2x_make_plan(int32_t kind, int64_t batch, int32_t t_or_n, int32_t leaf_hint,
                  f2x_plan *plan) {
    return f2x::plan_impl(kind, batch, t_or_n, leaf_hint, plan, nullptr);
}

double f2x_plan_cost(int32_t kind, int64_t batch, int32_t t_or_n, int32_t toom_levels) {
    if ((kind != F2X_KIND_FULL && kind != F2X_KIND_CYCLIC) || batch < 1 || t_or_n < 1 || toom_levels < 0 ||
        toom_levels > f2x::kMaxToom)
        return -1.0;
    const int t = kind == F2X_KIND_FULL ? t_or_n : (t_or_n + 63) / 64;
    int64_t M[f2x::kMaxToom + 1] = {0};
    int LF, K;
    double c;
    int wl;
    if (!f2x::plan_candidate(kind, t, toom_levels, 0, f2x::ceil_div(batch, 32), LF, K, M, c, wl)) return -1.0;
    return c;
}

int64_t f2x_workspace_bytes(int32_t kind, int64_t batch, int32_t t_or_n, int32_t leaf_hint) {
    f2x_plan pl;
    const int rc = f2x::plan_impl(kind, batch, t_or_n, leaf_hint, &pl, nullptr);
    return rc ? rc : pl.workspace_bytes;
}

int f2x_mul_full(const uint64_t *A, const uint64_t *B, uint64_t *C, int64_t batch, int32_t t,
                 void *workspace, size_t workspace_bytes, int32_t leaf_hint, void *stream) {
    return f2x::run(F2X_KIND_FULL, A, B, C, batch, t, workspace, workspace_bytes, leaf_hint,
                    nullptr, static_cast<cudaStream_t>(stream));
}

int f2x_mul_cyclic(const uint64_t *A, const uint64_t *B, uint64_t *C, int64_t batch, int32_t n,
                   void *workspace, size_t workspace_bytes, int32_t leaf_hint, uint32_t *d_err,
                   void *stream) {
    return f2x::run(F2X_KIND_CYCLIC, A, B, C, batch, n, workspace, workspace_bytes, leaf_hint,
                    d_err, static_cast<cudaStream_t>(stream));
}

int f2x_clmul64(const uint64_t *a, const uint64_t *b, uint64_t *lohi, int64_t lanes,
                void *workspace, size_t workspace_bytes, void *stream) {
    return f2x::run(F2X_KIND_FULL, a, b, lohi, lanes, 1, workspace, workspace_bytes, 0, nullptr,
                    static_cast<cudaStream_t>(stream));
}

int f2x_set_node_events(void *begin, void *end) {
    f2x::g_node_ev[0] = static_cast<cudaEvent_t>(begin);
    f2x::g_node_ev[1] = static_cast<cudaEvent_t>(end);
    return F2X_OK;
}

int f2x_bench_lop3(uint32_t *out, int32_t blocks, int32_t iters, void *stream) {
    if (!out || blocks < 1 || iters < 1) return F2X_EINVAL;
    f2x::lop3_peak<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(out, iters, 0x1234567u);
    const cudaError_t ce = cudaGetLastError();
    return ce == cudaSuccess ? F2X_OK : F2X_ECUDA - int(ce);
}

const char *f2x_strerror(int code) {
    if (code == F2X_OK) return "ok";
    if (code == F2X_EINVAL) return "invalid argument (batch/t/n < 1, null or misaligned pointer)";
    if (code == F2X_ENOSPC) return "workspace too small (see f2x_workspace_bytes)";
    if (code == F2X_ERANGE) return "operand size outside the supported envelope";
    if (code <= F2X_ECUDA) return cudaGetErrorString(static_cast<cudaError_t>(F2X_ECUDA - code));
    return "unknown error";
}

int f2x_version(void) { return 100; }

}  // extern "C"
