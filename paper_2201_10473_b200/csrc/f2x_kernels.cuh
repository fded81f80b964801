// Device code of the bitsliced GF(2)[X] engine (sm_100a).
//
// Data layout: products are processed in GROUPS of 32;
// a group's operand is BITSLICED -- uint32 word k holds coefficient k of the
// 32 products (bit p = product 32g+p).  Coefficients are stored in CHUNKS of
// LF (the leaf size) at a stride of LFS = round_up(LF, 4) words so that every
// Karatsuba half, leaf and quarter is a whole number of 16-byte quads.
//
// A bitsliced AND+XOR (one LOP3) performs 32 coefficient products, i.e. a
// 32x32 leaf costs exactly the 64*64/32 = 128 lane-ops per 64x64 block that
// the W_alg roofline charges; the Karatsuba additions are
// plain word XORs with no bit shifting, and the fold mod X^n-1 is pure index
// arithmetic.  No branch or address depends on operand bits.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace f2x {

__host__ __device__ constexpr int pow3c(int k) { return k <= 0 ? 1 : 3 * pow3c(k - 1); }

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

__device__ __forceinline__ void transpose32(uint32_t (&x)[32]) {
    tstage<16>(x);
    tstage<8>(x);
    tstage<4>(x);
    tstage<2>(x);
    tstage<1>(x);
}

// ----------------------------------------------------------- node kernel (K2)
struct K2Params {
    const uint32_t *Abs;  // [G][Ns] bitsliced, chunked
    const uint32_t *Bbs;
    uint32_t *Pout;       // [G][3^GL][2 Ss]
    int64_t Ns;           // storage words per operand per group
    int K;                // total Karatsuba levels
    int GL;               // global levels (paths = 3^GL)
    int paths;
};

template <int LF, int KC>
struct K2Cfg {
    static constexpr int LFS = (LF + 3) & ~3;
    static constexpr int Q = LFS / 4;                 // quads per chunk
    static constexpr int NLEAF = pow3c(KC);
    static constexpr int NT = NLEAF <= 32 ? 32 : ((NLEAF + 31) / 32) * 32;
    static constexpr int SQ = Q << KC;                // node operand, quads
    static constexpr int RQ = Q * NLEAF;              // region after KC levels
    static constexpr int NPOS = (pow3c(KC + 1) - 1) / 2;
    static constexpr size_t SMEM = size_t(2) * RQ * 16;
    static constexpr int REGS = 3 * LF + 14;
    static constexpr int MINB = REGS <= 64 ? 4 : (REGS <= 80 ? 3 : 2);
    static constexpr int LOAD_ITEMS = (SQ + NT - 1) / NT;
};

// Leaf: c[0..2LF-1) = a * b for bitsliced a, b of LF coefficients; a is
// streamed one quad at a time, b and c live in registers.  LF*LF LOP3.
template <int LF, int Q>
__device__ __forceinline__ void leaf_mul(uint4 *As, uint4 *Bs, int pq) {
    uint32_t b[LF];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const uint4 v = Bs[pq + q];
        const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int r = 0; r < 4; ++r)
            if (4 * q + r < LF) b[4 * q + r] = vv[r];
    }
    uint32_t c[2 * LF];
#pragma unroll
    for (int k = 0; k < 2 * LF; ++k) c[k] = 0u;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const uint4 v = As[pq + q];
        const uint32_t av[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int i = 4 * q + r;
            if (i < LF) {
#pragma unroll
                for (int j = 0; j < LF; ++j) c[i + j] ^= av[r] & b[j];
            }
        }
    }
    // lo chunk -> A slot, hi chunk -> B slot; pad words are zero.
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        uint32_t lo[4], hi[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int k = 4 * q + r;
            lo[r] = k < LF ? c[k] : 0u;
            hi[r] = k < LF ? c[LF + k] : 0u;  // c[2LF-1] == 0
        }
        As[pq + q] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        Bs[pq + q] = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    }
}

// One CTA = one (group, global path) node of S = LF*2^KC coefficients:
//   load   XOR of the path's 2^#mid input segments (global Karatsuba eval)
//   eval   KC breadth-first Karatsuba levels, mids appended (in-place layout)
//   leaf   3^KC register schoolbooks, products written over their operands
//   interp KC levels back up, elementwise in place
//   store  node product (2S coefficients) to global
template <int LF, int KC>
__global__ void __launch_bounds__(K2Cfg<LF, KC>::NT, K2Cfg<LF, KC>::MINB)
k2_node_mul(const K2Params p) {
    using C = K2Cfg<LF, KC>;
    extern __shared__ uint4 smem[];
    uint4 *As = smem;
    uint4 *Bs = smem + C::RQ;
    __shared__ uint16_t pos[C::NPOS];  // node positions (quads), level-major
    __shared__ uint32_t segoff[256];   // path segment offsets (quads), GL <= 8
    __shared__ int nseg_s;

    const int tid = threadIdx.x;
    const int64_t blk = blockIdx.x;
    const int64_t g = blk / p.paths;
    const int path = int(blk - g * p.paths);

    // --- position table: pos_j(nu) for j = 0..KC (public, data-independent)
    for (int e = tid; e < C::NPOS; e += C::NT) {
        int j = 0, T = 0, L = 1;
        while (e >= T + L) {
            T += L;
            L *= 3;
            ++j;
        }
        const int nu = e - T;
        int posq = 0, prefix = 0, div = L / 3;
        for (int l = 0; l < j; ++l) {
            const int d = (nu / div) % 3;
            const int hq = C::Q << (KC - l - 1);
            const int Rl = C::Q * (1 << (KC - l)) * pow3c(l);
            posq = d == 0 ? posq : (d == 1 ? posq + hq : Rl + prefix * hq);
            prefix = prefix * 3 + d;
            div /= 3;
        }
        pos[e] = (uint16_t)posq;
    }
    // --- path segments: chunk offsets of the global Karatsuba evaluation
    if (tid == 0) {
        int rem = path;
        int digits[16];
        for (int j = p.GL - 1; j >= 0; --j) {
            digits[j] = rem % 3;
            rem /= 3;
        }
        uint32_t base = 0, mids[16];
        int nm = 0;
        for (int j = 1; j <= p.GL; ++j) {
            const uint32_t hc = 1u << (p.K - j);  // half size in chunks
            if (digits[j - 1] == 1) base += hc;
            else if (digits[j - 1] == 2) mids[nm++] = hc;
        }
        for (int mask = 0; mask < (1 << nm); ++mask) {
            uint32_t o = base;
            for (int b = 0; b < nm; ++b)
                if ((mask >> b) & 1) o += mids[b];
            segoff[mask] = o * C::Q;
        }
        nseg_s = 1 << nm;
    }
    __syncthreads();

    // --- load: node operand = XOR of the path's segments
    {
        const int ns = nseg_s;
        const uint4 *Ag = reinterpret_cast<const uint4 *>(p.Abs) + g * (p.Ns / 4);
        const uint4 *Bg = reinterpret_cast<const uint4 *>(p.Bbs) + g * (p.Ns / 4);
        uint4 a[C::LOAD_ITEMS], b[C::LOAD_ITEMS];
#pragma unroll
        for (int i = 0; i < C::LOAD_ITEMS; ++i) a[i] = b[i] = make_uint4(0, 0, 0, 0);
        for (int s = 0; s < ns; ++s) {
            const uint32_t o = segoff[s];
#pragma unroll
            for (int i = 0; i < C::LOAD_ITEMS; ++i) {
                const int u = tid + i * C::NT;
                if (u < C::SQ) {
                    a[i] = a[i] ^ __ldg(Ag + o + u);
                    b[i] = b[i] ^ __ldg(Bg + o + u);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < C::LOAD_ITEMS; ++i) {
            const int u = tid + i * C::NT;
            if (u < C::SQ) {
                As[u] = a[i];
                Bs[u] = b[i];
            }
        }
    }
    __syncthreads();

    // --- eval: level j -> j+1, mids appended at R_j
#pragma unroll
    for (int j = 0; j < KC; ++j) {
        const int sh = KC - j - 1;
        const int hq = C::Q << sh;
        const int Rq = C::Q * (1 << (KC - j)) * pow3c(j);
        const int items = pow3c(j) * hq;
        const uint16_t *P = pos + (pow3c(j) - 1) / 2;
        for (int it = tid; it < items; it += C::NT) {
            const int nu = (it >> sh) / C::Q;
            const int u = it - nu * hq;
            const int s = P[nu];
            As[Rq + it] = As[s + u] ^ As[s + hq + u];
            Bs[Rq + it] = Bs[s + u] ^ Bs[s + hq + u];
        }
        __syncthreads();
    }

    // --- leaves
    if (tid < C::NLEAF) leaf_mul<LF, C::Q>(As, Bs, pos[(C::NLEAF - 1) / 2 + tid]);
    __syncthreads();

    // --- interp: level j+1 -> j, in place
#pragma unroll
    for (int j = KC - 1; j >= 0; --j) {
        const int sh = KC - j - 1;
        const int hq = C::Q << sh;
        const int Rq = C::Q * (1 << (KC - j)) * pow3c(j);
        const int items = pow3c(j) * hq;
        const uint16_t *P = pos + (pow3c(j) - 1) / 2;
        for (int it = tid; it < items; it += C::NT) {
            const int nu = (it >> sh) / C::Q;
            const int u = it - nu * hq;
            const int s = P[nu];
            const uint4 L0 = As[s + u], H0 = Bs[s + u];
            const uint4 L1 = As[s + hq + u], H1 = Bs[s + hq + u];
            const uint4 Ml = As[Rq + it], Mh = Bs[Rq + it];
            const uint4 T = H0 ^ L1;
            As[s + hq + u] = xor3(T, L0, Ml);
            Bs[s + u] = xor3(T, H1, Mh);
        }
        __syncthreads();
    }

    // --- store node product: lo half from A region, hi half from B region
    uint4 *out = reinterpret_cast<uint4 *>(p.Pout) + blk * (2 * C::SQ);
    for (int u = tid; u < C::SQ; u += C::NT) {
        out[u] = As[u];
        out[C::SQ + u] = Bs[u];
    }
}

template <int LF, int KC>
int launch_k2(const K2Params &p, int64_t blocks, cudaStream_t stream) {
    using C = K2Cfg<LF, KC>;
    static int configured_dev_mask = 0;  // benign race: attribute set is idempotent
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 31 && !(configured_dev_mask & (1 << dev))) {
        cudaError_t e = cudaFuncSetAttribute(k2_node_mul<LF, KC>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(C::SMEM));
        if (e != cudaSuccess) return -1000 - int(e);
        configured_dev_mask |= 1 << dev;
    }
    k2_node_mul<LF, KC><<<dim3(unsigned(blocks)), C::NT, C::SMEM, stream>>>(p);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : -1000 - int(e);
}

struct K2Entry {
    int LF, KC, threads;
    size_t smem;
    int (*launch)(const K2Params &, int64_t, cudaStream_t);
};

}  // namespace f2x
