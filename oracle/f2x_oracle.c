/* CPU ORACLE (C restatement) -- test infrastructure only, never the product.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs load this library, as the checker or the timed CPU
 * baseline.  The GPU engine never links it and has no CPU fallback.
 *
 * Restates the reference's word-level schoolbook (the counted route of
 * f2xmul.poly.schoolbook_mul, poly.py:493-514) with its multilane
 * integer-multiply carry-less base case (poly.py:269-302, 352-387), and the
 * SPEC ring fold.  Pinned against golden vectors
 * produced by the real reference (tests/golden/make_golden.py) in
 * tests/test_oracle.py.
 *
 * Layout (poly.py:4-8): row-major uint64[batch][t], little-endian words and
 * bits.  Rows are independent; a pthread pool spreads rows over host threads
 * (an atomic row counter, so uneven rows balance).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define M0 0x1111111111111111ULL
#define M1 0x2222222222222222ULL
#define M2 0x4444444444444444ULL
#define M3 0x8888888888888888ULL

/* 32x32 -> 64 carry-less via integer multiplies over 4-bit-spaced classes
 * (poly.py:275-291): column sums < 16, so each kept bit is the parity. */
static inline uint64_t k32(uint64_t x, uint64_t y) {
    uint64_t x0 = x & M0, x1 = x & M1, x2 = x & M2, x3 = x & M3;
    uint64_t y0 = y & M0, y1 = y & M1, y2 = y & M2, y3 = y & M3;
    uint64_t z0 = (x0 * y0) ^ (x1 * y3) ^ (x2 * y2) ^ (x3 * y1);
    uint64_t z1 = (x0 * y1) ^ (x1 * y0) ^ (x2 * y3) ^ (x3 * y2);
    uint64_t z2 = (x0 * y2) ^ (x1 * y1) ^ (x2 * y0) ^ (x3 * y3);
    uint64_t z3 = (x0 * y3) ^ (x1 * y2) ^ (x2 * y1) ^ (x3 * y0);
    return (z0 & M0) | (z1 & M1) | (z2 & M2) | (z3 & M3);
}

/* 64x64 -> 128: one Karatsuba step over 32-bit halves (poly.py:294-302,
 * 372-387). */
static inline void clmul64(uint64_t a, uint64_t b, uint64_t *lo, uint64_t *hi) {
    uint64_t al = a & 0xFFFFFFFFULL, ah = a >> 32;
    uint64_t bl = b & 0xFFFFFFFFULL, bh = b >> 32;
    uint64_t pll = k32(al, bl);
    uint64_t phh = k32(ah, bh);
    uint64_t pm = k32(al ^ ah, bl ^ bh) ^ pll ^ phh;
    *lo = pll ^ (pm << 32);
    *hi = phh ^ (pm >> 32);
}

/* Fixed 64-step masked shift-XOR (poly.py:261-266, 338-350). */
static inline void clmul64_portable(uint64_t a, uint64_t b, uint64_t *lo, uint64_t *hi) {
    uint64_t l = a & (0 - (b & 1)), h = 0;
    for (int k = 1; k < 64; ++k) {
        uint64_t m = 0 - ((b >> k) & 1);
        l ^= (a << k) & m;
        h ^= (a >> (64 - k)) & m;
    }
    *lo = l;
    *hi = h;
}

/* Word convolution: lo of (i,j) to word i+j, hi to i+j+1 (poly.py:503-511). */
static void conv_row(const uint64_t *a, const uint64_t *b, uint64_t *c, int t) {
    memset(c, 0, sizeof(uint64_t) * 2 * (size_t)t);
    for (int i = 0; i < t; ++i) {
        uint64_t ai = a[i];
        for (int j = 0; j < t; ++j) {
            uint64_t lo, hi;
            clmul64(ai, b[j], &lo, &hi);
            c[i + j] ^= lo;
            c[i + j + 1] ^= hi;
        }
    }
}

/* Fold mod X^n - 1: out[k] = P[k] ^ P[k+n] for bits k < n.
 * Word form with q = n/64, r = n%64: out[j] = P[j] ^ (P[q+j] >> r | P[q+j+1] << (64-r)),
 * top word masked to n - 64(t-1) bits. */
static void fold_row(const uint64_t *P, uint64_t *out, int n) {
    int t = (n + 63) / 64, q = n / 64, r = n % 64;
    for (int j = 0; j < t; ++j) {
        uint64_t lo = P[q + j];
        uint64_t hi = (q + j + 1 < 2 * t) ? P[q + j + 1] : 0;
        uint64_t sh = r ? ((lo >> r) | (hi << (64 - r))) : lo;
        out[j] = P[j] ^ sh;
    }
    int rb = n - 64 * (t - 1);
    if (rb < 64) out[t - 1] &= (1ULL << rb) - 1;
}

int f2x_oracle_threads(void) {
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

int f2x_oracle_clmul64(const uint64_t *a, const uint64_t *b, uint64_t *lo, uint64_t *hi,
                       int64_t lanes, int portable) {
    if (lanes < 0) return -1;
    for (int64_t i = 0; i < lanes; ++i) {
        if (portable) clmul64_portable(a[i], b[i], &lo[i], &hi[i]);
        else clmul64(a[i], b[i], &lo[i], &hi[i]);
    }
    return 0;
}

typedef struct {
    const uint64_t *A, *B;
    uint64_t *C;
    int64_t batch;
    int32_t t, n; /* n > 0: cyclic */
    int64_t next; /* shared row counter */
    int rc;
} job_t;

static void *worker(void *arg) {
    job_t *j = (job_t *)arg;
    int t = j->t;
    uint64_t *P = (uint64_t *)malloc(sizeof(uint64_t) * 2 * (size_t)t);
    if (!P) {
        __atomic_store_n(&j->rc, -3, __ATOMIC_RELAXED);
        return NULL;
    }
    for (;;) {
        int64_t r = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
        if (r >= j->batch) break;
        if (j->n > 0) {
            conv_row(j->A + r * t, j->B + r * t, P, t);
            fold_row(P, j->C + r * t, j->n);
        } else {
            conv_row(j->A + r * t, j->B + r * t, j->C + r * 2 * (int64_t)t, t);
        }
    }
    free(P);
    return NULL;
}

static int run_pool(job_t *j, int nthreads) {
    if (nthreads <= 0) nthreads = f2x_oracle_threads();
    if (nthreads > 256) nthreads = 256;
    if ((int64_t)nthreads > j->batch) nthreads = j->batch > 0 ? (int)j->batch : 1;
    pthread_t th[256];
    int started = 0;
    for (int i = 1; i < nthreads; ++i)
        if (pthread_create(&th[started], NULL, worker, j) == 0) ++started;
    worker(j); /* the caller's thread works too; rows still all get done */
    for (int i = 0; i < started; ++i) pthread_join(th[i], NULL);
    return j->rc;
}

/* C[batch][2t] = A[batch][t] * B[batch][t] over F2[X]. */
int f2x_oracle_mul_full(const uint64_t *A, const uint64_t *B, uint64_t *C,
                        int64_t batch, int32_t t, int32_t nthreads) {
    if (batch < 0 || t < 1) return -1;
    job_t j = {A, B, C, batch, t, 0, 0, 0};
    return run_pool(&j, nthreads);
}

/* C[batch][t] = A * B mod X^n - 1, t = ceil(n/64).  Returns -2 if an input
 * has bits >= n set (reject, never mask). */
int f2x_oracle_mul_cyclic(const uint64_t *A, const uint64_t *B, uint64_t *C,
                          int64_t batch, int32_t n, int32_t nthreads) {
    if (batch < 0 || n < 1) return -1;
    int t = (n + 63) / 64, rb = n - 64 * (t - 1);
    if (rb < 64) {
        uint64_t bad = 0;
        for (int64_t r = 0; r < batch; ++r)
            bad |= (A[r * t + t - 1] | B[r * t + t - 1]) >> rb;
        if (bad) return -2;
    }
    job_t j = {A, B, C, batch, t, n, 0, 0};
    return run_pool(&j, nthreads);
}
