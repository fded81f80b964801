/* f2x.h -- C ABI of the B200 batched dense GF(2)[X] multiply engine.
 *
 * Drop-in boundary for the reference's multiply entry points
 * (/root/reference/pkg/src/f2xmul/poly.py):
 *   f2x_mul_full    replaces schoolbook_mul          (poly.py:547-561)
 *                   batched over rows; each row is one PolyWords pair.
 *   f2x_mul_cyclic  replaces the SPEC's ring_mul
 *                   (absent from the reference package; restated there).
 *   f2x_clmul64     replaces clmul64_batch           (poly.py:451-480)
 *                   = f2x_mul_full with t = 1, lo/hi interleaved.
 *
 * Layout (poly.py:4-8, unchanged): row-major uint64[batch][t]; bit i of word
 * j of a row is the coefficient of X^(64 j + i).  All data pointers are
 * DEVICE pointers (cudaMalloc / torch CUDA tensors), non-aliasing; A, B, C
 * need only uint64 (8-byte) alignment, so any row view of a batch works; the
 * workspace must be 16-byte aligned.  Work runs on the stream's device.  Calls are asynchronous on `stream` (a cudaStream_t; NULL =
 * legacy default stream), reentrant, and allocate nothing: the caller passes
 * a device workspace of at least f2x_workspace_bytes() bytes.
 *
 * Return codes: 0 on success, negative F2X_E* on error (see f2x_strerror).
 * Errors mirror the reference's ValueError cases: unequal/zero lengths
 * (poly.py:84-85, 555-557), out-of-range operands.
 * Constant time: every launch shape, loop bound and address depends only on
 * (batch, t, n) -- never on operand bits.
 */
#ifndef F2X_H_
#define F2X_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define F2X_API __attribute__((visibility("default")))
#else
#define F2X_API
#endif

#define F2X_OK 0
#define F2X_EINVAL (-22)   /* bad batch / t / n / null pointer           */
#define F2X_ENOSPC (-28)   /* workspace too small                          */
#define F2X_ERANGE (-34)   /* size outside the supported envelope          */
#define F2X_ECUDA (-1000)  /* CUDA launch/runtime error (code - cudaError) */

#define F2X_KIND_FULL 0
#define F2X_KIND_CYCLIC 1

/* The multiplication plan the engine executes for a given call shape.
 * Operands are bitsliced 32 products per group; each operand is padded to
 * N = leaf_words * 2^levels coefficients and multiplied by 2-way Karatsuba:
 * `global_levels` levels across CTAs, `cta_levels` inside one CTA's shared
 * memory, then leaf_words x leaf_words schoolbook leaves in registers. */
typedef struct f2x_plan {
    int32_t kind;            /* F2X_KIND_FULL or F2X_KIND_CYCLIC              */
    int32_t t;               /* operand words                                 */
    int32_t n;               /* ring degree (cyclic) or 64 t (full)           */
    int32_t N;               /* padded coefficients per operand               */
    int64_t batch;
    int64_t groups;          /* ceil(batch / 32)                              */
    int32_t leaf_words;      /* LF                                            */
    int32_t leaf_stride;     /* chunk stride: 4 x odd #quads >= LF words     */
    int32_t levels;          /* K = global_levels + cta_levels                */
    int32_t cta_levels;      /* KC                                            */
    int32_t global_levels;   /* GL                                            */
    int32_t num_passes;      /* global interpolation passes                   */
    int32_t pass_levels[8];  /* levels per pass, bottom first                 */
    int32_t launches;        /* kernels launched per call                     */
    int32_t cta_threads;     /* threads per node CTA                          */
    int64_t node_ctas;       /* CTAs of the node kernel                       */
    int64_t node_smem_bytes; /* dynamic shared memory per node CTA            */
    int64_t workspace_bytes;
    double leaf_ops_per_product;    /* LOP3 in leaves / product (analytic)    */
    double karatsuba_ops_per_product; /* XOR ops of eval+interp / product     */
    int32_t eval_levels;     /* top global levels pre-evaluated by the slicing
                                kernel (node kernel runs on 3^eval_levels x
                                the groups with levels - eval_levels)        */
    int32_t toom_levels;     /* Toom-3 levels above the Karatsuba node problem
                                (node kernel runs on 5^toom_levels x groups) */
    int32_t toom_w;          /* Toom-3 point x = X^toom_w                      */
    int32_t toom_M[4];       /* part size (coefficients) of Toom level 1..     */
    int32_t toom_w_last;     /* w of the innermost Toom level (toom_w or 8): the
                                node problem holds toom_M[last] + 2 toom_w_last */
} f2x_plan;

/* Fill *plan for a call shape.  leaf_hint = 0 picks the default leaf;
 * otherwise it forces leaf_words (tuning).  Returns 0 or F2X_E*. */
F2X_API int f2x_make_plan(int32_t kind, int64_t batch, int32_t t_or_n, int32_t leaf_hint,
                  f2x_plan *plan);

/* Planner cost model (tests / tuning): modelled cost per 32-product group,
 * in leaf-LOP3 units, of the best plan with toom_levels Toom-3 levels for
 * this call shape; < 0 if no such plan exists.  f2x_make_plan takes the
 * cheapest level count among those it considers for the shape. */
F2X_API double f2x_plan_cost(int32_t kind, int64_t batch, int32_t t_or_n, int32_t toom_levels);

/* Workspace bytes for f2x_mul_full(batch, t) / f2x_mul_cyclic(batch, n). */
F2X_API int64_t f2x_workspace_bytes(int32_t kind, int64_t batch, int32_t t_or_n, int32_t leaf_hint);

/* C[batch][2t] = A[batch][t] * B[batch][t] over F2[X]  (schoolbook_mul). */
F2X_API int f2x_mul_full(const uint64_t *A, const uint64_t *B, uint64_t *C, int64_t batch,
                 int32_t t, void *workspace, size_t workspace_bytes, int32_t leaf_hint,
                 void *stream);

/* C[batch][t] = A * B mod X^n - 1, t = ceil(n/64)  (SPEC ring_mul).
 * If d_err (device uint32, nullable) is given, it is OR-ed with 1 when any
 * input has a bit >= n set; the caller checks it after synchronising and
 * rejects the call. */
F2X_API int f2x_mul_cyclic(const uint64_t *A, const uint64_t *B, uint64_t *C, int64_t batch,
                   int32_t n, void *workspace, size_t workspace_bytes, int32_t leaf_hint,
                   uint32_t *d_err, void *stream);

/* Lane-wise 64x64 -> 128 carry-less products (clmul64_batch):
 * LOHI[lanes][2] = {lo, hi}.  Uses the full-product path with t = 1. */
F2X_API int f2x_clmul64(const uint64_t *a, const uint64_t *b, uint64_t *lohi, int64_t lanes,
                void *workspace, size_t workspace_bytes, void *stream);

/* Measurement hooks (bench.py / profiling; not part of the reference API).
 * f2x_set_node_events: cudaEvent_t pair recorded on the call's stream right
 * before and after the node kernel of every later call from this thread
 * (NULL, NULL disables).  f2x_bench_lop3: integer-ALU peak microbenchmark,
 * blocks x 256 threads x iters x 128 LOP3 lane-ops; out needs
 * blocks*256 uint32. */
F2X_API int f2x_set_node_events(void *begin, void *end);
F2X_API int f2x_bench_lop3(uint32_t *out, int32_t blocks, int32_t iters, void *stream);

F2X_API const char *f2x_strerror(int code);
F2X_API int f2x_version(void);

#ifdef __cplusplus
}
#endif

#endif /* F2X_H_ */
