/* ozgpu.h -- C-ABI of the B200-native Ozaki-I FP64 GEMM (integer-slice
 * emulation, arXiv 2506.11277).  This is the drop-in boundary for the
 * reference library's GEMM path (ozmul, /root/reference/proj): every entry
 * point cites the reference interface it replaces.  Plain pointers and
 * sizes only; no C++ or torch types cross this boundary.
 *
 * Error codes (the reference's exception classes, scheme.cpp:221-239,
 * main.cpp:770-783):
 *   OZGPU_OK 0, OZGPU_INVALID_ARGUMENT 1 (std::invalid_argument),
 *   OZGPU_DOMAIN_ERROR 2 (std::domain_error), OZGPU_DEVICE_ERROR 3,
 *   OZGPU_INFEASIBLE 4 (SelectionInfeasible), OZGPU_OVERFLOW 5
 *   (MmaOverflowError), OZGPU_IO_ERROR 6 (std::runtime_error of the matrix
 *   file functions).  ozgpu_last_error() returns the calling thread's
 *   message for the last failing call, worded like the reference's.
 *
 * Enumerations match the reference headers:
 *   schedule: 0 kFull, 1 kReduced                       (scheme.hpp:30-33)
 *   strategy: 0 kFloatPerProduct, 1 kDiagonalInteger, 2 kLevelledExact
 *                                                        (scheme.hpp:45-49)
 *   mode:     0 kTruncate, 1 kNearest                    (slicing.hpp SliceMode)
 *   orientation: 0 rows (left factor), 1 columns (right factor)
 *
 * Threading: every call is safe from any number of host threads
 * (SPEC.md:91,363-364).  A context owns one workspace (slices, scales, chunk
 * planes, lockstep counters); every call orders its use of it after the
 * previous call's on the GPU (an event recorded where that call's work was
 * enqueued, waited on by this call's stream), so device-pointer calls on
 * different streams never overwrite each other's workspace -- on one context
 * they run one after the other.  Use one context per stream to overlap them.
 *
 * Operands: leading dimensions must be >= the row length (lda >= k,
 * ldb >= n, ldc >= n) and pointers non-null when the operand has elements,
 * else OZGPU_INVALID_ARGUMENT before anything is copied or launched.
 */
#ifndef OZGPU_H
#define OZGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OZGPU_OK 0
#define OZGPU_INVALID_ARGUMENT 1
#define OZGPU_DOMAIN_ERROR 2
#define OZGPU_DEVICE_ERROR 3
#define OZGPU_INFEASIBLE 4
#define OZGPU_OVERFLOW 5
#define OZGPU_IO_ERROR 6

#define OZGPU_MAX_LEVELS 128

/* MmaConfig (proj/include/ozmul/mma_sim.hpp:27-37): inputs in I_{t'},
 * accumulation in I_T.  int8_int32 = {7, 31}. */
typedef struct {
  int input_width; /* t' */
  int acc_width;   /* T  */
} ozgpu_mma_config;

/* MultiplyPlan (proj/include/ozmul/scheme.hpp:77-88) incl. Schedule and
 * LevelPlan (scheme.hpp:36-56). */
typedef struct {
  int slices_a;
  int slices_b;
  int width;          /* t */
  int schedule;       /* 0 full, 1 reduced */
  int diag_sum_limit; /* Schedule::diag_sum_limit; <= 0 means unset */
  int strategy;       /* 0 float-per-product, 1 diagonal-integer, 2 levelled-exact */
  int mode;           /* 0 truncate, 1 nearest */
  int precision;      /* p */
  int acc_bits_used;  /* T' = 2t + ceil(log2 k) */
  int num_levels;
  int levels[2 * OZGPU_MAX_LEVELS]; /* inclusive [first, last] diagonal pairs */
  long long level_inexact_adds;     /* LevelPlan::inexact_adds */
  long long psi;
} ozgpu_plan;

/* Diagnostics (proj/include/ozmul/scheme.hpp:97-106). */
typedef struct {
  int64_t products;
  int64_t integer_adds;
  int64_t float_adds;
  int64_t flushes;
  long long realized_psi;
  long long planned_psi;
  int width;
  int acc_bits_used;
} ozgpu_diag;

/* SliceSelection (proj/include/ozmul/analysis.hpp:86-92) and the
 * SelectionInfeasible payload (analysis.hpp:78-84). */
typedef struct {
  int slices_a;
  int slices_b;
  double lhs;
  double target;
  int64_t products;
  double gap; /* set when OZGPU_INFEASIBLE */
} ozgpu_selection;

/* ScalingProfile's scalar part (proj/include/ozmul/analysis.hpp:30-38). */
typedef struct {
  double kappa_a;
  double kappa_b;
  int a_has_zero_block;
  int b_has_zero_block;
} ozgpu_profile;

typedef struct ozgpu_ctx ozgpu_ctx;

/* ---- library / context ------------------------------------------------ */
const char* ozgpu_last_error(void);
const char* ozgpu_version(void);
/* Creates a context on CUDA device `device` (own stream + workspace).
 * Fails with OZGPU_DEVICE_ERROR when no sm_100 device is present: there is
 * no CPU fallback. */
int ozgpu_create(int device, ozgpu_ctx** out);
int ozgpu_destroy(ozgpu_ctx* ctx);
/* Number of this library's kernels launched through `ctx` so far. */
int64_t ozgpu_kernel_launches(const ozgpu_ctx* ctx);
/* The process-wide default context for `device` (created on first use). */
ozgpu_ctx* ozgpu_default_context(int device);
/* Per-stage device timing of the multiplies issued through `ctx` while
 * enabled: CUDA events recorded on the launching stream around the slicing
 * kernels, the tcgen05 pair-GEMM kernel and the combine kernel. */
int ozgpu_set_stage_timing(ozgpu_ctx* ctx, int enable);
/* Accumulated stage times since the last reset (synchronises the pending
 * events): ms3[0] slicing, ms3[1] pair GEMMs, ms3[2] combine; *calls =
 * number of timed multiplies. */
int ozgpu_stage_times(ozgpu_ctx* ctx, double* ms3, int64_t* calls, int reset);

/* ---- plan (host; O(s^2) scalar code) ---------------------------------- */
/* optimal_slice_width, proj/src/mma_sim.cpp:50-59 */
int ozgpu_optimal_slice_width(ozgpu_mma_config cfg, int64_t k, int* out);
/* max_inner_dim, proj/src/mma_sim.cpp:66-72 */
int ozgpu_max_inner_dim(ozgpu_mma_config cfg, int64_t* out);
/* chi, proj/src/scheme.cpp:46-52 */
int ozgpu_chi(int slices_a, int slices_b, int64_t* out);
/* spare_carries, proj/src/scheme.cpp:54-62 */
int ozgpu_spare_carries(int first_diag, int last_diag, int width, int64_t* out);
/* plan_levels, proj/src/scheme.cpp:64-95 (levels written into plan->levels) */
int ozgpu_plan_levels(int precision, int width, int acc_bits_used, int num_diagonals,
                      ozgpu_plan* out);
/* diagonal_flush_threshold, proj/src/scheme.cpp:97-106 */
int ozgpu_diagonal_flush_threshold(ozgpu_mma_config cfg, int width, int64_t k, int64_t* out);
/* make_plan, proj/src/scheme.cpp:127-168 */
int ozgpu_make_plan(ozgpu_mma_config cfg, int64_t k, int slices_a, int slices_b,
                    int schedule, int strategy, int mode, int precision, ozgpu_plan* out);

/* ---- estimator -------------------------------------------------------- */
/* select_slices, proj/src/analysis.cpp:142-207.  has_target=0 -> the
 * default target gamma_psi of each candidate's plan. */
int ozgpu_select_slices(double kappa_a, double kappa_b, int width, double u, int s_max,
                        int has_target, double target, int schedule, int strategy,
                        int acc_bits_used, int precision, ozgpu_selection* out);
/* scaling_profile, proj/src/analysis.cpp:58-68, computed on the GPU.
 * Host pointers; A m x k (lda), B k x n (ldb), row-major. */
int ozgpu_scaling_profile(ozgpu_ctx* ctx, int64_t m, int64_t k, int64_t n, const double* a,
                          int64_t lda, const double* b, int64_t ldb, ozgpu_profile* out);

/* block_ratios, proj/src/analysis.cpp:25-47, on the GPU: per-row
 * (orientation 0) or per-column (1) max / min-nonzero magnitude, 1.0 for an
 * all-zero block; *has_zero_block set when one exists.  ratios_out has rows
 * (orientation 0) or cols (1) entries. */
int ozgpu_block_ratios(ozgpu_ctx* ctx, int orientation, int64_t rows, int64_t cols,
                       const double* x, int64_t ldx, double* ratios_out, int* has_zero_block);
/* abs_product / gemm_reference, proj/src/matrix.cpp:31-54, on the GPU:
 * out(i,j) = sum_r op(a_ir) op(b_rj) in binary64, r ascending, zero a_ir
 * skipped, op = |.| when absolute != 0 (identical rounding sequence; tiled
 * through shared memory, one sequential sum per output). */
int ozgpu_fp64_gemm(ozgpu_ctx* ctx, int absolute, int64_t m, int64_t k, int64_t n,
                    const double* a, int64_t lda, const double* b, int64_t ldb, double* out,
                    int64_t ldo);

/* min_exact_slices, proj/src/slicing.cpp:212-249, on the GPU: the fewest
 * slices of `width` bits that hold every row (orientation 0) / column (1)
 * exactly (mode 0 truncate, 1 nearest). */
int ozgpu_min_exact_slices(ozgpu_ctx* ctx, int orientation, int64_t rows, int64_t cols,
                           const double* x, int64_t ldx, int width, int mode, int* out);
/* exact_gemm(a, b).to_matrix(), proj/src/oracle.cpp:223-232 + 157-180, on the
 * GPU: C = RN(AB) entrywise (the exact product rounded once), computed by the
 * Ozaki-I scheme with error-free slice counts and the full pair schedule.
 * Inputs as multiply() accepts them; OZGPU_DOMAIN_ERROR when their exponent
 * range needs an exact value wider than 1024 bits. */
int ozgpu_exact_gemm(ozgpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* a,
                     int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc);
/* Error metrics, proj/src/oracle.cpp:253-292 (+ frobenius_norm :64-68), on
 * the GPU against a reference matrix R = RN(exact): *max_elementwise = max
 * |c - r| / |r| (0 when both are 0, +inf when only r is), *sum_sq = sum
 * (c - r)^2; reference = NULL gives sum c^2.  Deterministic reduction order
 * (not the reference's sequential one). */
int ozgpu_error_metrics(ozgpu_ctx* ctx, int64_t m, int64_t n, const double* computed, int64_t ldc,
                        const double* reference, int64_t ldr, double* max_elementwise,
                        double* sum_sq);

/* ---- the GEMM (multiply, proj/src/scheme.cpp:219-361) ------------------ */
/* Host buffers: A m x k (lda), B k x n (ldb), C m x n (ldc), all row-major
 * binary64.  Copies in, runs slicing + int8 tcgen05 pair GEMMs + exact
 * epilogue on the GPU, copies C out.  diag may be NULL.  On an input error
 * (Inf / NaN / -0, scheme.cpp:223-225) C is left untouched, except that
 * page-locked buffers of a product >= 64 MiB stream C back block by block
 * while later blocks are still being checked: there its contents are then
 * unspecified. */
int ozgpu_dgemm(ozgpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* a, int64_t lda,
                const double* b, int64_t ldb, double* c, int64_t ldc, ozgpu_mma_config cfg,
                const ozgpu_plan* plan, ozgpu_diag* diag);
/* multiply_axpby, proj/src/scheme.cpp:363-372: D = alpha*(AB) + beta*C in
 * plain binary64 after the emulated product.  C is read from c_in (ldc),
 * D written to d_out (ldd); they may alias. */
int ozgpu_dgemm_axpby(ozgpu_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha,
                      const double* a, int64_t lda, const double* b, int64_t ldb, double beta,
                      const double* c_in, int64_t ldc, double* d_out, int64_t ldd,
                      ozgpu_mma_config cfg, const ozgpu_plan* plan, ozgpu_diag* diag);
/* The same multiply sharded over several contexts (one per GPU of the node,
 * or several on one GPU): C is split into p_r x p_c blocks (p_r >= p_c,
 * p_r * p_c = count, as square as possible: 1x1, 2x1, 2x2, 4x2); context r
 * computes block (r / p_c, r % p_c) with the full k from its A row-panel and
 * B column-panel, concurrently, each through its own blocked H2D / compute /
 * D2H pipeline.  Bit-identical to ozgpu_dgemm (scales are per row of A and
 * per column of B).  Errors: the first failing block's, in
 * context order. */
int ozgpu_dgemm_multi(ozgpu_ctx* const* ctxs, int count, int64_t m, int64_t n, int64_t k,
                      const double* a, int64_t lda, const double* b, int64_t ldb, double* c,
                      int64_t ldc, ozgpu_mma_config cfg, const ozgpu_plan* plan,
                      ozgpu_diag* diag);
/* Contexts for a list of device slots (e.g. OZGPU_DEVICES=0,1,2,3): the first
 * slot on a device gets its default context, repeated slots on the same
 * device get further process-wide contexts of their own (cached). */
int ozgpu_device_contexts(const int* devices, int count, ozgpu_ctx** out);
/* Device-resident twin: a, b, c are device pointers; the work is enqueued on
 * `stream` (a cudaStream_t; NULL is the legacy default stream) and the call returns without
 * synchronising.  Input validity (Inf/NaN/-0, scheme.cpp:223-225) is
 * reported through *dev_status (device int, may be NULL): 0 ok, nonzero dirty. */
int ozgpu_dgemm_device(ozgpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* a,
                       int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc,
                       ozgpu_mma_config cfg, const ozgpu_plan* plan, void* stream,
                       int* dev_status, ozgpu_diag* diag);
/* Device-resident sharding over the GPUs of the node (the
 * reference has no multi-device path -- scheme.cpp:219 is its one entry).
 * a, b, c are device pointers on src_device; C is split into the p_r x p_c
 * blocks of ozgpu_dgemm_multi.  A context on another device pulls its A
 * row-panel and B column-panel over NVLink (cudaMemcpy3DPeerAsync, peer
 * access enabled on first use), multiplies on its own stream and pushes its
 * C block back; a context on src_device reads its panels in place.  The work
 * is ordered after `stream` (a cudaStream_t on src_device) and `stream`
 * waits for every block, so the call returns without synchronising, like
 * ozgpu_dgemm_device.  dev_status: NULL or `count` device ints on
 * src_device, one per block (0 ok, nonzero: that block saw Inf / NaN / -0;
 * a product too small to split runs as one block, the other slots read 0).
 * Bit-identical to ozgpu_dgemm_device. */
int ozgpu_dgemm_device_multi(ozgpu_ctx* const* ctxs, int count, int src_device, int64_t m,
                             int64_t n, int64_t k, const double* a, int64_t lda, const double* b,
                             int64_t ldb, double* c, int64_t ldc, ozgpu_mma_config cfg,
                             const ozgpu_plan* plan, void* stream, int* dev_status,
                             ozgpu_diag* diag);

/* ---- debug hooks (bit-exact against the reference) --------------------- */
/* split_rows / split_cols, proj/src/slicing.cpp:67-132, on the GPU.
 * slices_out: [count][rows][cols] int64 (the reference's IntMatrix layout);
 * scales_out: rows (orientation 0) or cols (orientation 1) ints. */
int ozgpu_split(ozgpu_ctx* ctx, int orientation, int64_t rows, int64_t cols, const double* x,
                int64_t ldx, int width, int count, int mode, int64_t* slices_out,
                int* scales_out);
/* The production int8 slicer (the kernels ozgpu_dgemm* launch for its
 * operands: rowmax + streaming row slicer for A, column max + transposing
 * column slicer for B in truncate mode at t <= 7; generic kernels otherwise;
 * for small products, (m + n) k < 8M, multiply fuses both operands into two
 * launches that run the same row / column device code)
 * with its output as the GEMM reads it: slices_out [count][blocks][ld] int8,
 * K-major (blocks = rows for orientation 0, cols for 1; ld a multiple of 128
 * >= the block length, the tail zero-filled), scales_out per block.
 * Bit-exact against split_rows / split_cols (slicing.cpp:67-132). */
int ozgpu_split_i8(ozgpu_ctx* ctx, int orientation, int64_t rows, int64_t cols, const double* x,
                   int64_t ldx, int width, int count, int mode, int8_t* slices_out, int64_t ld,
                   int* scales_out);
/* The production pair GEMM's output before the combine: runs the slicing and
 * the tcgen05 pair-GEMM launch ozgpu_dgemm would make (same kernel choice,
 * chunk bins, lockstep and split-k tail; never row-blocked) and copies the
 * int32 chunk planes out.  Chunk c holds sum_{p < npairs} E_{l0+p, d+2-l0-p}
 * (integer_gemm of the slice pair, mma_sim.cpp:76-125, scheme.cpp:252-262).
 * *nchunks_out = chunk count; chunk_table (may be NULL) gets up to max_chunks
 * triples (d, l0, npairs); planes_out (NULL = query only) receives the window
 * rows [r0, r1) x columns [c0, c1) of every plane, [nchunks][r1-r0][c1-c0]. */
int ozgpu_pair_planes(ozgpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* a,
                      int64_t lda, const double* b, int64_t ldb, ozgpu_mma_config cfg,
                      const ozgpu_plan* plan, int* nchunks_out, int* chunk_table, int max_chunks,
                      int64_t r0, int64_t r1, int64_t c0, int64_t c1, int32_t* planes_out);
/* integer_gemm, proj/src/mma_sim.cpp:76-125: exact X (m x k) * Y (k x n)
 * on the tcgen05 int8 path (int32 accumulation in TMEM); when the inputs
 * do not fit int8 or the bound k*max|x|*max|y| can exceed I_T, an exact
 * CUDA-core path with per-MAC overflow checking (mma_sim.cpp:103-112) runs
 * instead.  c may be NULL (no accumulator input). */
int ozgpu_integer_gemm(ozgpu_ctx* ctx, int64_t m, int64_t k, int64_t n, const int64_t* x,
                       const int64_t* y, const int64_t* c, int64_t* out, ozgpu_mma_config cfg);

/* ---- "ozm1" matrix files (proj/include/ozmul/io.hpp:26-40; io.cpp:51-95) ----
 * format: 0 kHex (16 hex digits of the binary64 bits, bit-exact), 1 kDec
 * (shortest round-trip decimal).  Matrices are row-major. */
int ozgpu_matrix_file_shape(const char* path, int64_t* rows, int64_t* cols);
int ozgpu_read_matrix_file(const char* path, int format, int64_t rows, int64_t cols, double* out);
int ozgpu_write_matrix_file(const char* path, int format, int64_t rows, int64_t cols,
                            const double* a, int64_t ld);

#ifdef __cplusplus
}
#endif
#endif /* OZGPU_H */
