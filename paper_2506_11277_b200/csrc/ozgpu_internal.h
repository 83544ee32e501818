// Internal interface between the host orchestration (ozgpu_host.cpp) and
// the sm_100a kernels (ozgpu_kernels.cu).  Not installed; not part of the ABI.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ozgpu {

// GEMM tile geometry (tcgen05 kind::i8, one CTA per 128-row tile).
constexpr int kBlockM = 128;
constexpr int kBlockK = 128;  // bytes of K per pipeline stage (= 4 MMAs of K=32)
constexpr int kKPad = 128;    // slice rows are padded to a multiple of this

// One accumulation chunk: consecutive pairs (l0 + p, d + 2 - l0 - p),
// p in [0, npairs), all on diagonal d (shared scale 2^w(d)).  The exact
// combine adds the chunk's int32 sum shifted left by `shift` bits, with
// shift = (D - 1 - d) * t, so that the least significant diagonal has
// weight 2^0 (scheme.cpp:252-262).
struct ChunkDesc {
  int d;
  int l0;
  int npairs;
  int shift;
  int flush;  // sequential strategies: 1 = a reference chunk ends here (scheme.cpp:281-313)
};

struct GemmArgs {
  const ChunkDesc* chunks;
  int nchunks;
  int m, n;
  int kblocks;        // kp / kBlockK
  int tiles_m, tiles_n;
  int total_units;    // tiles_m * tiles_n * nchunks (split mode)
  int group;          // rasterisation: tile-rows per group (0 = 8)
  int pair_order;     // diagnostic: 1-CTA kernel walks 256-row pair tiles
  int l2_hint;        // CTA-pair kernel TMA cache policy: 0 none, 1 evict_last, 2 evict_normal
  // wave lockstep (CTA-pair kernel): the leader's producer publishes every
  // sync_g k-steps and waits until every cluster has passed the group
  // sync_d groups back, for its first sync_steps k-steps (all clusters run at
  // least that many).  sync = 64 zeroed counters, 128 bytes apart; null = off.
  int* sync;
  int sync_steps, sync_g, sync_d, sync_clusters, sync_prefetch;
  // split-k tail (CTA-pair kernel): units from tail_first on are the last
  // partial wave's units, each cut into tail_parts k-ranges whose partial
  // sums are added into the (pre-zeroed) plane; tail_parts = 0: off
  int tail_first, tail_parts;
  // measurement experiments only (OZGPU_DBG, results invalid): bit 0 maps
  // every unit of the CTA-pair kernel to tile 0 (ideal operand locality),
  // bit 1 drops its plane stores, bit 2 loads every B box twice (+L2 traffic)
  int dbg;
  // CTA-pair kernel tile width: 256 (256 x 256 tiles) or 512 (256 x 512)
  int pair_n;
  // kPN = 512: 1 = release the accumulator only once fully drained
  // (OZGPU_HALF_RELEASE=0, A/B of the half-by-half release)
  int no_half_release;
  // CTA-pair kernel: write the chunk planes with TMA bulk tensor stores
  int tma_store;
  // CTA-pair kernel cluster size: 2 (one pair) or 4 (two pairs stacked in M
  // sharing the B panel by multicast; pair_n 512 only)
  int cluster_ctas;
  int max_clusters;  // co-resident clusters to launch (0 = num_sms / cluster_ctas)
  int32_t* planes;    // [nchunks][m][ldp] int32 chunk sums
  int64_t plane_stride;
  int64_t ldp;
  // split mode with the exact combine folded into the last chunk's epilogue
  // (fused_words == 1): units run chunk-major in proc_order; the final
  // chunk's epilogue waits on tile_counters[tile] == nchunks - 1, then sums
  // the other chunks' planes diagonal by diagonal (diag_first) Horner-style,
  // rounds and stores C
  const int* proc_order;   // position -> chunk id (null = identity)
  const int* bin_first;    // split mode: bin b = positions [bin_first[b], bin_first[b+1]) (null = 1 chunk per unit)
  int final_chunk;
  int* tile_counters;
  const int* diag_first;   // diagonals + 1 entries
  int diagonals;
  int width;
  // fused exact epilogue (fused_words = W >= 2; units are tiles)
  int fused_words;
  uint64_t* scratch;  // per CTA: W x 256 x 128 words
  const int* qa;
  const int* qb;
  long w_last;
  double* c;
  int64_t ldc;
  int axpby;
  double alpha, beta;
  const double* cin;
  int64_t ldcin;
};

struct CombineArgs {
  const int32_t* planes;
  const ChunkDesc* chunks;
  int nchunks;
  int64_t plane_stride;
  int64_t ldp;
  const int* qa;
  const int* qb;
  int m, n;
  long w_last;         // exponent of the least significant diagonal: -(D+1)t (+2 nearest)
  int width;           // t
  int diagonals;       // D
  int hgroup;          // Horner combine: diagonals per int64 run (>= 1)
  int mode;            // 0 truncate, 1 nearest
  double* c;
  int64_t ldc;
  int* realized_psi;   // device int (atomicMax), sequential strategies only
  // optional axpby epilogue (scheme.cpp:363-372): d = alpha*c + beta*cin
  int axpby;
  double alpha, beta;
  const double* cin;
  int64_t ldcin;
};

// Launchers (return cudaError_t; 0 == success).  `launches` counts kernels.
cudaError_t launch_slice_rows(const double* a, int64_t lda, int64_t m, int64_t k, int64_t kp,
                              int width, int count, int mode, void* out, int out_is_i64,
                              int* scales, int* status, cudaStream_t st, int64_t* launches,
                              int64_t plane = 0);
cudaError_t launch_slice_cols(const double* b, int64_t ldb, int64_t k, int64_t n, int64_t kp,
                              int width, int count, int mode, void* out, int out_is_i64,
                              int* scales, unsigned long long* colmax, int* status,
                              cudaStream_t st, int64_t* launches, int64_t plane = 0);
// Small operands ((m + n) k < 8M entries, truncate mode, t = 7, 16-byte
// aligned A with an even lda, kp % 128 == 0): both operands' block maxima in
// one launch and both operands' slices in a second.  Returns false (nothing
// launched) when the shape does not qualify.
bool small_slicing_applies(int64_t m, int64_t n, int64_t k, int64_t kp, int width, int mode,
                           const double* a, int64_t lda);
cudaError_t launch_slice_small(const double* a, int64_t lda, int64_t m, const double* b,
                               int64_t ldb, int64_t n, int64_t k, int64_t kp, int count_a,
                               int count_b, int8_t* out_a, int64_t plane_a, int8_t* out_b,
                               int64_t plane_b, int* scales_a, int* scales_b,
                               unsigned long long* colmax, int* status, cudaStream_t st,
                               int64_t* launches);
// One persistent launch slicing A (rows) and / or B (columns) in truncate
// mode at width <= 7 into int8, reading each operand once from DRAM (ordered
// work queue over L2-sized panels).  a or b may be null (one operand only).
// work: slice_queue_work_ints(m, n, k, kp) ints of device scratch.
// upload copies a small host table to the device on `st` (graph-capture safe).
using UploadFn = void (*)(void* user, void* dst, const void* src, size_t bytes, cudaStream_t st);
int slice_queue_work_ints(int64_t m, int64_t n, int64_t k, int64_t kp);
cudaError_t launch_slice_queue(const double* a, int64_t lda, int64_t m, const double* b,
                               int64_t ldb, int64_t n, int64_t k, int64_t kp, int width,
                               int count_a, int count_b, int8_t* out_a, int64_t plane_a,
                               int8_t* out_b, int64_t plane_b, int* scales_a, int* scales_b,
                               unsigned long long* colmax, int* work, int* status,
                               UploadFn upload, void* upload_user, cudaStream_t st,
                               int64_t* launches);
cudaError_t launch_gemm_i8(const CUtensorMap* tma, const CUtensorMap* tmb, const GemmArgs& args,
                           int num_sms, cudaStream_t st, int64_t* launches);
cudaError_t launch_gemm_i8_mc(const CUtensorMap* tma, const CUtensorMap* tmb_half,
                              const GemmArgs& args, int num_sms, cudaStream_t st,
                              int64_t* launches);
// tmc: 3-D int32 tensor map over the chunk planes {n, m, nchunks}, box
// {32, 32, 1}, 128-byte swizzle (used when args.tma_store)
cudaError_t launch_gemm_i8_pair(const CUtensorMap* tma, const CUtensorMap* tmb,
                                const CUtensorMap* tmc, const GemmArgs& args, int num_sms,
                                cudaStream_t st, int64_t* launches);
int gemm_smem_bytes();
cudaError_t launch_combine_exact(const CombineArgs& args, int words, const ChunkDesc* host_chunks,
                                 cudaStream_t st, int64_t* launches);
cudaError_t launch_combine_sequential(const CombineArgs& args, cudaStream_t st,
                                      int64_t* launches);
cudaError_t launch_row_profile(const double* a, int64_t lda, int64_t m, int64_t k,
                               double* ratios, int* zero_flag, cudaStream_t st,
                               int64_t* launches);
cudaError_t launch_col_profile(const double* b, int64_t ldb, int64_t k, int64_t n,
                               unsigned long long* colmax, unsigned long long* colmin,
                               cudaStream_t st, int64_t* launches);
cudaError_t launch_fp64_gemm(int absolute, int64_t m, int64_t k, int64_t n, const double* a,
                             int64_t lda, const double* b, int64_t ldb, double* out, int64_t ldo,
                             cudaStream_t st, int64_t* launches);
// min_exact_slices bits (slicing.cpp:212-249): *bits_out = deepest fraction
// bit position holding a set bit over all rows (orientation 0) / columns (1).
cudaError_t launch_exact_bits(int orientation, const double* x, int64_t ldx, int64_t rows,
                              int64_t cols, unsigned long long* colmax, int* bits_out,
                              cudaStream_t st, int64_t* launches);
// error metrics: scratch[2P] = {max |c-r|/|r|, sum (c-r)^2} (r null: sum c^2)
int metric_scratch_doubles();
cudaError_t launch_error_metrics(const double* c, int64_t ldc, const double* r, int64_t ldr,
                                 int64_t m, int64_t n, double* scratch, cudaStream_t st,
                                 int64_t* launches);
cudaError_t launch_pack_i8(const int64_t* x, int64_t rows, int64_t cols, int transpose,
                           int64_t kp, int8_t* out, cudaStream_t st, int64_t* launches);
cudaError_t launch_integer_gemm_exact(const int64_t* x, const int64_t* y, const int64_t* c,
                                      int64_t* out, int64_t m, int64_t k, int64_t n,
                                      int acc_width, unsigned long long* first_overflow,
                                      cudaStream_t st, int64_t* launches);
cudaError_t launch_plane_to_i64(const int32_t* plane, int64_t ldp, const int64_t* c,
                                int64_t* out, int64_t m, int64_t n, cudaStream_t st,
                                int64_t* launches);

}  // namespace ozgpu
