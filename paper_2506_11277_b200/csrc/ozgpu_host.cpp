// Host orchestration and C-ABI of the B200-native Ozaki-I FP64 GEMM.
//
// ozgpu_dgemm* replace the reference's ozmul::multiply (proj/src/scheme.cpp:
// 219-361): validation in the reference's order, then three GPU stages on one
// stream -- slicing (HBM-bound), tcgen05 int8 pair GEMMs (tensor-bound) and
// the exact combine -- with no CPU fallback: a missing device is an error.
#include <cuda.h>
#include <cuda_runtime.h>

#include <unistd.h>
#include <immintrin.h>

#include <algorithm>
#include <map>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <mutex>
#include <set>
#include <thread>
#include <random>
#include <string>
#include <vector>

#include "ozgpu.h"
#include "ozgpu_internal.h"
#include "ozgpu_plan.h"

namespace ozgpu {
namespace {

thread_local std::string g_error;

}  // namespace

// for the C-ABI entry points defined in other translation units (ozgpu_io.cpp)
void set_last_error(const std::string& msg) { g_error = msg; }

namespace {

struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define OZ_CUDA(call)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw DeviceError(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + \
                        #call);                                                          \
  } while (0)

template <class F>
int guarded(F&& f) {
  try {
    f();
    return OZGPU_OK;
  } catch (const SelectionInfeasibleError& e) {
    g_error = e.what();
    return OZGPU_INFEASIBLE;
  } catch (const OverflowError& e) {
    g_error = e.what();
    return OZGPU_OVERFLOW;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return OZGPU_INVALID_ARGUMENT;
  } catch (const std::domain_error& e) {
    g_error = e.what();
    return OZGPU_DOMAIN_ERROR;
  } catch (const std::exception& e) {
    g_error = e.what();
    return OZGPU_DEVICE_ERROR;
  }
}

// Bumped whenever a workspace buffer is (re)allocated: captured CUDA graphs
// hold raw workspace pointers and are re-captured when it changes.
std::atomic<uint64_t> g_workspace_gen{0};

// A grow-only device allocation.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void* get(size_t want) {
    if (want > bytes) {
      g_workspace_gen.fetch_add(1);
      if (p) cudaFree(p);
      p = nullptr;
      bytes = 0;
      if (want) {
        cudaError_t e = cudaMalloc(&p, want);
        if (e != cudaSuccess) {
          cudaGetLastError();
          throw DeviceError("device allocation of " + std::to_string(want) +
                            " bytes failed: " + cudaGetErrorString(e));
        }
      }
      bytes = want;
    }
    return p;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

// Grow-only page-locked host buffer (staging of pageable caller buffers).
struct PinnedBuf {
  void* p = nullptr;
  size_t bytes = 0;
  // nullptr when the page-locked allocation fails (the caller then copies
  // from the pageable buffers directly); the runtime's sticky last error is
  // cleared so the failure cannot leak into a later, valid call.
  void* get(size_t want) {
    if (want > bytes) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      bytes = 0;
      if (cudaMallocHost(&p, want) != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
        return nullptr;
      }
      bytes = want;
    }
    return p;
  }
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
};

// A persistent fork-join pool for the host-side staging copies (one per
// context): run(nt, fn) calls fn(0..nt-1) on nt threads (the caller is one
// of them) and returns when all are done.
class CopyPool {
 public:
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      quit_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  template <class F>
  void run(int nt, F&& fn) {
    if (nt <= 1) {
      fn(0);
      return;
    }
    ensure(nt - 1);
    std::function<void(int)> task(std::forward<F>(fn));
    {
      std::lock_guard<std::mutex> lk(mu_);
      task_ = &task;
      parts_ = nt;
      next_ = 1;
      pending_ = nt - 1;
      ++gen_;
    }
    cv_.notify_all();
    task(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
    task_ = nullptr;
  }

 private:
  void ensure(int n) {
    while (static_cast<int>(workers_.size()) < n) workers_.emplace_back([this] { loop(); });
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::function<void(int)>* task = nullptr;
      int part = -1;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return quit_ || (gen_ != seen && task_ && next_ < parts_); });
        if (quit_) return;
        part = next_++;
        if (next_ >= parts_) seen = gen_;
        task = task_;
      }
      (*task)(part);
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0) done_cv_.notify_all();
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::function<void(int)>* task_ = nullptr;
  int parts_ = 0, next_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool quit_ = false;
};

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

}  // namespace
}  // namespace ozgpu

struct ozgpu_ctx {
  int device = 0;
  int num_sms = 0;
  size_t total_mem = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  std::atomic<int64_t> launches{0};
  ozgpu::EncodeTiledFn encode = nullptr;
  // workspace
  ozgpu::DevBuf slices_a, slices_b, qa, qb, colmax, colmin, status, planes, chunks, psi, scratch;
  ozgpu::DevBuf in_a, in_b, io_c, in_c2, ratios, i64a, i64b, i64c, i64o, ovf;
  std::vector<ozgpu::ChunkDesc> host_chunks;
  std::vector<int> host_aux;
  // CUDA-graph replay of ozgpu_dgemm_device (same shape, plan, pointers and
  // stream -> one cudaGraphLaunch): host-side tables uploaded by a captured
  // graph are staged in pinned buffers owned by the graph entry
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    uint64_t gen = 0;
    int64_t launches = 0;
    int uses = 0;
    std::vector<void*> pinned;
  };
  std::map<std::string, GraphEntry> graphs;
  GraphEntry* capturing = nullptr;
  ozgpu::DevBuf aux, counters, sync, qwork;
  // row-blocked H2D / compute / D2H pipeline of ozgpu_dgemm
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  // B's slicing runs on a forked stream, joined before the GEMM
  cudaStream_t fork_stream = nullptr;
  cudaEvent_t fork_ev[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> pipe_events;
  // pinned staging of pageable host A / B / C (ozgpu_dgemm)
  ozgpu::PinnedBuf stage_a, stage_b, stage_c;
  ozgpu::CopyPool copy_pool;  // staging copies (pageable <-> pinned)
  // Workspace ordering across streams: every call that touches the
  // workspace first makes its stream wait on ws_done (recorded where the
  // previous call's last use of the workspace was enqueued), and records it
  // again after its own enqueue.  ozgpu_dgemm_device returns without
  // synchronising, so without this a call on another stream (or the host
  // path on ctx->stream) could overwrite slices / planes still in use.
  cudaEvent_t ws_done = nullptr;
  bool ws_recorded = false;
  // ozgpu_dgemm_device_multi: this context's stream, and its A row-panel,
  // B column-panel, C block and status int when the operands live on
  // another device (pulled / pushed over NVLink by peer copies)
  std::mutex multi_mu;
  cudaStream_t multi_stream = nullptr;
  ozgpu::DevBuf peer_a, peer_b, peer_c, peer_status;
  // debug hook ozgpu_pair_planes: run_multiply stops after the pair GEMM
  // (split mode, no row blocking) and leaves the int32 chunk planes in
  // `planes` with this geometry
  bool debug_planes = false;
  int64_t dbg_plane_stride = 0, dbg_ldp = 0;
  // stage timing (ozgpu_set_stage_timing)
  bool timing = false;
  std::vector<std::array<cudaEvent_t, 4>> pending_events;
  std::vector<cudaEvent_t> event_pool;
  double stage_ms[3] = {0, 0, 0};
  int64_t timed_calls = 0;
};

namespace ozgpu {
namespace {

void init_ctx(ozgpu_ctx* ctx, int device) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    throw DeviceError("no CUDA device available (the Ozaki-I path has no CPU fallback)");
  }
  if (device < 0 || device >= count) throw std::invalid_argument("ozgpu_create: bad device index");
  cudaDeviceProp prop{};
  OZ_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10 || prop.minor != 0)
    throw DeviceError("device " + std::to_string(device) + " (" + prop.name + ", sm_" +
                      std::to_string(prop.major) + std::to_string(prop.minor) +
                      ") is not sm_100: kernels are built for sm_100a only");
  ctx->device = device;
  ctx->num_sms = prop.multiProcessorCount;
  ctx->total_mem = prop.totalGlobalMem;
  OZ_CUDA(cudaSetDevice(device));
  OZ_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  OZ_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess)
    throw DeviceError("cuTensorMapEncodeTiled unavailable from the driver");
  ctx->encode = reinterpret_cast<EncodeTiledFn>(fn);
}

// The one-launch queue slicer (launch_slice_queue, OZGPU_SLICE_QUEUE=1) for
// truncate-mode int8 operands.  Opt-in: measured on B200 it reads A and B
// 1.67x instead of 2x from DRAM (the slice pass's L2 re-reads still miss 65%
// with ~16 MB panels while the 1.6 GB of slice writes stream through L2) and
// is issue-bound like the two-kernel path, 1.11 vs 0.97 ms at 8192^2 (12,12)
// and 4.1 vs 3.4 ms at 16384^2 (13,12) inside the power-capped step
// (DESIGN.md 4).
bool use_slice_queue(int mode, int t, int64_t ld) {
  if (mode != 0 || t < 1 || t > 7 || ld % kKPad) return false;
  const char* env = std::getenv("OZGPU_SLICE_QUEUE");
  return env && std::string(env) == "1";
}

void upload_table(ozgpu_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st);

// UploadFn for the queue slicer's segment table
void upload_cb(void* user, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  upload_table(static_cast<ozgpu_ctx*>(user), dst, src, bytes, st);
}

int* queue_work(ozgpu_ctx* ctx, int64_t m, int64_t n, int64_t k, int64_t ld) {
  return static_cast<int*>(
      ctx->qwork.get(sizeof(int) * static_cast<size_t>(slice_queue_work_ints(m, n, k, ld))));
}

// Orders this call's use of the context workspace after every earlier
// call's (caller holds ctx->mu; `st` is the stream the call enqueues its
// first workspace access on -- helper streams fork from it by events).
void acquire_workspace(ozgpu_ctx* ctx, cudaStream_t st) {
  if (ctx->ws_recorded) OZ_CUDA(cudaStreamWaitEvent(st, ctx->ws_done, 0));
}

// Marks the end of this call's workspace use on `st` (every helper stream
// has been joined back into `st` by then).
void release_workspace(ozgpu_ctx* ctx, cudaStream_t st) {
  if (!ctx->ws_done) OZ_CUDA(cudaEventCreateWithFlags(&ctx->ws_done, cudaEventDisableTiming));
  OZ_CUDA(cudaEventRecord(ctx->ws_done, st));
  ctx->ws_recorded = true;
}

// TMA L2 sector promotion of the slice loads (OZGPU_L2_PROMO=0/64/128/256).
CUtensorMapL2promotion l2_promotion() {
  if (const char* env = std::getenv("OZGPU_L2_PROMO")) {
    const int v = std::atoi(env);
    if (v == 0) return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    if (v == 64) return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    if (v == 128) return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  }
  return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}

// 3-D int8 tensor map over slices [count][rows][kp], box {128, box_rows, 1},
// 128-byte swizzle (matches the UMMA SW128 K-major descriptor).
CUtensorMap make_slice_map(ozgpu_ctx* ctx, const void* base, int64_t kp, int64_t rows,
                           int count, int box_rows, int64_t plane = 0, int64_t ld = 0) {
  CUtensorMap m;
  if (ld == 0) ld = kp;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(kp), static_cast<cuuint64_t>(rows),
                        static_cast<cuuint64_t>(count)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld),
                           static_cast<cuuint64_t>(plane ? plane : ld * rows)};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(kBlockK), static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = ctx->encode(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, l2_promotion(),
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw DeviceError("cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// 3-D int32 tensor map over the chunk planes [nchunks][m][ldp] (element
// strides ldp and plane), box {32 columns, 32 rows, 1}, 128-byte swizzle:
// the pair GEMM's epilogue TMA-stores 32 x 32 tiles through it; the map's
// extent {n, m} clips the ragged edges.
CUtensorMap make_plane_map(ozgpu_ctx* ctx, int32_t* planes, int64_t n, int64_t m, int64_t ldp,
                           int nchunks, int64_t plane) {
  CUtensorMap map;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(m),
                        static_cast<cuuint64_t>(nchunks)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ldp * 4), static_cast<cuuint64_t>(plane * 4)};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = ctx->encode(&map, CU_TENSOR_MAP_DATA_TYPE_INT32, 3, planes, dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw DeviceError("cuTensorMapEncodeTiled (planes) failed: " + std::to_string(r));
  return map;
}

// Row stride of the slice buffers: the K extent kp (a multiple of 128) plus
// an optional pad (OZGPU_KPAD bytes, multiple of 128; the pad is zero-filled
// by the slicing kernels and never read by the GEMM).
int64_t slice_ld(int64_t kp) {
  int64_t pad = 0;
  if (const char* env = std::getenv("OZGPU_KPAD")) pad = round_up(std::max<int64_t>(0, std::atoll(env)), 128);
  return kp + pad;
}

cudaEvent_t take_event(ozgpu_ctx* ctx) {
  if (!ctx->event_pool.empty()) {
    cudaEvent_t e = ctx->event_pool.back();
    ctx->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  OZ_CUDA(cudaEventCreate(&e));
  return e;
}

// Resolves pending stage events into ctx->stage_ms (caller holds ctx->mu).
void drain_events(ozgpu_ctx* ctx) {
  for (auto& ev : ctx->pending_events) {
    OZ_CUDA(cudaEventSynchronize(ev[3]));
    for (int s = 0; s < 3; ++s) {
      float ms = 0.f;
      OZ_CUDA(cudaEventElapsedTime(&ms, ev[s], ev[s + 1]));
      ctx->stage_ms[s] += ms;
    }
    ++ctx->timed_calls;
    for (cudaEvent_t e : ev) ctx->event_pool.push_back(e);
  }
  ctx->pending_events.clear();
}

// Chunking of the scheduled pairs.  Levelled-exact: the int32 capacity of the
// tensor-core accumulator bounds the pairs per chunk (the result is order-
// independent).  Float-per-product: one pair per chunk.  Diagonal-integer:
// the reference's flush grouping (scheme.cpp:281-313), split further only if
// a reference chunk could exceed int32 (flush_after marks the end of a
// reference chunk).
struct ChunkPlan {
  std::vector<ChunkDesc> chunks;
  int diagonals = 0;
};

ChunkPlan build_chunks(const ozgpu_plan& p, const ozgpu_mma_config& cfg, int64_t k) {
  ChunkPlan cp;
  cp.diagonals = max_diag_sum(p) - 1;
  const int t = p.width;
  const int64_t maxs = (int64_t{1} << t) - 1;
  const int64_t prod_bound = k * maxs * maxs;
  int64_t cap32 = std::max<int64_t>(1, (int64_t{2147483647}) / std::max<int64_t>(prod_bound, 1));
  int64_t ref_flush = 0;
  if (p.strategy == 1) {
    ref_flush = diagonal_flush_threshold(cfg, t, k);
    if (p.precision < cfg.acc_width)
      ref_flush = std::min(ref_flush, int64_t{1} << std::max(0, p.precision - 2 * t - ceil_log2(k)));
  }
  for (int d = 0; d < cp.diagonals; ++d) {
    int w = diagonal_width(d, p.slices_a, p.slices_b);
    if (w == 0) continue;
    int l0 = diagonal_first_l(d, p.slices_b);
    int shift = (cp.diagonals - 1 - d) * t;
    if (p.strategy == 2) {
      for (int s = 0; s < w; s += static_cast<int>(cap32)) {
        int np = static_cast<int>(std::min<int64_t>(cap32, w - s));
        cp.chunks.push_back({d, l0 + s, np, shift, 1});
      }
    } else if (p.strategy == 0) {
      for (int s = 0; s < w; ++s) cp.chunks.push_back({d, l0 + s, 1, shift, 1});
    } else {
      for (int s = 0; s < w; s += static_cast<int>(std::min<int64_t>(ref_flush, w))) {
        int ref_len = static_cast<int>(std::min<int64_t>(ref_flush, w - s));
        for (int u = 0; u < ref_len; u += static_cast<int>(cap32)) {
          int np = static_cast<int>(std::min<int64_t>(cap32, ref_len - u));
          cp.chunks.push_back({d, l0 + s + u, np, shift, u + np >= ref_len ? 1 : 0});
        }
      }
    }
  }
  return cp;
}

// Bins of the split-mode GEMM: chunks packed (first-fit decreasing) into
// runs with the same total pair count, so every unit of the pair GEMM has the
// same length and the CTAs of a wave stay in step (they then stream the same
// slice pair at the same time and share it through L2).  Tries bin sizes
// from the largest chunk upward and keeps the first packing in which every
// bin is full, then consecutive cuts (below).  For the reduced schedule the
// diagonals 1..L pair up as (1, L), (2, L-1), ... into bins of L + 1.
bool build_bins(const std::vector<ChunkDesc>& chunks, std::vector<int>& order,
                std::vector<int>& first) {
  const int nc = static_cast<int>(chunks.size());
  if (nc < 2) return false;
  int total = 0, maxlen = 0;
  for (const auto& c : chunks) {
    total += c.npairs;
    maxlen = std::max(maxlen, c.npairs);
  }
  std::vector<int> idx(nc);
  for (int i = 0; i < nc; ++i) idx[i] = i;
  std::stable_sort(idx.begin(), idx.end(),
                   [&](int a, int b) { return chunks[a].npairs > chunks[b].npairs; });
  for (int cap = maxlen; cap <= 2 * maxlen; ++cap) {
    if (total % cap) continue;
    std::vector<std::vector<int>> bins;
    std::vector<int> fill;
    for (int i : idx) {
      size_t b = 0;
      while (b < bins.size() && fill[b] + chunks[i].npairs > cap) ++b;
      if (b == bins.size()) {
        bins.emplace_back();
        fill.push_back(0);
      }
      bins[b].push_back(i);
      fill[b] += chunks[i].npairs;
    }
    if (static_cast<int>(bins.size()) * cap != total) continue;
    order.clear();
    first.clear();
    for (auto& b : bins) {
      first.push_back(static_cast<int>(order.size()));
      order.insert(order.end(), b.begin(), b.end());
    }
    first.push_back(static_cast<int>(order.size()));
    return true;
  }
  // No first-fit packing (e.g. k = 32768: int32 capacity 4 pairs per chunk,
  // lengths 1..4): cut the chunks in diagonal order into consecutive runs of
  // equal length -- the smallest length that divides the pair count and
  // falls on chunk boundaries; at worst one bin holds every chunk (a unit is
  // then a whole tile, still equal-length).
  for (int len = maxlen; len <= total; ++len) {
    if (total % len) continue;
    std::vector<int> cut{0};
    int acc = 0;
    bool ok = true;
    for (int c = 0; c < nc && ok; ++c) {
      acc += chunks[c].npairs;
      if (acc == len) {
        cut.push_back(c + 1);
        acc = 0;
      } else if (acc > len) {
        ok = false;
      }
    }
    if (!ok || acc != 0) continue;
    order.resize(nc);
    for (int c = 0; c < nc; ++c) order[c] = c;
    first = cut;
    return true;
  }
  return false;
}

// Co-resident clusters of the CTA-pair kernel: 4-CTA clusters cannot tile
// every GPC of the 148-SM part (33 fit, OZGPU_QUAD_CLUSTERS overrides).
int max_pair_clusters(int num_sms, int cluster_ctas) {
  if (cluster_ctas != 4) return num_sms / 2;
  if (const char* env = std::getenv("OZGPU_QUAD_CLUSTERS")) return std::max(1, std::atoi(env));
  return num_sms * 33 / 148;
}

// Wave lockstep of the 2-CTA GEMM kernels (GemmArgs::sync): equal-length
// units (bins) only; OZGPU_SYNC=0/1, OZGPU_SYNC_G / OZGPU_SYNC_D override the
// group size and the allowed lag in groups.
void setup_lockstep(ozgpu_ctx* ctx, GemmArgs& g, const ChunkPlan& cp, const std::vector<int>& aux,
                    const std::vector<int>& bfirst, cudaStream_t st, DevBuf& sync_buf) {
  if (!g.bin_first || bfirst.size() < 2) return;
  bool sync = true;
  if (const char* env = std::getenv("OZGPU_SYNC")) sync = std::string(env) == "1";
  if (!sync) return;
  const int clusters = std::min(max_pair_clusters(ctx->num_sms, g.cluster_ctas), g.total_units);
  int bin_pairs = 0;
  for (int q = bfirst[0]; q < bfirst[1]; ++q) bin_pairs += cp.chunks[aux[q]].npairs;
  g.sync = static_cast<int*>(sync_buf.get(sizeof(int) * 64 * 32));
  OZ_CUDA(cudaMemsetAsync(g.sync, 0, sizeof(int) * 64 * 32, st));
  g.sync_clusters = clusters;
  g.sync_steps = (g.total_units / clusters) * bin_pairs * g.kblocks;
  g.sync_g = g.pair_n == 512 ? 32 : 64;  // k-steps per lockstep group (measured per tile width)
  g.sync_d = 1;
  if (const char* env = std::getenv("OZGPU_SYNC_G")) g.sync_g = std::max(1, std::atoi(env));
  if (const char* env = std::getenv("OZGPU_SYNC_D")) g.sync_d = std::max(1, std::atoi(env));
  g.sync_prefetch = 1;
  if (const char* env = std::getenv("OZGPU_SYNC_PREFETCH")) g.sync_prefetch = std::atoi(env);
}

// Diagnostics exactly as the reference accumulates them (scheme.cpp:246-359).
ozgpu_diag make_diag(const ozgpu_plan& p, const ozgpu_mma_config& cfg, int64_t m, int64_t n,
                     int64_t k, long long realized_psi) {
  ozgpu_diag d{};
  d.width = p.width;
  d.acc_bits_used = 2 * p.width + ceil_log2(k);
  d.planned_psi = p.psi;
  const uint64_t mn = static_cast<uint64_t>(m) * static_cast<uint64_t>(n);
  const int diagonals = max_diag_sum(p) - 1;
  uint64_t products = 0, iadds = 0, fadds = 0, flushes = 0;
  if (p.strategy == 1) {
    int64_t flush = diagonal_flush_threshold(cfg, p.width, k);
    if (p.precision < cfg.acc_width)
      flush = std::min(flush, int64_t{1} << std::max(0, p.precision - d.acc_bits_used));
    for (int dd = 0; dd < diagonals; ++dd) {
      int64_t w = diagonal_width(dd, p.slices_a, p.slices_b);
      int64_t chunks = 0;
      for (int64_t taken = 0; taken < w;) {
        int64_t in_chain = std::min<int64_t>(flush, w - taken);
        products += in_chain;
        iadds += static_cast<uint64_t>(k - 1) * mn + static_cast<uint64_t>(in_chain - 1) *
                                                          static_cast<uint64_t>(k) * mn;
        fadds += 1;
        taken += in_chain;
        ++chunks;
      }
      if (chunks > 1) flushes += chunks - 1;
    }
  } else {
    for (int dd = 0; dd < diagonals; ++dd) {
      int64_t w = diagonal_width(dd, p.slices_a, p.slices_b);
      products += w;
      iadds += static_cast<uint64_t>(w) * static_cast<uint64_t>(k - 1) * mn;
      fadds += w;
    }
    if (p.strategy == 2) {
      // level count as multiply() re-derives it when the plan's levels do
      // not tile the diagonals (scheme.cpp:316-320)
      int nlev = p.num_levels;
      if (nlev == 0 || p.levels[0] != 0 || p.levels[2 * (nlev - 1) + 1] != diagonals - 1)
        nlev = static_cast<int>(plan_levels(p.precision, p.width, d.acc_bits_used, diagonals)
                                    .levels.size());
      if (nlev > 1) fadds += nlev - 1;
    }
  }
  d.products = static_cast<int64_t>(products);
  d.integer_adds = static_cast<int64_t>(iadds);
  d.float_adds = static_cast<int64_t>(fadds);
  d.flushes = static_cast<int64_t>(flushes);
  d.realized_psi = realized_psi;
  return d;
}

struct ValidationResult {
  bool capacity_error = false;
  bool precision_error = false;
  std::string message;
};

// scheme.cpp:221-239 (minus the clean-input scan, which runs on the GPU)
ValidationResult host_validation(const ozgpu_mma_config& cfg, const ozgpu_plan& p, int64_t k) {
  validate_cfg(cfg);
  ValidationResult v;
  const int t = p.width;
  if (k >= 1) {
    if (2 * t + ceil_log2(k) > cfg.acc_width) {
      v.capacity_error = true;
      v.message = "multiply: inner dimension " + std::to_string(k) +
                  " exceeds the capacity limit " + std::to_string(max_inner_dim(cfg)) +
                  " of this unit";
    } else if (p.precision < 2 * t + ceil_log2(k)) {
      v.precision_error = true;
      v.message = "multiply: accumulation format too narrow for exact conversion; needs " +
                  std::to_string(2 * t + ceil_log2(k)) + " bits";
    }
  }
  return v;
}

int exact_words(int diagonals, int width, size_t nchunks) {
  int bits = (diagonals - 1) * width + 32 + ceil_log2(static_cast<int64_t>(nchunks) + 1) + 2;
  int w = (bits + 63) / 64;
  for (int cand : {2, 3, 4, 6, 8, 12, 16})
    if (w <= cand) return cand;
  throw std::invalid_argument("multiply: exact accumulator wider than 1024 bits");
}

// Host -> device copy of a small host-built table on `st`.  Inside a graph
// capture the source is first staged in pinned memory owned by the graph, so
// the captured copy node stays valid for every replay.
void upload_table(ozgpu_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (ctx->capturing) {
    void* pin = nullptr;
    OZ_CUDA(cudaMallocHost(&pin, bytes));
    std::memcpy(pin, src, bytes);
    ctx->capturing->pinned.push_back(pin);
    src = pin;
  }
  OZ_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
}

// Operands already sliced by the caller (the blocked pipeline of
// host_multiply): a row range of the [count][rows][kp] slice buffers, with
// the full buffers' plane stride, and the matching scales.
struct Presliced {
  const int8_t* a;
  int64_t plane_a;
  const int* qa;
  const int8_t* b;
  int64_t plane_b;
  const int* qb;
  int64_t ld;  // row stride of the slice buffers
};

// The device-resident core of multiply(): everything is enqueued on `st`.
// Returns the realized psi device pointer (sequential strategies) or null.
int* run_multiply(ozgpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* da, int64_t lda,
                  const double* db, int64_t ldb, double* dc, int64_t ldc,
                  const ozgpu_mma_config& cfg, const ozgpu_plan& p, cudaStream_t st,
                  int* dev_status, bool axpby, double alpha, double beta, const double* dcin,
                  int64_t ldcin, const Presliced* pre = nullptr) {
  int64_t launches = 0;
  std::array<cudaEvent_t, 4> ev{};
  if (ctx->timing) {
    for (auto& e : ev) e = take_event(ctx);
    OZ_CUDA(cudaEventRecord(ev[0], st));
  }
  const int t = p.width;
  if (t > 7)
    throw std::invalid_argument("multiply: slice width " + std::to_string(t) +
                                " exceeds the int8 tensor-core operand (t <= 7)");
  if (t < 1 || t > 62) throw std::invalid_argument("split: width out of range");
  if (p.mode == 1 && t < 2) throw std::invalid_argument("split: nearest mode needs width >= 2");
  const int sa = p.slices_a, sb = p.slices_b;
  const int64_t kp = round_up(k, kKPad);
  const int64_t ld = pre ? pre->ld : slice_ld(kp);
  ChunkPlan cp = build_chunks(p, cfg, k);

  const int8_t* slA;
  const int8_t* slB;
  const int* qa;
  const int* qb;
  int64_t plane_a = m * ld, plane_b = n * ld;
  if (pre) {
    slA = pre->a;
    slB = pre->b;
    qa = pre->qa;
    qb = pre->qb;
    plane_a = pre->plane_a;
    plane_b = pre->plane_b;
  } else {
    int8_t* wa = static_cast<int8_t*>(ctx->slices_a.get(static_cast<size_t>(sa) * m * ld + 1));
    int8_t* wb = static_cast<int8_t*>(ctx->slices_b.get(static_cast<size_t>(sb) * n * ld + 1));
    int* wqa = static_cast<int*>(ctx->qa.get(sizeof(int) * (m + 1)));
    int* wqb = static_cast<int*>(ctx->qb.get(sizeof(int) * (n + 1)));
    auto* colmax = static_cast<unsigned long long*>(ctx->colmax.get(8 * (n + 1)));
    int* status = dev_status ? dev_status : static_cast<int*>(ctx->status.get(sizeof(int)));
    OZ_CUDA(cudaMemsetAsync(status, 0, sizeof(int), st));
    if (use_slice_queue(p.mode, t, ld)) {
      // both operands in one launch, each read once from DRAM
      OZ_CUDA(launch_slice_queue(da, lda, m, db, ldb, n, k, ld, t, sa, sb, wa, 0, wb, 0, wqa, wqb,
                                 colmax, queue_work(ctx, m, n, k, ld), status, upload_cb, ctx, st,
                                 &launches));
      slA = wa;
      slB = wb;
      qa = wqa;
      qb = wqb;
    } else if (small_slicing_applies(m, n, k, ld, t, p.mode, da, lda)) {
      // small operands: two launches cover both (launch latency dominates)
      OZ_CUDA(launch_slice_small(da, lda, m, db, ldb, n, k, ld, sa, sb, wa, m * ld, wb, n * ld, wqa,
                                 wqb, colmax, status, st, &launches));
      slA = wa;
      slB = wb;
      qa = wqa;
      qb = wqb;
    } else {
    // A's and B's slicing are independent: B's runs on a forked stream so
    // the two HBM-bound chains overlap (their tails and the short memsets
    // hide each other); joined before the GEMM.  OZGPU_SLICE_FORK=0: serial.
    const char* fv = std::getenv("OZGPU_SLICE_FORK");
    // (small operands: the fork / join costs more than the overlap saves)
    const bool fork = !(fv && std::string(fv) == "0") && m > 0 && n > 0 &&
                      (m + n) * k >= (int64_t{8} << 20);
    cudaStream_t sb_st = st;
    if (fork) {
      if (!ctx->fork_stream) {
        OZ_CUDA(cudaStreamCreateWithFlags(&ctx->fork_stream, cudaStreamNonBlocking));
        OZ_CUDA(cudaEventCreateWithFlags(&ctx->fork_ev[0], cudaEventDisableTiming));
        OZ_CUDA(cudaEventCreateWithFlags(&ctx->fork_ev[1], cudaEventDisableTiming));
      }
      OZ_CUDA(cudaEventRecord(ctx->fork_ev[0], st));
      OZ_CUDA(cudaStreamWaitEvent(ctx->fork_stream, ctx->fork_ev[0], 0));
      sb_st = ctx->fork_stream;
    }
    OZ_CUDA(launch_slice_cols(db, ldb, k, n, ld, t, sb, p.mode, wb, 0, wqb, colmax, status, sb_st,
                              &launches));
    OZ_CUDA(launch_slice_rows(da, lda, m, k, ld, t, sa, p.mode, wa, 0, wqa, status, st,
                              &launches));
    if (fork) {
      OZ_CUDA(cudaEventRecord(ctx->fork_ev[1], sb_st));
      OZ_CUDA(cudaStreamWaitEvent(st, ctx->fork_ev[1], 0));
    }
    slA = wa;
    slB = wb;
    qa = wqa;
    qb = wqb;
    }
  }
  if (ctx->timing) OZ_CUDA(cudaEventRecord(ev[1], st));

  // Chunk-plane memory budget: the int32 planes cost 4 * chunks * m * n
  // bytes (72 GiB for 32768^3 at (13,12)); beyond the budget the GEMM +
  // combine run over row blocks of C against the slices already in HBM
  // (blocking is exact: scales are per row of A / column of B).
  if (p.strategy == 2 && m > 512 && n > 0 && !cp.chunks.empty() && !ctx->debug_planes) {
    const int64_t ldp_b = round_up(n, 4);
    const double plane_bytes = 4.0 * static_cast<double>(cp.chunks.size()) * m * ldp_b;
    double budget = 0.0;
    if (const char* env = std::getenv("OZGPU_PLANE_BUDGET_GB")) {
      budget = std::atof(env) * 1073741824.0;
    } else {
      budget = 0.25 * static_cast<double>(ctx->total_mem);  // no per-call driver query
    }
    if (plane_bytes > budget) {
      const double per_row = 4.0 * static_cast<double>(cp.chunks.size()) * ldp_b;
      int64_t rows = static_cast<int64_t>(budget / per_row) / 256 * 256;
      rows = std::max<int64_t>(rows, 256);
      const bool timing = ctx->timing;
      ctx->timing = false;  // the blocks' GEMM + combine are timed as one stage
      for (int64_t r0 = 0; r0 < m; r0 += rows) {
        const int64_t r1 = std::min(m, r0 + rows);
        Presliced sub{slA + r0 * ld, plane_a, qa + r0, slB, plane_b, qb, ld};
        run_multiply(ctx, r1 - r0, n, k, nullptr, 0, nullptr, 0, dc + r0 * ldc, ldc, cfg, p, st,
                     nullptr, axpby, alpha, beta, dcin ? dcin + r0 * ldcin : nullptr, ldcin, &sub);
      }
      ctx->timing = timing;
      if (ctx->timing) {
        OZ_CUDA(cudaEventRecord(ev[2], st));
        OZ_CUDA(cudaEventRecord(ev[3], st));
        ctx->pending_events.push_back(ev);
      }
      ctx->launches += launches;
      return nullptr;
    }
  }

  int* psi_dev = nullptr;
  if (m > 0 && n > 0 && !cp.chunks.empty()) {
    const int tiles_m = static_cast<int>((m + kBlockM - 1) / kBlockM);
    const int tiles_n = static_cast<int>((n + 255) / 256);
    const int64_t tiles = static_cast<int64_t>(tiles_m) * tiles_n;
    const long w_last = -static_cast<long>(cp.diagonals + 1) * t + (p.mode == 1 ? 2 : 0);
    // Default: split units over (tile, chunk) writing int32 chunk planes, then
    // the bandwidth-bound exact combine.  The fused exact epilogue (W-word
    // RMW in a CTA-private scratch) is opt-in (OZGPU_EPILOGUE=fused): measured
    // on B200 at 8192^3 (12,12) its scratch traffic evicts operand panels from
    // L2 (105 GB vs 66 GB DRAM per launch) and loses to split + combine.
    int words = p.strategy == 2 ? exact_words(cp.diagonals, t, cp.chunks.size()) : 0;
    bool fused = false;
    if (const char* env = ctx->debug_planes ? nullptr : std::getenv("OZGPU_EPILOGUE")) {
      if (std::string(env) == "split") fused = false;
      if (std::string(env) == "fused" && p.strategy == 2 && words <= 3) fused = true;
    }
    if (fused) {
      if (words < 2) words = 2;
      // Alternate long and short chunks so the epilogue of a short chunk
      // overlaps the MMAs of a long one (the exact sum is order-free).
      std::vector<ChunkDesc> sorted = cp.chunks;
      std::stable_sort(sorted.begin(), sorted.end(),
                       [](const ChunkDesc& x, const ChunkDesc& y) { return x.npairs > y.npairs; });
      std::vector<ChunkDesc> order;
      for (size_t lo = 0, hi = sorted.size(); lo < hi;) {
        order.push_back(sorted[lo++]);
        if (lo < hi) order.push_back(sorted[--hi]);
      }
      cp.chunks = order;
    }
    ChunkDesc* dchunks =
        static_cast<ChunkDesc*>(ctx->chunks.get(sizeof(ChunkDesc) * cp.chunks.size()));
    upload_table(ctx, dchunks, cp.chunks.data(), sizeof(ChunkDesc) * cp.chunks.size(), st);
    ctx->host_chunks = cp.chunks;

    CUtensorMap tma = make_slice_map(ctx, slA, kp, m, sa, kBlockM, plane_a, ld);
    CUtensorMap tmb = make_slice_map(ctx, slB, kp, n, sb, 256, plane_b, ld);
    GemmArgs g{};
    g.chunks = dchunks;
    g.nchunks = static_cast<int>(cp.chunks.size());
    g.m = static_cast<int>(m);
    g.n = static_cast<int>(n);
    g.kblocks = static_cast<int>(kp / kBlockK);
    g.tiles_m = tiles_m;
    g.tiles_n = tiles_n;
    if (const char* env = std::getenv("OZGPU_RASTER_G")) g.group = std::atoi(env);
    if (const char* env = std::getenv("OZGPU_L2_HINT")) g.l2_hint = std::atoi(env);
    if (const char* env = std::getenv("OZGPU_DBG")) g.dbg = std::atoi(env);
    if (const char* env = std::getenv("OZGPU_HALF_RELEASE")) g.no_half_release = std::atoi(env) == 0;
    if (const char* env = std::getenv("OZGPU_PAIR_ORDER"))
      g.pair_order = std::string(env) == "1" && tiles_m % 2 == 0;
    if (fused) {
      g.total_units = static_cast<int>(tiles);
      g.fused_words = words;
      const int grid = static_cast<int>(std::min<int64_t>(tiles, ctx->num_sms));
      g.scratch = static_cast<uint64_t*>(
          ctx->scratch.get(sizeof(uint64_t) * static_cast<size_t>(grid) * words * 256 * kBlockM));
      g.qa = qa;
      g.qb = qb;
      g.w_last = w_last;
      g.c = dc;
      g.ldc = ldc;
      g.axpby = axpby ? 1 : 0;
      g.alpha = alpha;
      g.beta = beta;
      g.cin = dcin;
      g.ldcin = ldcin;
      OZ_CUDA(launch_gemm_i8(&tma, &tmb, g, ctx->num_sms, st, &launches));
      if (ctx->timing) {
        OZ_CUDA(cudaEventRecord(ev[2], st));
        OZ_CUDA(cudaEventRecord(ev[3], st));
        ctx->pending_events.push_back(ev);
      }
      ctx->launches += launches;
      return nullptr;
    }
    const int64_t ldp = round_up(n, 4);
    // chunk planes are skewed by 4352 bytes so the combine's concurrent
    // per-plane streams do not sit a power of two apart (OZGPU_PLANE_SKEW ints)
    int64_t skew = 1088;
    if (const char* env = std::getenv("OZGPU_PLANE_SKEW")) skew = std::atoll(env) & ~int64_t{3};
    const int64_t plane = m * ldp + skew;
    int32_t* planes = static_cast<int32_t*>(
        ctx->planes.get(sizeof(int32_t) * static_cast<size_t>(plane) * cp.chunks.size()));
    g.planes = planes;
    g.plane_stride = plane;
    g.ldp = ldp;
    // Default: the CTA-pair kernel (cta_group::2, 256 x 256 tiles, 6-stage
    // ring) with equal-length bins and wave lockstep.  Measured on B200 at
    // 8192^3 (12,12), interleaved and power-capped: 29.2 ms per launch vs
    // 30.4 ms for the B-multicast 1-CTA kernel (OZGPU_CTA_PAIR=0) and 30.8 ms
    // without lockstep; DRAM reads 46 GB, tensor pipe 93 % active at the base
    // clock.  Without lockstep the deep ring lets the CTAs of a wave drift
    // apart and DRAM reads grow 2-3.5x.
    bool pair = m >= 256;
    if (const char* env = std::getenv("OZGPU_CTA_PAIR")) pair = std::string(env) == "1" && m >= 256;
    // Pair tile width (OZGPU_PAIR_N = 256 / 512).  256 x 512 tiles by default:
    // each wave of 74 CTA pairs then covers twice the C area per slice byte
    // it reads, and at the power cap the saved DRAM / L2 traffic buys clock.
    // Measured on B200 (tools/gemm_ab.py, interleaved, bitwise identical):
    // 8192^3 (12,12) 29.3 -> 27.1 ms, 16384^3 (13,12) 276.8 -> 244.3 ms,
    // 32768^3 2141 -> 1949 ms, 4096^3 (16,17) 6.04 -> 5.72 ms, 65536 x 2048^2
    // (12,11) 14.62 -> 14.42 ms.
    // Small products keep 256-wide tiles (enough units to fill two waves of
    // CTA pairs: at 1024^3 (4,4) 0.027 vs 0.039 ms).
    const int64_t units512 = ((m + 255) / 256) * ((n + 511) / 512) * static_cast<int64_t>(g.nchunks);
    int pair_n = n > 256 && units512 >= ctx->num_sms ? 512 : 256;
    if (const char* env = std::getenv("OZGPU_PAIR_N")) pair_n = std::atoi(env) == 512 ? 512 : 256;
    // One launch of the CTA-pair kernel over C rows [row0, row0 + rows) with
    // clusters of `cl` CTAs (2: one pair; 4: two pairs stacked in M sharing
    // the B panel by multicast, 512-wide tiles only), its own lockstep
    // counters and split-k tail.
    bool bins_ok = false;  // set below, before the launches
    std::vector<int> bfirst;
    int* daux = nullptr;
    auto launch_pair_part = [&](int64_t row0, int64_t rows, int cl, cudaStream_t pst,
                                DevBuf& sync_buf) {
      GemmArgs gp = g;
      const int unit_rows = 128 * cl;  // 256 per CTA pair
      const int pair_tiles_n = static_cast<int>((n + pair_n - 1) / pair_n);
      const int pair_tiles =
          static_cast<int>(((rows + unit_rows - 1) / unit_rows) * pair_tiles_n);
      gp.m = static_cast<int>(rows);
      gp.pair_n = pair_n;
      gp.cluster_ctas = cl;
      gp.max_clusters = max_pair_clusters(ctx->num_sms, cl);
      gp.tiles_n = pair_tiles_n;
      gp.tiles_m = static_cast<int>((rows + unit_rows - 1) / unit_rows);
      // raster groups of 16 tile rows balance a wave's A and B footprint for
      // 256 x 512 tiles on large squares; 8 on narrow / small grids (measured)
      if (!std::getenv("OZGPU_RASTER_G") && pair_n == 512)
        gp.group = cl == 4 ? (gp.tiles_m >= 16 && gp.tiles_n >= 16 ? 8 : 4)
                           : (gp.tiles_m >= 32 && gp.tiles_n >= 16 ? 16 : 8);
      gp.total_units = pair_tiles * gp.nchunks;
      bool bins = static_cast<int64_t>(pair_tiles) * gp.nchunks >= 2 * static_cast<int64_t>(ctx->num_sms);
      if (const char* env = std::getenv("OZGPU_BINS")) bins = std::string(env) == "1";
      std::vector<int>& aux = ctx->host_aux;
      std::vector<int> no_bins;
      const std::vector<int>& bf = bins && bins_ok ? bfirst : no_bins;
      if (bins && bins_ok) {
        const size_t nb = bfirst.size() - 1;
        gp.proc_order = daux;
        gp.bin_first = daux + gp.nchunks;
        gp.total_units = static_cast<int>(static_cast<int64_t>(pair_tiles) * nb);
      }
      setup_lockstep(ctx, gp, cp, aux, bf, pst, sync_buf);
      // Split-k tail (OZGPU_TAIL_SPLIT=0 turns it off): the R units of the
      // last partial wave (equal-length units on C clusters, R = U mod C) are
      // each cut into P = C / R k-ranges that run side by side and add their
      // exact int32 partial sums into the plane (zeroed here over the tail
      // tiles' bounding box; the other tiles in the box are stored later in
      // the same launch).  At 8192^3 (12,12): 6144 units on 74 pairs leave 2
      // units for a whole unit time.
      {
        bool tail = true;
        if (const char* env = std::getenv("OZGPU_TAIL_SPLIT")) tail = std::string(env) == "1";
        const int clusters = std::min(max_pair_clusters(ctx->num_sms, cl), gp.total_units);
        const int U = gp.total_units;
        const int R = clusters > 0 ? U % clusters : 0;
        // at most 512 (part, chunk) plane tiles of atomic adds (32 M int32
        // adds): bins of many short chunks (k = 32768) get fewer parts
        const int nc_last = bf.size() >= 2 ? bf[bf.size() - 1] - bf[bf.size() - 2] : 1;
        // P parts per tail unit take ceil(R P / C) rounds of 1/P unit each;
        // pick the P that minimises that (a half-full last wave, R > C / 2,
        // gains from several rounds of short parts: R = 38 of C = 74 at
        // 8192^3 (12,12) runs 0.6 instead of 1 unit length at P = 5).
        // OZGPU_TAIL_MULTI=0: one round only, P = C / R.
        const int pmax = R ? std::min(512 / (R * std::max(1, nc_last)), gp.kblocks) : 0;
        int P = R ? std::min(clusters / R, pmax) : 0;
        const char* tm_env = std::getenv("OZGPU_TAIL_MULTI");
        if (R && !(tm_env && std::atoi(tm_env) == 0)) {
          double best = P >= 2 ? 1.0 / P : 1.0;
          for (int q = 2; q <= pmax; ++q) {
            const double t = static_cast<double>((R * q + clusters - 1) / clusters) / q;
            if (t < best - 1e-9) {
              best = t;
              P = q;
            }
          }
        }
        if (tail && gp.bin_first && R && P >= 2 && pair_tiles >= R && gp.kblocks >= P &&
            U >= clusters) {
          const int G = gp.group > 0 ? gp.group : 8;
          int r0 = INT32_MAX, r1 = 0, q0 = INT32_MAX, q1 = 0;
          for (int u = U - R; u < U; ++u) {
            const int tile = u % pair_tiles;  // the last bin (R <= pair_tiles)
            const int group_size = G * gp.tiles_n;
            const int grp = tile / group_size, first_m = grp * G;
            const int gsz = std::min(G, gp.tiles_m - first_m);
            const int in_group = tile - grp * group_size;
            const int tm = first_m + in_group % gsz, tn = in_group / gsz;
            r0 = std::min(r0, tm * unit_rows);
            r1 = std::max(r1, tm * unit_rows + unit_rows);
            q0 = std::min(q0, tn * pair_n);
            q1 = std::max(q1, tn * pair_n + pair_n);
          }
          r1 = static_cast<int>(std::min<int64_t>(r1, rows));
          q1 = static_cast<int>(std::min<int64_t>(q1, n));
          const size_t nb = bf.size() - 1;
          for (int q = bf[nb - 1]; q < bf[nb]; ++q)
            OZ_CUDA(cudaMemset2DAsync(planes + static_cast<int64_t>(aux[q]) * plane +
                                          (row0 + static_cast<int64_t>(r0)) * ldp + q0,
                                      sizeof(int32_t) * ldp, 0, sizeof(int32_t) * (q1 - q0),
                                      r1 - r0, pst));
          gp.tail_first = U - R;
          gp.tail_parts = P;
          gp.total_units = U - R + R * P;
        }
      }
      CUtensorMap tma_p = make_slice_map(ctx, slA + row0 * ld, kp, rows, sa, kBlockM, plane_a, ld);
      CUtensorMap tmb2 = make_slice_map(ctx, slB, kp, n, sb, 128, plane_b, ld);
      // chunk planes as a TMA store target (OZGPU_TMA_STORE=0: plain stores)
      CUtensorMap tmc{};
      gp.tma_store = 1;
      if (const char* env = std::getenv("OZGPU_TMA_STORE")) gp.tma_store = std::atoi(env) != 0;
      gp.planes = planes + row0 * ldp;
      if (gp.tma_store) tmc = make_plane_map(ctx, gp.planes, n, rows, ldp, gp.nchunks, plane);
      OZ_CUDA(launch_gemm_i8_pair(&tma_p, &tmb2, &tmc, gp, ctx->num_sms, pst, &launches));
    };
    if (pair) {
      // the bin table (built and uploaded once)
      bins_ok = build_bins(cp.chunks, ctx->host_aux, bfirst);
      if (bins_ok) {
        std::vector<int>& aux = ctx->host_aux;
        aux.insert(aux.end(), bfirst.begin(), bfirst.end());
        daux = static_cast<int*>(ctx->aux.get(sizeof(int) * aux.size()));
        upload_table(ctx, daux, aux.data(), sizeof(int) * aux.size(), st);
      }
      // OZGPU_QUAD=1 (opt-in): 4-CTA clusters, two CTA pairs stacked in M
      // sharing the B panel by multicast.  Measured on B200 at 8192^3 (12,12):
      // the multicast saves energy (SM clock 1436 -> 1507 MHz at the cap) but
      // only 33 such clusters fit on the 148 SMs (132 used): 28.6 vs 27.1 ms.
      // Running the last rows concurrently on 2-CTA clusters over the 16 idle
      // SMs was bitwise exact but 46 ms -- the hardware places the second
      // kernel's clusters on SMs the first one needs, stalling its lockstep.
      int quad = 0;
      if (const char* env = std::getenv("OZGPU_QUAD")) quad = std::atoi(env);
      if (quad == 1 && pair_n == 512 && m >= 512) {
        launch_pair_part(0, m, 4, st, ctx->sync);
      } else {
        launch_pair_part(0, m, 2, st, ctx->sync);
      }
    } else {
      g.total_units = static_cast<int>(tiles * g.nchunks);
      // Opt-in (OZGPU_EPILOGUE=final): the exact combine folded into the
      // GEMM -- the largest chunk runs last and its epilogue sums the tile's
      // other planes (Horner, 128-bit).  Bit-exact, but measured ~3% slower
      // than split + the combine kernel under the B200 power cap (the heavy
      // epilogue competes with the MMAs for power), so not the default.
      bool final_mode = false;
      if (const char* env = ctx->debug_planes ? nullptr : std::getenv("OZGPU_EPILOGUE"))
        final_mode = std::string(env) == "final" && p.strategy == 2 && g.nchunks >= 2 &&
                     cp.diagonals <= 64 &&
                     static_cast<int64_t>(cp.diagonals - 1) * t + 40 <= 126;
      if (final_mode) {
        int fin = 0;
        for (int c = 1; c < g.nchunks; ++c)
          if (cp.chunks[c].npairs >= cp.chunks[fin].npairs) fin = c;
        std::vector<int>& aux = ctx->host_aux;
        aux.clear();
        for (int c = 0; c < g.nchunks; ++c)
          if (c != fin) aux.push_back(c);
        aux.push_back(fin);
        int cc = 0;
        for (int d = 0; d <= cp.diagonals; ++d) {
          while (cc < g.nchunks && cp.chunks[cc].d < d) ++cc;
          aux.push_back(d == cp.diagonals ? g.nchunks : cc);
        }
        int* daux = static_cast<int*>(ctx->aux.get(sizeof(int) * aux.size()));
        upload_table(ctx, daux, aux.data(), sizeof(int) * aux.size(), st);
        int* counters = static_cast<int*>(ctx->counters.get(sizeof(int) * tiles));
        OZ_CUDA(cudaMemsetAsync(counters, 0, sizeof(int) * tiles, st));
        g.proc_order = daux;
        g.diag_first = daux + g.nchunks;
        g.final_chunk = fin;
        g.tile_counters = counters;
        g.diagonals = cp.diagonals;
        g.width = t;
        g.fused_words = 1;
        g.qa = qa;
        g.qb = qb;
        g.w_last = w_last;
        g.c = dc;
        g.ldc = ldc;
        g.axpby = axpby ? 1 : 0;
        g.alpha = alpha;
        g.beta = beta;
        g.cin = dcin;
        g.ldcin = ldcin;
        OZ_CUDA(launch_gemm_i8(&tma, &tmb, g, ctx->num_sms, st, &launches));
        if (ctx->timing) {
          OZ_CUDA(cudaEventRecord(ev[2], st));
          OZ_CUDA(cudaEventRecord(ev[3], st));
          ctx->pending_events.push_back(ev);
        }
        ctx->launches += launches;
        return nullptr;
      }
      // Equal-length bins of chunks per unit (default when every CTA gets
      // several units; OZGPU_BINS=0/1 overrides).
      bool bins = tiles * g.nchunks >= 4 * static_cast<int64_t>(ctx->num_sms);
      if (const char* env = std::getenv("OZGPU_BINS")) bins = std::string(env) == "1";
      std::vector<int>& aux = ctx->host_aux;
      std::vector<int> bfirst;
      if (bins && build_bins(cp.chunks, aux, bfirst)) {
        const size_t nb = bfirst.size() - 1;
        aux.insert(aux.end(), bfirst.begin(), bfirst.end());
        int* daux = static_cast<int*>(ctx->aux.get(sizeof(int) * aux.size()));
        upload_table(ctx, daux, aux.data(), sizeof(int) * aux.size(), st);
        g.proc_order = daux;
        g.bin_first = daux + g.nchunks;
        g.total_units = static_cast<int>(tiles * static_cast<int64_t>(nb));
      }
      // 2-CTA clusters multicasting the shared B panel (default; OZGPU_MC=0
      // selects the plain 1-CTA launch): measured on B200 at 8192^3 (12,12)
      // under the power cap, 30.3 vs 34.4 ms per pair-GEMM launch (8
      // interleaved rounds) -- a third less L2->SM operand traffic lets the
      // SM clock run ~5% higher at the same board power.
      bool mc = tiles_m >= 2;
      if (const char* env = std::getenv("OZGPU_MC")) mc = std::string(env) == "1" && tiles_m >= 2;
      if (mc) {
        const int64_t super_tiles = static_cast<int64_t>((tiles_m + 1) / 2) * tiles_n;
        g.total_units = static_cast<int>(g.total_units / tiles * super_tiles);
        setup_lockstep(ctx, g, cp, aux, bfirst, st, ctx->sync);
        CUtensorMap tmb_half = make_slice_map(ctx, slB, kp, n, sb, 128, plane_b, ld);
        OZ_CUDA(launch_gemm_i8_mc(&tma, &tmb_half, g, ctx->num_sms, st, &launches));
      } else {
        OZ_CUDA(launch_gemm_i8(&tma, &tmb, g, ctx->num_sms, st, &launches));
      }
    }
    if (ctx->timing) OZ_CUDA(cudaEventRecord(ev[2], st));
    if (ctx->debug_planes) {
      ctx->dbg_plane_stride = plane;
      ctx->dbg_ldp = ldp;
      if (ctx->timing) {
        OZ_CUDA(cudaEventRecord(ev[3], st));
        ctx->pending_events.push_back(ev);
      }
      ctx->launches += launches;
      return nullptr;
    }

    CombineArgs c{};
    c.planes = planes;
    c.chunks = dchunks;
    c.nchunks = g.nchunks;
    c.plane_stride = plane;
    c.ldp = ldp;
    c.qa = qa;
    c.qb = qb;
    c.m = static_cast<int>(m);
    c.n = static_cast<int>(n);
    c.width = t;
    c.diagonals = cp.diagonals;
    c.mode = p.mode;
    c.w_last = -static_cast<long>(cp.diagonals + 1) * t + (p.mode == 1 ? 2 : 0);
    c.c = dc;
    c.ldc = ldc;
    c.axpby = axpby ? 1 : 0;
    c.alpha = alpha;
    c.beta = beta;
    c.cin = dcin;
    c.ldcin = ldcin;
    if (p.strategy == 2) {
      OZ_CUDA(launch_combine_exact(c, exact_words(cp.diagonals, t, cp.chunks.size()),
                                   cp.chunks.data(), st, &launches));
    } else {
      psi_dev = static_cast<int*>(ctx->psi.get(sizeof(int)));
      OZ_CUDA(cudaMemsetAsync(psi_dev, 0, sizeof(int), st));
      c.realized_psi = psi_dev;
      OZ_CUDA(launch_combine_sequential(c, st, &launches));
    }
  } else if (m > 0 && n > 0) {
    // no scheduled products: C = 0 (+ beta*C for axpby) -- cannot happen for
    // valid plans (max_diag_sum >= 2), kept for completeness
    OZ_CUDA(cudaMemset2DAsync(dc, ldc * sizeof(double), 0, n * sizeof(double), m, st));
  }
  if (ctx->timing) {
    if (!(m > 0 && n > 0 && !cp.chunks.empty())) OZ_CUDA(cudaEventRecord(ev[2], st));
    OZ_CUDA(cudaEventRecord(ev[3], st));
    ctx->pending_events.push_back(ev);
  }
  ctx->launches += launches;
  return psi_dev;
}

// Copies a row-major host matrix (ld) into a dense device buffer (ld = cols).
void h2d(void* dst, const double* src, int64_t rows, int64_t cols, int64_t ld, cudaStream_t st) {
  if (rows == 0 || cols == 0) return;
  OZ_CUDA(cudaMemcpy2DAsync(dst, cols * sizeof(double), src, ld * sizeof(double),
                            cols * sizeof(double), rows, cudaMemcpyHostToDevice, st));
}
void d2h(double* dst, int64_t ld, const void* src, int64_t rows, int64_t cols, cudaStream_t st) {
  if (rows == 0 || cols == 0) return;
  OZ_CUDA(cudaMemcpy2DAsync(dst, ld * sizeof(double), src, cols * sizeof(double),
                            cols * sizeof(double), rows, cudaMemcpyDeviceToHost, st));
}

void check_plan(const ozgpu_plan* plan) {
  if (!plan) throw std::invalid_argument("multiply: null plan");
  if (plan->strategy < 0 || plan->strategy > 2)
    throw std::invalid_argument("multiply: unknown accumulation strategy");
}

// C-ABI operand checks (no reference counterpart: its Matrix carries its own
// shape): leading dimensions cover the rows, pointers are non-null whenever
// the operand has elements.  Raised before any copy or launch.
void check_operands(const char* fn, int64_t m, int64_t n, int64_t k, const void* a, int64_t lda,
                    const void* b, int64_t ldb, const void* c, int64_t ldc) {
  const std::string f(fn);
  if (m < 0 || n < 0 || k < 0) throw std::invalid_argument(f + ": shape mismatch");
  if (lda < k)
    throw std::invalid_argument(f + ": leading dimension of A (" + std::to_string(lda) +
                                ") is smaller than k (" + std::to_string(k) + ")");
  if (ldb < n)
    throw std::invalid_argument(f + ": leading dimension of B (" + std::to_string(ldb) +
                                ") is smaller than n (" + std::to_string(n) + ")");
  if (ldc < n)
    throw std::invalid_argument(f + ": leading dimension of C (" + std::to_string(ldc) +
                                ") is smaller than n (" + std::to_string(n) + ")");
  if ((m > 0 && k > 0 && !a) || (k > 0 && n > 0 && !b) || (m > 0 && n > 0 && !c))
    throw std::invalid_argument(f + ": null matrix pointer");
}

// Errors the reference raises from split() after multiply's own validation
// (slicing.cpp:69-72), plus the int8 operand limit of the tensor-core path.
std::string plan_error(const ozgpu_plan& p) {
  if (p.width < 1 || p.width > 62) return "split: width out of range";
  if (p.slices_a < 1 || p.slices_b < 1) return "split: need at least one slice";
  if (p.mode == 1 && p.width < 2) return "split: nearest mode needs width >= 2";
  if (p.width > 7)
    return "multiply: slice width " + std::to_string(p.width) +
           " exceeds the int8 tensor-core operand (t <= 7)";
  return {};
}

// The caller's pageable buffers behind a staged pipeline call (the pinned
// staging buffers are passed as a / b / c with dense leading dimensions).
struct HostStage {
  const double* a;
  int64_t lda;
  const double* b;
  int64_t ldb;
  double* c;
  int64_t ldc;
};

// Host-pointer multiply / multiply_axpby.
void host_multiply_locked(ozgpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* a,
                          int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc,
                          const ozgpu_mma_config& cfg, const ozgpu_plan& p, ozgpu_diag* diag,
                          bool axpby, double alpha, double beta, const double* cin,
                          int64_t ldcin, const HostStage* hs = nullptr);

int pipe_env(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

// Whether host_multiply_locked takes the blocked H2D / compute / D2H pipeline.
bool pipeline_eligible(const ozgpu_mma_config& cfg, const ozgpu_plan& p, int64_t m, int64_t n,
                       int64_t k, bool axpby) {
  const ValidationResult v = host_validation(cfg, p, k);
  const bool failing = k < 1 || v.capacity_error || v.precision_error || !plan_error(p).empty();
  const int64_t bytes = 8 * (m * k + k * n + m * n);
  return !failing && !axpby && p.strategy == 2 && m >= 2048 && n >= 1024 && bytes >= (64 << 20) &&
         pipe_env("OZGPU_PIPE", 1) == 1;
}

bool is_pageable(const void* ptr) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return at.type == cudaMemoryTypeUnregistered;
}

// rows x cols doubles copied on the context's pool with `nt` threads; the
// copy also ORs the clean-input status bits of every value it moves (1 =
// Inf / NaN, 2 = -0, the GPU slicer's definition, matrix.cpp:22-29) into
// *dirty, so a staged call knows its inputs' verdict on the host as soon as
// they are staged.
// One row: copy + status bits.  AVX2 when the CPU has it (streaming stores:
// the pinned destination is read next by the DMA engine, not by the CPU).
int copy_check_scalar(uint64_t* out, const uint64_t* in, int64_t n) {
  uint64_t bi = 0, bz = 0;
  for (int64_t j = 0; j < n; ++j) {
    const uint64_t x = in[j];
    out[j] = x;
    bi |= static_cast<uint64_t>((x & 0x7FF0000000000000ULL) == 0x7FF0000000000000ULL);
    bz |= static_cast<uint64_t>(x == 0x8000000000000000ULL);
  }
  return (bi ? 1 : 0) | (bz ? 2 : 0);
}

__attribute__((target("avx2"))) int copy_check_avx2(uint64_t* out, const uint64_t* in,
                                                     int64_t n) {
  int64_t j = 0;
  int bits = 0;
  while (j < n && (reinterpret_cast<uintptr_t>(out + j) & 31)) {
    bits |= copy_check_scalar(out + j, in + j, 1);
    ++j;
  }
  const __m256i em = _mm256_set1_epi64x(0x7FF0000000000000LL);
  const __m256i nz = _mm256_set1_epi64x(static_cast<long long>(0x8000000000000000ULL));
  __m256i acc_i = _mm256_setzero_si256(), acc_z = _mm256_setzero_si256();
  for (; j + 4 <= n; j += 4) {
    const __m256i x = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(in + j));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(out + j), x);
    acc_i = _mm256_or_si256(acc_i, _mm256_cmpeq_epi64(_mm256_and_si256(x, em), em));
    acc_z = _mm256_or_si256(acc_z, _mm256_cmpeq_epi64(x, nz));
  }
  if (j < n) bits |= copy_check_scalar(out + j, in + j, n - j);
  _mm_sfence();
  if (!_mm256_testz_si256(acc_i, acc_i)) bits |= 1;
  if (!_mm256_testz_si256(acc_z, acc_z)) bits |= 2;
  return bits;
}

void pool_copy_check(CopyPool& pool, int nt, double* dst, int64_t ldd, const double* src,
                     int64_t lds, int64_t rows, int64_t cols, std::atomic<int>* dirty) {
  if (rows == 0 || cols == 0) return;
  nt = static_cast<int>(std::clamp<int64_t>(nt, 1, rows));
  static const bool avx2 = __builtin_cpu_supports("avx2");
  pool.run(nt, [&](int t) {
    const int64_t r0 = rows * t / nt, r1 = rows * (t + 1) / nt;
    int bits = 0;
    for (int64_t r = r0; r < r1; ++r) {
      const uint64_t* in = reinterpret_cast<const uint64_t*>(src + r * lds);
      uint64_t* out = reinterpret_cast<uint64_t*>(dst + r * ldd);
      if (dirty)
        bits |= avx2 ? copy_check_avx2(out, in, cols) : copy_check_scalar(out, in, cols);
      else
        std::memcpy(out, in, static_cast<size_t>(cols) * 8);
    }
    if (dirty && bits) dirty->fetch_or(bits);
  });
}

// rows x cols doubles between strided host buffers, rows split over threads
// (one per 16 MiB up to min(cores, 16); `threads` > 0 forces the count)
void parallel_copy(double* dst, int64_t ldd, const double* src, int64_t lds, int64_t rows,
                   int64_t cols, int threads = 0) {
  if (rows == 0 || cols == 0) return;
  const int64_t bytes = rows * cols * 8;
  const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  const int nt = threads > 0 ? static_cast<int>(std::clamp<int64_t>(threads, 1, std::max<int64_t>(1, rows)))
                             : static_cast<int>(std::clamp<int64_t>(bytes >> 24, 1, std::min(hw, 16)));
  auto work = [&](int t) {
    const int64_t r0 = rows * t / nt, r1 = rows * (t + 1) / nt;
    if (ldd == cols && lds == cols) {
      std::memcpy(dst + r0 * cols, src + r0 * cols, static_cast<size_t>((r1 - r0) * cols * 8));
    } else {
      for (int64_t r = r0; r < r1; ++r)
        std::memcpy(dst + r * ldd, src + r * lds, static_cast<size_t>(cols * 8));
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
}

// Host-pointer multiply / multiply_axpby.  Pageable caller buffers (the
// reference's Matrix is a std::vector) copy at ~10 GB/s through the driver's
// own staging (157 ms vs 36 ms pinned at 8192^3, tools/pageable_probe.py), so
// large ones are first copied by host threads into the context's pinned
// buffers (OZGPU_STAGE=0 turns this off; OZGPU_STAGE_MIN = byte threshold).
void host_multiply(ozgpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* a, int64_t lda,
                   const double* b, int64_t ldb, double* c, int64_t ldc,
                   const ozgpu_mma_config& cfg, const ozgpu_plan& p, ozgpu_diag* diag,
                   bool axpby, double alpha, double beta, const double* cin, int64_t ldcin) {
  std::lock_guard<std::mutex> lock(ctx->mu);
  OZ_CUDA(cudaSetDevice(ctx->device));
  bool stage = !axpby && m > 0 && n > 0 && k > 0;
  if (const char* env = std::getenv("OZGPU_STAGE")) stage = stage && std::string(env) == "1";
  int64_t min_bytes = 64 << 20;
  if (const char* env = std::getenv("OZGPU_STAGE_MIN")) min_bytes = std::atoll(env);
  stage = stage && 8 * (m * k + k * n + m * n) >= min_bytes &&
          (is_pageable(a) || is_pageable(b) || is_pageable(c));
  if (!stage) {
    host_multiply_locked(ctx, m, n, k, a, lda, b, ldb, c, ldc, cfg, p, diag, axpby, alpha, beta,
                         cin, ldcin);
    return;
  }
  double* sa = static_cast<double*>(ctx->stage_a.get(sizeof(double) * m * k));
  double* sb = static_cast<double*>(ctx->stage_b.get(sizeof(double) * k * n));
  double* sc = static_cast<double*>(ctx->stage_c.get(sizeof(double) * m * n));
  if (!sa || !sb || !sc) {  // no page-locked memory: the driver's own staging
    host_multiply_locked(ctx, m, n, k, a, lda, b, ldb, c, ldc, cfg, p, diag, axpby, alpha, beta,
                         cin, ldcin);
    return;
  }
  if (pipeline_eligible(cfg, p, m, n, k, axpby) && pipe_env("OZGPU_STAGE_OVERLAP", 1) == 1) {
    // the pipeline stages each A block / B panel just before its H2D copy
    // and unstages each C block as soon as it is back (and the inputs were
    // found clean), so the host copies overlap PCIe and the GEMMs
    const HostStage hs{a, lda, b, ldb, c, ldc};
    host_multiply_locked(ctx, m, n, k, sa, k, sb, n, sc, n, cfg, p, diag, axpby, alpha, beta, cin,
                         ldcin, &hs);
    return;
  }
  std::thread tb([&] { parallel_copy(sb, n, b, ldb, k, n); });
  parallel_copy(sa, k, a, lda, m, k);
  tb.join();
  host_multiply_locked(ctx, m, n, k, sa, k, sb, n, sc, n, cfg, p, diag, axpby, alpha, beta, cin,
                       ldcin);
  parallel_copy(c, ldc, sc, n, m, n);
}

void host_multiply_locked(ozgpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* a,
                          int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc,
                          const ozgpu_mma_config& cfg, const ozgpu_plan& p, ozgpu_diag* diag,
                          bool axpby, double alpha, double beta, const double* cin,
                          int64_t ldcin, const HostStage* hs) {
  cudaStream_t st = ctx->stream;
  acquire_workspace(ctx, st);
  ValidationResult v = host_validation(cfg, p, k);
  double* da = static_cast<double*>(ctx->in_a.get(sizeof(double) * m * k + 8));
  double* db = static_cast<double*>(ctx->in_b.get(sizeof(double) * k * n + 8));
  const std::string perr = plan_error(p);
  const bool failing = k < 1 || v.capacity_error || v.precision_error || !perr.empty();
  // Blocked H2D / compute / D2H pipeline for large products.  A arrives in
  // row blocks; the first row block is multiplied against B column panel by
  // column panel as the panels land (so the tensor cores start after one A
  // block + one B panel instead of all of B), the other row blocks against
  // the whole of B, the last one in column halves so that only a small C
  // block is left to copy back after the final GEMM.  Every block's C goes
  // back on the D2H stream as soon as its combine is done.  Blocking is
  // exact: scales are per row of A and per column of B.
  auto env_int = pipe_env;
  const bool pipeline = pipeline_eligible(cfg, p, m, n, k, axpby);
  if (hs && !pipeline) throw std::logic_error("host_multiply: staged overlap needs the pipeline");
  if (pipeline) {
    // ~2048-row blocks of A and ~2048-column panels of B (at least 4 each),
    // measured on B200 (PCIe ~55 GB/s each way): 8192^3 4 x 4 (35.5 ms),
    // 16384^3 8 x 8 (277 vs 307 ms with 4 x 4), 65536 x 2048^2 32 row blocks
    // (24.5 vs 31.7 ms with 4).  OZGPU_PIPE_FIRST=f makes the first row block
    // and the first column panel 1/f of the others (less to copy before the
    // tensor cores start).
    const int rows_default = static_cast<int>(std::clamp<int64_t>((m + 1024) / 2048, 4, 32));
    const int pan_default = static_cast<int>(std::clamp<int64_t>((n + 1024) / 2048, 4, 16));
    const int nblk = std::max(1, env_int("OZGPU_PIPE_ROWS", rows_default));
    const int npan = std::max(1, env_int("OZGPU_PIPE_PANELS", pan_default));
    // measured at 8192^3: first blocks of half size and the final row block
    // in 4 column parts, 36.2 -> 34.6 ms (16384^3: 4 parts cost 5 ms, so 2)
    const int last_default = n <= 8192 ? static_cast<int>(std::clamp<int64_t>(n / 2048, 2, 4)) : 2;
    const int nlast = std::max(1, env_int("OZGPU_PIPE_LAST", last_default));
    const int first = std::max(1, env_int("OZGPU_PIPE_FIRST", 2));
    if (!ctx->h2d_stream) {
      OZ_CUDA(cudaStreamCreateWithFlags(&ctx->h2d_stream, cudaStreamNonBlocking));
      OZ_CUDA(cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking));
    }
    const int t = p.width;
    const int64_t kp = slice_ld(round_up(k, kKPad));  // slice row stride
    double* dc = static_cast<double*>(ctx->io_c.get(sizeof(double) * m * n + 8));
    int8_t* slA =
        static_cast<int8_t*>(ctx->slices_a.get(static_cast<size_t>(p.slices_a) * m * kp + 1));
    int8_t* slB =
        static_cast<int8_t*>(ctx->slices_b.get(static_cast<size_t>(p.slices_b) * n * kp + 1));
    int* qa = static_cast<int*>(ctx->qa.get(sizeof(int) * (m + 1)));
    int* qb = static_cast<int*>(ctx->qb.get(sizeof(int) * (n + 1)));
    auto* colmax = static_cast<unsigned long long*>(ctx->colmax.get(8 * (n + 1)));
    int* status = static_cast<int*>(ctx->status.get(sizeof(int)));
    // row blocks (multiples of 256 rows) and column panels (multiples of 256)
    std::vector<int64_t> rb{0}, cb{0};
    const int64_t rows = round_up((m + nblk - 1) / nblk, 256);
    if (first > 1) rb.push_back(std::min(m, std::max<int64_t>(256, round_up(rows / first, 256))));
    while (rb.back() < m) rb.push_back(std::min(m, rb.back() + rows));
    auto split_cols = [&](int parts, int lead) {
      std::vector<int64_t> e{0};
      const int64_t w = round_up((n + parts - 1) / parts, 256);
      if (lead > 1) e.push_back(std::min(n, std::max<int64_t>(256, round_up(w / lead, 256))));
      while (e.back() < n) e.push_back(std::min(n, e.back() + w));
      return e;
    };
    cb = split_cols(npan, first);
    const std::vector<int64_t> cl = split_cols(nlast, 1);
    const size_t nr = rb.size() - 1, nc = cb.size() - 1;
    const size_t nev = 2 + nr + nc + 2 * (nr * std::max(nc, cl.size()) + 4);
    while (ctx->pipe_events.size() < nev) {
      cudaEvent_t e;
      OZ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ctx->pipe_events.push_back(e);
    }
    size_t evi = 0;
    auto next_event = [&]() { return ctx->pipe_events[evi++]; };
    // OZGPU_PIPE_TRACE=1: timing events on every step, printed to stderr
    const bool trace = env_int("OZGPU_PIPE_TRACE", 0) == 1;
    std::vector<std::pair<std::string, cudaEvent_t>> marks;
    auto mark = [&](const std::string& what, cudaStream_t s) {
      if (!trace) return;
      cudaEvent_t e;
      OZ_CUDA(cudaEventCreate(&e));
      OZ_CUDA(cudaEventRecord(e, s));
      marks.emplace_back(what, e);
    };
    // inputs: A block 0, then the B panels, then the other A blocks
    cudaEvent_t start = next_event();
    OZ_CUDA(cudaMemsetAsync(status, 0, sizeof(int), st));
    OZ_CUDA(cudaEventRecord(start, st));  // after earlier work on the compute stream
    OZ_CUDA(cudaStreamWaitEvent(ctx->h2d_stream, start, 0));
    mark("start", ctx->h2d_stream);
    std::vector<cudaEvent_t> a_in(nr), b_in(nc);
    // Default (OZGPU_PIPE_MODE=rect): A blocks and B panels alternate on the copy
    // stream (A0 B0 B1 A1 B2 A2 ...) and each arrival releases the rectangle
    // of C it completes (a growing square), so the tensor cores are fed
    // while the inputs are still crossing PCIe
    const char* pm = std::getenv("OZGPU_PIPE_MODE");
    const bool rect = !(pm && std::string(pm) == "panels");  // measured 36.0 vs 37.0 ms at 8192^3
    std::vector<std::pair<char, size_t>> arrivals;
    if (rect) {
      size_t ia = 0, jb = 0;
      arrivals.push_back({'A', ia++});
      while (ia < nr || jb < nc) {
        if (jb < nc) arrivals.push_back({'B', jb++});
        if (jb < nc && jb == 1) arrivals.push_back({'B', jb++});
        if (ia < nr) arrivals.push_back({'A', ia++});
      }
    } else {
      arrivals.push_back({'A', 0});
      for (size_t j = 0; j < nc; ++j) arrivals.push_back({'B', j});
      for (size_t i = 1; i < nr; ++i) arrivals.push_back({'A', i});
    }
    // Staged call (pageable caller buffers): a host thread copies the inputs
    // into the pinned staging buffers a / b in arrival order; each H2D copy
    // waits only for its own block.
    std::atomic<size_t> staged{0};
    std::atomic<bool> stop_staging{false};
    std::atomic<int> host_dirty{0};  // clean-input bits seen by the staging copies
    std::mutex stage_mu;
    std::condition_variable stage_cv;
    std::thread stager;
    // the staging copies are memory-latency bound: two threads per core
    // (capped at 32) measured 40.4 vs 41.5 ms at 8192^3, 53 vs 59 ms at
    // 65536 x 2048^2 against one per core on the 16-core B200 host
    const int stage_threads = std::max(
        1, pipe_env("OZGPU_STAGE_THREADS",
                    static_cast<int>(std::min(32u, 2 * std::max(1u, std::thread::hardware_concurrency())))));
    if (hs) {
      stager = std::thread([&] {
        for (size_t q = 0; q < arrivals.size() && !stop_staging.load(); ++q) {
          const size_t x = arrivals[q].second;
          if (arrivals[q].first == 'A')
            pool_copy_check(ctx->copy_pool, stage_threads, const_cast<double*>(a) + rb[x] * lda,
                            lda, hs->a + rb[x] * hs->lda, hs->lda, rb[x + 1] - rb[x], k,
                            &host_dirty);
          else
            pool_copy_check(ctx->copy_pool, stage_threads, const_cast<double*>(b) + cb[x], ldb,
                            hs->b + cb[x], hs->ldb, k, cb[x + 1] - cb[x], &host_dirty);
          {
            std::lock_guard<std::mutex> lk(stage_mu);
            staged.store(q + 1);
          }
          stage_cv.notify_all();
        }
      });
    }
    struct StagerJoin {
      std::thread& th;
      std::atomic<bool>& stop;
      ~StagerJoin() {
        stop.store(true);
        if (th.joinable()) th.join();
      }
    } stager_join{stager, stop_staging};
    std::vector<size_t> arrival_of_a(nr), arrival_of_b(nc);
    for (size_t q = 0; q < arrivals.size(); ++q)
      (arrivals[q].first == 'A' ? arrival_of_a : arrival_of_b)[arrivals[q].second] = q;
    auto wait_staged = [&](size_t q) {
      if (!hs) return;
      std::unique_lock<std::mutex> lk(stage_mu);
      stage_cv.wait(lk, [&] { return staged.load() > q; });
    };
    auto copy_a = [&](size_t i) {
      wait_staged(arrival_of_a[i]);
      h2d(da + rb[i] * k, a + rb[i] * lda, rb[i + 1] - rb[i], k, lda, ctx->h2d_stream);
      a_in[i] = next_event();
      OZ_CUDA(cudaEventRecord(a_in[i], ctx->h2d_stream));
      mark("h2d A" + std::to_string(i), ctx->h2d_stream);
    };
    auto copy_b = [&](size_t j) {  // panel j: k x nj, dense at db + k * c0
      wait_staged(arrival_of_b[j]);
      h2d(db + k * cb[j], b + cb[j], k, cb[j + 1] - cb[j], ldb, ctx->h2d_stream);
      b_in[j] = next_event();
      OZ_CUDA(cudaEventRecord(b_in[j], ctx->h2d_stream));
      mark("h2d B" + std::to_string(j), ctx->h2d_stream);
    };
    // rect: each arrival's copy is enqueued right before its compute (the
    // copy stream's order is unchanged; a staged call then never holds back
    // the compute of blocks already staged); panels: all copies first
    if (!rect)
      for (auto& ar : arrivals) ar.first == 'A' ? copy_a(ar.second) : copy_b(ar.second);
    int64_t launches = 0;
    struct CBlock {
      int64_t r0, r1, c0, c1;
      cudaEvent_t back;
    };
    std::vector<CBlock> cblocks;
    const bool queue = use_slice_queue(p.mode, t, kp);
    int* qwork = queue ? queue_work(ctx, m, n, k, kp) : nullptr;
    auto slice_a = [&](size_t i) {
      OZ_CUDA(cudaStreamWaitEvent(st, a_in[i], 0));
      if (queue)
        OZ_CUDA(launch_slice_queue(da + rb[i] * k, k, rb[i + 1] - rb[i], nullptr, 0, 0, k, kp, t,
                                   p.slices_a, 0, slA + rb[i] * kp, m * kp, nullptr, 0,
                                   qa + rb[i], nullptr, nullptr, qwork, status, upload_cb, ctx, st,
                                   &launches));
      else
        OZ_CUDA(launch_slice_rows(da + rb[i] * k, k, rb[i + 1] - rb[i], k, kp, t, p.slices_a,
                                  p.mode, slA + rb[i] * kp, 0, qa + rb[i], status, st, &launches,
                                  m * kp));
      mark("slice A" + std::to_string(i), st);
    };
    auto block = [&](int64_t r0, int64_t r1, int64_t c0, int64_t c1) {
      Presliced pre{slA + r0 * kp, m * kp, qa + r0, slB + c0 * kp, n * kp, qb + c0, kp};
      run_multiply(ctx, r1 - r0, c1 - c0, k, nullptr, 0, nullptr, 0, dc + r0 * n + c0, n, cfg, p,
                   st, nullptr, false, 1.0, 0.0, nullptr, 0, &pre);
      cudaEvent_t done = next_event();
      OZ_CUDA(cudaEventRecord(done, st));
      const std::string tag = "C[" + std::to_string(r0) + ":" + std::to_string(r1) + "," +
                              std::to_string(c0) + ":" + std::to_string(c1) + "]";
      mark("gemm " + tag, st);
      OZ_CUDA(cudaStreamWaitEvent(ctx->d2h_stream, done, 0));
      OZ_CUDA(cudaMemcpy2DAsync(c + r0 * ldc + c0, ldc * sizeof(double), dc + r0 * n + c0,
                                n * sizeof(double), (c1 - c0) * sizeof(double), r1 - r0,
                                cudaMemcpyDeviceToHost, ctx->d2h_stream));
      mark("d2h " + tag, ctx->d2h_stream);
      if (hs) {
        cudaEvent_t back = next_event();
        OZ_CUDA(cudaEventRecord(back, ctx->d2h_stream));
        cblocks.push_back({r0, r1, c0, c1, back});
      }
    };
    auto slice_b = [&](size_t j) {
      const int64_t nj = cb[j + 1] - cb[j];
      OZ_CUDA(cudaStreamWaitEvent(st, b_in[j], 0));
      if (queue)
        OZ_CUDA(launch_slice_queue(nullptr, 0, 0, db + k * cb[j], nj, nj, k, kp, t, 0, p.slices_b,
                                   nullptr, 0, slB + cb[j] * kp, n * kp, nullptr, qb + cb[j],
                                   colmax + cb[j], qwork, status, upload_cb, ctx, st, &launches));
      else
        OZ_CUDA(launch_slice_cols(db + k * cb[j], nj, k, nj, kp, t, p.slices_b, p.mode,
                                  slB + cb[j] * kp, 0, qb + cb[j], colmax + cb[j], status, st,
                                  &launches, n * kp));
    };
    if (rect) {
      size_t na = 0, nbp = 0;  // A blocks / B panels sliced so far
      for (size_t q = 0; q < arrivals.size(); ++q) {
        const auto& ar = arrivals[q];
        const bool last = q + 1 == arrivals.size();
        ar.first == 'A' ? copy_a(ar.second) : copy_b(ar.second);
        if (ar.first == 'A') {
          slice_a(ar.second);
          na = ar.second + 1;
          if (nbp == 0) continue;
          const size_t i = ar.second;
          if (last && nbp == nc) {  // final row block: two column halves shorten the D2H tail
            for (size_t j = 0; j + 1 < cl.size(); ++j) block(rb[i], rb[i + 1], cl[j], cl[j + 1]);
          } else {
            block(rb[i], rb[i + 1], 0, cb[nbp]);
          }
        } else {
          slice_b(ar.second);
          nbp = ar.second + 1;
          if (na == 0) continue;
          const size_t j = ar.second;
          if (last && na == nr && na > 1) {  // final column panel: split its rows
            const size_t half = nr / 2;
            block(rb[0], rb[half], cb[j], cb[j + 1]);
            block(rb[half], rb[nr], cb[j], cb[j + 1]);
          } else {
            block(rb[0], rb[na], cb[j], cb[j + 1]);
          }
        }
      }
    } else {
    slice_a(0);
    for (size_t j = 0; j < nc; ++j) {
      slice_b(j);
      block(rb[0], rb[1], cb[j], cb[j + 1]);
    }
    for (size_t i = 1; i < nr; ++i) {
      slice_a(i);
      if (i + 1 == nr && nr > 1) {
        for (size_t j = 0; j + 1 < cl.size(); ++j) block(rb[i], rb[i + 1], cl[j], cl[j + 1]);
      } else {
        block(rb[i], rb[i + 1], 0, n);
      }
    }
    }
    ctx->launches += launches;
    if (hs) {
      // Unstage C block by block as each lands, once the inputs are known
      // clean: the staging copies checked every input value on the host, so
      // the verdict is in as soon as the last block is staged (the GPU's own
      // status, read below, must agree).
      wait_staged(arrivals.size() - 1);
      if (host_dirty.load() == 0)
        for (const CBlock& cbk : cblocks) {
          OZ_CUDA(cudaEventSynchronize(cbk.back));
          pool_copy_check(ctx->copy_pool, stage_threads, hs->c + cbk.r0 * hs->ldc + cbk.c0,
                          hs->ldc, c + cbk.r0 * ldc + cbk.c0, ldc, cbk.r1 - cbk.r0,
                          cbk.c1 - cbk.c0, nullptr);
        }
    }
    int hs_status = 0;
    OZ_CUDA(cudaMemcpyAsync(&hs_status, status, sizeof(int), cudaMemcpyDeviceToHost,
                            ctx->d2h_stream));
    OZ_CUDA(cudaStreamSynchronize(ctx->d2h_stream));
    OZ_CUDA(cudaStreamSynchronize(st));
    if (trace) {
      for (auto& mk : marks) {
        float ms = 0.f;
        OZ_CUDA(cudaEventElapsedTime(&ms, marks[0].second, mk.second));
        std::fprintf(stderr, "[ozgpu pipe] %8.3f ms  %s\n", ms, mk.first.c_str());
      }
      for (auto& mk : marks) cudaEventDestroy(mk.second);
    }
    if (hs && (hs_status != 0) != (host_dirty.load() != 0))
      throw std::logic_error("multiply: host and device input checks disagree");
    if (hs_status)
      throw std::invalid_argument("multiply: inputs must be finite with no negative zeros");
    if (diag) *diag = make_diag(p, cfg, m, n, k, 0);
    return;
  }
  h2d(da, a, m, k, lda, st);
  h2d(db, b, k, n, ldb, st);
  if (failing) {
    // the clean-input check precedes these errors (scheme.cpp:223-239, then
    // split()'s argument checks, slicing.cpp:69-72)
    int* status = static_cast<int*>(ctx->status.get(sizeof(int)));
    OZ_CUDA(cudaMemsetAsync(status, 0, sizeof(int), st));
    int64_t launches = 0;
    auto* colmax = static_cast<unsigned long long*>(ctx->colmax.get(8 * (n + 1)));
    int* qa = static_cast<int*>(ctx->qa.get(sizeof(int) * (m + 1)));
    int* qb = static_cast<int*>(ctx->qb.get(sizeof(int) * (n + 1)));
    int64_t kp8 = round_up(std::max<int64_t>(k, 1), 8);
    int8_t* sA = static_cast<int8_t*>(ctx->slices_a.get(static_cast<size_t>(m) * kp8 + 1));
    int8_t* sB = static_cast<int8_t*>(ctx->slices_b.get(static_cast<size_t>(n) * kp8 + 1));
    if (k >= 1) {
      OZ_CUDA(launch_slice_rows(da, k, m, k, kp8, 1, 1, 0, sA, 0, qa, status, st, &launches));
      OZ_CUDA(launch_slice_cols(db, n, k, n, kp8, 1, 1, 0, sB, 0, qb, colmax, status, st,
                                &launches));
    }
    int hs = 0;
    OZ_CUDA(cudaMemcpyAsync(&hs, status, sizeof(int), cudaMemcpyDeviceToHost, st));
    OZ_CUDA(cudaStreamSynchronize(st));
    ctx->launches += launches;
    if (hs) throw std::invalid_argument("multiply: inputs must be finite with no negative zeros");
    if (k < 1) throw std::invalid_argument("multiply: empty inner dimension");
    if (v.capacity_error || v.precision_error) throw std::domain_error(v.message);
    throw std::invalid_argument(perr);
  }
  double* dc = static_cast<double*>(ctx->io_c.get(sizeof(double) * m * n + 8));
  const double* dcin = nullptr;
  if (axpby) {
    double* t = static_cast<double*>(ctx->in_c2.get(sizeof(double) * m * n + 8));
    h2d(t, cin, m, n, ldcin, st);
    dcin = t;
  }
  int* psi_dev = run_multiply(ctx, m, n, k, da, k, db, n, dc, n, cfg, p, st, nullptr, axpby,
                              alpha, beta, dcin, n);
  int dirty = 0, hpsi = 0;
  OZ_CUDA(cudaMemcpyAsync(&dirty, ctx->status.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (psi_dev) OZ_CUDA(cudaMemcpyAsync(&hpsi, psi_dev, sizeof(int), cudaMemcpyDeviceToHost, st));
  OZ_CUDA(cudaStreamSynchronize(st));
  // the reference throws before producing output (scheme.cpp:223-225): C is
  // copied back only for clean inputs
  if (dirty) throw std::invalid_argument("multiply: inputs must be finite with no negative zeros");
  d2h(c, ldc, dc, m, n, st);
  OZ_CUDA(cudaStreamSynchronize(st));
  if (diag) *diag = make_diag(p, cfg, m, n, k, hpsi);
}

ozgpu_ctx* g_default[64];
std::mutex g_default_mu;

}  // namespace

// analysis.cpp:142-207
ozgpu_selection select_slices(double kappa_a, double kappa_b, int width, double u, int s_max,
                              bool has_target, double target, int schedule, int strategy,
                              int acc_bits_used, int precision) {
  if (width < 1 || s_max < 1 || s_max > 64 || !(u > 0.0) || !(u < 1.0))
    throw std::invalid_argument("select_slices: bad arguments");
  if (!(kappa_a > 0.0) || !(kappa_b > 0.0))
    throw std::invalid_argument("select_slices: kappas must be positive");
  bool found = false;
  ozgpu_selection best{};
  double best_lhs_any = std::numeric_limits<double>::infinity();
  double target_at_best = 0.0;
  for (int sa = 1; sa <= s_max; ++sa)
    for (int sb = 1; sb <= s_max; ++sb) {
      double lhs = std::ldexp(kappa_a, -sa * width) + std::ldexp(kappa_b, -sb * width);
      double tgt;
      if (has_target) {
        tgt = target;
      } else {
        int diagonals = schedule == 0 ? sa + sb - 1 : std::max(sa, sb);
        long long psi;
        if (strategy == 2)
          psi = plan_levels(precision, width, acc_bits_used, diagonals).inexact_adds;
        else if (strategy == 1)
          psi = diagonals - 1;
        else
          psi = (schedule == 0 ? static_cast<int64_t>(sa) * sb : chi(sa, sb)) - 1;
        tgt = gamma_factor(std::max(psi, 1LL), u);
      }
      if (lhs < best_lhs_any) {
        best_lhs_any = lhs;
        target_at_best = tgt;
      }
      if (lhs > tgt) continue;
      int64_t cost = chi(sa, sb);
      bool better;
      if (!found)
        better = true;
      else if (cost != best.products)
        better = cost < best.products;
      else if (std::max(sa, sb) != std::max(best.slices_a, best.slices_b))
        better = std::max(sa, sb) < std::max(best.slices_a, best.slices_b);
      else
        better = sa < best.slices_a;
      if (better) {
        best = {sa, sb, lhs, tgt, cost, 0.0};
        found = true;
      }
    }
  if (!found) {
    double gap = best_lhs_any / std::max(target_at_best, std::numeric_limits<double>::min());
    throw SelectionInfeasibleError(
        "select_slices: no feasible pair within s_max = " + std::to_string(s_max) +
            "; best achievable term exceeds the target by a factor " + std::to_string(gap),
        gap, best_lhs_any, target_at_best);
  }
  return best;
}

}  // namespace ozgpu

using namespace ozgpu;

extern "C" {

const char* ozgpu_last_error(void) { return g_error.c_str(); }
const char* ozgpu_version(void) { return "ozgpu 0.1 (sm_100a, tcgen05 kind::i8)"; }

int ozgpu_create(int device, ozgpu_ctx** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("ozgpu_create: null output");
    auto ctx = std::make_unique<ozgpu_ctx>();
    init_ctx(ctx.get(), device);
    *out = ctx.release();
  });
}

int ozgpu_destroy(ozgpu_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    if (ctx->h2d_stream) {
      cudaStreamSynchronize(ctx->h2d_stream);
      cudaStreamSynchronize(ctx->d2h_stream);
      cudaStreamDestroy(ctx->h2d_stream);
      cudaStreamDestroy(ctx->d2h_stream);
    }
    for (cudaEvent_t e : ctx->pipe_events) cudaEventDestroy(e);
    if (ctx->multi_stream) {
      cudaStreamSynchronize(ctx->multi_stream);
      cudaStreamDestroy(ctx->multi_stream);
    }
    if (ctx->fork_stream) {
      cudaStreamSynchronize(ctx->fork_stream);
      cudaStreamDestroy(ctx->fork_stream);
      cudaEventDestroy(ctx->fork_ev[0]);
      cudaEventDestroy(ctx->fork_ev[1]);
    }
    for (auto& ev : ctx->pending_events)
      for (cudaEvent_t e : ev) cudaEventDestroy(e);
    for (auto& kv : ctx->graphs) {
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
      for (void* pp : kv.second.pinned) cudaFreeHost(pp);
    }
    for (cudaEvent_t e : ctx->event_pool) cudaEventDestroy(e);
    delete ctx;
  });
}

int64_t ozgpu_kernel_launches(const ozgpu_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

int ozgpu_set_stage_timing(ozgpu_ctx* ctx, int enable) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("ozgpu_set_stage_timing: null context");
    std::lock_guard<std::mutex> lock(ctx->mu);
    ctx->timing = enable != 0;
  });
}

int ozgpu_stage_times(ozgpu_ctx* ctx, double* ms3, int64_t* calls, int reset) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("ozgpu_stage_times: null context");
    std::lock_guard<std::mutex> lock(ctx->mu);
    OZ_CUDA(cudaSetDevice(ctx->device));
    drain_events(ctx);
    if (ms3)
      for (int s = 0; s < 3; ++s) ms3[s] = ctx->stage_ms[s];
    if (calls) *calls = ctx->timed_calls;
    if (reset) {
      ctx->stage_ms[0] = ctx->stage_ms[1] = ctx->stage_ms[2] = 0;
      ctx->timed_calls = 0;
    }
  });
}

ozgpu_ctx* ozgpu_default_context(int device) {
  if (device < 0 || device >= 64) {
    g_error = "ozgpu_default_context: bad device index";
    return nullptr;
  }
  std::lock_guard<std::mutex> lock(g_default_mu);
  if (!g_default[device]) {
    ozgpu_ctx* c = nullptr;
    if (ozgpu_create(device, &c) != OZGPU_OK) return nullptr;
    g_default[device] = c;
  }
  return g_default[device];
}

int ozgpu_optimal_slice_width(ozgpu_mma_config cfg, int64_t k, int* out) {
  return guarded([&] { *out = optimal_slice_width(cfg, k); });
}
int ozgpu_max_inner_dim(ozgpu_mma_config cfg, int64_t* out) {
  return guarded([&] { *out = max_inner_dim(cfg); });
}
int ozgpu_chi(int sa, int sb, int64_t* out) {
  return guarded([&] { *out = chi(sa, sb); });
}
int ozgpu_spare_carries(int first, int last, int width, int64_t* out) {
  return guarded([&] { *out = spare_carries(first, last, width); });
}
int ozgpu_plan_levels(int precision, int width, int acc_bits_used, int diagonals,
                      ozgpu_plan* out) {
  return guarded([&] {
    Levels lv = plan_levels(precision, width, acc_bits_used, diagonals);
    if (lv.levels.size() > OZGPU_MAX_LEVELS)
      throw std::invalid_argument("plan_levels: more than 128 levels");
    set_levels(*out, lv);
  });
}
int ozgpu_diagonal_flush_threshold(ozgpu_mma_config cfg, int width, int64_t k, int64_t* out) {
  return guarded([&] { *out = diagonal_flush_threshold(cfg, width, k); });
}
int ozgpu_make_plan(ozgpu_mma_config cfg, int64_t k, int sa, int sb, int schedule, int strategy,
                    int mode, int precision, ozgpu_plan* out) {
  return guarded([&] { *out = make_plan(cfg, k, sa, sb, schedule, strategy, mode, precision); });
}

int ozgpu_select_slices(double kappa_a, double kappa_b, int width, double u, int s_max,
                        int has_target, double target, int schedule, int strategy,
                        int acc_bits_used, int precision, ozgpu_selection* out) {
  return guarded([&] {
    try {
      *out = select_slices(kappa_a, kappa_b, width, u, s_max, has_target != 0, target, schedule,
                           strategy, acc_bits_used, precision);
    } catch (const SelectionInfeasibleError& e) {
      out->gap = e.gap;
      out->lhs = e.best_lhs;
      out->target = e.target;
      throw;
    }
  });
}

int ozgpu_scaling_profile(ozgpu_ctx* ctx, int64_t m, int64_t k, int64_t n, const double* a,
                          int64_t lda, const double* b, int64_t ldb, ozgpu_profile* out) {
  return guarded([&] {
    if (!ctx || !out) throw std::invalid_argument("scaling_profile: null argument");
    std::lock_guard<std::mutex> lock(ctx->mu);
    OZ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    acquire_workspace(ctx, st);
    int64_t launches = 0;
    double* da = static_cast<double*>(ctx->in_a.get(sizeof(double) * m * k + 8));
    double* db = static_cast<double*>(ctx->in_b.get(sizeof(double) * k * n + 8));
    h2d(da, a, m, k, lda, st);
    h2d(db, b, k, n, ldb, st);
    double* ratios = static_cast<double*>(ctx->ratios.get(sizeof(double) * (m + 1)));
    int* zf = static_cast<int*>(ctx->status.get(sizeof(int)));
    auto* cmax = static_cast<unsigned long long*>(ctx->colmax.get(8 * (n + 1)));
    auto* cmin = static_cast<unsigned long long*>(ctx->colmin.get(8 * (n + 1)));
    OZ_CUDA(cudaMemsetAsync(zf, 0, sizeof(int), st));
    OZ_CUDA(launch_row_profile(da, k, m, k, ratios, zf, st, &launches));
    OZ_CUDA(launch_col_profile(db, n, k, n, cmax, cmin, st, &launches));
    std::vector<double> hr(m);
    std::vector<unsigned long long> hmax(n), hmin(n);
    int hz = 0;
    if (m) OZ_CUDA(cudaMemcpyAsync(hr.data(), ratios, sizeof(double) * m, cudaMemcpyDeviceToHost, st));
    if (n) {
      OZ_CUDA(cudaMemcpyAsync(hmax.data(), cmax, 8 * n, cudaMemcpyDeviceToHost, st));
      OZ_CUDA(cudaMemcpyAsync(hmin.data(), cmin, 8 * n, cudaMemcpyDeviceToHost, st));
    }
    OZ_CUDA(cudaMemcpyAsync(&hz, zf, sizeof(int), cudaMemcpyDeviceToHost, st));
    OZ_CUDA(cudaStreamSynchronize(st));
    ctx->launches += launches;
    double wa = 1.0, wb = 1.0;
    for (double r : hr) wa = std::max(wa, r);
    int bz = 0;
    for (int64_t j = 0; j < n; ++j) {
      if (hmax[j] == 0) {
        bz = 1;
        continue;
      }
      double mx, mn;
      std::memcpy(&mx, &hmax[j], 8);
      std::memcpy(&mn, &hmin[j], 8);
      wb = std::max(wb, mx / mn);
    }
    out->kappa_a = 2.0 * wa;
    out->kappa_b = 2.0 * wb;
    out->a_has_zero_block = hz;
    out->b_has_zero_block = bz;
  });
}

int ozgpu_block_ratios(ozgpu_ctx* ctx, int orientation, int64_t rows, int64_t cols,
                       const double* x, int64_t ldx, double* ratios_out, int* has_zero_block) {
  return guarded([&] {
    if (!ctx || !ratios_out || !has_zero_block)
      throw std::invalid_argument("block_ratios: null argument");
    std::lock_guard<std::mutex> lock(ctx->mu);
    OZ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    acquire_workspace(ctx, st);
    int64_t launches = 0;
    double* dx = static_cast<double*>(ctx->in_a.get(sizeof(double) * rows * cols + 8));
    h2d(dx, x, rows, cols, ldx, st);
    *has_zero_block = 0;
    if (orientation == 0) {
      double* ratios = static_cast<double*>(ctx->ratios.get(sizeof(double) * (rows + 1)));
      int* zf = static_cast<int*>(ctx->status.get(sizeof(int)));
      OZ_CUDA(cudaMemsetAsync(zf, 0, sizeof(int), st));
      OZ_CUDA(launch_row_profile(dx, cols, rows, cols, ratios, zf, st, &launches));
      if (rows)
        OZ_CUDA(cudaMemcpyAsync(ratios_out, ratios, sizeof(double) * rows, cudaMemcpyDeviceToHost,
                                st));
      OZ_CUDA(cudaMemcpyAsync(has_zero_block, zf, sizeof(int), cudaMemcpyDeviceToHost, st));
      OZ_CUDA(cudaStreamSynchronize(st));
    } else {
      auto* cmax = static_cast<unsigned long long*>(ctx->colmax.get(8 * (cols + 1)));
      auto* cmin = static_cast<unsigned long long*>(ctx->colmin.get(8 * (cols + 1)));
      OZ_CUDA(launch_col_profile(dx, cols, rows, cols, cmax, cmin, st, &launches));
      std::vector<unsigned long long> hmax(cols), hmin(cols);
      if (cols) {
        OZ_CUDA(cudaMemcpyAsync(hmax.data(), cmax, 8 * cols, cudaMemcpyDeviceToHost, st));
        OZ_CUDA(cudaMemcpyAsync(hmin.data(), cmin, 8 * cols, cudaMemcpyDeviceToHost, st));
      }
      OZ_CUDA(cudaStreamSynchronize(st));
      for (int64_t j = 0; j < cols; ++j) {
        if (hmax[j] == 0) {
          ratios_out[j] = 1.0;
          *has_zero_block = 1;
          continue;
        }
        double mx, mn;
        std::memcpy(&mx, &hmax[j], 8);
        std::memcpy(&mn, &hmin[j], 8);
        ratios_out[j] = mx / mn;
      }
    }
    ctx->launches += launches;
  });
}

int ozgpu_fp64_gemm(ozgpu_ctx* ctx, int absolute, int64_t m, int64_t k, int64_t n,
                    const double* a, int64_t lda, const double* b, int64_t ldb, double* out,
                    int64_t ldo) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("fp64_gemm: null context");
    if (m < 0 || n < 0 || k < 0) throw std::invalid_argument("fp64_gemm: shape mismatch");
    std::lock_guard<std::mutex> lock(ctx->mu);
    OZ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    acquire_workspace(ctx, st);
    int64_t launches = 0;
    double* da = static_cast<double*>(ctx->in_a.get(sizeof(double) * m * k + 8));
    double* db = static_cast<double*>(ctx->in_b.get(sizeof(double) * k * n + 8));
    double* dc = static_cast<double*>(ctx->io_c.get(sizeof(double) * m * n + 8));
    h2d(da, a, m, k, lda, st);
    h2d(db, b, k, n, ldb, st);
    OZ_CUDA(launch_fp64_gemm(absolute, m, k, n, da, k, db, n, dc, n, st, &launches));
    d2h(out, ldo, dc, m, n, st);
    OZ_CUDA(cudaStreamSynchronize(st));
    ctx->launches += launches;
  });
}

int ozgpu_min_exact_slices(ozgpu_ctx* ctx, int orientation, int64_t rows, int64_t cols,
                           const double* x, int64_t ldx, int width, int mode, int* out) {
  return guarded([&] {
    if (!ctx || !out) throw std::invalid_argument("min_exact_slices: null argument");
    if (width < 1) throw std::invalid_argument("min_exact_slices: width must be >= 1");
    if (rows < 0 || cols < 0 || ldx < cols || (rows * cols > 0 && !x))
      throw std::invalid_argument("min_exact_slices: bad matrix");
    std::lock_guard<std::mutex> lock(ctx->mu);
    OZ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    acquire_workspace(ctx, st);
    int64_t launches = 0;
    double* dx = static_cast<double*>(ctx->in_a.get(sizeof(double) * rows * cols + 8));
    h2d(dx, x, rows, cols, ldx, st);
    int* bits = static_cast<int*>(ctx->status.get(sizeof(int)));
    auto* colmax = static_cast<unsigned long long*>(ctx->colmax.get(8 * (cols + 1)));
    OZ_CUDA(launch_exact_bits(orientation, dx, cols, rows, cols, colmax, bits, st, &launches));
    int hb = 0;
    OZ_CUDA(cudaMemcpyAsync(&hb, bits, sizeof(int), cudaMemcpyDeviceToHost, st));
    OZ_CUDA(cudaStreamSynchronize(st));
    ctx->launches += launches;
    // slicing.cpp:236-240
    *out = mode == 1 ? std::max(1, (hb + 1 + width - 1) / width) : std::max(1, (hb + width - 1) / width);
  });
}

// exact_gemm(a, b).to_matrix() (oracle.cpp:223-232, 157-180) on the GPU: the
// Ozaki-I scheme itself with slices that hold A and B exactly (the minimal
// truncate-mode counts, found by the GPU scan above) and the full pair
// schedule is error-free, and the levelled-exact combine rounds the exact
// sum once: C = RN(AB) for every entry.
int ozgpu_exact_gemm(ozgpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* a,
                     int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("exact_gemm: null context");
    check_operands("exact_gemm", m, n, k, a, lda, b, ldb, c, ldc);
    if (m == 0 || n == 0) return;
    if (k == 0) {
      for (int64_t i = 0; i < m; ++i) std::fill(c + i * ldc, c + i * ldc + n, 0.0);
      return;
    }
    const ozgpu_mma_config cfg{7, 31};
    const int t = optimal_slice_width(cfg, k);
    int sa = 0, sb = 0;
    if (ozgpu_min_exact_slices(ctx, 0, m, k, a, lda, t, 0, &sa) != OZGPU_OK ||
        ozgpu_min_exact_slices(ctx, 1, k, n, b, ldb, t, 0, &sb) != OZGPU_OK)
      throw std::runtime_error(g_error);
    const ozgpu_plan plan = make_plan(cfg, k, sa, sb, 0, 2, 0, 53);
    const ChunkPlan cp = build_chunks(plan, cfg, k);
    try {
      (void)exact_words(cp.diagonals, t, cp.chunks.size());
    } catch (const std::invalid_argument&) {
      throw std::domain_error("exact_gemm: the exponent range of the inputs needs " +
                              std::to_string(sa) + " x " + std::to_string(sb) +
                              " exact slices, beyond the 1024-bit exact combine");
    }
    std::lock_guard<std::mutex> lock(ctx->mu);
    OZ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    acquire_workspace(ctx, st);
    double* da = static_cast<double*>(ctx->in_a.get(sizeof(double) * m * k + 8));
    double* db = static_cast<double*>(ctx->in_b.get(sizeof(double) * k * n + 8));
    double* dc = static_cast<double*>(ctx->io_c.get(sizeof(double) * m * n + 8));
    h2d(da, a, m, k, lda, st);
    h2d(db, b, k, n, ldb, st);
    run_multiply(ctx, m, n, k, da, k, db, n, dc, n, cfg, plan, st, nullptr, false, 1.0, 0.0,
                 nullptr, 0);
    int hs = 0;
    OZ_CUDA(cudaMemcpyAsync(&hs, ctx->status.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    OZ_CUDA(cudaStreamSynchronize(st));
    if (hs) throw std::invalid_argument("exact_gemm: inputs must be finite with no negative zeros");
    d2h(c, ldc, dc, m, n, st);
    OZ_CUDA(cudaStreamSynchronize(st));
  });
}

int ozgpu_error_metrics(ozgpu_ctx* ctx, int64_t m, int64_t n, const double* computed, int64_t ldc,
                        const double* reference, int64_t ldr, double* max_elementwise,
                        double* sum_sq) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("error_metrics: null context");
    if (m < 0 || n < 0 || ldc < n || (reference && ldr < n) || (m * n > 0 && !computed))
      throw std::invalid_argument("error_metrics: bad matrix");
    std::lock_guard<std::mutex> lock(ctx->mu);
    OZ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    acquire_workspace(ctx, st);
    int64_t launches = 0;
    double* dcm = static_cast<double*>(ctx->in_a.get(sizeof(double) * m * n + 8));
    h2d(dcm, computed, m, n, ldc, st);
    double* dr = nullptr;
    if (reference) {
      dr = static_cast<double*>(ctx->in_b.get(sizeof(double) * m * n + 8));
      h2d(dr, reference, m, n, ldr, st);
    }
    const int sd = metric_scratch_doubles();
    double* scratch = static_cast<double*>(ctx->ratios.get(sizeof(double) * sd));
    OZ_CUDA(launch_error_metrics(dcm, n, dr, n, m, n, scratch, st, &launches));
    double h[2] = {0.0, 0.0};
    OZ_CUDA(cudaMemcpyAsync(h, scratch + sd - 2, sizeof h, cudaMemcpyDeviceToHost, st));
    OZ_CUDA(cudaStreamSynchronize(st));
    ctx->launches += launches;
    if (max_elementwise) *max_elementwise = h[0];
    if (sum_sq) *sum_sq = h[1];
  });
}

int ozgpu_dgemm(ozgpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* a, int64_t lda,
                const double* b, int64_t ldb, double* c, int64_t ldc, ozgpu_mma_config cfg,
                const ozgpu_plan* plan, ozgpu_diag* diag) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("multiply: null context");
    check_plan(plan);
    check_operands("multiply", m, n, k, a, lda, b, ldb, c, ldc);
    host_multiply(ctx, m, n, k, a, lda, b, ldb, c, ldc, cfg, *plan, diag, false, 1.0, 0.0,
                  nullptr, 0);
  });
}

int ozgpu_dgemm_axpby(ozgpu_ctx* ctx, int64_t m, int64_t n, int64_t k, double alpha,
                      const double* a, int64_t lda, const double* b, int64_t ldb, double beta,
                      const double* c_in, int64_t ldc, double* d_out, int64_t ldd,
                      ozgpu_mma_config cfg, const ozgpu_plan* plan, ozgpu_diag* diag) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("multiply_axpby: null context");
    check_plan(plan);
    check_operands("multiply_axpby", m, n, k, a, lda, b, ldb, d_out, ldd);
    if (ldc < n) throw std::invalid_argument("multiply_axpby: leading dimension of C_in is smaller than n");
    if (m > 0 && n > 0 && !c_in) throw std::invalid_argument("multiply_axpby: null matrix pointer");
    host_multiply(ctx, m, n, k, a, lda, b, ldb, d_out, ldd, cfg, *plan, diag, true, alpha, beta,
                  c_in, ldc);
  });
}

int ozgpu_dgemm_device(ozgpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* a,
                       int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc,
                       ozgpu_mma_config cfg, const ozgpu_plan* plan, void* stream,
                       int* dev_status, ozgpu_diag* diag) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("multiply: null context");
    check_plan(plan);
    check_operands("multiply", m, n, k, a, lda, b, ldb, c, ldc);
    if (k < 1) throw std::invalid_argument("multiply: empty inner dimension");
    ValidationResult v = host_validation(cfg, *plan, k);
    if (v.capacity_error || v.precision_error) throw std::domain_error(v.message);
    const std::string perr = plan_error(*plan);
    if (!perr.empty()) throw std::invalid_argument(perr);
    std::lock_guard<std::mutex> lock(ctx->mu);
    OZ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);  // NULL = legacy default stream
    acquire_workspace(ctx, st);
    // Repeated calls with the same shape, plan, pointers and stream replay a
    // captured CUDA graph (one launch instead of ~10 enqueues and the host
    // planning); the first call runs eagerly (it also sizes the workspace),
    // the second captures.  Off with OZGPU_GRAPH=0, under stage timing, on
    // the legacy default stream, and for the sequential strategies.
    const char* genv = std::getenv("OZGPU_GRAPH");
    const bool graphs = !(genv && std::string(genv) == "0") && !ctx->timing && st != nullptr &&
                        plan->strategy == 2;
    if (graphs) {
      char key[512];
      std::snprintf(key, sizeof key, "%p|%lld|%lld|%lld|%p|%lld|%p|%lld|%p|%lld|%p|%d|%d|%d|%d|%d|%d|%d|%d|%d|%d",
                    stream, (long long)m, (long long)n, (long long)k, (const void*)a, (long long)lda,
                    (const void*)b, (long long)ldb, (void*)c, (long long)ldc, (void*)dev_status,
                    cfg.input_width, cfg.acc_width, plan->slices_a, plan->slices_b, plan->width,
                    plan->schedule, plan->strategy, plan->mode, plan->precision,
                    plan->diag_sum_limit);
      // the OZGPU_* knobs select kernels at capture time: part of the key
      std::string gkey(key);
      for (char** ev = environ; ev && *ev; ++ev)
        if (std::strncmp(*ev, "OZGPU_", 6) == 0) gkey += std::string("|") + *ev;
      if (ctx->graphs.size() >= 64 && !ctx->graphs.count(gkey)) {  // bound the cache
        OZ_CUDA(cudaDeviceSynchronize());  // pinned table copies may still be in flight
        for (auto& kv : ctx->graphs) {
          if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
          for (void* pp : kv.second.pinned) cudaFreeHost(pp);
        }
        ctx->graphs.clear();
      }
      auto& e = ctx->graphs[gkey];
      const uint64_t gen = g_workspace_gen.load();
      if (e.exec && e.gen == gen) {
        OZ_CUDA(cudaGraphLaunch(e.exec, st));
        release_workspace(ctx, st);
        ctx->launches += e.launches;
        if (diag) *diag = make_diag(*plan, cfg, m, n, k, 0);
        return;
      }
      if (e.exec) {  // stale: the workspace moved
        OZ_CUDA(cudaDeviceSynchronize());  // its pinned table copies may still be in flight
        cudaGraphExecDestroy(e.exec);
        e.exec = nullptr;
        for (void* pp : e.pinned) cudaFreeHost(pp);
        e.pinned.clear();
      }
      if (e.uses++ >= 1) {
        cudaGraph_t graph = nullptr;
        const int64_t before = ctx->launches.load();
        ctx->capturing = &e;
        OZ_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
        try {
          run_multiply(ctx, m, n, k, a, lda, b, ldb, c, ldc, cfg, *plan, st, dev_status, false,
                       1.0, 0.0, nullptr, 0);
        } catch (...) {
          ctx->capturing = nullptr;
          cudaStreamEndCapture(st, &graph);
          if (graph) cudaGraphDestroy(graph);
          throw;
        }
        ctx->capturing = nullptr;
        OZ_CUDA(cudaStreamEndCapture(st, &graph));
        e.launches = ctx->launches.load() - before;
        ctx->launches -= e.launches;  // counted when replayed
        OZ_CUDA(cudaGraphInstantiate(&e.exec, graph, 0));
        cudaGraphDestroy(graph);
        e.gen = g_workspace_gen.load();
        if (e.gen != gen) {  // the capture itself grew the workspace: do not trust it
          cudaGraphExecDestroy(e.exec);
          e.exec = nullptr;
          e.uses = 1;
        } else {
          OZ_CUDA(cudaGraphLaunch(e.exec, st));
          release_workspace(ctx, st);
          ctx->launches += e.launches;
          if (diag) *diag = make_diag(*plan, cfg, m, n, k, 0);
          return;
        }
      }
    }
    try {
      run_multiply(ctx, m, n, k, a, lda, b, ldb, c, ldc, cfg, *plan, st, dev_status, false, 1.0,
                   0.0, nullptr, 0);
    } catch (...) {
      release_workspace(ctx, st);  // whatever was enqueued still orders later calls
      throw;
    }
    release_workspace(ctx, st);
    if (diag) *diag = make_diag(*plan, cfg, m, n, k, 0);
  });
}

int ozgpu_split(ozgpu_ctx* ctx, int orientation, int64_t rows, int64_t cols, const double* x,
                int64_t ldx, int width, int count, int mode, int64_t* slices_out,
                int* scales_out) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("split: null context");
    if (width < 1 || width > 62) throw std::invalid_argument("split: width out of range");
    if (count < 1) throw std::invalid_argument("split: need at least one slice");
    if (mode == 1 && width < 2) throw std::invalid_argument("split: nearest mode needs width >= 2");
    std::lock_guard<std::mutex> lock(ctx->mu);
    OZ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    acquire_workspace(ctx, st);
    int64_t launches = 0;
    double* dx = static_cast<double*>(ctx->in_a.get(sizeof(double) * rows * cols + 8));
    h2d(dx, x, rows, cols, ldx, st);
    int* status = static_cast<int*>(ctx->status.get(sizeof(int)));
    OZ_CUDA(cudaMemsetAsync(status, 0, sizeof(int), st));
    const int64_t blocks = orientation == 0 ? rows : cols;
    const int64_t len = orientation == 0 ? cols : rows;
    const int64_t kp = round_up(std::max<int64_t>(len, 1), 8);
    int64_t* out = static_cast<int64_t*>(
        ctx->i64o.get(sizeof(int64_t) * static_cast<size_t>(count) * blocks * kp + 8));
    int* scales = static_cast<int*>(ctx->qa.get(sizeof(int) * (blocks + 1)));
    if (orientation == 0) {
      OZ_CUDA(launch_slice_rows(dx, cols, rows, cols, kp, width, count, mode, out, 1, scales,
                                status, st, &launches));
    } else {
      auto* colmax = static_cast<unsigned long long*>(ctx->colmax.get(8 * (cols + 1)));
      OZ_CUDA(launch_slice_cols(dx, cols, rows, cols, kp, width, count, mode, out, 1, scales,
                                colmax, status, st, &launches));
    }
    std::vector<int64_t> host(static_cast<size_t>(count) * blocks * kp);
    int hs = 0;
    if (!host.empty())
      OZ_CUDA(cudaMemcpyAsync(host.data(), out, sizeof(int64_t) * host.size(),
                              cudaMemcpyDeviceToHost, st));
    if (blocks)
      OZ_CUDA(cudaMemcpyAsync(scales_out, scales, sizeof(int) * blocks, cudaMemcpyDeviceToHost, st));
    OZ_CUDA(cudaMemcpyAsync(&hs, status, sizeof(int), cudaMemcpyDeviceToHost, st));
    OZ_CUDA(cudaStreamSynchronize(st));
    ctx->launches += launches;
    if (hs & 1) throw std::invalid_argument("split: non-finite entry");
    for (int l = 0; l < count; ++l)
      for (int64_t bb = 0; bb < blocks; ++bb)
        for (int64_t j = 0; j < len; ++j) {
          int64_t v = host[(static_cast<size_t>(l) * blocks + bb) * kp + j];
          int64_t r = orientation == 0 ? bb : j, c = orientation == 0 ? j : bb;
          slices_out[(static_cast<size_t>(l) * rows + r) * cols + c] = v;
        }
  });
}

int ozgpu_device_contexts(const int* devices, int count, ozgpu_ctx** out) {
  return guarded([&] {
    if (!devices || !out || count < 1) throw std::invalid_argument("device_contexts: bad arguments");
    static std::mutex mu;
    static std::map<std::pair<int, int>, ozgpu_ctx*> extra;  // (device, occurrence > 0)
    std::lock_guard<std::mutex> lock(mu);
    std::map<int, int> seen;
    for (int s = 0; s < count; ++s) {
      const int dev = devices[s];
      const int occ = seen[dev]++;
      if (occ == 0) {
        out[s] = ozgpu_default_context(dev);
        if (!out[s]) throw DeviceError(g_error);
        continue;
      }
      auto& c = extra[{dev, occ}];
      if (!c) {
        ozgpu_ctx* made = nullptr;
        if (ozgpu_create(dev, &made) != OZGPU_OK) throw DeviceError(g_error);
        c = made;
      }
      out[s] = c;
    }
  });
}

namespace ozgpu {
namespace {

// p_r >= p_c, p_r * p_c == count, as square as possible (1x1, 2x1, 2x2, 4x2)
void shard_grid(int count, int& pr, int& pc) {
  pr = count;
  pc = 1;
  for (int q = 1; q <= count; ++q)
    if (count % q == 0 && count / q >= q) {
      pr = count / q;
      pc = q;
    }
}

void shard_range(int64_t len, int parts, int idx, int64_t& lo, int64_t& hi) {
  const int64_t base = len / parts, rem = len % parts;
  lo = idx * base + std::min<int64_t>(idx, rem);
  hi = lo + base + (idx < rem ? 1 : 0);
}

// Pitched copy of a rows x width_bytes window between (possibly different)
// devices: NVLink P2P when peer access is on, a device-to-device copy when
// both sides are the same device.
void peer_copy_2d(void* dst, size_t dpitch, int ddev, const void* src, size_t spitch, int sdev,
                  size_t width_bytes, size_t rows, cudaStream_t st) {
  if (!width_bytes || !rows) return;
  cudaMemcpy3DPeerParms p{};
  p.srcPtr = make_cudaPitchedPtr(const_cast<void*>(src), spitch, width_bytes, rows);
  p.srcDevice = sdev;
  p.dstPtr = make_cudaPitchedPtr(dst, dpitch, width_bytes, rows);
  p.dstDevice = ddev;
  p.extent = make_cudaExtent(width_bytes, rows, 1);
  OZ_CUDA(cudaMemcpy3DPeerAsync(&p, st));
}

void enable_peer(int from, int to) {
  if (from == to) return;
  static std::mutex mu;
  static std::set<std::pair<int, int>> done;
  std::lock_guard<std::mutex> lock(mu);
  if (!done.insert({from, to}).second) return;
  int can = 0;
  OZ_CUDA(cudaDeviceCanAccessPeer(&can, from, to));
  if (!can) return;  // the copies still work, staged by the driver
  int cur = 0;
  OZ_CUDA(cudaGetDevice(&cur));
  OZ_CUDA(cudaSetDevice(from));
  cudaError_t e = cudaDeviceEnablePeerAccess(to, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
  else OZ_CUDA(e);
  OZ_CUDA(cudaSetDevice(cur));
}

}  // namespace
}  // namespace ozgpu

// 2-D C-tile sharding of one host-pointer multiply over several contexts
// (SURVEY.md 8e): context r computes C block (i, j) = divmod(r, p_c) with the
// full k from its A row-panel and B column-panel, pulled from the caller's
// host buffers over its own PCIe link by its own blocked pipeline.  Scales
// are per row of A / column of B, so the blocks are bit-identical to the
// single-context result; no device-to-device exchange is
// needed because every panel starts on the host.
int ozgpu_dgemm_multi(ozgpu_ctx* const* ctxs, int count, int64_t m, int64_t n, int64_t k,
                      const double* a, int64_t lda, const double* b, int64_t ldb, double* c,
                      int64_t ldc, ozgpu_mma_config cfg, const ozgpu_plan* plan,
                      ozgpu_diag* diag) {
  int pr = 1, pc = 1;
  int rc = guarded([&] {
    if (!ctxs || count < 1) throw std::invalid_argument("multiply: no contexts");
    for (int r = 0; r < count; ++r)
      if (!ctxs[r]) throw std::invalid_argument("multiply: null context");
    check_plan(plan);
    check_operands("multiply", m, n, k, a, lda, b, ldb, c, ldc);
    shard_grid(count, pr, pc);
  });
  if (rc != OZGPU_OK) return rc;
  if (count == 1 || m < pr || n < pc)  // nothing to shard (every block must be non-empty)
    return ozgpu_dgemm(ctxs[0], m, n, k, a, lda, b, ldb, c, ldc, cfg, plan, diag);
  std::vector<int> codes(count, OZGPU_OK);
  std::vector<std::string> msgs(count);
  std::vector<ozgpu_diag> diags(count);
  std::vector<std::thread> pool;
  for (int r = 0; r < count; ++r)
    pool.emplace_back([&, r] {
      int64_t r0, r1, c0, c1;
      shard_range(m, pr, r / pc, r0, r1);
      shard_range(n, pc, r % pc, c0, c1);
      codes[r] = ozgpu_dgemm(ctxs[r], r1 - r0, c1 - c0, k, a + r0 * lda, lda, b + c0, ldb,
                             c + r0 * ldc + c0, ldc, cfg, plan, &diags[r]);
      if (codes[r] != OZGPU_OK) msgs[r] = g_error;  // thread-local: copy out
    });
  for (auto& th : pool) th.join();
  for (int r = 0; r < count; ++r)
    if (codes[r] != OZGPU_OK) {  // first failing block in rank order
      g_error = msgs[r];
      return codes[r];
    }
  return guarded([&] {
    long long psi = 0;
    for (const auto& d : diags) psi = std::max(psi, d.realized_psi);
    if (diag) *diag = make_diag(*plan, cfg, m, n, k, psi);
  });
}


// Device-resident 2-D C-tile sharding: A, B and C live on
// src_device; context r computes C block (r / p_c, r % p_c) with the full k.
// A context on another device pulls its A row-panel and B column-panel over
// NVLink (peer copies), multiplies on its own stream and pushes its C block
// back; a context on src_device reads the panels in place.  Only the panels
// a block needs move, once each -- no collective, since scales are per row
// of A / column of B and every block is independent (bit-identical to
// ozgpu_dgemm_device).  Ordered after the caller's stream and before its
// later work by events; the call does not synchronise.
int ozgpu_dgemm_device_multi(ozgpu_ctx* const* ctxs, int count, int src_device, int64_t m,
                             int64_t n, int64_t k, const double* a, int64_t lda, const double* b,
                             int64_t ldb, double* c, int64_t ldc, ozgpu_mma_config cfg,
                             const ozgpu_plan* plan, void* stream, int* dev_status,
                             ozgpu_diag* diag) {
  int pr = 1, pc = 1;
  bool force_peer = false;
  int rc = guarded([&] {
    if (!ctxs || count < 1) throw std::invalid_argument("multiply: no contexts");
    for (int r = 0; r < count; ++r)
      if (!ctxs[r]) throw std::invalid_argument("multiply: null context");
    check_plan(plan);
    check_operands("multiply", m, n, k, a, lda, b, ldb, c, ldc);
    if (k < 1) throw std::invalid_argument("multiply: empty inner dimension");
    int ndev = 0;
    OZ_CUDA(cudaGetDeviceCount(&ndev));
    if (src_device < 0 || src_device >= ndev)
      throw std::invalid_argument("multiply: bad source device");
    shard_grid(count, pr, pc);
    // test hook: treat contexts on src_device as remote (exercises the
    // panel copies on a one-GPU box)
    const char* fe = std::getenv("OZGPU_MULTI_PEER");
    force_peer = fe && std::string(fe) == "1";
  });
  if (rc != OZGPU_OK) return rc;
  const int slots = count;
  if (m < pr || n < pc) {  // every block must be non-empty: one context does it all
    count = 1;
    pr = pc = 1;
  }
  std::vector<long long> psi(count, 0);
  int failed = OZGPU_OK;
  rc = guarded([&] {
    cudaStream_t caller = static_cast<cudaStream_t>(stream);
    OZ_CUDA(cudaSetDevice(src_device));
    // every slot reads 0 unless its block sees a bad input (slots past the
    // block count when the product is too small to split stay 0)
    if (dev_status) OZ_CUDA(cudaMemsetAsync(dev_status, 0, sizeof(int) * slots, caller));
    cudaEvent_t ready = nullptr;
    OZ_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    std::unique_ptr<CUevent_st, decltype(&cudaEventDestroy)> ready_guard(ready, &cudaEventDestroy);
    OZ_CUDA(cudaEventRecord(ready, caller));
    for (int r = 0; r < count; ++r) {
      ozgpu_ctx* x = ctxs[r];
      int64_t r0, r1, c0, c1;
      shard_range(m, pr, r / pc, r0, r1);
      shard_range(n, pc, r % pc, c0, c1);
      const int64_t rows = r1 - r0, cols = c1 - c0;
      const bool local = x->device == src_device && !force_peer;
      std::lock_guard<std::mutex> lock(x->multi_mu);
      OZ_CUDA(cudaSetDevice(x->device));
      if (!x->multi_stream) OZ_CUDA(cudaStreamCreateWithFlags(&x->multi_stream, cudaStreamNonBlocking));
      cudaStream_t s = x->multi_stream;
      OZ_CUDA(cudaStreamWaitEvent(s, ready, 0));
      int* slot = dev_status ? dev_status + r : nullptr;
      ozgpu_diag d{};
      int code;
      if (local) {
        code = ozgpu_dgemm_device(x, rows, cols, k, a + r0 * lda, lda, b + c0, ldb,
                                  c + r0 * ldc + c0, ldc, cfg, plan, s, slot, &d);
      } else {
        enable_peer(x->device, src_device);
        enable_peer(src_device, x->device);
        const size_t ba = sizeof(double) * rows * k, bb = sizeof(double) * k * cols,
                     bc = sizeof(double) * rows * cols;
        if (ba > x->peer_a.bytes || bb > x->peer_b.bytes || bc > x->peer_c.bytes)
          OZ_CUDA(cudaStreamSynchronize(s));  // regrowing: earlier calls' panels in flight
        auto* pa = static_cast<double*>(x->peer_a.get(ba));
        auto* pb = static_cast<double*>(x->peer_b.get(bb));
        auto* pcb = static_cast<double*>(x->peer_c.get(bc));
        int* pst = slot ? static_cast<int*>(x->peer_status.get(sizeof(int))) : nullptr;
        OZ_CUDA(cudaSetDevice(x->device));
        peer_copy_2d(pa, sizeof(double) * k, x->device, a + r0 * lda, sizeof(double) * lda,
                     src_device, sizeof(double) * k, rows, s);
        peer_copy_2d(pb, sizeof(double) * cols, x->device, b + c0, sizeof(double) * ldb,
                     src_device, sizeof(double) * cols, k, s);
        code = ozgpu_dgemm_device(x, rows, cols, k, pa, k, pb, cols, pcb, cols, cfg, plan, s, pst,
                                  &d);
        if (code == OZGPU_OK) {
          OZ_CUDA(cudaSetDevice(x->device));
          peer_copy_2d(c + r0 * ldc + c0, sizeof(double) * ldc, src_device, pcb,
                       sizeof(double) * cols, x->device, sizeof(double) * cols, rows, s);
          if (slot) OZ_CUDA(cudaMemcpyPeerAsync(slot, src_device, pst, x->device, sizeof(int), s));
        }
      }
      if (code != OZGPU_OK) {  // g_error already says why; blocks before it stay enqueued
        failed = code;
        cudaSetDevice(src_device);
        return;
      }
      psi[r] = d.realized_psi;
      // the caller's stream continues once this block (and its copies) is done
      OZ_CUDA(cudaSetDevice(x->device));
      cudaEvent_t done = nullptr;
      OZ_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
      OZ_CUDA(cudaEventRecord(done, s));
      cudaError_t we = cudaStreamWaitEvent(caller, done, 0);
      cudaEventDestroy(done);  // released once it completes
      OZ_CUDA(we);
    }
    OZ_CUDA(cudaSetDevice(src_device));
    if (diag) *diag = make_diag(*plan, cfg, m, n, k, *std::max_element(psi.begin(), psi.end()));
  });
  return rc != OZGPU_OK ? rc : failed;
}

int ozgpu_split_i8(ozgpu_ctx* ctx, int orientation, int64_t rows, int64_t cols, const double* x,
                   int64_t ldx, int width, int count, int mode, int8_t* slices_out, int64_t ld,
                   int* scales_out) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("split: null context");
    if (width < 1 || width > 62) throw std::invalid_argument("split: width out of range");
    if (count < 1) throw std::invalid_argument("split: need at least one slice");
    if (mode == 1 && width < 2) throw std::invalid_argument("split: nearest mode needs width >= 2");
    if (width > 7)
      throw std::invalid_argument("split_i8: width " + std::to_string(width) +
                                  " does not fit the int8 operand");
    if (rows < 0 || cols < 0 || ldx < cols) throw std::invalid_argument("split_i8: bad shape");
    const int64_t blocks = orientation == 0 ? rows : cols;
    const int64_t len = orientation == 0 ? cols : rows;
    if (ld < round_up(std::max<int64_t>(len, 1), kKPad) || ld % kKPad)
      throw std::invalid_argument("split_i8: ld must be a multiple of 128 covering the block length");
    if ((rows * cols > 0 && !x) || (blocks > 0 && (!slices_out || !scales_out)))
      throw std::invalid_argument("split_i8: null pointer");
    std::lock_guard<std::mutex> lock(ctx->mu);
    OZ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    acquire_workspace(ctx, st);
    int64_t launches = 0;
    double* dx = static_cast<double*>(ctx->in_a.get(sizeof(double) * rows * cols + 8));
    h2d(dx, x, rows, cols, ldx, st);
    int* status = static_cast<int*>(ctx->status.get(sizeof(int)));
    OZ_CUDA(cudaMemsetAsync(status, 0, sizeof(int), st));
    const size_t bytes = static_cast<size_t>(count) * blocks * ld;
    int8_t* out = static_cast<int8_t*>(ctx->slices_a.get(bytes + 1));
    int* scales = static_cast<int*>(ctx->qa.get(sizeof(int) * (blocks + 1)));
    // exactly the launches run_multiply makes for its operands
    auto* colmax = static_cast<unsigned long long*>(ctx->colmax.get(8 * (cols + 1)));
    if (use_slice_queue(mode, width, ld)) {
      int* qw = queue_work(ctx, rows, cols, len, ld);
      if (orientation == 0)
        OZ_CUDA(launch_slice_queue(dx, cols, rows, nullptr, 0, 0, cols, ld, width, count, 0, out,
                                   0, nullptr, 0, scales, nullptr, nullptr, qw, status, upload_cb,
                                   ctx, st, &launches));
      else
        OZ_CUDA(launch_slice_queue(nullptr, 0, 0, dx, cols, cols, rows, ld, width, 0, count,
                                   nullptr, 0, out, 0, nullptr, scales, colmax, qw, status, upload_cb,
                                   ctx, st, &launches));
    } else if (orientation == 0) {
      OZ_CUDA(launch_slice_rows(dx, cols, rows, cols, ld, width, count, mode, out, 0, scales,
                                status, st, &launches));
    } else {
      OZ_CUDA(launch_slice_cols(dx, cols, rows, cols, ld, width, count, mode, out, 0, scales,
                                colmax, status, st, &launches));
    }
    int hs = 0;
    if (bytes) OZ_CUDA(cudaMemcpyAsync(slices_out, out, bytes, cudaMemcpyDeviceToHost, st));
    if (blocks)
      OZ_CUDA(cudaMemcpyAsync(scales_out, scales, sizeof(int) * blocks, cudaMemcpyDeviceToHost, st));
    OZ_CUDA(cudaMemcpyAsync(&hs, status, sizeof(int), cudaMemcpyDeviceToHost, st));
    OZ_CUDA(cudaStreamSynchronize(st));
    ctx->launches += launches;
    if (hs & 1) throw std::invalid_argument("split: non-finite entry");
  });
}

int ozgpu_pair_planes(ozgpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* a,
                      int64_t lda, const double* b, int64_t ldb, ozgpu_mma_config cfg,
                      const ozgpu_plan* plan, int* nchunks_out, int* chunk_table, int max_chunks,
                      int64_t r0, int64_t r1, int64_t c0, int64_t c1, int32_t* planes_out) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("pair_planes: null context");
    check_plan(plan);
    if (!nchunks_out) throw std::invalid_argument("pair_planes: null argument");
    check_operands("pair_planes", m, n, k, a, lda, b, ldb, planes_out ? static_cast<const void*>(planes_out) : static_cast<const void*>(a), n);
    if (k < 1) throw std::invalid_argument("multiply: empty inner dimension");
    ValidationResult v = host_validation(cfg, *plan, k);
    if (v.capacity_error || v.precision_error) throw std::domain_error(v.message);
    const std::string perr = plan_error(*plan);
    if (!perr.empty()) throw std::invalid_argument(perr);
    const ChunkPlan cp = build_chunks(*plan, cfg, k);
    const int nc = static_cast<int>(cp.chunks.size());
    *nchunks_out = nc;
    if (chunk_table)
      for (int c = 0; c < std::min(nc, max_chunks); ++c) {
        chunk_table[3 * c] = cp.chunks[c].d;
        chunk_table[3 * c + 1] = cp.chunks[c].l0;
        chunk_table[3 * c + 2] = cp.chunks[c].npairs;
      }
    if (!planes_out || m == 0 || n == 0 || nc == 0) return;
    if (r0 < 0 || r1 > m || r0 >= r1 || c0 < 0 || c1 > n || c0 >= c1)
      throw std::invalid_argument("pair_planes: window outside C");
    std::lock_guard<std::mutex> lock(ctx->mu);
    OZ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    acquire_workspace(ctx, st);
    double* da = static_cast<double*>(ctx->in_a.get(sizeof(double) * m * k + 8));
    double* db = static_cast<double*>(ctx->in_b.get(sizeof(double) * k * n + 8));
    double* dc = static_cast<double*>(ctx->io_c.get(sizeof(double) * m * n + 8));
    h2d(da, a, m, k, lda, st);
    h2d(db, b, k, n, ldb, st);
    struct Guard {
      ozgpu_ctx* c;
      ~Guard() { c->debug_planes = false; }
    } guard{ctx};
    ctx->debug_planes = true;
    run_multiply(ctx, m, n, k, da, k, db, n, dc, n, cfg, *plan, st, nullptr, false, 1.0, 0.0,
                 nullptr, 0);
    const int32_t* planes = static_cast<const int32_t*>(ctx->planes.p);
    const int64_t wr = r1 - r0, wc = c1 - c0;
    for (int c = 0; c < nc; ++c)
      OZ_CUDA(cudaMemcpy2DAsync(planes_out + static_cast<int64_t>(c) * wr * wc,
                                wc * sizeof(int32_t),
                                planes + c * ctx->dbg_plane_stride + r0 * ctx->dbg_ldp + c0,
                                ctx->dbg_ldp * sizeof(int32_t), wc * sizeof(int32_t), wr,
                                cudaMemcpyDeviceToHost, st));
    int hs = 0;
    OZ_CUDA(cudaMemcpyAsync(&hs, ctx->status.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    OZ_CUDA(cudaStreamSynchronize(st));
    if (hs) throw std::invalid_argument("multiply: inputs must be finite with no negative zeros");
  });
}

int ozgpu_integer_gemm(ozgpu_ctx* ctx, int64_t m, int64_t k, int64_t n, const int64_t* x,
                       const int64_t* y, const int64_t* c, int64_t* out, ozgpu_mma_config cfg) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("integer_gemm: null context");
    validate_cfg(cfg);
    const int64_t in_lo = -(int64_t{1} << cfg.input_width), in_hi = (int64_t{1} << cfg.input_width) - 1;
    const int64_t acc_lo = -(int64_t{1} << cfg.acc_width), acc_hi = (int64_t{1} << cfg.acc_width) - 1;
    int64_t mx = 0, my = 0, mc = 0;
    for (int64_t i = 0; i < m * k; ++i) {
      if (x[i] < in_lo || x[i] > in_hi)
        throw std::domain_error("integer_gemm: left operand entry outside I_" +
                                std::to_string(cfg.input_width));
      mx = std::max(mx, x[i] < 0 ? -x[i] : x[i]);
    }
    for (int64_t i = 0; i < k * n; ++i) {
      if (y[i] < in_lo || y[i] > in_hi)
        throw std::domain_error("integer_gemm: right operand entry outside I_" +
                                std::to_string(cfg.input_width));
      my = std::max(my, y[i] < 0 ? -y[i] : y[i]);
    }
    if (c)
      for (int64_t i = 0; i < m * n; ++i) {
        if (c[i] < acc_lo || c[i] > acc_hi)
          throw std::domain_error("integer_gemm: accumulator input outside I_" +
                                  std::to_string(cfg.acc_width));
        mc = std::max(mc, c[i] < 0 ? -c[i] : c[i]);
      }
    std::lock_guard<std::mutex> lock(ctx->mu);
    OZ_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    acquire_workspace(ctx, st);
    int64_t launches = 0;
    if (m == 0 || n == 0) return;
    int64_t* dx = static_cast<int64_t*>(ctx->i64a.get(sizeof(int64_t) * m * k + 8));
    int64_t* dy = static_cast<int64_t*>(ctx->i64b.get(sizeof(int64_t) * k * n + 8));
    int64_t* dc = c ? static_cast<int64_t*>(ctx->i64c.get(sizeof(int64_t) * m * n + 8)) : nullptr;
    int64_t* dout = static_cast<int64_t*>(ctx->i64o.get(sizeof(int64_t) * m * n + 8));
    if (m * k > 0) OZ_CUDA(cudaMemcpyAsync(dx, x, sizeof(int64_t) * m * k, cudaMemcpyHostToDevice, st));
    if (k * n > 0) OZ_CUDA(cudaMemcpyAsync(dy, y, sizeof(int64_t) * k * n, cudaMemcpyHostToDevice, st));
    if (c) OZ_CUDA(cudaMemcpyAsync(dc, c, sizeof(int64_t) * m * n, cudaMemcpyHostToDevice, st));
    // Tensor-core path when int8 holds the operands and no partial sum can
    // leave I_T nor int32; otherwise the exact per-MAC checked path.
    const __int128 bound = static_cast<__int128>(k) * mx * my + mc;
    const bool tc = cfg.input_width <= 7 && k >= 1 && bound <= acc_hi &&
                    bound <= static_cast<__int128>(2147483647);
    if (tc) {
      const int64_t kp = round_up(k, kKPad);
      int8_t* sA = static_cast<int8_t*>(ctx->slices_a.get(static_cast<size_t>(m) * kp));
      int8_t* sB = static_cast<int8_t*>(ctx->slices_b.get(static_cast<size_t>(n) * kp));
      OZ_CUDA(launch_pack_i8(dx, m, k, 0, kp, sA, st, &launches));
      OZ_CUDA(launch_pack_i8(dy, k, n, 1, kp, sB, st, &launches));
      const int64_t ldp = round_up(n, 4);
      int32_t* plane = static_cast<int32_t*>(ctx->planes.get(sizeof(int32_t) * m * ldp));
      ChunkDesc one{0, 1, 1, 0, 1};
      ChunkDesc* dch = static_cast<ChunkDesc*>(ctx->chunks.get(sizeof(ChunkDesc)));
      OZ_CUDA(cudaMemcpyAsync(dch, &one, sizeof one, cudaMemcpyHostToDevice, st));
      CUtensorMap tma = make_slice_map(ctx, sA, kp, m, 1, kBlockM);
      CUtensorMap tmb = make_slice_map(ctx, sB, kp, n, 1, 256);
      GemmArgs g{};
      g.chunks = dch;
      g.nchunks = 1;
      g.m = static_cast<int>(m);
      g.n = static_cast<int>(n);
      g.kblocks = static_cast<int>(kp / kBlockK);
      g.tiles_m = static_cast<int>((m + kBlockM - 1) / kBlockM);
      g.tiles_n = static_cast<int>((n + 255) / 256);
      g.total_units = g.tiles_m * g.tiles_n;
      g.planes = plane;
      g.plane_stride = m * ldp;
      g.ldp = ldp;
      OZ_CUDA(launch_gemm_i8(&tma, &tmb, g, ctx->num_sms, st, &launches));
      OZ_CUDA(launch_plane_to_i64(plane, ldp, dc, dout, m, n, st, &launches));
      OZ_CUDA(cudaMemcpyAsync(out, dout, sizeof(int64_t) * m * n, cudaMemcpyDeviceToHost, st));
      OZ_CUDA(cudaStreamSynchronize(st));
    } else {
      auto* first = static_cast<unsigned long long*>(ctx->ovf.get(8));
      OZ_CUDA(cudaMemsetAsync(first, 0xFF, 8, st));
      OZ_CUDA(launch_integer_gemm_exact(dx, dy, dc, dout, m, k, n, cfg.acc_width, first, st,
                                        &launches));
      unsigned long long hf = 0;
      OZ_CUDA(cudaMemcpyAsync(&hf, first, 8, cudaMemcpyDeviceToHost, st));
      OZ_CUDA(cudaMemcpyAsync(out, dout, sizeof(int64_t) * m * n, cudaMemcpyDeviceToHost, st));
      OZ_CUDA(cudaStreamSynchronize(st));
      if (hf != ~0ULL)
        throw OverflowError("integer accumulator overflow at (" + std::to_string(hf / n) + ", " +
                            std::to_string(hf % n) + "): value left I_" +
                            std::to_string(cfg.acc_width));
    }
    ctx->launches += launches;
  });
}

}  // extern "C"
