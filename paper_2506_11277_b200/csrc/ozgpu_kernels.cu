// sm_100a kernels of the B200-native Ozaki-I FP64 GEMM.
//
//   slice_rows / colmax + slice_cols   HBM-bound slicing (slicing.cpp:67-132)
//   gemm_i8                            tcgen05 kind::i8 pair GEMMs, TMA-fed,
//                                      int32 accumulators in TMEM (mma_sim.cpp:76-114)
//   combine_exact                      exact multi-word accumulation of the chunk
//                                      sums + one rounding (scheme.cpp:314-355,
//                                      oracle.cpp:157-180)
//   combine_sequential                 FP64 accumulation in the reference's order
//                                      for the non-default strategies (scheme.cpp:267-313)
//   row/col_profile                    kappa reductions (analysis.cpp:25-68)
//
// Compiled only for sm_100a (-gencode arch=compute_100a,code=sm_100a).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ozgpu_internal.h"
#include "ozgpu_numeric.h"

namespace ozgpu {

// ----------------------------------------------------------------------------
// Slicing (proj/src/slicing.cpp:67-132; fpcore.cpp:58-87)
// ----------------------------------------------------------------------------

// Absolute value bits of a double; positive doubles order like their bits.
__device__ __forceinline__ unsigned long long abs_bits(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x)) & 0x7FFFFFFFFFFFFFFFULL;
}

// Input status bits: 1 = Inf/NaN (split rejects these, slicing.cpp:88),
// 2 = negative zero (multiply also rejects these, matrix.cpp:22-29).
__device__ __forceinline__ int dirty(double x) {
  unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  return (((b >> 52) & 0x7FF) == 0x7FF ? 1 : 0) | (b == 0x8000000000000000ULL ? 2 : 0);
}

// Block-scale exponent from the max |x| bits: ilogb(max) + 1, 0 for a zero
// block (slicing.cpp:92, fpcore.cpp:83-87).  Handles subnormal maxima.
__device__ __forceinline__ int scale_from_maxbits(unsigned long long mb) {
  if (mb == 0) return 0;
  int be = static_cast<int>(mb >> 52);
  if (be > 0) return be - 1023 + 1;
  int top = 63 - __clzll(static_cast<long long>(mb));  // frac's leading bit
  return top - 1074 + 1;
}

// Writes the `count` slices of 8 consecutive entries (values v[0..8)) of
// one row / column with block exponent q.  Out layout: out[l * plane + off + e].
template <typename OutT>
__device__ __forceinline__ void emit_slices8(const double* v, int q, int width, int count,
                                             int mode, OutT* out, int64_t plane, int64_t off) {
  SliceEntry ent[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) ent[e] = make_slice_entry(v[e], q, width, count, mode);
  for (int l = 0; l < count; ++l) {
    if constexpr (sizeof(OutT) == 1) {
      unsigned long long packed = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        long long s = slice_of(ent[e], l, width, count, mode);
        packed |= (static_cast<unsigned long long>(s) & 0xFFULL) << (8 * e);
      }
      *reinterpret_cast<unsigned long long*>(out + l * plane + off) = packed;
    } else {
      long long s[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) s[e] = slice_of(ent[e], l, width, count, mode);
      longlong2* dst = reinterpret_cast<longlong2*>(out + l * plane + off);
#pragma unroll
      for (int e = 0; e < 4; ++e) dst[e] = make_longlong2(s[2 * e], s[2 * e + 1]);
    }
  }
}

// One CTA per row (grid-stride).  Pass 1: max |a| + cleanliness over the
// row; pass 2: s slices of 8 consecutive entries per thread, written as
// K-major rows of length kp (zero padded past k).
template <typename OutT>
__global__ void __launch_bounds__(256) slice_rows_kernel(const double* __restrict__ a,
                                                         int64_t lda, int64_t m, int64_t k,
                                                         int64_t kp, int width, int count,
                                                         int mode, OutT* __restrict__ out,
                                                         int* __restrict__ scales,
                                                         int* __restrict__ status) {
  __shared__ unsigned long long red[8];
  const int64_t plane = m * kp;
  for (int64_t row = blockIdx.x; row < m; row += gridDim.x) {
    const double* ar = a + row * lda;
    unsigned long long mx = 0;
    int bad = 0;
    for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
      double x = __ldg(ar + j);
      bad |= dirty(x);
      unsigned long long b = abs_bits(x);
      mx = b > mx ? b : mx;
    }
    if (bad) atomicOr(status, bad);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      unsigned long long t = __shfl_xor_sync(0xFFFFFFFFu, mx, o);
      mx = t > mx ? t : mx;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
      unsigned long long t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        unsigned long long u = __shfl_xor_sync(0xFFFFFFFFu, t, o);
        t = u > t ? u : t;
      }
      if (threadIdx.x == 0) red[0] = t;
    }
    __syncthreads();
    const int q = scale_from_maxbits(red[0]);
    if (threadIdx.x == 0) scales[row] = q;
    for (int64_t g = threadIdx.x; g < kp / 8; g += blockDim.x) {
      double v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        int64_t j = g * 8 + e;
        v[e] = j < k ? __ldg(ar + j) : 0.0;
      }
      emit_slices8<OutT>(v, q, width, count, mode, out, plane, row * kp + g * 8);
    }
    __syncthreads();
  }
}

// Column max |b| + cleanliness: thread per column, rows split over gridDim.y.
__global__ void __launch_bounds__(256) colmax_kernel(const double* __restrict__ b, int64_t ldb,
                                                     int64_t k, int64_t n, int64_t rows_per,
                                                     unsigned long long* __restrict__ colmax,
                                                     int* __restrict__ status) {
  int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  int64_t r0 = static_cast<int64_t>(blockIdx.y) * rows_per;
  int64_t r1 = r0 + rows_per < k ? r0 + rows_per : k;
  unsigned long long mx = 0;
  int bad = 0;
  for (int64_t r = r0; r < r1; ++r) {
    double x = __ldg(b + r * ldb + j);
    bad |= dirty(x);
    unsigned long long t = abs_bits(x);
    mx = t > mx ? t : mx;
  }
  if (bad) atomicOr(status, bad);
  if (mx) atomicMax(colmax + j, mx);
}

// 64 (k) x 64 (n) tile transpose-and-slice: B is k x n row-major; slices are
// written K-major as out[l][n][kp] (the tcgen05 B operand layout).
template <typename OutT>
__global__ void __launch_bounds__(256) slice_cols_kernel(
    const double* __restrict__ b, int64_t ldb, int64_t k, int64_t n, int64_t kp, int width,
    int count, int mode, const unsigned long long* __restrict__ colmax, OutT* __restrict__ out,
    int* __restrict__ scales) {
  __shared__ double tile[64][65];
  const int64_t k0 = static_cast<int64_t>(blockIdx.x) * 64;
  const int64_t n0 = static_cast<int64_t>(blockIdx.y) * 64;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  for (int rr = ty; rr < 64; rr += 4) {
    int64_t r = k0 + rr, c = n0 + tx;
    tile[tx][rr] = (r < k && c < n) ? __ldg(b + r * ldb + c) : 0.0;
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x < 64 && n0 + threadIdx.x < n)
    scales[n0 + threadIdx.x] = scale_from_maxbits(colmax[n0 + threadIdx.x]);
  const int64_t plane = n * kp;
  for (int item = threadIdx.x; item < 64 * 8; item += blockDim.x) {
    int nl = item >> 3, g = item & 7;
    int64_t col = n0 + nl;
    if (col >= n) continue;
    int64_t kk = k0 + g * 8;
    if (kk >= kp) continue;
    int q = scale_from_maxbits(colmax[col]);
    double v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = tile[nl][g * 8 + e];
    emit_slices8<OutT>(v, q, width, count, mode, out, plane, col * kp + kk);
  }
}

// ----------------------------------------------------------------------------
// tcgen05 / TMA / mbarrier primitives (inline PTX, sm_100a)
// ----------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_addr(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 32 lanes x 32 columns of 32-bit TMEM -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row core
// groups 1024 bytes apart (SBO), sm_100 descriptor version 1.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>(1) << 16;              // LBO (ignored for SW128 K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;      // SBO
  d |= static_cast<uint64_t>(1) << 46;              // version
  d |= static_cast<uint64_t>(2) << 61;              // SWIZZLE_128B
  return d;
}

// Instruction descriptor, kind::i8: s8 x s8 -> s32, both K-major.
template <int M, int N>
__host__ __device__ constexpr uint32_t idesc_i8() {
  return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

// ----------------------------------------------------------------------------
// Pair GEMM: persistent, warp-specialised, one 128 x BN tile per work unit.
//   warp 0: TMA producer   warp 1: MMA issuer   warp 2: TMEM allocator
//   warps 4..7: epilogue (TMEM -> registers -> global int32 chunk plane)
// ----------------------------------------------------------------------------

constexpr int kBN = 256;
constexpr int kStages = 4;
constexpr int kABytes = kBlockM * kBlockK;   // 16 KB
constexpr int kBBytes = kBN * kBlockK;       // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kTmemCols = 2 * kBN;           // double-buffered accumulator
constexpr int kGemmThreads = 256;
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;

int gemm_smem_bytes() { return kSmemBytes; }

struct UnitCoord {
  int tm, tn, chunk;
};

// Grouped rasterisation: consecutive units walk 8 tile-rows at a time so
// concurrently running CTAs share A and B slice panels in L2.
__device__ __forceinline__ UnitCoord decode_unit(int unit, const GemmArgs& p) {
  const int tiles = p.tiles_m * p.tiles_n;
  UnitCoord u;
  u.chunk = unit / tiles;
  int t = unit - u.chunk * tiles;
  const int G = 8;
  int group_size = G * p.tiles_n;
  int group = t / group_size;
  int first_m = group * G;
  int gsz = p.tiles_m - first_m < G ? p.tiles_m - first_m : G;
  int in_group = t - group * group_size;
  u.tm = first_m + in_group % gsz;
  u.tn = in_group / gsz;
  return u;
}

__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_i8_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb,
                   const GemmArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmb)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_addr(tmem_holder)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    int stage = 0;
    uint32_t phase = 0;
    for (int unit = blockIdx.x; unit < p.total_units; unit += gridDim.x) {
      UnitCoord u = decode_unit(unit, p);
      const ChunkDesc cd = p.chunks[u.chunk];
      for (int pr = 0; pr < cd.npairs; ++pr) {
        const int l = cd.l0 + pr;
        const int h = cd.d + 2 - l;
        for (int kb = 0; kb < p.kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], kStageBytes);
          tma_load_3d(sA + stage * kABytes, &tma, &full[stage], kb * kBlockK, u.tm * kBlockM, l - 1);
          tma_load_3d(sB + stage * kBBytes, &tmb, &full[stage], kb * kBlockK, u.tn * kBN, h - 1);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer (single thread) ----------------
    constexpr uint32_t idesc = idesc_i8<kBlockM, kBN>();
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int unit = blockIdx.x; unit < p.total_units; unit += gridDim.x, ++it) {
      UnitCoord u = decode_unit(unit, p);
      const ChunkDesc cd = p.chunks[u.chunk];
      const int acc = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      mbar_wait(&tempty[acc], aphase ^ 1);
      tc_fence_after();
      const uint32_t tmem_d = tmem_base + acc * kBN;
      const int total = cd.npairs * p.kblocks;
      for (int i = 0; i < total; ++i) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint64_t ad = sdesc_sw128(smem_addr(sA + stage * kABytes));
        const uint64_t bd = sdesc_sw128(smem_addr(sB + stage * kBBytes));
#pragma unroll
        for (int kk = 0; kk < kBlockK / 32; ++kk)
          tc_mma_i8(tmem_d, ad + 2 * kk, bd + 2 * kk, idesc, (i | kk) != 0);
        tc_commit(&empty[stage]);
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      tc_commit(&tfull[acc]);
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> int32 chunk plane ----------------
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    int it = 0;
    for (int unit = blockIdx.x; unit < p.total_units; unit += gridDim.x, ++it) {
      UnitCoord u = decode_unit(unit, p);
      const int acc = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const int row = u.tm * kBlockM + q * 32 + lane;
      int32_t* dst = p.planes + static_cast<int64_t>(u.chunk) * p.plane_stride +
                     static_cast<int64_t>(row) * p.ldp;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * kBN;
#pragma unroll 1
      for (int c0 = 0; c0 < kBN; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(taddr + c0, r);
        const int col0 = u.tn * kBN + c0;
        if (row < p.m) {
          if (col0 + 32 <= p.n && (p.ldp & 3) == 0) {
            int4* d4 = reinterpret_cast<int4*>(dst + col0);
#pragma unroll
            for (int v = 0; v < 8; ++v)
              d4[v] = make_int4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
          } else {
            for (int v = 0; v < 32; ++v)
              if (col0 + v < p.n) dst[col0 + v] = static_cast<int32_t>(r[v]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols)
                 : "memory");
  }
}

// ----------------------------------------------------------------------------
// Exact combine: V = sum_chunks S_c << shift_c as a W-word two's-complement
// integer, C = RN(V * 2^(qa_i + qb_j + w_last)) exactly as ExactValue::to_double.
// ----------------------------------------------------------------------------

template <int W>
__global__ void __launch_bounds__(256) combine_exact_kernel(const CombineArgs p) {
  const int64_t total = static_cast<int64_t>(p.m) * p.n;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx / p.n, j = idx - i * p.n;
    uint64_t v[W];
#pragma unroll
    for (int w = 0; w < W; ++w) v[w] = 0;
    const int32_t* src = p.planes + i * p.ldp + j;
    for (int c = 0; c < p.nchunks; ++c) {
      const int32_t s = __ldg(src + c * p.plane_stride);
      if (s != 0) words_add_shifted<W>(v, s, p.chunks[c].shift);
    }
    const long e = static_cast<long>(__ldg(p.qa + i)) + __ldg(p.qb + j) + p.w_last;
    double r = round_words<W>(v, e);
    if (p.axpby)  // two roundings, no FMA contraction (scheme.cpp:369-370)
      r = __dadd_rn(__dmul_rn(p.alpha, r), __dmul_rn(p.beta, p.cin[i * p.ldcin + j]));
    p.c[i * p.ldc + j] = r;
  }
}

// Sequential FP64 accumulation in the reference order (d ascending, l
// ascending) with the TwoSum inexact counter (scheme.cpp:173-215).
__global__ void __launch_bounds__(256) combine_sequential_kernel(const CombineArgs p) {
  const int64_t total = static_cast<int64_t>(p.m) * p.n;
  int local_max = 0;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx / p.n, j = idx - i * p.n;
    const int32_t* src = p.planes + i * p.ldp + j;
    const long qe = static_cast<long>(__ldg(p.qa + i)) + __ldg(p.qb + j);
    double acc = 0.0;
    int inexact = 0;
    long long pending = 0;  // integer chain of one reference chunk
    for (int c = 0; c < p.nchunks; ++c) {
      pending += __ldg(src + c * p.plane_stride);
      const ChunkDesc cd = p.chunks[c];
      if (!cd.flush) continue;
      const long long s = pending;
      pending = 0;
      const long wexp = -static_cast<long>(cd.d + 2) * p.width + (p.mode == 1 ? 2 : 0);
      double term = s != 0 ? ldexp_rn(__ll2double_rn(s), qe + wexp) : 0.0;
      double sum = __dadd_rn(acc, term);
      double bp = __dsub_rn(sum, acc);
      double err = __dadd_rn(__dsub_rn(acc, __dsub_rn(sum, bp)), __dsub_rn(term, bp));
      inexact += err != 0.0;
      acc = sum;
    }
    local_max = inexact > local_max ? inexact : local_max;
    double r = acc;
    if (p.axpby)  // two roundings, no FMA contraction (scheme.cpp:369-370)
      r = __dadd_rn(__dmul_rn(p.alpha, r), __dmul_rn(p.beta, p.cin[i * p.ldcin + j]));
    p.c[i * p.ldc + j] = r;
  }
  if (local_max) atomicMax(p.realized_psi, local_max);
}

// ----------------------------------------------------------------------------
// kappa profile (analysis.cpp:25-47): per-row / per-column max and min
// nonzero magnitude.
// ----------------------------------------------------------------------------

__global__ void __launch_bounds__(256) row_profile_kernel(const double* __restrict__ a,
                                                          int64_t lda, int64_t m, int64_t k,
                                                          double* __restrict__ ratios,
                                                          int* __restrict__ zero_flag) {
  __shared__ unsigned long long rmax[8], rmin[8];
  for (int64_t row = blockIdx.x; row < m; row += gridDim.x) {
    unsigned long long mx = 0, mn = ~0ULL;
    for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
      unsigned long long b = abs_bits(__ldg(a + row * lda + j));
      if (b) {
        mx = b > mx ? b : mx;
        mn = b < mn ? b : mn;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      unsigned long long t = __shfl_xor_sync(0xFFFFFFFFu, mx, o);
      unsigned long long u = __shfl_xor_sync(0xFFFFFFFFu, mn, o);
      mx = t > mx ? t : mx;
      mn = u < mn ? u : mn;
    }
    if ((threadIdx.x & 31) == 0) {
      rmax[threadIdx.x >> 5] = mx;
      rmin[threadIdx.x >> 5] = mn;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
        mx = rmax[w] > mx ? rmax[w] : mx;
        mn = rmin[w] < mn ? rmin[w] : mn;
      }
      if (mx == 0) {
        ratios[row] = 1.0;
        *zero_flag = 1;
      } else {
        ratios[row] = __ddiv_rn(__longlong_as_double(static_cast<long long>(mx)),
                                __longlong_as_double(static_cast<long long>(mn)));
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) col_profile_kernel(const double* __restrict__ b,
                                                          int64_t ldb, int64_t k, int64_t n,
                                                          int64_t rows_per,
                                                          unsigned long long* __restrict__ colmax,
                                                          unsigned long long* __restrict__ colmin) {
  int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  int64_t r0 = static_cast<int64_t>(blockIdx.y) * rows_per;
  int64_t r1 = r0 + rows_per < k ? r0 + rows_per : k;
  unsigned long long mx = 0, mn = ~0ULL;
  for (int64_t r = r0; r < r1; ++r) {
    unsigned long long t = abs_bits(__ldg(b + r * ldb + j));
    if (t) {
      mx = t > mx ? t : mx;
      mn = t < mn ? t : mn;
    }
  }
  if (mx) atomicMax(colmax + j, mx);
  if (mn != ~0ULL) atomicMin(colmin + j, mn);
}

// ----------------------------------------------------------------------------
// integer_gemm debug hook helpers (mma_sim.cpp:76-125)
// ----------------------------------------------------------------------------

// int64 (rows x cols) -> int8 K-major rows of length kp: transpose=0 keeps
// rows (X, m x k -> [m][kp]); transpose=1 emits columns (Y, k x n -> [n][kp]).
__global__ void pack_i8_kernel(const int64_t* __restrict__ x, int64_t rows, int64_t cols,
                               int transpose, int64_t kp, int8_t* __restrict__ out) {
  const int64_t outer = transpose ? cols : rows;
  const int64_t total = outer * kp;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t o = idx / kp, kk = idx - o * kp;
    int64_t inner = transpose ? rows : cols;
    int8_t v = 0;
    if (kk < inner) v = static_cast<int8_t>(transpose ? x[kk * cols + o] : x[o * cols + kk]);
    out[idx] = v;
  }
}

// Exact CUDA-core integer GEMM with the reference's per-MAC range check
// (mma_sim.cpp:103-112); records the first overflowing (row-major) element.
__global__ void integer_gemm_exact_kernel(const int64_t* __restrict__ x,
                                          const int64_t* __restrict__ y,
                                          const int64_t* __restrict__ c, int64_t* __restrict__ out,
                                          int64_t m, int64_t k, int64_t n, int acc_width,
                                          unsigned long long* first_overflow) {
  const int64_t total = m * n;
  const __int128 lo = -(static_cast<__int128>(1) << acc_width);
  const __int128 hi = (static_cast<__int128>(1) << acc_width) - 1;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t i = idx / n, j = idx - i * n;
    __int128 acc = c ? c[idx] : 0;
    bool ovf = false;
    for (int64_t r = 0; r < k; ++r) {
      acc += static_cast<__int128>(x[i * k + r]) * y[r * n + j];
      if (acc < lo || acc > hi) {
        ovf = true;
        break;
      }
    }
    if (ovf)
      atomicMin(first_overflow, static_cast<unsigned long long>(idx));
    else
      out[idx] = static_cast<int64_t>(acc);
  }
}

__global__ void plane_to_i64_kernel(const int32_t* __restrict__ plane, int64_t ldp,
                                    const int64_t* __restrict__ c, int64_t* __restrict__ out,
                                    int64_t m, int64_t n) {
  const int64_t total = m * n;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t i = idx / n, j = idx - i * n;
    out[idx] = static_cast<int64_t>(plane[i * ldp + j]) + (c ? c[idx] : 0);
  }
}

// ----------------------------------------------------------------------------
// Launchers
// ----------------------------------------------------------------------------

static inline int grid_for(int64_t work, int per_block, int cap = 148 * 16) {
  int64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  return static_cast<int>(g < cap ? g : cap);
}

cudaError_t launch_slice_rows(const double* a, int64_t lda, int64_t m, int64_t k, int64_t kp,
                              int width, int count, int mode, void* out, int out_is_i64,
                              int* scales, int* status, cudaStream_t st, int64_t* launches) {
  if (m == 0) return cudaSuccess;
  int grid = static_cast<int>(m < 148 * 32 ? m : 148 * 32);
  if (out_is_i64)
    slice_rows_kernel<long long><<<grid, 256, 0, st>>>(a, lda, m, k, kp, width, count, mode,
                                                       static_cast<long long*>(out), scales,
                                                       status);
  else
    slice_rows_kernel<int8_t><<<grid, 256, 0, st>>>(a, lda, m, k, kp, width, count, mode,
                                                    static_cast<int8_t*>(out), scales, status);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_slice_cols(const double* b, int64_t ldb, int64_t k, int64_t n, int64_t kp,
                              int width, int count, int mode, void* out, int out_is_i64,
                              int* scales, unsigned long long* colmax, int* status,
                              cudaStream_t st, int64_t* launches) {
  if (n == 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(colmax, 0, sizeof(unsigned long long) * n, st);
  if (e != cudaSuccess) return e;
  {
    int64_t col_blocks = (n + 255) / 256;
    int64_t splits = (148 * 8 + col_blocks - 1) / col_blocks;
    if (splits > k) splits = k > 0 ? k : 1;
    if (splits > 65535) splits = 65535;
    int64_t rows_per = k > 0 ? (k + splits - 1) / splits : 0;
    dim3 grid(static_cast<unsigned>(col_blocks), static_cast<unsigned>(splits));
    colmax_kernel<<<grid, 256, 0, st>>>(b, ldb, k, n, rows_per, colmax, status);
    ++*launches;
  }
  dim3 grid2(static_cast<unsigned>((kp + 63) / 64), static_cast<unsigned>((n + 63) / 64));
  if (out_is_i64)
    slice_cols_kernel<long long><<<grid2, 256, 0, st>>>(b, ldb, k, n, kp, width, count, mode,
                                                        colmax, static_cast<long long*>(out),
                                                        scales);
  else
    slice_cols_kernel<int8_t><<<grid2, 256, 0, st>>>(b, ldb, k, n, kp, width, count, mode,
                                                     colmax, static_cast<int8_t*>(out), scales);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_gemm_i8(const CUtensorMap* tma, const CUtensorMap* tmb, const GemmArgs& args,
                           int num_sms, cudaStream_t st, int64_t* launches) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(gemm_i8_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  int grid = args.total_units < num_sms ? args.total_units : num_sms;
  if (grid < 1) return cudaSuccess;
  gemm_i8_kernel<<<grid, kGemmThreads, kSmemBytes, st>>>(*tma, *tmb, args);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_combine_exact(const CombineArgs& args, int words, cudaStream_t st,
                                 int64_t* launches) {
  int64_t total = static_cast<int64_t>(args.m) * args.n;
  if (total == 0) return cudaSuccess;
  int grid = grid_for(total, 256);
  switch (words) {
    case 2: combine_exact_kernel<2><<<grid, 256, 0, st>>>(args); break;
    case 3: combine_exact_kernel<3><<<grid, 256, 0, st>>>(args); break;
    case 4: combine_exact_kernel<4><<<grid, 256, 0, st>>>(args); break;
    case 6: combine_exact_kernel<6><<<grid, 256, 0, st>>>(args); break;
    case 8: combine_exact_kernel<8><<<grid, 256, 0, st>>>(args); break;
    case 12: combine_exact_kernel<12><<<grid, 256, 0, st>>>(args); break;
    case 16: combine_exact_kernel<16><<<grid, 256, 0, st>>>(args); break;
    default: return cudaErrorInvalidValue;
  }
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_combine_sequential(const CombineArgs& args, cudaStream_t st,
                                      int64_t* launches) {
  int64_t total = static_cast<int64_t>(args.m) * args.n;
  if (total == 0) return cudaSuccess;
  combine_sequential_kernel<<<grid_for(total, 256), 256, 0, st>>>(args);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_row_profile(const double* a, int64_t lda, int64_t m, int64_t k,
                               double* ratios, int* zero_flag, cudaStream_t st,
                               int64_t* launches) {
  if (m == 0) return cudaSuccess;
  int grid = static_cast<int>(m < 148 * 32 ? m : 148 * 32);
  row_profile_kernel<<<grid, 256, 0, st>>>(a, lda, m, k, ratios, zero_flag);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_col_profile(const double* b, int64_t ldb, int64_t k, int64_t n,
                               unsigned long long* colmax, unsigned long long* colmin,
                               cudaStream_t st, int64_t* launches) {
  if (n == 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(colmax, 0, sizeof(unsigned long long) * n, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(colmin, 0xFF, sizeof(unsigned long long) * n, st);
  if (e != cudaSuccess) return e;
  int64_t col_blocks = (n + 255) / 256;
  int64_t splits = (148 * 8 + col_blocks - 1) / col_blocks;
  if (splits > k) splits = k > 0 ? k : 1;
  if (splits > 65535) splits = 65535;
  int64_t rows_per = k > 0 ? (k + splits - 1) / splits : 0;
  dim3 grid(static_cast<unsigned>(col_blocks), static_cast<unsigned>(splits));
  col_profile_kernel<<<grid, 256, 0, st>>>(b, ldb, k, n, rows_per, colmax, colmin);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_pack_i8(const int64_t* x, int64_t rows, int64_t cols, int transpose,
                           int64_t kp, int8_t* out, cudaStream_t st, int64_t* launches) {
  int64_t total = (transpose ? cols : rows) * kp;
  if (total == 0) return cudaSuccess;
  pack_i8_kernel<<<grid_for(total, 256), 256, 0, st>>>(x, rows, cols, transpose, kp, out);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_integer_gemm_exact(const int64_t* x, const int64_t* y, const int64_t* c,
                                      int64_t* out, int64_t m, int64_t k, int64_t n,
                                      int acc_width, unsigned long long* first_overflow,
                                      cudaStream_t st, int64_t* launches) {
  if (m * n == 0) return cudaSuccess;
  integer_gemm_exact_kernel<<<grid_for(m * n, 128), 128, 0, st>>>(x, y, c, out, m, k, n,
                                                                  acc_width, first_overflow);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_plane_to_i64(const int32_t* plane, int64_t ldp, const int64_t* c,
                                int64_t* out, int64_t m, int64_t n, cudaStream_t st,
                                int64_t* launches) {
  if (m * n == 0) return cudaSuccess;
  plane_to_i64_kernel<<<grid_for(m * n, 256), 256, 0, st>>>(plane, ldp, c, out, m, n);
  ++*launches;
  return cudaGetLastError();
}

}  // namespace ozgpu
