// Combine, kappa-profile and integer_gemm helper kernels of the B200-native
// Ozaki-I FP64 GEMM (scheme.cpp:267-355, analysis.cpp:25-68, mma_sim.cpp:76-125).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>
#include <cstdlib>
#include <string>

#include "ozgpu_internal.h"
#include "ozgpu_numeric.h"

namespace ozgpu {

__device__ __forceinline__ unsigned long long abs_bits_m(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x)) & 0x7FFFFFFFFFFFFFFFULL;
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

// Vectorised exact combine: 4 consecutive columns per thread (int4 plane
// loads, chunk loads issued ahead of the multi-word adds), chunk shifts in
// the parameter space.  Used when n % 4 == 0 and nchunks <= 64.
struct ShiftTable {
  int shift[64];
};

template <int W>
__global__ void __launch_bounds__(256) combine_exact_v4_kernel(const CombineArgs p,
                                                               const ShiftTable sh) {
  const int64_t groups_per_row = p.n / 4;
  const int64_t total = static_cast<int64_t>(p.m) * groups_per_row;
  const bool vec_c = (p.ldc & 1) == 0 && (reinterpret_cast<uintptr_t>(p.c) & 15) == 0;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx / groups_per_row, j = (idx - i * groups_per_row) * 4;
    uint64_t v[4][W];
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
      for (int w = 0; w < W; ++w) v[e][w] = 0;
    const int4* src = reinterpret_cast<const int4*>(p.planes + i * p.ldp + j);
    const int64_t stride4 = p.plane_stride / 4;
    int c = 0;
    for (; c + 4 <= p.nchunks; c += 4) {
      int4 s[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) s[u] = __ldcs(src + (c + u) * stride4);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int shf = sh.shift[c + u];
        words_add_shifted<W>(v[0], s[u].x, shf);
        words_add_shifted<W>(v[1], s[u].y, shf);
        words_add_shifted<W>(v[2], s[u].z, shf);
        words_add_shifted<W>(v[3], s[u].w, shf);
      }
    }
    for (; c < p.nchunks; ++c) {
      const int4 s = __ldcs(src + c * stride4);
      const int shf = sh.shift[c];
      words_add_shifted<W>(v[0], s.x, shf);
      words_add_shifted<W>(v[1], s.y, shf);
      words_add_shifted<W>(v[2], s.z, shf);
      words_add_shifted<W>(v[3], s.w, shf);
    }
    const long qi = static_cast<long>(__ldg(p.qa + i)) + p.w_last;
    const int4 qb = __ldg(reinterpret_cast<const int4*>(p.qb + j));
    double r[4];
    r[0] = round_words<W>(v[0], qi + qb.x);
    r[1] = round_words<W>(v[1], qi + qb.y);
    r[2] = round_words<W>(v[2], qi + qb.z);
    r[3] = round_words<W>(v[3], qi + qb.w);
    if (p.axpby) {  // two roundings, no FMA contraction (scheme.cpp:369-370)
#pragma unroll
      for (int e = 0; e < 4; ++e)
        r[e] = __dadd_rn(__dmul_rn(p.alpha, r[e]), __dmul_rn(p.beta, p.cin[i * p.ldcin + j + e]));
    }
    double* dst = p.c + i * p.ldc + j;
    if (vec_c) {
      __stcs(reinterpret_cast<double2*>(dst), make_double2(r[0], r[1]));
      __stcs(reinterpret_cast<double2*>(dst) + 1, make_double2(r[2], r[3]));
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) dst[e] = r[e];
    }
  }
}

// Horner form of the exact combine for values that fit 127 bits:
// V = (...((S_0 << t) + S_1) << t ...) + S_{D-1}, with S_d the int64 sum of
// diagonal d's chunk planes (chunks are stored diagonal-major).  One 128-bit
// shift-add per diagonal instead of a multi-word add per chunk.
struct DiagTable {
  int first_chunk[65];  // chunks of diagonal d: [first_chunk[d], first_chunk[d + 1])
};

__global__ void __launch_bounds__(256) combine_horner_v4_kernel(const CombineArgs p,
                                                                const DiagTable dt) {
  const int64_t groups_per_row = p.n / 4;
  const int64_t total = static_cast<int64_t>(p.m) * groups_per_row;
  const bool vec_c = (p.ldc & 1) == 0 && (reinterpret_cast<uintptr_t>(p.c) & 15) == 0;
  const int64_t stride4 = p.plane_stride / 4;
  const int t = p.width;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx / groups_per_row, j = (idx - i * groups_per_row) * 4;
    const int4* src = reinterpret_cast<const int4*>(p.planes + i * p.ldp + j);
    unsigned __int128 v0 = 0, v1 = 0, v2 = 0, v3 = 0;
    // Diagonals in runs of p.hgroup: a run is Horner-summed in int64 (the
    // multiply-by-2^t runs on the FMA pipe; the host sizes the run so it
    // cannot overflow), then folded into the 128-bit value with one shift-add.
    const long long radix = 1LL << t;
    for (int d0 = 0; d0 < p.diagonals; d0 += p.hgroup) {
      const int d1 = min(p.diagonals, d0 + p.hgroup);
      long long a0 = 0, a1 = 0, a2 = 0, a3 = 0;
      for (int d = d0; d < d1; ++d) {
        long long s0 = 0, s1 = 0, s2 = 0, s3 = 0;
        for (int c = dt.first_chunk[d]; c < dt.first_chunk[d + 1]; ++c) {
          const int4 s = __ldcs(src + c * stride4);
          s0 += s.x;
          s1 += s.y;
          s2 += s.z;
          s3 += s.w;
        }
        a0 = a0 * radix + s0;
        a1 = a1 * radix + s1;
        a2 = a2 * radix + s2;
        a3 = a3 * radix + s3;
      }
      const int sh = t * (d1 - d0);
      v0 = (v0 << sh) + static_cast<unsigned __int128>(static_cast<__int128>(a0));
      v1 = (v1 << sh) + static_cast<unsigned __int128>(static_cast<__int128>(a1));
      v2 = (v2 << sh) + static_cast<unsigned __int128>(static_cast<__int128>(a2));
      v3 = (v3 << sh) + static_cast<unsigned __int128>(static_cast<__int128>(a3));
    }
    const long qi = static_cast<long>(__ldg(p.qa + i)) + p.w_last;
    const int4 qb = __ldg(reinterpret_cast<const int4*>(p.qb + j));
    double r[4];
    r[0] = round_i128(v0, qi + qb.x);
    r[1] = round_i128(v1, qi + qb.y);
    r[2] = round_i128(v2, qi + qb.z);
    r[3] = round_i128(v3, qi + qb.w);
    if (p.axpby) {  // two roundings, no FMA contraction (scheme.cpp:369-370)
#pragma unroll
      for (int e = 0; e < 4; ++e)
        r[e] = __dadd_rn(__dmul_rn(p.alpha, r[e]), __dmul_rn(p.beta, p.cin[i * p.ldcin + j + e]));
    }
    double* dst = p.c + i * p.ldc + j;
    if (vec_c) {
      __stcs(reinterpret_cast<double2*>(dst), make_double2(r[0], r[1]));
      __stcs(reinterpret_cast<double2*>(dst) + 1, make_double2(r[2], r[3]));
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) dst[e] = r[e];
    }
  }
}

// Straight-line variant of the Horner combine: the chunk loads of a batch of
// 16 are all issued before any arithmetic (static register indexing), and a
// host-built program says per chunk whether it opens a new diagonal
// (int64 run *= 2^t) or closes a run (fold into 128 bits, shift given).
struct HornerProgram {
  int flags[64];       // bit0: opens a new diagonal, bit1: fold the run first
  int fold_shift[64];  // bits to shift the 128-bit value by when folding
  int final_shift;     // fold of the last run
};

__global__ void __launch_bounds__(256) combine_horner2_v4_kernel(const CombineArgs p,
                                                                 const HornerProgram hp) {
  const int64_t groups_per_row = p.n / 4;
  const int64_t total = static_cast<int64_t>(p.m) * groups_per_row;
  const bool vec_c = (p.ldc & 1) == 0 && (reinterpret_cast<uintptr_t>(p.c) & 15) == 0;
  const int64_t stride4 = p.plane_stride / 4;
  const long long radix = 1LL << p.width;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx / groups_per_row, j = (idx - i * groups_per_row) * 4;
    const int4* src = reinterpret_cast<const int4*>(p.planes + i * p.ldp + j);
    unsigned __int128 v0 = 0, v1 = 0, v2 = 0, v3 = 0;
    long long a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    for (int cb = 0; cb < p.nchunks; cb += 16) {
      int4 s[16];
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (cb + u < p.nchunks) s[u] = __ldcs(src + (cb + u) * stride4);
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int c = cb + u;
        if (c < p.nchunks) {
          const int f = hp.flags[c];
          if (f & 2) {
            const int sh = hp.fold_shift[c];
            v0 = (v0 << sh) + static_cast<unsigned __int128>(static_cast<__int128>(a0));
            v1 = (v1 << sh) + static_cast<unsigned __int128>(static_cast<__int128>(a1));
            v2 = (v2 << sh) + static_cast<unsigned __int128>(static_cast<__int128>(a2));
            v3 = (v3 << sh) + static_cast<unsigned __int128>(static_cast<__int128>(a3));
            a0 = a1 = a2 = a3 = 0;
          } else if (f & 1) {
            a0 *= radix;
            a1 *= radix;
            a2 *= radix;
            a3 *= radix;
          }
          a0 += s[u].x;
          a1 += s[u].y;
          a2 += s[u].z;
          a3 += s[u].w;
        }
      }
    }
    const int sh = hp.final_shift;
    v0 = (v0 << sh) + static_cast<unsigned __int128>(static_cast<__int128>(a0));
    v1 = (v1 << sh) + static_cast<unsigned __int128>(static_cast<__int128>(a1));
    v2 = (v2 << sh) + static_cast<unsigned __int128>(static_cast<__int128>(a2));
    v3 = (v3 << sh) + static_cast<unsigned __int128>(static_cast<__int128>(a3));
    const long qi = static_cast<long>(__ldg(p.qa + i)) + p.w_last;
    const int4 qb = __ldg(reinterpret_cast<const int4*>(p.qb + j));
    double r[4];
    r[0] = round_i128(v0, qi + qb.x);
    r[1] = round_i128(v1, qi + qb.y);
    r[2] = round_i128(v2, qi + qb.z);
    r[3] = round_i128(v3, qi + qb.w);
    if (p.axpby) {  // two roundings, no FMA contraction (scheme.cpp:369-370)
#pragma unroll
      for (int e = 0; e < 4; ++e)
        r[e] = __dadd_rn(__dmul_rn(p.alpha, r[e]), __dmul_rn(p.beta, p.cin[i * p.ldcin + j + e]));
    }
    double* dst = p.c + i * p.ldc + j;
    if (vec_c) {
      __stcs(reinterpret_cast<double2*>(dst), make_double2(r[0], r[1]));
      __stcs(reinterpret_cast<double2*>(dst) + 1, make_double2(r[2], r[3]));
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) dst[e] = r[e];
    }
  }
}

// Exact combine, Horner form with the arithmetic split across pipes:
// diagonals are accumulated in int64 runs, a = a * 2^(t gap) + S_c, as two
// integer multiply-adds on the FMA pipe (mad.wide.u32 + mad.lo.u32, the
// chunk value as the 64-bit addend), and a run is folded into the 128-bit
// (hi, lo) value with a funnel shift and a carry-chained add on the ALU only
// every few diagonals; the final rounding (round_hilo) is two exact
// conversions and one FMA on the FP64 pipe.  A host-built program gives, per
// chunk (diagonal-major order), the fold and multiply shifts (uniform
// branches).  The integer pipe was the limiter of the plain 128-bit Horner.
struct HiloProgram {
  int fold_shift[64];  // > 0: before chunk c, V = (V << (fold_shift - 1)) + a, a = 0
  int mul_shift[64];   // a = a * 2^mul_shift + S_c
  int end_shift;       // after the last chunk: V = (V << end_shift) + a
  int final_shift;     // then V <<= final_shift (empty trailing diagonals)
};

// W-word (W = 2, 3) little-endian two's-complement value: v <<= sh (0 < sh < 64)
template <int W>
__device__ __forceinline__ void words_shift(uint64_t (&v)[W], int sh) {
#pragma unroll
  for (int i = W - 1; i > 0; --i) v[i] = (v[i] << sh) | (v[i - 1] >> (64 - sh));
  v[0] <<= sh;
}
// v += a (sign-extended), one carry chain
template <int W>
__device__ __forceinline__ void words_add64(uint64_t (&v)[W], int64_t a) {
  const uint64_t ext = static_cast<uint64_t>(a >> 63);
  if constexpr (W == 2) {
    asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;"
        : "+l"(v[0]), "+l"(v[1])
        : "l"(static_cast<uint64_t>(a)), "l"(ext));
  } else {
    asm("add.cc.u64 %0, %0, %3;\n\taddc.cc.u64 %1, %1, %4;\n\taddc.u64 %2, %2, %4;"
        : "+l"(v[0]), "+l"(v[1]), "+l"(v[2])
        : "l"(static_cast<uint64_t>(a)), "l"(ext));
  }
}
// a * r + s (r < 2^32) on the FMA pipe
__device__ __forceinline__ int64_t mad_run(int64_t a, uint32_t r, int32_t s) {
  uint64_t res;
  asm("{\n\t.reg .u32 alo, ahi, shi, rlo, rhi;\n\t"
      "mov.b64 {alo, ahi}, %1;\n\t"
      "shr.s32 shi, %3, 31;\n\t"
      "mov.b64 %0, {%3, shi};\n\t"
      "mad.wide.u32 %0, alo, %2, %0;\n\t"
      "mov.b64 {rlo, rhi}, %0;\n\t"
      "mad.lo.u32 rhi, ahi, %2, rhi;\n\t"
      "mov.b64 %0, {rlo, rhi};\n\t}"
      : "=l"(res)
      : "l"(a), "r"(r), "r"(s));
  return static_cast<int64_t>(res);
}

template <int BATCH, int MINB, int W>
__global__ void __launch_bounds__(256, MINB) combine_hilo_v4_kernel(const CombineArgs p,
                                                                    const HiloProgram hp) {
  // 2-D grid: x covers a row's 4-column groups, y strides over rows (no
  // per-element index division)
  const int groups_per_row = p.n / 4;
  const bool vec_c = (p.ldc & 1) == 0 && (reinterpret_cast<uintptr_t>(p.c) & 15) == 0;
  const int64_t stride4 = p.plane_stride / 4;
  const int jg = blockIdx.x * blockDim.x + threadIdx.x;
  if (jg >= groups_per_row) return;
  for (int64_t i = blockIdx.y; i < p.m; i += gridDim.y) {
    const int64_t j = static_cast<int64_t>(jg) * 4;
    const int4* src = reinterpret_cast<const int4*>(p.planes + i * p.ldp + j);
    uint64_t v[4][W];
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
      for (int w = 0; w < W; ++w) v[e][w] = 0;
    int64_t a[4] = {0, 0, 0, 0};
    for (int cb = 0; cb < p.nchunks; cb += BATCH) {
      int4 s[BATCH];
#pragma unroll
      for (int u = 0; u < BATCH; ++u)
        if (cb + u < p.nchunks) s[u] = __ldcs(src + (cb + u) * stride4);
#pragma unroll
      for (int u = 0; u < BATCH; ++u) {
        if (cb + u < p.nchunks) {
          const int fs = hp.fold_shift[cb + u];
          if (fs) {  // uniform branch
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              if (fs > 1) words_shift<W>(v[e], fs - 1);
              words_add64<W>(v[e], a[e]);
              a[e] = 0;
            }
          }
          const uint32_t r = 1u << hp.mul_shift[cb + u];
          a[0] = mad_run(a[0], r, s[u].x);
          a[1] = mad_run(a[1], r, s[u].y);
          a[2] = mad_run(a[2], r, s[u].z);
          a[3] = mad_run(a[3], r, s[u].w);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (hp.end_shift) words_shift<W>(v[e], hp.end_shift);
      words_add64<W>(v[e], a[e]);
      if (hp.final_shift) words_shift<W>(v[e], hp.final_shift);
    }
    const long qi = static_cast<long>(__ldg(p.qa + i)) + p.w_last;
    const int4 qb = __ldg(reinterpret_cast<const int4*>(p.qb + j));
    const long qe[4] = {qi + qb.x, qi + qb.y, qi + qb.z, qi + qb.w};
    double r[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if constexpr (W == 2)
        r[e] = round_hilo(v[e][1], v[e][0], qe[e]);
      else
        r[e] = round_w3(v[e][2], v[e][1], v[e][0], qe[e]);
    }
    if (p.axpby) {  // two roundings, no FMA contraction (scheme.cpp:369-370)
#pragma unroll
      for (int e = 0; e < 4; ++e)
        r[e] = __dadd_rn(__dmul_rn(p.alpha, r[e]), __dmul_rn(p.beta, p.cin[i * p.ldcin + j + e]));
    }
    double* dst = p.c + i * p.ldc + j;
    if (vec_c) {
      __stcs(reinterpret_cast<double2*>(dst), make_double2(r[0], r[1]));
      __stcs(reinterpret_cast<double2*>(dst) + 1, make_double2(r[2], r[3]));
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) dst[e] = r[e];
    }
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

// abs_product / gemm_reference (matrix.cpp:31-54): out(i,j) = sum_r op(a_ir)
// op(b_rj) with r ascending, zero a_ir skipped, a separate multiply and add
// rounding per term (the reference's loop, no FMA contraction).  Each output
// keeps that exact sequence; the parallelism is across outputs: 64 x 64
// output tiles per CTA (4 x 4 per thread) with 16-deep K slabs of A and B
// staged in shared memory, so A and B are read from DRAM once per tile row /
// column instead of once per output.
template <bool ABS>
__global__ void __launch_bounds__(256) fp64_gemm_tiled_kernel(int64_t m, int64_t k, int64_t n,
                                                              const double* __restrict__ a,
                                                              int64_t lda,
                                                              const double* __restrict__ b,
                                                              int64_t ldb, double* __restrict__ out,
                                                              int64_t ldo) {
  constexpr int TM = 64, TN = 64, TK = 16;
  __shared__ __align__(16) double As[TK][TM + 2];  // As[r][i]
  __shared__ __align__(16) double Bs[TK][TN];      // Bs[r][j]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t i0 = static_cast<int64_t>(blockIdx.y) * TM, j0 = static_cast<int64_t>(blockIdx.x) * TN;
  double acc[4][4];
#pragma unroll
  for (int ii = 0; ii < 4; ++ii)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) acc[ii][jj] = 0.0;
  for (int64_t r0 = 0; r0 < k; r0 += TK) {
#pragma unroll
    for (int q = 0; q < (TM * TK) / 256; ++q) {
      const int e = tid + 256 * q, ii = e / TK, rr = e % TK;
      const int64_t gi = i0 + ii, gr = r0 + rr;
      const double v = (gi < m && gr < k) ? __ldg(a + gi * lda + gr) : 0.0;
      As[rr][ii] = ABS ? fabs(v) : v;
    }
#pragma unroll
    for (int q = 0; q < (TK * TN) / 256; ++q) {
      const int e = tid + 256 * q, rr = e / TN, jj = e % TN;
      const int64_t gr = r0 + rr, gj = j0 + jj;
      const double v = (gr < k && gj < n) ? __ldg(b + gr * ldb + gj) : 0.0;
      Bs[rr][jj] = ABS ? fabs(v) : v;
    }
    __syncthreads();
    const int kk = k - r0 < TK ? static_cast<int>(k - r0) : TK;
    for (int rr = 0; rr < kk; ++rr) {
      double av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        av[u] = As[rr][ty * 4 + u];
        bv[u] = Bs[rr][tx * 4 + u];
      }
#pragma unroll
      for (int ii = 0; ii < 4; ++ii) {
        if (av[ii] == 0.0) continue;  // matrix.cpp:36-37
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc[ii][jj] = __dadd_rn(acc[ii][jj], __dmul_rn(av[ii], bv[jj]));
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int ii = 0; ii < 4; ++ii) {
    const int64_t gi = i0 + ty * 4 + ii;
    if (gi >= m) continue;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int64_t gj = j0 + tx * 4 + jj;
      if (gj < n) out[gi * ldo + gj] = acc[ii][jj];
    }
  }
}

cudaError_t launch_fp64_gemm(int absolute, int64_t m, int64_t k, int64_t n, const double* a,
                             int64_t lda, const double* b, int64_t ldb, double* out, int64_t ldo,
                             cudaStream_t st, int64_t* launches) {
  if (m * n == 0) return cudaSuccess;
  if ((m + 63) / 64 > 65535) return cudaErrorInvalidValue;
  dim3 grid(static_cast<unsigned>((n + 63) / 64), static_cast<unsigned>((m + 63) / 64));
  if (k == 0) return cudaMemset2DAsync(out, ldo * sizeof(double), 0, n * sizeof(double), m, st);
  if (absolute)
    fp64_gemm_tiled_kernel<true><<<grid, 256, 0, st>>>(m, k, n, a, lda, b, ldb, out, ldo);
  else
    fp64_gemm_tiled_kernel<false><<<grid, 256, 0, st>>>(m, k, n, a, lda, b, ldb, out, ldo);
  ++*launches;
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------
// min_exact_slices (slicing.cpp:212-249): the deepest fraction bit position
// holding a set bit, lsb_pos = q + 52 - e - ctz(significand), over every
// block (row / column) with q = ilogb(max |x|) + 1 of its block.
// ----------------------------------------------------------------------------

__device__ __forceinline__ int deepest_bit(double v, int q) {
  const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(v)) & 0x7FFFFFFFFFFFFFFFULL;
  if (bits == 0) return 0;
  const uint64_t biased = bits >> 52, frac = bits & 0xFFFFFFFFFFFFFULL;
  const uint64_t sig = biased ? (frac | 0x10000000000000ULL) : frac;
  const int ex = biased ? static_cast<int>(biased) - 1023 : -1022;
  return q + 52 - ex - (__ffsll(static_cast<long long>(sig)) - 1);
}

__device__ __forceinline__ int q_of_maxbits(unsigned long long mb) {
  if (mb == 0) return 0;
  const int be = static_cast<int>(mb >> 52);
  if (be > 0) return be - 1023 + 1;
  return (63 - __clzll(static_cast<long long>(mb))) - 1074 + 1;
}

// one warp per row: max, then the deepest set bit against the row's q
__global__ void __launch_bounds__(256) exact_bits_rows_kernel(const double* __restrict__ a,
                                                              int64_t lda, int64_t m, int64_t k,
                                                              int* __restrict__ bits_out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  int deepest = 0;
  for (int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
       row < m; row += warps) {
    unsigned long long mx = 0;
    for (int64_t j = lane; j < k; j += 32) {
      const unsigned long long t = abs_bits_m(__ldg(a + row * lda + j));
      mx = t > mx ? t : mx;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const unsigned long long t = __shfl_xor_sync(0xFFFFFFFFu, mx, o);
      mx = t > mx ? t : mx;
    }
    if (mx == 0) continue;
    const int q = q_of_maxbits(mx);
    for (int64_t j = lane; j < k; j += 32) deepest = max(deepest, deepest_bit(__ldg(a + row * lda + j), q));
  }
  deepest = __reduce_max_sync(0xFFFFFFFFu, deepest);
  if (lane == 0 && deepest > 0) atomicMax(bits_out, deepest);
}

// thread per column, the column max precomputed (colmax)
__global__ void __launch_bounds__(256) exact_bits_cols_kernel(
    const double* __restrict__ b, int64_t ldb, int64_t k, int64_t n,
    const unsigned long long* __restrict__ colmax, int* __restrict__ bits_out) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int deepest = 0;
  if (j < n && colmax[j] != 0) {
    const int q = q_of_maxbits(colmax[j]);
    for (int64_t r = blockIdx.y; r < k; r += gridDim.y) deepest = max(deepest, deepest_bit(__ldg(b + r * ldb + j), q));
  }
  deepest = __reduce_max_sync(0xFFFFFFFFu, deepest);
  if ((threadIdx.x & 31) == 0 && deepest > 0) atomicMax(bits_out, deepest);
}

__global__ void __launch_bounds__(256) colmax_plain_kernel(const double* __restrict__ b,
                                                           int64_t ldb, int64_t k, int64_t n,
                                                           unsigned long long* __restrict__ colmax) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  unsigned long long mx = 0;
  for (int64_t r = blockIdx.y; r < k; r += gridDim.y) {
    const unsigned long long t = abs_bits_m(__ldg(b + r * ldb + j));
    mx = t > mx ? t : mx;
  }
  if (mx) atomicMax(colmax + j, mx);
}

cudaError_t launch_exact_bits(int orientation, const double* x, int64_t ldx, int64_t rows,
                              int64_t cols, unsigned long long* colmax, int* bits_out,
                              cudaStream_t st, int64_t* launches) {
  cudaError_t e = cudaMemsetAsync(bits_out, 0, sizeof(int), st);
  if (e != cudaSuccess || rows == 0 || cols == 0) return e;
  if (orientation == 0) {
    const int64_t g = (rows + 7) / 8;
    exact_bits_rows_kernel<<<static_cast<int>(g < 148 * 16 ? g : 148 * 16), 256, 0, st>>>(
        x, ldx, rows, cols, bits_out);
    ++*launches;
  } else {
    e = cudaMemsetAsync(colmax, 0, sizeof(unsigned long long) * cols, st);
    if (e != cudaSuccess) return e;
    const int64_t gy = rows < 64 ? rows : 64;
    dim3 grid(static_cast<unsigned>((cols + 255) / 256), static_cast<unsigned>(gy));
    colmax_plain_kernel<<<grid, 256, 0, st>>>(x, ldx, rows, cols, colmax);
    exact_bits_cols_kernel<<<grid, 256, 0, st>>>(x, ldx, rows, cols, colmax, bits_out);
    *launches += 2;
  }
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------
// Error metrics (oracle.cpp:253-292) against a reference matrix r (RN of the
// exact product): the worst |c - r| / |r| (0 / 0 -> 0, x / 0 -> inf) and
// sum (c - r)^2 (r = null: sum c^2, for frobenius_norm, oracle.cpp:64-68).
// Deterministic: fixed grid, per-CTA partials summed in order by one CTA.
// ----------------------------------------------------------------------------

constexpr int kMetricCtas = 592;

__global__ void __launch_bounds__(256) metric_partials_kernel(const double* __restrict__ c,
                                                              int64_t ldc,
                                                              const double* __restrict__ r,
                                                              int64_t ldr, int64_t m, int64_t n,
                                                              double* __restrict__ part_sum,
                                                              double* __restrict__ part_max) {
  __shared__ double ssum[8], smax[8];
  double sum = 0.0, worst = 0.0;
  const int64_t total = m * n;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx / n, j = idx - i * n;
    const double cv = c[i * ldc + j];
    if (r) {
      const double rv = r[i * ldr + j];
      const double d = __dadd_rn(cv, -rv);
      sum = __dadd_rn(sum, __dmul_rn(d, d));
      double fe;
      if (rv == 0.0)
        fe = cv == 0.0 ? 0.0 : __longlong_as_double(0x7FF0000000000000LL);
      else
        fe = fabs(d) / fabs(rv);
      worst = fe > worst ? fe : worst;
    } else {
      sum = __dadd_rn(sum, __dmul_rn(cv, cv));
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sum = __dadd_rn(sum, __shfl_down_sync(0xFFFFFFFFu, sum, o));
    const double w = __shfl_down_sync(0xFFFFFFFFu, worst, o);
    worst = w > worst ? w : worst;
  }
  if ((threadIdx.x & 31) == 0) {
    ssum[threadIdx.x >> 5] = sum;
    smax[threadIdx.x >> 5] = worst;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0, w = 0.0;
    for (int q = 0; q < 8; ++q) {
      s = __dadd_rn(s, ssum[q]);
      w = smax[q] > w ? smax[q] : w;
    }
    part_sum[blockIdx.x] = s;
    part_max[blockIdx.x] = w;
  }
}

__global__ void metric_final_kernel(const double* __restrict__ part_sum,
                                    const double* __restrict__ part_max, int parts,
                                    double* __restrict__ out2) {
  if (threadIdx.x != 0) return;
  double s = 0.0, w = 0.0;
  for (int q = 0; q < parts; ++q) {
    s = __dadd_rn(s, part_sum[q]);
    w = part_max[q] > w ? part_max[q] : w;
  }
  out2[0] = w;
  out2[1] = s;
}

int metric_scratch_doubles() { return 2 * kMetricCtas + 2; }

cudaError_t launch_error_metrics(const double* c, int64_t ldc, const double* r, int64_t ldr,
                                 int64_t m, int64_t n, double* scratch, cudaStream_t st,
                                 int64_t* launches) {
  metric_partials_kernel<<<kMetricCtas, 256, 0, st>>>(c, ldc, r, ldr, m, n, scratch,
                                                      scratch + kMetricCtas);
  metric_final_kernel<<<1, 32, 0, st>>>(scratch, scratch + kMetricCtas, kMetricCtas,
                                        scratch + 2 * kMetricCtas);
  *launches += 2;
  return cudaGetLastError();
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
      unsigned long long b = abs_bits_m(__ldg(a + row * lda + j));
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
    unsigned long long t = abs_bits_m(__ldg(b + r * ldb + j));
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

static inline int grid_for(int64_t work, int per_block, int cap = 148 * 16) {
  int64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  return static_cast<int>(g < cap ? g : cap);
}


cudaError_t launch_combine_exact(const CombineArgs& args, int words, const ChunkDesc* host_chunks,
                                 cudaStream_t st, int64_t* launches) {
  int64_t total = static_cast<int64_t>(args.m) * args.n;
  if (total == 0) return cudaSuccess;
  const int64_t vbits = static_cast<int64_t>(args.diagonals - 1) * args.width + 40;
  if (args.n % 4 == 0 && args.ldp % 4 == 0 && args.diagonals <= 64 &&
      ((words == 2 && vbits <= 126) || (words == 3 && vbits <= 190))) {
    // chunks are stored diagonal-major (build_chunks): tabulate each diagonal's range
    DiagTable dt{};
    int c = 0;
    for (int d = 0; d <= args.diagonals; ++d) {
      while (c < args.nchunks && host_chunks[c].d < d) ++c;
      dt.first_chunk[d] = c;
    }
    dt.first_chunk[args.diagonals] = args.nchunks;
    bool sorted = true;
    for (int q = 1; q < args.nchunks; ++q) sorted &= host_chunks[q - 1].d <= host_chunks[q].d;
    if (sorted) {
      // run length so an int64 Horner run cannot overflow:
      // bits(S_d) + t (len - 1) + 1 <= 63, bits(S_d) = 31 + ceil(log2 chunks_d)
      int maxc = 1;
      for (int d = 0; d < args.diagonals; ++d)
        maxc = std::max(maxc, dt.first_chunk[d + 1] - dt.first_chunk[d]);
      int lg = 0;
      while ((1 << lg) < maxc) ++lg;
      CombineArgs a2 = args;
      a2.hgroup = std::max(1, 1 + (62 - (31 + lg)) / std::max(1, args.width));
      const int grid = grid_for(total / 4, 256, 148 * 8);
      const char* hv = std::getenv("OZGPU_COMBINE");
      const bool w3 = vbits > 126;
      if (args.nchunks <= 64 && args.width < 64 && !(hv && std::string(hv) == "horner")) {
        // runs: an int64 run may span run_bits_max bits above one chunk value
        // (31 bits) plus the chunk-count growth of a diagonal, sign included
        int maxc2 = 1;
        for (int d = 0; d < args.diagonals; ++d)
          maxc2 = std::max(maxc2, dt.first_chunk[d + 1] - dt.first_chunk[d]);
        int lg2 = 0;
        while ((1 << lg2) < maxc2) ++lg2;
        const int run_bits_max = 30 - lg2;
        HiloProgram hp{};
        bool ok = run_bits_max >= 0;
        int vd = host_chunks[0].d, run_bits = 0;
        for (int c = 1; c < args.nchunks && ok; ++c) {
          const int gap = host_chunks[c].d - host_chunks[c - 1].d;
          if (gap == 0) continue;
          if (run_bits + gap * args.width <= run_bits_max && gap * args.width < 32) {
            hp.mul_shift[c] = gap * args.width;
            run_bits += gap * args.width;
          } else {
            // fold the run (aligned at d_{c-1}) into V (aligned at vd); the
            // gap to d_c is covered by the next fold, measured from d_{c-1}
            hp.fold_shift[c] = 1 + (host_chunks[c - 1].d - vd) * args.width;
            vd = host_chunks[c - 1].d;
            run_bits = 0;
            hp.mul_shift[c] = 0;
          }
        }
        const int dl = host_chunks[args.nchunks - 1].d;
        hp.end_shift = (dl - vd) * args.width;
        hp.final_shift = (args.diagonals - 1 - dl) * args.width;
        for (int c = 0; c < args.nchunks; ++c)
          ok &= hp.fold_shift[c] >= 0 && hp.fold_shift[c] <= 64 && hp.mul_shift[c] < 32;
        ok &= hp.end_shift < 64 && hp.final_shift < 64;
        if (ok) {
          // 4 chunk loads in flight per batch, 4 CTAs / SM: measured best of
          // {4,6,8,12} x {2,3,4} on B200 (OZGPU_COMBINE_CFG=83 selects 8 / 3)
          const char* cv = std::getenv("OZGPU_COMBINE_CFG");
          const int cfg = cv ? std::atoi(cv) : 44;
          const int gx = (args.n / 4 + 255) / 256;
          const int gy = static_cast<int>(std::min<int64_t>(args.m, std::max(1, 148 * 16 / gx)));
          const dim3 grid2(gx, gy);
          if (w3)
            combine_hilo_v4_kernel<4, 3, 3><<<grid2, 256, 0, st>>>(args, hp);
          else if (cfg == 83)
            combine_hilo_v4_kernel<8, 3, 2><<<grid2, 256, 0, st>>>(args, hp);
          else
            combine_hilo_v4_kernel<4, 4, 2><<<grid2, 256, 0, st>>>(args, hp);
          ++*launches;
          return cudaGetLastError();
        }
      }
      if (!w3) {  // 3-word values without the fast path: generic kernel below
        if (args.nchunks <= 64) {
          HornerProgram hp{};
          int run_len = 0;
          for (int c = 0; c < args.nchunks; ++c) {
            const bool newdiag = c == 0 || host_chunks[c].d != host_chunks[c - 1].d;
            if (c > 0 && newdiag) {
              if (run_len == a2.hgroup) {
                hp.flags[c] = 2;
                hp.fold_shift[c] = args.width * run_len;
                run_len = 0;
              } else {
                hp.flags[c] = 1;
              }
            }
            if (newdiag) ++run_len;
          }
          hp.final_shift = args.width * run_len;
          combine_horner2_v4_kernel<<<grid, 256, 0, st>>>(a2, hp);
        } else {
          combine_horner_v4_kernel<<<grid, 256, 0, st>>>(a2, dt);
        }
        ++*launches;
        return cudaGetLastError();
      }
    }
  }
  if (args.n % 4 == 0 && args.nchunks <= 64 && args.ldp % 4 == 0 && words <= 3) {
    ShiftTable sh{};
    for (int c = 0; c < args.nchunks; ++c) sh.shift[c] = host_chunks[c].shift;
    const int grid = grid_for(total / 4, 256, 148 * 8);
    if (words == 2)
      combine_exact_v4_kernel<2><<<grid, 256, 0, st>>>(args, sh);
    else
      combine_exact_v4_kernel<3><<<grid, 256, 0, st>>>(args, sh);
    ++*launches;
    return cudaGetLastError();
  }
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

