// Slicing kernels of the B200-native Ozaki-I FP64 GEMM (HBM-bound):
// per-row / per-column block scales and the FP64 -> int8 slice split
// (proj/src/slicing.cpp:67-132, fpcore.cpp:58-87).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

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
                                                         int64_t kp, int64_t plane, int width,
                                                         int count,
                                                         int mode, OutT* __restrict__ out,
                                                         int* __restrict__ scales,
                                                         int* __restrict__ status) {
  __shared__ unsigned long long red[8];
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
    const double* __restrict__ b, int64_t ldb, int64_t k, int64_t n, int64_t kp, int64_t plane,
    int width,
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
// Fast path (the product's default: truncate mode, t <= 7, int8 slices).
// The fraction bits of |x| / 2^q are cut into 63-bit windows holding
// 63 / T whole slices each, so every slice is one constant shift + mask of a
// window instead of a per-slice variable-shift field extraction; signs are
// applied to 4 packed bytes at a time.  Bit-identical to slice_of() in
// truncate mode (extract_field, slicing.cpp:35-45).
// ----------------------------------------------------------------------------

// The t = 7 slicer with a known slice count (the production case), cut for
// the integer ALU pipe, which bounds the slicing kernels (ncu: ALU 88 %,
// issue 60 %):
//  * the two 63-bit windows come from one pre-shifted significand:
//    W0 = floor(|x| 2^(63-q)) = (sig << 10) >> a0 and L = the next 64 bits of
//    (sig << 10):0 >> a0 (window 1 = L >> 1, so its digits sit one bit
//    higher in L); the hidden bit and the subnormal exponent come from one
//    max-and-add, sig_hi = |hi| - max(biased - 1, 0) * 2^20;
//  * each digit is moved to its byte by a constant shift chosen per
//    (digit, byte): left shifts compile to IMAD.SHL on the FMA pipe, and the
//    mask and merge are one LOP3 (XOR-accumulate);
//  * signs: the accumulator starts at m & 0x7F per negative byte, so after
//    the merge a negative byte holds 127 - d; adding m & 0x01 (no carry
//    leaves a byte: 127 - d + 1 <= 128) and XOR-ing m & 0x80 gives 256 - d.
// Needs q >= -1000 (then a0 = 1021 + q - max(biased - 1, 0) >= 0 for every
// entry |x| < 2^q); tinier blocks take emit8_trunc_i8.  Bit-identical to
// emit8_trunc_i8<7> (and so to slice_of(), slicing.cpp:35-45).
// x >> c for a constant 0 <= c < 32 as the high word of x * 2^(32-c): an
// IMAD.HI on the FMA pipe, which the ALU-bound slicers leave mostly idle.
__device__ __forceinline__ uint32_t shr_fma(uint32_t x, int c) {
  if (c == 0) return x;
  uint32_t r;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(1u << (32 - c)));
  return r;
}

template <bool CS, int FC>
__device__ __forceinline__ void emit8_t7(const double (&v)[8], int q, int8_t* __restrict__ out,
                                         int64_t plane, int64_t off) {
  static_assert(FC >= 1 && FC <= 18, "two 63-bit windows hold 18 slices");
  constexpr bool kTwo = FC > 9;
  constexpr bool kTwoLo = FC > 13;  // slices 9..12 sit in the high word of L
  uint32_t w0h[8], w0l[8], lh[8], ll[8];
  uint32_t hw[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const uint64_t bits = dbl_bits(v[e]);
    hw[e] = static_cast<uint32_t>(bits >> 32);
    const uint32_t habs = hw[e] & 0x7FFFFFFFu;
    const int b1m1 = max(static_cast<int>(habs >> 20) - 1, 0);
    const uint32_t sig_hi = habs - (static_cast<uint32_t>(b1m1) << 20);
    const uint64_t sig10 = ((static_cast<uint64_t>(sig_hi) << 32) | static_cast<uint32_t>(bits)) << 10;
    const uint32_t a0 = static_cast<uint32_t>(1021 + q - b1m1);
    uint64_t w0;
    asm("shr.b64 %0, %1, %2;" : "=l"(w0) : "l"(sig10), "r"(a0));
    w0h[e] = static_cast<uint32_t>(w0 >> 32);
    w0l[e] = static_cast<uint32_t>(w0);
    if constexpr (kTwo) {
      // a0 <= 64: sig10 << (64 - a0); a0 > 64: sig10 >> (a0 - 64).  The
      // other shift's amount wraps past 64, which PTX clamps to a zero
      // result, so an OR selects (both equal sig10 at a0 = 64).
      if constexpr (kTwoLo) {
        uint64_t left, right;
        asm("shl.b64 %0, %1, %2;" : "=l"(left) : "l"(sig10), "r"(64u - a0));
        asm("shr.b64 %0, %1, %2;" : "=l"(right) : "l"(sig10), "r"(a0 - 64u));
        const uint64_t l = left | right;
        lh[e] = static_cast<uint32_t>(l >> 32);
        ll[e] = static_cast<uint32_t>(l);
      } else {  // only the high word of L (its low word is dead code)
        uint64_t left;
        uint32_t right;
        asm("shl.b64 %0, %1, %2;" : "=l"(left) : "l"(sig10), "r"(64u - a0));
        asm("shr.b32 %0, %1, %2;" : "=r"(right) : "r"(static_cast<uint32_t>(sig10 >> 32)), "r"(a0 - 64u));
        lh[e] = static_cast<uint32_t>(left >> 32) | right;
        ll[e] = 0;
      }
    }
  }
  // per-byte sign masks of entries 0..3 / 4..7 (byte e = 0xFF if v[e] < 0)
  uint32_t m[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    // prmt selector nibble 0xB / 0xF: byte 3 of the first / second source
    // with its sign bit replicated over the byte
    uint32_t t01, t23;
    asm("prmt.b32 %0, %1, %2, 0x00FB;" : "=r"(t01) : "r"(hw[4 * h]), "r"(hw[4 * h + 1]));
    asm("prmt.b32 %0, %1, %2, 0x00FB;" : "=r"(t23) : "r"(hw[4 * h + 2]), "r"(hw[4 * h + 3]));
    m[h] = __byte_perm(t01, t23, 0x5410);
  }
  const uint32_t m7f[2] = {m[0] & 0x7F7F7F7Fu, m[1] & 0x7F7F7F7Fu};
  const uint32_t m01[2] = {m[0] & 0x01010101u, m[1] & 0x01010101u};
  const uint32_t m80[2] = {m[0] & 0x80808080u, m[1] & 0x80808080u};
  int8_t* base = out + off;
#pragma unroll
  for (int l = 0; l < FC; ++l) {
    const int j = l / 9, i = l % 9;
    const int P = 56 - 7 * i + j;  // digit bit position in its 64-bit window
    uint32_t word[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t acc = m7f[h];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int e = 4 * h + b;
        const uint32_t hi = j ? lh[e] : w0h[e], lo = j ? ll[e] : w0l[e];
        uint32_t src;
        if (P >= 32) {
          const int p = P - 32;
          src = p >= 8 * b ? shr_fma(hi, p - 8 * b) : hi << (8 * b - p);
        } else if (P + 7 <= 32) {
          src = P >= 8 * b ? shr_fma(lo, P - 8 * b) : lo << (8 * b - P);
        } else {  // straddles the halves: funnel shift
          src = __funnelshift_r(lo, hi, P - 8 * b);
        }
        // acc = (src & mask) ^ acc as one explicit LOP3 (left to itself the
        // compiler masks the first byte and XORs m7f in as extra ops)
        asm("lop3.b32 %0, %1, %2, %0, 0x6A;" : "+r"(acc) : "r"(src), "r"(0x7Fu << (8 * b)));
      }
      word[h] = (acc + m01[h]) ^ m80[h];
    }
    int8_t* dst = base + l * plane;
    if constexpr (CS)
      __stcs(reinterpret_cast<uint2*>(dst), make_uint2(word[0], word[1]));
    else
      *reinterpret_cast<uint2*>(dst) = make_uint2(word[0], word[1]);
  }
}

// FC > 0: the slice count is a compile-time constant (the common counts get
// their own instantiation: fully unrolled windows and constant store offsets)
template <int T, bool CS = false, int FC = 0>
__device__ __forceinline__ void emit8_trunc_i8(const double (&v)[8], int q, int count_rt,
                                               int8_t* __restrict__ out, int64_t plane,
                                               int64_t off) {
  if constexpr (T == 7 && FC > 0) {
    if (q >= -1000) {
      emit8_t7<CS, FC>(v, q, out, plane, off);
      return;
    }
  }
  const int count = FC > 0 ? FC : count_rt;
  constexpr int SPW = 63 / T;  // slices per window
  constexpr int WB = SPW * T;  // window bits
  constexpr uint64_t WMASK = (WB == 64) ? ~0ULL : ((1ULL << WB) - 1);
  constexpr uint32_t TMASK = (1u << T) - 1;
  uint64_t sig[8];
  int lsb[8];
  uint32_t neg_lo = 0, neg_hi = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    uint64_t bits = dbl_bits(v[e]);
    if (bits >> 63) {
      if (e < 4)
        neg_lo |= 0xFFu << (8 * e);
      else
        neg_hi |= 0xFFu << (8 * (e - 4));
    }
    bits &= 0x7FFFFFFFFFFFFFFFULL;
    const uint64_t biased = bits >> 52;
    const uint64_t frac = bits & 0xFFFFFFFFFFFFFULL;
    sig[e] = biased ? (frac | 0x10000000000000ULL) : frac;
    const int ex = biased ? static_cast<int>(biased) - 1023 : -1022;
    lsb[e] = q + 52 - ex;
  }
  auto window = [&](int j) {
    uint64_t w[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      // branch-free: PTX 64-bit shifts clamp amounts >= 64 to a zero result
      const int sh = WB * (j + 1) - lsb[e];
      uint64_t l, r;
      asm("shl.b64 %0, %1, %2;" : "=l"(l) : "l"(sig[e]), "r"(static_cast<uint32_t>(max(sh, 0))));
      asm("shr.b64 %0, %1, %2;" : "=l"(r) : "l"(sig[e]), "r"(static_cast<uint32_t>(max(-sh, 0))));
      w[e] = (sh >= 0 ? l : r) & WMASK;
    }
#pragma unroll
    for (int i = 0; i < SPW; ++i) {
      const int l = j * SPW + i;
      if (l >= count) break;
      const int s = WB - T * (i + 1);
      uint32_t lo = 0, hi = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        lo |= (static_cast<uint32_t>(w[e] >> s) & TMASK) << (8 * e);
        hi |= (static_cast<uint32_t>(w[e + 4] >> s) & TMASK) << (8 * e);
      }
      lo = __vsub4(lo ^ neg_lo, neg_lo);
      hi = __vsub4(hi ^ neg_hi, neg_hi);
      if constexpr (CS)  // streaming store: keep L2 for the panels awaiting their slice pass
        __stcs(reinterpret_cast<uint2*>(out + l * plane + off), make_uint2(lo, hi));
      else
        *reinterpret_cast<uint2*>(out + l * plane + off) = make_uint2(lo, hi);
    }
  };
  if constexpr (FC > 0) {
#pragma unroll
    for (int j = 0; j < (FC + SPW - 1) / SPW; ++j) window(j);
  } else {
    for (int j = 0; j * SPW < count; ++j) window(j);
  }
}

// Two-kernel row path (no dependence between the row reduction and the
// slice stores, so both kernels stream at HBM rate): rowmax_kernel computes
// the block scales (one warp per row, 16-byte loads), slice_rows_stream_kernel
// then slices 8 consecutive entries per thread over the whole matrix.
// (bodies take the block index and block count, so the small-operand
// kernel below can run them side by side in one launch)
template <bool VEC>
__device__ __forceinline__ void rowmax_body(int64_t blk, int64_t nblk, const double* __restrict__ a,
                                            int64_t lda, int64_t m, int64_t k,
                                            int* __restrict__ scales, int* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = nblk * (blockDim.x >> 5);
  for (int64_t row = blk * (blockDim.x >> 5) + (threadIdx.x >> 5); row < m; row += warps) {
    const double* ar = a + row * lda;
    unsigned long long mx = 0;
    int bad = 0;
    int64_t j = 0;
    if (VEC) {
      const double2* a2 = reinterpret_cast<const double2*>(ar);
      const int64_t k2 = k / 2;
      int64_t u = lane;
      for (; u + 96 < k2; u += 128) {
        double2 x[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) x[q] = __ldcs(a2 + u + 32 * q);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          bad |= dirty(x[q].x) | dirty(x[q].y);
          const unsigned long long b0 = abs_bits(x[q].x), b1 = abs_bits(x[q].y);
          mx = b0 > mx ? b0 : mx;
          mx = b1 > mx ? b1 : mx;
        }
      }
      for (; u < k2; u += 32) {
        const double2 x = __ldcs(a2 + u);
        bad |= dirty(x.x) | dirty(x.y);
        const unsigned long long b0 = abs_bits(x.x), b1 = abs_bits(x.y);
        mx = b0 > mx ? b0 : mx;
        mx = b1 > mx ? b1 : mx;
      }
      j = 2 * k2 + lane;
    } else {
      j = lane;
    }
    for (; j < k; j += 32) {
      const double x = __ldcs(ar + j);
      bad |= dirty(x);
      const unsigned long long b = abs_bits(x);
      mx = b > mx ? b : mx;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const unsigned long long t = __shfl_xor_sync(0xFFFFFFFFu, mx, o);
      mx = t > mx ? t : mx;
    }
    bad = __reduce_or_sync(0xFFFFFFFFu, bad);
    if (lane == 0) {
      if (bad) atomicOr(status, bad);
      scales[row] = scale_from_maxbits(mx);
    }
  }
}

template <bool VEC>
__global__ void __launch_bounds__(256) rowmax_kernel(const double* __restrict__ a, int64_t lda,
                                                     int64_t m, int64_t k,
                                                     int* __restrict__ scales,
                                                     int* __restrict__ status) {
  rowmax_body<VEC>(blockIdx.x, gridDim.x, a, lda, m, k, scales, status);
}

template <int T, bool VEC, int FC>
__device__ __forceinline__ void slice_rows_body(int64_t blk, int64_t nblk,
                                                const double* __restrict__ a, int64_t lda,
                                                int64_t m, int64_t k, int64_t kp, int64_t plane,
                                                int count, const int* __restrict__ scales,
                                                int8_t* __restrict__ out) {
  const int64_t groups = kp / 8;
  const int64_t total = m * groups;
  for (int64_t idx = blk * blockDim.x + threadIdx.x; idx < total; idx += nblk * blockDim.x) {
    const int64_t row = idx / groups, g = idx - row * groups;
    const double* ar = a + row * lda;
    const int64_t j0 = g * 8;
    double v[8];
    if (VEC && j0 + 8 <= k) {
      const double2* p2 = reinterpret_cast<const double2*>(ar + j0);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double2 t2 = __ldcs(p2 + u);
        v[2 * u] = t2.x;
        v[2 * u + 1] = t2.y;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = j0 + e < k ? __ldcs(ar + j0 + e) : 0.0;
    }
    emit8_trunc_i8<T, false, FC>(v, __ldg(scales + row), count, out, plane, row * kp + j0);
  }
}

template <int T, bool VEC, int MINB, int FC = 0>
__global__ void __launch_bounds__(256, MINB) slice_rows_stream_kernel(
    const double* __restrict__ a, int64_t lda, int64_t m, int64_t k, int64_t kp, int64_t plane,
    int count, const int* __restrict__ scales, int8_t* __restrict__ out) {
  slice_rows_body<T, VEC, FC>(blockIdx.x, gridDim.x, a, lda, m, k, kp, plane, count, scales, out);
}

// 128 (k) x 32 (n) tile transpose-and-slice into K-major [l][n][kp] int8.
// Smem holds the tile column-major in 16-byte units with an XOR swizzle so
// both the row-wise fill and the 8-entry column reads are conflict-light.
constexpr int kColTileK = 128, kColTileN = 32, kColTileStride = kColTileK + 2;

template <int T, int FC>
__device__ __forceinline__ void slice_cols_tile(int64_t bx, int64_t by, double* __restrict__ tile,
                                                const double* __restrict__ b, int64_t ldb,
                                                int64_t k, int64_t n, int64_t kp, int64_t plane,
                                                int count,
                                                const unsigned long long* __restrict__ colmax,
                                                int8_t* __restrict__ out,
                                                int* __restrict__ scales) {
  constexpr int TK = kColTileK, TN = kColTileN, STRIDE = kColTileStride;  // doubles per column (padded)
  const int64_t k0 = bx * TK;
  const int64_t n0 = by * TN;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // swizzled position of row r in column c: 16-byte unit (r >> 1) ^ ((r >> 3) & 7)
  auto pos = [](int c, int r) {
    int u = r >> 1;
    return c * STRIDE + ((u ^ ((u >> 2) & 7)) << 1) + (r & 1);
  };
  // each warp loads 8 row pairs (all 16 loads in flight), then stores each
  // column's pair as one 16-byte word: lane c hits 16-byte slot c + const
  // (mod 8) -- 4 wavefronts per 512 bytes, no bank conflicts
  {
    double v[16];
    const int64_t c = n0 + lane;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = 2 * (warp + 8 * i);
      const int64_t kr = k0 + r;
      v[2 * i] = (kr < k && c < n) ? __ldcs(b + kr * ldb + c) : 0.0;
      v[2 * i + 1] = (kr + 1 < k && c < n) ? __ldcs(b + (kr + 1) * ldb + c) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = 2 * (warp + 8 * i);
      *reinterpret_cast<double2*>(&tile[pos(lane, r)]) = make_double2(v[2 * i], v[2 * i + 1]);
    }
  }
  if (bx == 0 && threadIdx.x < TN && n0 + threadIdx.x < n)
    scales[n0 + threadIdx.x] = scale_from_maxbits(colmax[n0 + threadIdx.x]);
  __syncthreads();
  // item = (column, group of 8 rows); groups fastest so a warp writes 2
  // columns x 128 contiguous bytes per slice
  for (int item = threadIdx.x; item < TN * (TK / 8); item += blockDim.x) {
    const int c = item / (TK / 8), g = item % (TK / 8);
    const int64_t col = n0 + c, kk = k0 + g * 8;
    if (col >= n || kk >= kp) continue;
    const int q = scale_from_maxbits(colmax[col]);
    double v[8];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double2 t2 = *reinterpret_cast<const double2*>(&tile[pos(c, g * 8 + 2 * u)]);
      v[2 * u] = t2.x;
      v[2 * u + 1] = t2.y;
    }
    emit8_trunc_i8<T, false, FC>(v, q, count, out, plane, col * kp + kk);
  }
}

template <int T, int FC = 0>
__global__ void __launch_bounds__(256) slice_cols_fast_kernel(
    const double* __restrict__ b, int64_t ldb, int64_t k, int64_t n, int64_t kp, int64_t plane,
    int count,
    const unsigned long long* __restrict__ colmax, int8_t* __restrict__ out,
    int* __restrict__ scales) {
  __shared__ __align__(16) double tile[kColTileN * kColTileStride];
  slice_cols_tile<T, FC>(blockIdx.x, blockIdx.y, tile, b, ldb, k, n, kp, plane, count, colmax, out,
                         scales);
}

// ----------------------------------------------------------------------------
// Small operands ((m + n) k below ~8M entries): the four slicing launches
// (row max, column max, row slices, column slices) cost more in launch
// latency and ramp-up than in memory time, so they run as two launches that
// each cover both operands -- blocks [0, ga) work on A, the rest on B (the
// column maxima of 64-row slices meet in an atomicMax).  Equal slice counts
// use the compile-time-count emit, unequal ones the runtime count.
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) maxes_small_kernel(
    const double* __restrict__ a, int64_t lda, int64_t m, const double* __restrict__ b,
    int64_t ldb, int64_t n, int64_t k, int ga, int gbx, int64_t rows_per,
    int* __restrict__ scales_a, unsigned long long* __restrict__ colmax, int* __restrict__ status) {
  if (static_cast<int>(blockIdx.x) < ga) {
    rowmax_body<true>(blockIdx.x, ga, a, lda, m, k, scales_a, status);
    return;
  }
  // B: 32 columns x 8 row groups per block over a slice of rows_per rows;
  // the warp reads 32 consecutive columns of one row (256 contiguous bytes)
  __shared__ unsigned long long red[8][32];
  const int bb = blockIdx.x - ga;
  const int c = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t col = static_cast<int64_t>(bb % gbx) * 32 + c;
  const int64_t r0 = static_cast<int64_t>(bb / gbx) * rows_per;
  const int64_t r1 = r0 + rows_per < k ? r0 + rows_per : k;
  unsigned long long mx = 0;
  int bad = 0;
  if (col < n) {
#pragma unroll 4
    for (int64_t r = r0 + g; r < r1; r += 8) {
      const double x = __ldcs(b + r * ldb + col);
      bad |= dirty(x);
      const unsigned long long v = abs_bits(x);
      mx = v > mx ? v : mx;
    }
  }
  red[g][c] = mx;
  bad = __reduce_or_sync(0xFFFFFFFFu, bad);
  if (bad && c == 0) atomicOr(status, bad);
  __syncthreads();
  if (g == 0 && col < n) {
#pragma unroll
    for (int u = 1; u < 8; ++u) mx = red[u][c] > mx ? red[u][c] : mx;
    if (mx) atomicMax(colmax + col, mx);
  }
}

template <int T, int FC>
__global__ void __launch_bounds__(256) slices_small_kernel(
    const double* __restrict__ a, int64_t lda, int64_t m, const double* __restrict__ b,
    int64_t ldb, int64_t n, int64_t k, int64_t kp, int count_a, int count_b, int64_t plane_a,
    int64_t plane_b, int ga, int gbx, const int* __restrict__ scales_a,
    const unsigned long long* __restrict__ colmax, int8_t* __restrict__ out_a,
    int8_t* __restrict__ out_b, int* __restrict__ scales_b) {
  __shared__ __align__(16) double tile[kColTileN * kColTileStride];
  if (static_cast<int>(blockIdx.x) < ga) {
    slice_rows_body<T, true, FC>(blockIdx.x, ga, a, lda, m, k, kp, plane_a, count_a, scales_a,
                                 out_a);
    return;
  }
  const int bb = blockIdx.x - ga;
  slice_cols_tile<T, FC>(bb % gbx, bb / gbx, tile, b, ldb, k, n, kp, plane_b, count_b, colmax,
                         out_b, scales_b);
}

// ----------------------------------------------------------------------------
// One launch slicing both operands through an ordered work queue.
//
// The block scale of a row of A (a column of B) depends on the whole row
// (column), so the two-kernel path above reads each operand twice from DRAM.
// Here each operand is cut into panels of ~16 MB and one persistent launch
// takes work items from a global ticket in a fixed order
//     max(P0), max(P1), slice(P0), max(P2), slice(P1), ..., slice(P_last)
// (the panels of A, then those of B).  A slice item of panel p first waits
// until every max item of p has finished (a per-panel counter); tickets are
// handed out in order and max items never wait, so a wait always ends.  The
// slice pass re-reads a panel about one panel-time after its max pass, from
// L2, so DRAM reads each operand once.
// ----------------------------------------------------------------------------

struct SliceQueueOp {
  const double* x;  // A: blocks x len rows (ldx); B: len x blocks (ldx)
  int64_t ldx;
  int64_t blocks;   // rows of A / columns of B
  int64_t len;      // k
  int64_t kp;       // output row stride (multiple of 128), zero-filled past len
  int64_t plane;
  int8_t* out;
  int* scales;
  unsigned long long* colmax;  // B: zeroed before the launch
  int count;
  int panel;        // blocks per panel (A: multiple of 8; B: multiple of 32)
  int npanels;
  int max_items;    // per panel
  int slice_items;  // per panel
  int rb;           // B: rows per max item
  int cw;           // B: columns per max item (32..256, divides 256 and the panel)
  int vec;          // A: 16-byte loads are legal
};

struct SliceQueueArgs {
  SliceQueueOp op[2];  // 0 = A (rows), 1 = B (columns)
  int* ticket;         // ticket[0]: next item; ticket[1 + g]: finished max items of panel g
  const int* seg_start;  // nseg + 1 ascending ticket offsets of the queue's segments
  const int* seg_info;   // per segment: 2 * panel + (1 = slice items, 0 = max items)
  int nseg;
  int* status;
  int total;
};

constexpr int kQueueGroups = 2048;  // A slice item: 2048 groups of 8 entries (128 KB of A)

__device__ __forceinline__ int q_ld_acquire(const int* ptr) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ptr) : "memory");
  return v;
}

// ticket -> (is_slice, global panel g, item within the panel's max / slice set)
__device__ __forceinline__ void queue_item(const SliceQueueArgs& p, int t, int& is_slice, int& g,
                                           int& item) {
  int lo = 0, hi = p.nseg - 1;  // last segment with start <= t
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(p.seg_start + mid) <= t) lo = mid;
    else hi = mid - 1;
  }
  const int info = __ldg(p.seg_info + lo);
  is_slice = info & 1;
  g = info >> 1;
  item = t - __ldg(p.seg_start + lo);
}

template <int T>
__global__ void __launch_bounds__(256, 3) slice_queue_kernel(const SliceQueueArgs p) {
  constexpr int TK = 128, TN = 32, STRIDE = TK + 2;
  __shared__ __align__(16) double tile[TN * STRIDE];
  __shared__ int s_ticket;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (;;) {
    if (tid == 0) s_ticket = atomicAdd(p.ticket, 1);
    __syncthreads();
    const int t = s_ticket;
    __syncthreads();  // s_ticket is rewritten next round
    if (t >= p.total) return;
    int is_slice, g, item;
    queue_item(p, t, is_slice, g, item);
    const int o = g < p.op[0].npanels ? 0 : 1;
    const SliceQueueOp& op = p.op[o];
    const int pg = o == 0 ? g : g - p.op[0].npanels;  // panel within the operand
    const int64_t b0 = static_cast<int64_t>(pg) * op.panel;
    const int64_t b1 = b0 + op.panel < op.blocks ? b0 + op.panel : op.blocks;
    if (!is_slice) {
      if (o == 0) {
        // ---- max of 8 rows of A, one warp per row (16-byte loads) ----
        const int64_t row = b0 + static_cast<int64_t>(item) * 8 + warp;
        if (row < b1) {
          const double* ar = op.x + row * op.ldx;
          unsigned long long mx = 0;
          int bad = 0;
          int64_t j = 0;
          if (op.vec) {
            const double2* a2 = reinterpret_cast<const double2*>(ar);
            const int64_t k2 = op.len / 2;
            int64_t u = lane;
            for (; u + 224 < k2; u += 256) {
              double2 x[8];
#pragma unroll
              for (int q = 0; q < 8; ++q) x[q] = __ldcg(a2 + u + 32 * q);
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                bad |= dirty(x[q].x) | dirty(x[q].y);
                const unsigned long long c0 = abs_bits(x[q].x), c1 = abs_bits(x[q].y);
                mx = c0 > mx ? c0 : mx;
                mx = c1 > mx ? c1 : mx;
              }
            }
            for (; u < k2; u += 32) {
              const double2 x = __ldcg(a2 + u);
              bad |= dirty(x.x) | dirty(x.y);
              const unsigned long long c0 = abs_bits(x.x), c1 = abs_bits(x.y);
              mx = c0 > mx ? c0 : mx;
              mx = c1 > mx ? c1 : mx;
            }
            j = 2 * k2 + lane;
          } else {
            j = lane;
          }
          for (; j < op.len; j += 32) {
            const double x = __ldcg(ar + j);
            bad |= dirty(x);
            const unsigned long long c = abs_bits(x);
            mx = c > mx ? c : mx;
          }
#pragma unroll
          for (int sft = 16; sft; sft >>= 1) {
            const unsigned long long u2 = __shfl_xor_sync(0xFFFFFFFFu, mx, sft);
            mx = u2 > mx ? u2 : mx;
          }
          bad = __reduce_or_sync(0xFFFFFFFFu, bad);
          if (lane == 0) {
            if (bad) atomicOr(p.status, bad);
            op.scales[row] = scale_from_maxbits(mx);
          }
        }
      } else {
        // ---- column max over rb rows x cw columns of B ----
        const int subs = op.panel / op.cw;
        const int sub = item % subs, rc = item / subs;
        const int col_in = tid % op.cw, rg = tid / op.cw, ngroups = 256 / op.cw;
        const int64_t col = b0 + static_cast<int64_t>(sub) * op.cw + col_in;
        const int64_t r0 = static_cast<int64_t>(rc) * op.rb;
        const int64_t r1 = r0 + op.rb < op.len ? r0 + op.rb : op.len;
        if (col < b1) {
          unsigned long long mx = 0;
          int bad = 0;
          int64_t r = r0 + rg;
          for (; r + 7 * ngroups < r1; r += 8 * ngroups) {
            double x[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) x[q] = __ldcg(op.x + (r + q * ngroups) * op.ldx + col);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              bad |= dirty(x[q]);
              const unsigned long long c = abs_bits(x[q]);
              mx = c > mx ? c : mx;
            }
          }
          for (; r < r1; r += ngroups) {
            const double x = __ldcg(op.x + r * op.ldx + col);
            bad |= dirty(x);
            const unsigned long long c = abs_bits(x);
            mx = c > mx ? c : mx;
          }
          if (bad) atomicOr(p.status, bad);
          if (mx) atomicMax(op.colmax + col, mx);
        }
      }
      __syncthreads();  // every thread's scale / colmax update precedes the release
      if (tid == 0) {
        __threadfence();
        atomicAdd(p.ticket + 1 + g, 1);
      }
      continue;
    }
    // slice item: wait for the panel's scales
    if (tid == 0)
      while (q_ld_acquire(p.ticket + 1 + g) < op.max_items) __nanosleep(64);
    __syncthreads();
    if (o == 0) {
      // ---- slice rows of A: 2048 groups of 8 entries, 8 per thread ----
      const int64_t gpr = op.kp / 8;
      const int64_t e_end0 = (b1 - b0) * gpr;
      const int64_t e0 = static_cast<int64_t>(item) * kQueueGroups;
      const int64_t e1 = e0 + kQueueGroups < e_end0 ? e0 + kQueueGroups : e_end0;
      for (int64_t e = e0 + tid; e < e1; e += 256) {
        const int64_t row = b0 + e / gpr, j0 = (e % gpr) * 8;
        const double* ar = op.x + row * op.ldx;
        double v[8];
        if (op.vec && j0 + 8 <= op.len) {
          const double2* p2 = reinterpret_cast<const double2*>(ar + j0);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double2 t2 = __ldcs(p2 + u);  // last use of A: evict first
            v[2 * u] = t2.x;
            v[2 * u + 1] = t2.y;
          }
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = j0 + q < op.len ? __ldcs(ar + j0 + q) : 0.0;
        }
        emit8_trunc_i8<T, true>(v, __ldcg(op.scales + row), op.count, op.out, op.plane,
                                row * op.kp + j0);
      }
    } else {
      // ---- slice a 128 (k) x 32 (n) tile of B, transposed through smem ----
      const int ktiles = static_cast<int>(op.kp / TK);
      const int kt = item % ktiles, nt = item / ktiles;
      const int64_t k0 = static_cast<int64_t>(kt) * TK;
      const int64_t n0 = b0 + static_cast<int64_t>(nt) * TN;
      auto pos = [](int c, int r) {
        int u = r >> 1;
        return c * STRIDE + ((u ^ ((u >> 2) & 7)) << 1) + (r & 1);
      };
      {
        double v[16];
        const int64_t c = n0 + lane;
        const bool cok = c < b1;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = 2 * (warp + 8 * i);
          const int64_t kr = k0 + r;
          v[2 * i] = (kr < op.len && cok) ? __ldcs(op.x + kr * op.ldx + c) : 0.0;
          v[2 * i + 1] = (kr + 1 < op.len && cok) ? __ldcs(op.x + (kr + 1) * op.ldx + c) : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = 2 * (warp + 8 * i);
          *reinterpret_cast<double2*>(&tile[pos(lane, r)]) = make_double2(v[2 * i], v[2 * i + 1]);
        }
      }
      if (kt == 0 && tid < TN && n0 + tid < b1)
        op.scales[n0 + tid] = scale_from_maxbits(__ldcg(op.colmax + n0 + tid));
      __syncthreads();
      for (int it = tid; it < TN * (TK / 8); it += 256) {
        const int c = it / (TK / 8), gq = it % (TK / 8);
        const int64_t col = n0 + c, kk = k0 + gq * 8;
        if (col >= b1) continue;
        const int q = scale_from_maxbits(__ldcg(op.colmax + col));
        double v[8];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double2 t2 = *reinterpret_cast<const double2*>(&tile[pos(c, gq * 8 + 2 * u)]);
          v[2 * u] = t2.x;
          v[2 * u + 1] = t2.y;
        }
        emit8_trunc_i8<T, true>(v, q, op.count, op.out, op.plane, col * op.kp + kk);
      }
      __syncthreads();  // the tile is refilled by the next item
    }
  }
}

// Panel geometry of the queue launch (host side).  ~16 MB panels
// (OZGPU_SLICE_PANEL_MB): two of them in flight stay well inside L2.
static void plan_queue_op(SliceQueueOp& q, bool rows) {
  double mb = 16.0;
  if (const char* env = std::getenv("OZGPU_SLICE_PANEL_MB")) mb = std::max(1.0, std::atof(env));
  const int64_t per = static_cast<int64_t>(mb * 1048576.0 / (8.0 * std::max<int64_t>(q.len, 1)));
  if (q.blocks <= 0) {
    q.npanels = 0, q.max_items = 0, q.slice_items = 0, q.panel = 8;
    return;
  }
  if (rows) {
    int64_t pr = std::max<int64_t>(8, per / 8 * 8);
    pr = std::min<int64_t>(pr, (q.blocks + 7) / 8 * 8);
    q.panel = static_cast<int>(pr);
    q.max_items = static_cast<int>(pr / 8);
    q.slice_items = static_cast<int>((pr * (q.kp / 8) + kQueueGroups - 1) / kQueueGroups);
  } else {
    int64_t pc = std::max<int64_t>(32, per / 32 * 32);
    pc = std::min<int64_t>(pc, (q.blocks + 31) / 32 * 32);
    int cw;
    if (pc >= 256) {
      pc = pc / 256 * 256;
      cw = 256;
    } else {
      cw = pc >= 128 ? 128 : pc >= 64 ? 64 : 32;
      pc = cw;
    }
    q.panel = static_cast<int>(pc);
    q.cw = cw;
    q.rb = static_cast<int>(std::max<int64_t>(8, 32768 / cw));  // ~256 KB of B per max item
    q.max_items = static_cast<int>((pc / cw) * ((q.len + q.rb - 1) / q.rb));
    q.slice_items = static_cast<int>((q.kp / 128) * (pc / 32));
  }
  q.npanels = static_cast<int>((q.blocks + q.panel - 1) / q.panel);
}

int slice_queue_work_ints(int64_t m, int64_t n, int64_t k, int64_t kp) {
  SliceQueueOp a{}, b{};
  a.blocks = m, a.len = k, a.kp = kp;
  b.blocks = n, b.len = k, b.kp = kp;
  plan_queue_op(a, true);
  plan_queue_op(b, false);
  const int P = a.npanels + b.npanels;
  return 1 + P + (2 * P + 1) + 2 * P;  // counters, segment starts, segment infos
}

template <int T>
static void launch_queue_t(const SliceQueueArgs& qa, int grid, cudaStream_t st) {
  slice_queue_kernel<T><<<grid, 256, 0, st>>>(qa);
}

cudaError_t launch_slice_queue(const double* a, int64_t lda, int64_t m, const double* b,
                               int64_t ldb, int64_t n, int64_t k, int64_t kp, int width,
                               int count_a, int count_b, int8_t* out_a, int64_t plane_a,
                               int8_t* out_b, int64_t plane_b, int* scales_a, int* scales_b,
                               unsigned long long* colmax, int* work, int* status,
                               UploadFn upload, void* upload_user, cudaStream_t st,
                               int64_t* launches) {
  SliceQueueArgs q{};
  SliceQueueOp& A = q.op[0];
  SliceQueueOp& B = q.op[1];
  A.x = a, A.ldx = lda, A.blocks = a ? m : 0, A.len = k, A.kp = kp;
  A.plane = plane_a ? plane_a : m * kp, A.out = out_a, A.scales = scales_a, A.count = count_a;
  A.vec = (reinterpret_cast<uintptr_t>(a) & 15) == 0 && (lda & 1) == 0;
  B.x = b, B.ldx = ldb, B.blocks = b ? n : 0, B.len = k, B.kp = kp;
  B.plane = plane_b ? plane_b : n * kp, B.out = out_b, B.scales = scales_b, B.colmax = colmax;
  B.count = count_b;
  plan_queue_op(A, true);
  plan_queue_op(B, false);
  const int P = A.npanels + B.npanels;
  if (P == 0) return cudaSuccess;
  // Queue order with a lookahead of L panels: max(0..L-1), then max(h),
  // slice(h - L) for h = L..P-1, then the last L slices.  L is sized so that
  // a panel's slice items are handed out only after about one full wave of
  // other items followed its max items (OZGPU_SLICE_LOOKAHEAD).
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int ctas = 3 * sms;
  auto mi = [&](int g) { return g < A.npanels ? A.max_items : B.max_items; };
  auto si = [&](int g) { return g < A.npanels ? A.slice_items : B.slice_items; };
  int L = 0;
  if (const char* env = std::getenv("OZGPU_SLICE_LOOKAHEAD")) {
    L = std::max(1, std::atoi(env));
  } else {
    const int per = std::max(1, std::min(A.npanels ? A.max_items + A.slice_items : 1 << 30,
                                         B.npanels ? B.max_items + B.slice_items : 1 << 30));
    L = std::max(1, (ctas + per - 1) / per);
  }
  L = std::min(L, P);
  std::vector<int> table;  // [nseg + 1 starts][nseg infos]
  std::vector<int> starts, infos;
  int pos = 0;
  auto seg = [&](int g, int kind) {
    const int cnt = kind ? si(g) : mi(g);
    if (cnt <= 0) return;
    starts.push_back(pos);
    infos.push_back(2 * g + kind);
    pos += cnt;
  };
  for (int h = 0; h < L; ++h) seg(h, 0);
  for (int h = L; h < P; ++h) {
    seg(h, 0);
    seg(h - L, 1);
  }
  for (int h = P - L; h < P; ++h) seg(h, 1);
  const int nseg = static_cast<int>(infos.size());
  starts.push_back(pos);
  table.insert(table.end(), starts.begin(), starts.end());
  table.insert(table.end(), infos.begin(), infos.end());
  q.total = pos;
  q.ticket = work;
  q.seg_start = work + 1 + P;
  q.seg_info = work + 1 + P + nseg + 1;
  q.nseg = nseg;
  q.status = status;
  upload(upload_user, work + 1 + P, table.data(), sizeof(int) * table.size(), st);
  cudaError_t e = cudaMemsetAsync(work, 0, sizeof(int) * (1 + P), st);
  if (e == cudaSuccess && B.blocks > 0)
    e = cudaMemsetAsync(colmax, 0, sizeof(unsigned long long) * n, st);
  if (e != cudaSuccess) return e;
  const int grid = std::min(q.total, ctas);
  switch (width) {
    case 7: launch_queue_t<7>(q, grid, st); break;
    case 6: launch_queue_t<6>(q, grid, st); break;
    case 5: launch_queue_t<5>(q, grid, st); break;
    case 4: launch_queue_t<4>(q, grid, st); break;
    case 3: launch_queue_t<3>(q, grid, st); break;
    case 2: launch_queue_t<2>(q, grid, st); break;
    default: launch_queue_t<1>(q, grid, st); break;
  }
  ++*launches;
  return cudaGetLastError();
}

static inline int grid_for(int64_t work, int per_block, int cap = 148 * 16) {
  int64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  return static_cast<int>(g < cap ? g : cap);
}

// OZGPU_SLICE_FC=0: runtime slice count everywhere (A/B of the instantiations)
static bool fixed_counts() {
  const char* env = std::getenv("OZGPU_SLICE_FC");
  return !(env && std::atoi(env) == 0);
}

template <int T, int FC>
static void rows_fc(int grid2, cudaStream_t st, const double* a, int64_t lda, int64_t m, int64_t k,
                    int64_t kp, int64_t plane, const int* scales, int8_t* out) {
  slice_rows_stream_kernel<T, true, 4, FC><<<grid2, 256, 0, st>>>(a, lda, m, k, kp, plane, FC,
                                                                  scales, out);
}

template <int T>
static void launch_rows_fc(int count, int grid2, cudaStream_t st, const double* a, int64_t lda,
                           int64_t m, int64_t k, int64_t kp, int64_t plane, const int* scales,
                           int8_t* out) {
  switch (count) {
#define OZ_FC(c) case c: rows_fc<T, c>(grid2, st, a, lda, m, k, kp, plane, scales, out); break;
    OZ_FC(1) OZ_FC(2) OZ_FC(3) OZ_FC(4) OZ_FC(5) OZ_FC(6) OZ_FC(7) OZ_FC(8) OZ_FC(9)
    OZ_FC(10) OZ_FC(11) OZ_FC(12) OZ_FC(13) OZ_FC(14) OZ_FC(15) OZ_FC(16) OZ_FC(17)
#undef OZ_FC
    default: break;
  }
}

template <int T, int FC>
static void cols_fc(dim3 grid, cudaStream_t st, const double* b, int64_t ldb, int64_t k, int64_t n,
                    int64_t kp, int64_t plane, const unsigned long long* colmax, int8_t* out,
                    int* scales) {
  slice_cols_fast_kernel<T, FC><<<grid, 256, 0, st>>>(b, ldb, k, n, kp, plane, FC, colmax, out,
                                                      scales);
}

template <int T>
static bool launch_cols_fc(int count, dim3 grid, cudaStream_t st, const double* b, int64_t ldb,
                           int64_t k, int64_t n, int64_t kp, int64_t plane,
                           const unsigned long long* colmax, int8_t* out, int* scales) {
  switch (count) {
#define OZ_FC(c) case c: cols_fc<T, c>(grid, st, b, ldb, k, n, kp, plane, colmax, out, scales); return true;
    OZ_FC(1) OZ_FC(2) OZ_FC(3) OZ_FC(4) OZ_FC(5) OZ_FC(6) OZ_FC(7) OZ_FC(8) OZ_FC(9)
    OZ_FC(10) OZ_FC(11) OZ_FC(12) OZ_FC(13) OZ_FC(14) OZ_FC(15) OZ_FC(16) OZ_FC(17)
#undef OZ_FC
    default: return false;
  }
}

template <int T>
static int launch_rows_fast_t(const double* a, int64_t lda, int64_t m, int64_t k, int64_t kp,
                               int64_t plane, int count, int8_t* out, int* scales, int* status,
                               cudaStream_t st) {
  const bool vec = (reinterpret_cast<uintptr_t>(a) & 15) == 0 && (lda & 1) == 0;
  const int grid = grid_for(m, 8, 148 * 16);
  const int grid2 = grid_for(m * (kp / 8), 256, 148 * 16);
  // 4 CTAs / SM (64 registers, measured ~3% faster than 3 / SM on B200)
  const char* mb = std::getenv("OZGPU_SLICE_MINB");
  const bool four = !(mb && std::atoi(mb) == 1);
  if (vec) {
    rowmax_kernel<true><<<grid, 256, 0, st>>>(a, lda, m, k, scales, status);
    bool done = false;
    if constexpr (T == 7) {
      if (four && fixed_counts() && count >= 1 && count <= 17) {
        launch_rows_fc<T>(count, grid2, st, a, lda, m, k, kp, plane, scales, out);
        done = true;
      }
    }
    if (done) {
    } else if (four)
      slice_rows_stream_kernel<T, true, 4><<<grid2, 256, 0, st>>>(a, lda, m, k, kp, plane, count,
                                                                  scales, out);
    else
      slice_rows_stream_kernel<T, true, 1><<<grid2, 256, 0, st>>>(a, lda, m, k, kp, plane, count,
                                                                  scales, out);
  } else {
    rowmax_kernel<false><<<grid, 256, 0, st>>>(a, lda, m, k, scales, status);
    slice_rows_stream_kernel<T, false, 1><<<grid2, 256, 0, st>>>(a, lda, m, k, kp, plane, count,
                                                                 scales, out);
  }
  return 2;
}

template <int T>
static void launch_cols_fast_t(const double* b, int64_t ldb, int64_t k, int64_t n, int64_t kp,
                               int64_t plane, int count, const unsigned long long* colmax,
                               int8_t* out, int* scales, cudaStream_t st) {
  dim3 grid(static_cast<unsigned>((kp + 127) / 128), static_cast<unsigned>((n + 31) / 32));
  if constexpr (T == 7) {
    if (fixed_counts() &&
        launch_cols_fc<T>(count, grid, st, b, ldb, k, n, kp, plane, colmax, out, scales))
      return;
  }
  slice_cols_fast_kernel<T><<<grid, 256, 0, st>>>(b, ldb, k, n, kp, plane, count, colmax, out,
                                                  scales);
}

bool small_slicing_applies(int64_t m, int64_t n, int64_t k, int64_t kp, int width, int mode,
                           const double* a, int64_t lda) {
  const char* env = std::getenv("OZGPU_SLICE_SMALL");
  if (env && std::atoi(env) == 0) return false;
  return m > 0 && n > 0 && k > 0 && mode == 0 && width == 7 && kp % 128 == 0 &&
         (m + n) * k < (int64_t{8} << 20) && (reinterpret_cast<uintptr_t>(a) & 15) == 0 &&
         (lda & 1) == 0;
}

cudaError_t launch_slice_small(const double* a, int64_t lda, int64_t m, const double* b,
                               int64_t ldb, int64_t n, int64_t k, int64_t kp, int count_a,
                               int count_b, int8_t* out_a, int64_t plane_a, int8_t* out_b,
                               int64_t plane_b, int* scales_a, int* scales_b,
                               unsigned long long* colmax, int* status, cudaStream_t st,
                               int64_t* launches) {
  cudaError_t e = cudaMemsetAsync(colmax, 0, sizeof(unsigned long long) * n, st);
  if (e != cudaSuccess) return e;
  const int ga = grid_for(m, 8, 148 * 16);
  const int gb = static_cast<int>((n + 31) / 32);
  const int64_t rows_per = 64;  // 8 rows per thread
  const int splits = static_cast<int>((k + rows_per - 1) / rows_per);
  maxes_small_kernel<<<ga + gb * splits, 256, 0, st>>>(a, lda, m, b, ldb, n, k, ga, gb, rows_per,
                                                        scales_a, colmax, status);
  const int ga2 = grid_for(m * (kp / 8), 256, 148 * 16);
  const int gbx = static_cast<int>(kp / kColTileK);
  // equal slice counts (the common square plans) get the compile-time-count emit
  const int fc = (count_a == count_b && fixed_counts()) ? count_a : 0;
  switch (fc) {
#define OZ_FC(c)                                                                              \
  case c:                                                                                     \
    slices_small_kernel<7, c><<<ga2 + gbx * gb, 256, 0, st>>>(                                \
        a, lda, m, b, ldb, n, k, kp, count_a, count_b, plane_a, plane_b, ga2, gbx, scales_a,   \
        colmax, out_a, out_b, scales_b);                                                      \
    break;
    OZ_FC(1) OZ_FC(2) OZ_FC(3) OZ_FC(4) OZ_FC(5) OZ_FC(6) OZ_FC(7) OZ_FC(8) OZ_FC(9)
    OZ_FC(10) OZ_FC(11) OZ_FC(12) OZ_FC(13) OZ_FC(14) OZ_FC(15) OZ_FC(16) OZ_FC(17)
#undef OZ_FC
    default:
      slices_small_kernel<7, 0><<<ga2 + gbx * gb, 256, 0, st>>>(
          a, lda, m, b, ldb, n, k, kp, count_a, count_b, plane_a, plane_b, ga2, gbx, scales_a,
          colmax, out_a, out_b, scales_b);
      break;
  }
  *launches += 2;
  return cudaGetLastError();
}

cudaError_t launch_slice_rows(const double* a, int64_t lda, int64_t m, int64_t k, int64_t kp,
                              int width, int count, int mode, void* out, int out_is_i64,
                              int* scales, int* status, cudaStream_t st, int64_t* launches,
                              int64_t plane) {
  if (m == 0) return cudaSuccess;
  if (plane == 0) plane = m * kp;
  if (!out_is_i64 && mode == 0 && width >= 1 && width <= 7) {
    int8_t* o = static_cast<int8_t*>(out);
    int n_launch = 0;
    switch (width) {
      case 7: n_launch = launch_rows_fast_t<7>(a, lda, m, k, kp, plane, count, o, scales, status, st); break;
      case 6: n_launch = launch_rows_fast_t<6>(a, lda, m, k, kp, plane, count, o, scales, status, st); break;
      case 5: n_launch = launch_rows_fast_t<5>(a, lda, m, k, kp, plane, count, o, scales, status, st); break;
      case 4: n_launch = launch_rows_fast_t<4>(a, lda, m, k, kp, plane, count, o, scales, status, st); break;
      case 3: n_launch = launch_rows_fast_t<3>(a, lda, m, k, kp, plane, count, o, scales, status, st); break;
      case 2: n_launch = launch_rows_fast_t<2>(a, lda, m, k, kp, plane, count, o, scales, status, st); break;
      default: n_launch = launch_rows_fast_t<1>(a, lda, m, k, kp, plane, count, o, scales, status, st); break;
    }
    *launches += n_launch;  // single-pass kernel, or rowmax + stream slicing
    return cudaGetLastError();
  }
  int grid = static_cast<int>(m < 148 * 32 ? m : 148 * 32);
  if (out_is_i64)
    slice_rows_kernel<long long><<<grid, 256, 0, st>>>(a, lda, m, k, kp, plane, width, count, mode,
                                                       static_cast<long long*>(out), scales,
                                                       status);
  else
    slice_rows_kernel<int8_t><<<grid, 256, 0, st>>>(a, lda, m, k, kp, plane, width, count, mode,
                                                    static_cast<int8_t*>(out), scales, status);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_slice_cols(const double* b, int64_t ldb, int64_t k, int64_t n, int64_t kp,
                              int width, int count, int mode, void* out, int out_is_i64,
                              int* scales, unsigned long long* colmax, int* status,
                              cudaStream_t st, int64_t* launches, int64_t plane) {
  if (n == 0) return cudaSuccess;
  if (plane == 0) plane = n * kp;
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
  if (!out_is_i64 && mode == 0 && width >= 1 && width <= 7 && kp % 128 == 0) {
    int8_t* o = static_cast<int8_t*>(out);
    switch (width) {
      case 7: launch_cols_fast_t<7>(b, ldb, k, n, kp, plane, count, colmax, o, scales, st); break;
      case 6: launch_cols_fast_t<6>(b, ldb, k, n, kp, plane, count, colmax, o, scales, st); break;
      case 5: launch_cols_fast_t<5>(b, ldb, k, n, kp, plane, count, colmax, o, scales, st); break;
      case 4: launch_cols_fast_t<4>(b, ldb, k, n, kp, plane, count, colmax, o, scales, st); break;
      case 3: launch_cols_fast_t<3>(b, ldb, k, n, kp, plane, count, colmax, o, scales, st); break;
      case 2: launch_cols_fast_t<2>(b, ldb, k, n, kp, plane, count, colmax, o, scales, st); break;
      default: launch_cols_fast_t<1>(b, ldb, k, n, kp, plane, count, colmax, o, scales, st); break;
    }
    ++*launches;
    return cudaGetLastError();
  }
  dim3 grid2(static_cast<unsigned>((kp + 63) / 64), static_cast<unsigned>((n + 63) / 64));
  if (out_is_i64)
    slice_cols_kernel<long long><<<grid2, 256, 0, st>>>(b, ldb, k, n, kp, plane, width, count, mode,
                                                        colmax, static_cast<long long*>(out),
                                                        scales);
  else
    slice_cols_kernel<int8_t><<<grid2, 256, 0, st>>>(b, ldb, k, n, kp, plane, width, count, mode,
                                                     colmax, static_cast<int8_t*>(out), scales);
  ++*launches;
  return cudaGetLastError();
}

}  // namespace ozgpu
