// Bit-level numerics shared by the slicing and combine kernels.  Written as
// __host__ __device__ so the same code is unit-tested on the host build
// (tests/test_numeric_host.py compiles tools/numeric_selftest.cpp) — the
// product itself only runs them on the GPU.
#pragma once

#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define OZ_HD __host__ __device__ __forceinline__
#else
#define OZ_HD inline
#endif

namespace ozgpu {

OZ_HD uint64_t dbl_bits(double x) {
#ifdef __CUDA_ARCH__
  return static_cast<uint64_t>(__double_as_longlong(x));
#else
  uint64_t b;
  memcpy(&b, &x, sizeof b);
  return b;
#endif
}
OZ_HD double bits_dbl(uint64_t b) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double(static_cast<long long>(b));
#else
  double x;
  memcpy(&x, &b, sizeof x);
  return x;
#endif
}
OZ_HD int clz64(uint64_t x) {
#ifdef __CUDA_ARCH__
  return __clzll(static_cast<long long>(x));
#else
  return x ? __builtin_clzll(x) : 64;
#endif
}
OZ_HD double u64_to_double_rn(uint64_t x) {
#ifdef __CUDA_ARCH__
  return __ull2double_rn(x);
#else
  return static_cast<double>(x);
#endif
}

// proj/src/slicing.cpp:35-45 (extract_field)
OZ_HD uint64_t extract_field(uint64_t sig, int lsb_pos, int end, int nbits) {
  uint64_t mask = (static_cast<uint64_t>(1) << nbits) - 1;
  int shift = end - lsb_pos;
  if (shift >= 0) {
    if (shift >= nbits) return 0;
    return (sig & (mask >> shift)) << shift;
  }
  int down = -shift;
  if (down >= 64) return 0;
  return (sig >> down) & mask;
}

// Per-entry slicing state: significand view (fpcore.cpp:58-74) in the
// block fixed-point frame (slicing.cpp:97-104) plus, in nearest mode, the
// value rounded at the last kept bit (slicing.cpp:112-128: RN-even with the
// carry rippling upward; slice 0 absorbs the final carry).
struct SliceEntry {
  uint64_t sig;
  uint64_t rounded;  // nearest mode with dropped bits: RN(|x| 2^(end_last-q))
  int lsb_pos;
  int neg;
  int has_rounded;
};

OZ_HD SliceEntry make_slice_entry(double x, int q, int width, int count, int mode) {
  SliceEntry s;
  uint64_t bits = dbl_bits(x);
  s.neg = static_cast<int>(bits >> 63);
  bits &= 0x7FFFFFFFFFFFFFFFULL;
  uint64_t biased = bits >> 52;
  uint64_t frac = bits & ((static_cast<uint64_t>(1) << 52) - 1);
  int e;
  if (biased == 0) {
    s.sig = frac;
    e = -1022;
  } else {
    s.sig = frac | (static_cast<uint64_t>(1) << 52);
    e = static_cast<int>(biased) - 1023;
  }
  s.lsb_pos = q + 52 - e;
  s.has_rounded = 0;
  s.rounded = 0;
  if (mode == 1 && s.sig != 0) {
    int end_last = count * width - 1;
    int dropped = s.lsb_pos - end_last;
    if (dropped > 0) {
      uint64_t kept, rem, half;
      bool can_round;
      if (dropped >= 64) {
        kept = 0;
        rem = s.sig;
        can_round = dropped - 1 < 64;
        half = can_round ? (static_cast<uint64_t>(1) << (dropped - 1)) : 0;
      } else {
        kept = s.sig >> dropped;
        rem = s.sig & ((static_cast<uint64_t>(1) << dropped) - 1);
        half = static_cast<uint64_t>(1) << (dropped - 1);
        can_round = true;
      }
      bool up = can_round && (rem > half || (rem == half && (kept & 1)));
      s.rounded = kept + (up ? 1 : 0);
      s.has_rounded = 1;
    }
  }
  return s;
}

// Slice l (0 = most significant) of an entry, sign applied
// (slicing.cpp:95-111 truncate; :112-128 nearest).
OZ_HD long long slice_of(const SliceEntry& s, int l, int width, int count, int mode) {
  if (s.sig == 0) return 0;
  uint64_t v;
  if (mode == 0) {
    v = extract_field(s.sig, s.lsb_pos, (l + 1) * width, width);
  } else {
    int end = (l + 1) * width - 1;
    int start = l == 0 ? 1 : l * width;
    int nbits = end - start + 1;
    if (!s.has_rounded) {
      v = extract_field(s.sig, s.lsb_pos, end, nbits);
    } else {
      int sh = (count * width - 1) - end;
      v = sh >= 64 ? 0 : (s.rounded >> sh);
      if (l > 0) v &= (static_cast<uint64_t>(1) << nbits) - 1;
    }
  }
  long long r = static_cast<long long>(v);
  return s.neg ? -r : r;
}

// ldexp with IEEE round-to-nearest-even on underflow and +-inf on overflow
// (the std::ldexp the reference uses, scheme.cpp:213, oracle.cpp:178).
// d must be finite.
OZ_HD double ldexp_rn(double d, long e) {
  uint64_t bits = dbl_bits(d);
  uint64_t sign = bits & 0x8000000000000000ULL;
  bits &= 0x7FFFFFFFFFFFFFFFULL;
  if (bits == 0) return d;
  long be = static_cast<long>(bits >> 52);
  uint64_t sig = bits & ((static_cast<uint64_t>(1) << 52) - 1);
  if (be == 0) {  // subnormal input: normalise
    int lead = 63 - clz64(sig);
    int up = 52 - lead;
    sig <<= up;
    be = 1 - up;
    sig &= (static_cast<uint64_t>(1) << 52) - 1;
  }
  sig |= static_cast<uint64_t>(1) << 52;
  long ne = be + e;
  if (ne >= 2047) return bits_dbl(sign | 0x7FF0000000000000ULL);
  if (ne >= 1) return bits_dbl(sign | (static_cast<uint64_t>(ne) << 52) | (sig & ((static_cast<uint64_t>(1) << 52) - 1)));
  long sh = 1 - ne;  // >= 1
  if (sh > 54) return bits_dbl(sign);
  uint64_t q = sig >> sh;
  uint64_t rem = sig & ((static_cast<uint64_t>(1) << sh) - 1);
  uint64_t half = static_cast<uint64_t>(1) << (sh - 1);
  if (rem > half || (rem == half && (q & 1))) ++q;
  return bits_dbl(sign | q);
}

// v += s * 2^shift on a W-word little-endian two's-complement integer.
template <int W>
OZ_HD void words_add_shifted(uint64_t (&v)[W], int32_t s, int shift) {
  const int w0 = shift >> 6, b = shift & 63;
  const int64_t s64 = s;
  const uint64_t lo = static_cast<uint64_t>(s64) << b;
  const uint64_t ext = s64 < 0 ? ~static_cast<uint64_t>(0) : 0;
  const uint64_t hi = b ? static_cast<uint64_t>(s64 >> (64 - b)) : ext;
  uint64_t carry = 0;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    uint64_t add = w < w0 ? 0 : (w == w0 ? lo : (w == w0 + 1 ? hi : ext));
    uint64_t t = v[w] + add;
    uint64_t c1 = t < v[w];
    uint64_t t2 = t + carry;
    uint64_t c2 = t2 < t;
    v[w] = w < w0 ? v[w] : t2;
    carry = w < w0 ? 0 : (c1 | c2);
  }
}

// RN(v * 2^e) exactly as ExactValue::to_double (oracle.cpp:157-180): keep
// 55 bits, fold the rest into a sticky low bit, convert once, then ldexp.
template <int W>
OZ_HD double round_words(const uint64_t (&v)[W], long e) {
  const bool neg = (v[W - 1] >> 63) != 0;
  uint64_t mag[W];
  uint64_t carry = 1;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    if (neg) {
      uint64_t t = ~v[w] + carry;
      carry = (carry && t == 0) ? 1 : 0;
      mag[w] = t;
    } else {
      mag[w] = v[w];
    }
  }
  int top = -1;
#pragma unroll
  for (int w = 0; w < W; ++w)
    if (mag[w]) top = w;
  if (top < 0) return 0.0;
  uint64_t topw = 0;
#pragma unroll
  for (int w = 0; w < W; ++w)
    if (w == top) topw = mag[w];
  const int nbits = top * 64 + (64 - clz64(topw));
  uint64_t low;
  if (nbits > 55) {
    const int drop = nbits - 55;
    const int w0 = drop >> 6, b0 = drop & 63;
    bool sticky = false;
    uint64_t a = 0, bnext = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      if (w < w0 && mag[w]) sticky = true;
      if (w == w0) {
        a = mag[w];
        if (b0 && (mag[w] & ((static_cast<uint64_t>(1) << b0) - 1))) sticky = true;
      }
      if (w == w0 + 1) bnext = mag[w];
    }
    low = b0 ? ((a >> b0) | (bnext << (64 - b0))) : a;
    low &= (static_cast<uint64_t>(1) << 55) - 1;
    e += drop;
    if (sticky && (low & 1) == 0) low += 1;
  } else {
    low = mag[0];
  }
  double d = ldexp_rn(u64_to_double_rn(low), e);
  return neg ? -d : d;
}

// round_words<2> specialised for a signed 128-bit value (the Horner combine):
// same result, roughly a third of the instructions.
OZ_HD double round_i128(unsigned __int128 v, long e) {
  const bool neg = static_cast<int64_t>(static_cast<uint64_t>(v >> 64)) < 0;
  if (neg) v = ~v + 1;
  const uint64_t hi = static_cast<uint64_t>(v >> 64), lo = static_cast<uint64_t>(v);
  if ((hi | lo) == 0) return 0.0;
  const int nbits = hi ? 128 - clz64(hi) : 64 - clz64(lo);
  uint64_t low;
  if (nbits > 55) {
    const int drop = nbits - 55;
    low = static_cast<uint64_t>(v >> drop);
    const bool sticky = (v << (128 - drop)) != 0;
    e += drop;
    if (sticky) low |= 1;  // round-to-odd at 55 bits == the reference's +1 on even
  } else {
    low = lo;
  }
  // |value| = low * 2^e with low < 2^55: convert (RN-even) then scale; the
  // common case (normal result) is a plain exponent add.
  const double d = u64_to_double_rn(low);
  const uint64_t bits = dbl_bits(d);
  const long ne = static_cast<long>(bits >> 52) + e;
  double r;
  if (ne >= 1 && ne <= 2046)
    r = bits_dbl((bits & 0x800FFFFFFFFFFFFFULL) | (static_cast<uint64_t>(ne) << 52));
  else
    r = ldexp_rn(d, e);
  return neg ? -r : r;
}

// The rare path of round_hilo, kept out of line so the combine kernel's
// common path stays small in registers.
#ifdef __CUDACC__
static __host__ __device__ __noinline__
#else
static inline
#endif
double round_hilo_slow(uint64_t hi, uint64_t lo, long e) {
  const unsigned __int128 v = (static_cast<unsigned __int128>(hi) << 64) | lo;
  return round_i128(v, e);
}

// 2^x as a double, x in [-1022, 1023] (normal range only).
OZ_HD double pow2_normal(long x) { return bits_dbl(static_cast<uint64_t>(x + 1023) << 52); }

// RN(v * 2^e) for the signed 128-bit value v = hi * 2^64 + lo (lo unsigned)
// -- the same result as round_i128 (and so ExactValue::to_double,
// oracle.cpp:157-180) but with two exact conversions and one rounding IEEE
// operation on the common path:
//   v = H + L with H = hi * 2^64 and L = lo.  Rounding L to odd at
//   granularity 2^12, L' = ((lo >> 12) | sticky) * 2^12, commutes with adding
//   H (a multiple of 2^13).  When |v| >= 2^66 (hi >= 4 or hi <= -5) the
//   result's ulp is >= 2^14 = 4 * 2^12, so RN(H + L') == RN(v) (round-to-odd
//   with two extra bits, Boldo-Melquiond).  hi (|hi| < 2^51) and lo >> 12
//   (52 bits) convert exactly with the 2^52 magic-number trick on the FP64
//   pipe (no integer->double conversion unit), the scale 2^e is applied to
//   both terms exactly while -1034 <= e <= 900, and one FMA rounds once.
//   Everything else takes round_i128.
OZ_HD double round_hilo(uint64_t hi, uint64_t lo, long e) {
  const int64_t h = static_cast<int64_t>(hi);
  const int64_t l = static_cast<int64_t>(lo);
  if (h == (l >> 63) && e >= -1000 && e <= 900) {
    // v fits in int64 (few diagonals, e.g. s = 3): one correctly rounded
    // conversion (exact below 2^51 via the magic number), then an exact
    // power-of-two scale -- the result is normal for these e
    if (l == 0) return 0.0;
    double d;
    if (l < (int64_t{1} << 51) && l > -(int64_t{1} << 51)) {
#ifdef __CUDA_ARCH__
      d = __dsub_rn(bits_dbl(0x4338000000000000ULL + static_cast<uint64_t>(l)), 6755399441055744.0);
#else
      d = bits_dbl(0x4338000000000000ULL + static_cast<uint64_t>(l)) - 6755399441055744.0;
#endif
    } else {
#ifdef __CUDA_ARCH__
      d = __ll2double_rn(l);
#else
      d = static_cast<double>(l);
#endif
    }
#ifdef __CUDA_ARCH__
    return __dmul_rn(d, pow2_normal(e));
#else
    return d * pow2_normal(e);
#endif
  }
  const bool big = (h >= 4 || h <= -5) && h < (int64_t{1} << 51) && h > -(int64_t{1} << 51);
  if (big && e >= -1034 && e <= 900) {
    const uint64_t lr = (lo >> 12) | ((lo & 0xFFF) != 0);
    // exact: 0x1.8p52 + h and 0x1p52 + lr are representable, their
    // differences with the magic constants are exact
#ifdef __CUDA_ARCH__
    const double hf = __dsub_rn(bits_dbl(0x4338000000000000ULL + static_cast<uint64_t>(h)),
                                6755399441055744.0);
    const double lf = __dsub_rn(bits_dbl(0x4330000000000000ULL | lr), 4503599627370496.0);
    return __fma_rn(hf, pow2_normal(64 + e), __dmul_rn(lf, pow2_normal(12 + e)));
#else
    const double hf = bits_dbl(0x4338000000000000ULL + static_cast<uint64_t>(h)) -
                      6755399441055744.0;
    const double lf = bits_dbl(0x4330000000000000ULL | lr) - 4503599627370496.0;
    return __builtin_fma(hf, pow2_normal(64 + e), lf * pow2_normal(12 + e));
#endif
  }
  return round_hilo_slow(hi, lo, e);
}

// The 192-bit counterpart of round_hilo for v = w2 * 2^128 + w1 * 2^64 + w0
// (w1, w0 unsigned): values that fit 128 bits go through round_hilo; for
// |v| >= 2^130 (w2 >= 4 or w2 <= -5) the low 128 bits are rounded to odd at
// granularity 2^76 (52 bits, exact in a double) and added to w2 * 2^128 with
// one FMA -- the same argument as round_hilo, two guard bits.  The rest goes
// through round_words<3>.
#ifdef __CUDACC__
static __host__ __device__ __noinline__
#else
static inline
#endif
double round_w3_rest(uint64_t w2, uint64_t w1, uint64_t w0, long e);

OZ_HD double round_w3(uint64_t w2, uint64_t w1, uint64_t w0, long e) {
  const int64_t h = static_cast<int64_t>(w2);
  if (h == (static_cast<int64_t>(w1) >> 63)) return round_hilo(w1, w0, e);
  const bool big = (h >= 4 || h <= -5) && h < (int64_t{1} << 51) && h > -(int64_t{1} << 51);
  if (big && e >= -1098 && e <= 844) {
    const uint64_t lr = (w1 >> 12) | (((w1 & 0xFFF) | w0) != 0);
#ifdef __CUDA_ARCH__
    const double hf = __dsub_rn(bits_dbl(0x4338000000000000ULL + static_cast<uint64_t>(h)),
                                6755399441055744.0);
    const double lf = __dsub_rn(bits_dbl(0x4330000000000000ULL | lr), 4503599627370496.0);
    return __fma_rn(hf, pow2_normal(128 + e), __dmul_rn(lf, pow2_normal(76 + e)));
#else
    const double hf = bits_dbl(0x4338000000000000ULL + static_cast<uint64_t>(h)) -
                      6755399441055744.0;
    const double lf = bits_dbl(0x4330000000000000ULL | lr) - 4503599627370496.0;
    return __builtin_fma(hf, pow2_normal(128 + e), lf * pow2_normal(76 + e));
#endif
  }
  return round_w3_rest(w2, w1, w0, e);
}

#ifdef __CUDACC__
static __host__ __device__ __noinline__
#else
static inline
#endif
double round_w3_rest(uint64_t w2, uint64_t w1, uint64_t w0, long e) {
  const uint64_t v[3] = {w0, w1, w2};
  return round_words<3>(v, e);
}

}  // namespace ozgpu
