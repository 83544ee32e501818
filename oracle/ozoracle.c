/* ozoracle.c -- plain-C CPU restatement of the reference's Ozaki-I hot path
 * (arxiv/paper_2506_11277, proj/).  TEST INFRASTRUCTURE ONLY: see ozoracle.h.
 *
 * Every function cites the reference file:line it restates.  Parity of this
 * restatement is pinned in tests/test_oracle.py against the reference's own
 * golden vectors and against the compiled reference (oracle/_ref).
 */
#include "ozoracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef __int128 i128;
typedef unsigned __int128 u128;

/* ---------------------------------------------------------------- helpers */

/* ceil(log2 k) for k >= 1: std::bit_width(k - 1) (proj/src/mma_sim.cpp:27-30) */
static int ceil_log2_i64(int64_t k) {
  uint64_t u = (uint64_t)k - 1;
  int w = 0;
  while (u) {
    ++w;
    u >>= 1;
  }
  return w;
}

static int imax(int a, int b) { return a > b ? a : b; }
static int imin(int a, int b) { return a < b ? a : b; }

/* proj/src/fpcore.cpp:58-74 (significand_view) */
static void significand_view(double x, uint64_t* sig, int* exponent, int* negative) {
  uint64_t bits;
  memcpy(&bits, &x, sizeof bits);
  *negative = (int)(bits >> 63);
  bits &= ~(UINT64_C(1) << 63);
  uint64_t biased = bits >> 52;
  uint64_t frac = bits & ((UINT64_C(1) << 52) - 1);
  if (biased == 0) {
    *sig = frac;
    *exponent = -1022;
  } else {
    *sig = frac | (UINT64_C(1) << 52);
    *exponent = (int)biased - 1023;
  }
}

/* proj/src/fpcore.cpp:83-87 (scale_exponent_direct = ilogb(m) + 1) */
static int scale_exponent_direct(double m) { return ilogb(m) + 1; }

/* ------------------------------------------------------------------- plan */

/* proj/src/mma_sim.cpp:50-59 */
int ozo_optimal_slice_width(int t_in, int t_acc, int64_t k) {
  int t = (t_acc - ceil_log2_i64(k)) / 2;
  return t_in < t ? t_in : t;
}

/* proj/src/scheme.cpp:46-52 */
int64_t ozo_chi(int sa, int sb) {
  int64_t lo = imin(sa, sb), hi = imax(sa, sb);
  return lo * (2 * hi - lo + 1) / 2;
}

/* proj/src/scheme.cpp:54-62 */
int64_t ozo_spare_carries(int first, int last, int width) {
  i128 span = last - first + 1;
  i128 value = span * (((i128)1 << (width + 1)) - last - first) / 2;
  return (int64_t)value;
}

/* proj/src/scheme.cpp:64-95 */
int ozo_plan_levels(int precision, int width, int acc_bits_used, int diagonals,
                    int* levels_out, int max_levels) {
  if (diagonals < 1) return 0;
  int extra = 0;
  if (diagonals >= 2) {
    int64_t eta = ozo_spare_carries(1, diagonals - 1, width);
    if (eta < 0) extra = ceil_log2_i64(-eta);
  }
  int headroom = precision - acc_bits_used - 1 - extra;
  int per_level = headroom >= 0 ? headroom / width : 0;
  int first = 0, count = 0, initial = 1;
  while (first < diagonals) {
    int size = initial ? per_level + 1 : imax(per_level, 1);
    int last = imin(first + size - 1, diagonals - 1);
    if (count < max_levels && levels_out) {
      levels_out[2 * count] = first;
      levels_out[2 * count + 1] = last;
    }
    ++count;
    first = last + 1;
    initial = 0;
  }
  return count;
}

/* proj/src/scheme.cpp:39-44 */
int ozo_max_diag_sum(int schedule, int diag_sum_limit, int sa, int sb) {
  int base = schedule == 0 ? sa + sb : imax(sa, sb) + 1;
  if (diag_sum_limit > 0) base = imin(base, diag_sum_limit);
  return imax(base, 2);
}

/* ---------------------------------------------------------------- slicing */

/* proj/src/slicing.cpp:28-31 */
static int start_bit(int index, int width, int mode) {
  if (mode == 1) return index == 0 ? 1 : index * width;
  return index * width + 1;
}
/* proj/include/ozmul/slicing.hpp:59-62 */
static int end_bit(int index, int width, int mode) {
  int last = (index + 1) * width;
  return mode == 1 ? last - 1 : last;
}

/* proj/src/slicing.cpp:35-45 */
static uint64_t extract_field(uint64_t significand, int lsb_pos, int end, int nbits) {
  uint64_t mask = (UINT64_C(1) << nbits) - 1;
  int shift = end - lsb_pos;
  if (shift >= 0) {
    if (shift >= nbits) return 0;
    return (significand & (mask >> shift)) << shift;
  }
  int down = -shift;
  if (down >= 64) return 0;
  return (significand >> down) & mask;
}

/* proj/src/slicing.cpp:50-65 */
static int rounds_up(uint64_t significand, int lsb_pos, int kept_end, int kept_lsb_odd) {
  int dropped = lsb_pos - kept_end;
  if (dropped <= 0) return 0;
  uint64_t rem, half;
  if (dropped >= 64) {
    if (dropped - 1 >= 64) return 0;
    rem = significand;
    half = UINT64_C(1) << (dropped - 1);
  } else {
    rem = significand & ((UINT64_C(1) << dropped) - 1);
    half = UINT64_C(1) << (dropped - 1);
  }
  if (rem > half) return 1;
  if (rem < half) return 0;
  return kept_lsb_odd;
}

/* proj/src/slicing.cpp:67-132 */
int ozo_split(int orientation, int64_t rows, int64_t cols, const double* x, int width,
              int count, int mode, int64_t* slices_out, int* scales_out) {
  if (width < 1 || width > 62 || count < 1) return 1;
  if (mode == 1 && width < 2) return 1;
  int64_t blocks = orientation == 0 ? rows : cols;
  int64_t len = orientation == 0 ? cols : rows;
  int64_t plane = rows * cols;
  memset(slices_out, 0, sizeof(int64_t) * (size_t)(plane * count));
  for (int64_t b = 0; b < blocks; ++b) {
    double max_abs = 0.0;
    for (int64_t j = 0; j < len; ++j) {
      double v = orientation == 0 ? x[b * cols + j] : x[j * cols + b];
      if (!isfinite(v)) return 1;
      if (fabs(v) > max_abs) max_abs = fabs(v);
    }
    int q = max_abs == 0.0 ? 0 : scale_exponent_direct(max_abs);
    scales_out[b] = q;
    for (int64_t j = 0; j < len; ++j) {
      int64_t r = orientation == 0 ? b : j;
      int64_t c = orientation == 0 ? j : b;
      uint64_t sig;
      int e, neg;
      significand_view(x[r * cols + c], &sig, &e, &neg);
      if (sig == 0) continue;
      int lsb_pos = q + 52 - e;
      int64_t sign = neg ? -1 : 1;
      for (int l = 0; l < count; ++l) {
        int end = end_bit(l, width, mode);
        int nbits = end - start_bit(l, width, mode) + 1;
        uint64_t v = extract_field(sig, lsb_pos, end, nbits);
        slices_out[l * plane + r * cols + c] = sign * (int64_t)v;
      }
      if (mode == 1) {
        int last = count - 1;
        int64_t last_v = llabs(slices_out[last * plane + r * cols + c]);
        if (rounds_up(sig, lsb_pos, end_bit(last, width, mode), (last_v & 1) != 0)) {
          for (int l = last; l >= 0; --l) {
            int nbits = end_bit(l, width, mode) - start_bit(l, width, mode) + 1;
            int64_t cap = (int64_t)1 << nbits;
            int64_t v = llabs(slices_out[l * plane + r * cols + c]) + 1;
            if (v < cap || l == 0) {
              slices_out[l * plane + r * cols + c] = sign * v;
              break;
            }
            slices_out[l * plane + r * cols + c] = 0;
          }
        }
      }
    }
  }
  return 0;
}

/* ------------------------------------------------------- integer products */

/* proj/src/mma_sim.cpp:76-114 */
int ozo_integer_gemm(int64_t m, int64_t k, int64_t n, const int64_t* x, const int64_t* y,
                     int64_t* out, int t_in, int t_acc) {
  int64_t in_lo = -((int64_t)1 << t_in), in_hi = ((int64_t)1 << t_in) - 1;
  for (int64_t i = 0; i < m * k; ++i)
    if (x[i] < in_lo || x[i] > in_hi) return 2;
  for (int64_t i = 0; i < k * n; ++i)
    if (y[i] < in_lo || y[i] > in_hi) return 2;
  i128 lo = -((i128)1 << t_acc), hi = ((i128)1 << t_acc) - 1;
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      i128 acc = 0;
      for (int64_t r = 0; r < k; ++r) {
        acc += (i128)x[i * k + r] * y[r * n + j];
        if (acc < lo || acc > hi) return 5;
      }
      out[i * n + j] = (int64_t)acc;
    }
  return 0;
}

/* ------------------------------------------------------ exact rounding */

/* proj/src/oracle.cpp:157-180 (ExactValue::to_double): keep 55 bits, fold
 * the rest into a sticky (round-to-odd), convert, then ldexp. */
double ozo_round_words(const uint64_t* v, int words, long exp) {
  uint64_t* mag = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)words);
  int neg = (int)(v[words - 1] >> 63);
  if (neg) {
    uint64_t carry = 1;
    for (int w = 0; w < words; ++w) {
      uint64_t t = ~v[w];
      mag[w] = t + carry;
      carry = (carry && mag[w] == 0) ? 1 : 0;
    }
  } else {
    memcpy(mag, v, sizeof(uint64_t) * (size_t)words);
  }
  int top = -1;
  for (int w = words - 1; w >= 0; --w)
    if (mag[w]) {
      top = w;
      break;
    }
  if (top < 0) {
    free(mag);
    return 0.0;
  }
  int nbits = top * 64 + (64 - __builtin_clzll(mag[top]));
  uint64_t low;
  if (nbits > 55) {
    int drop = nbits - 55;
    int sticky = 0;
    for (int w = 0; w < words && w * 64 < drop; ++w) {
      int hi_bit = drop - w * 64; /* bits [w*64, w*64+hi_bit) are dropped */
      uint64_t mask = hi_bit >= 64 ? ~UINT64_C(0) : ((UINT64_C(1) << hi_bit) - 1);
      if (mag[w] & mask) sticky = 1;
    }
    int w0 = drop / 64, b0 = drop % 64;
    low = mag[w0] >> b0;
    if (b0 && w0 + 1 < words) low |= mag[w0 + 1] << (64 - b0);
    exp += drop;
    if (sticky && (low & 1) == 0) low += 1;
  } else {
    low = mag[0];
  }
  free(mag);
  double d = (double)low;
  double r = ldexp(d, (int)exp);
  return neg ? -r : r;
}

/* signed add of (s << shift) into the two's-complement word vector */
static void words_add_shifted(uint64_t* v, int words, i128 s, int shift) {
  if (s == 0) return;
  int w0 = shift / 64, b = shift % 64;
  /* s << b as a 192-bit signed quantity in three words */
  u128 lo_part = (u128)s << b; /* low 128 bits of s<<b */
  uint64_t parts[3];
  parts[0] = (uint64_t)lo_part;
  parts[1] = (uint64_t)(lo_part >> 64);
  /* bits above 128: arithmetic shift of s by (128 - b) */
  i128 hi = b ? (s >> (127 - b)) >> 1 : (s < 0 ? -1 : 0);
  parts[2] = (uint64_t)hi;
  uint64_t ext = s < 0 ? ~UINT64_C(0) : 0;
  uint64_t carry = 0;
  for (int w = w0; w < words; ++w) {
    int idx = w - w0;
    uint64_t add = idx < 3 ? parts[idx] : ext;
    uint64_t t = v[w] + add;
    uint64_t c1 = t < v[w];
    uint64_t t2 = t + carry;
    uint64_t c2 = t2 < t;
    v[w] = t2;
    carry = c1 | c2;
  }
}

/* The levelled-exact multiply (proj/src/scheme.cpp:219-361, kLevelledExact,
 * level sums exact by the plan and combined by ExactValue with one final
 * rounding, scheme.cpp:339-354) restated as RN of the exact scheduled sum. */
int ozo_multiply_exact(int64_t m, int64_t n, int64_t k, const double* a, const double* b,
                       double* c, int sa, int sb, int schedule, int diag_sum_limit, int mode,
                       int width) {
  /* validation order: scheme.cpp:221-239 */
  for (int64_t i = 0; i < m * k; ++i) {
    double v = a[i];
    if (!isfinite(v) || (v == 0.0 && signbit(v))) return 1;
  }
  for (int64_t i = 0; i < k * n; ++i) {
    double v = b[i];
    if (!isfinite(v) || (v == 0.0 && signbit(v))) return 1;
  }
  if (k < 1) return 1;
  if (2 * width + ceil_log2_i64(k) > 31) return 2;
  if (sa < 1 || sb < 1) return 1;

  int64_t* sla = (int64_t*)malloc(sizeof(int64_t) * (size_t)(sa * m * k));
  int64_t* slb = (int64_t*)malloc(sizeof(int64_t) * (size_t)(sb * k * n));
  int* qa = (int*)malloc(sizeof(int) * (size_t)(m ? m : 1));
  int* qb = (int*)malloc(sizeof(int) * (size_t)(n ? n : 1));
  int rc = ozo_split(0, m, k, a, width, sa, mode, sla, qa);
  if (!rc) rc = ozo_split(1, k, n, b, width, sb, mode, slb, qb);
  if (rc) {
    free(sla), free(slb), free(qa), free(qb);
    return rc;
  }
  int diagonals = ozo_max_diag_sum(schedule, diag_sum_limit, sa, sb) - 1;
  int words = ((diagonals - 1) * width + 70) / 64 + 2;
  uint64_t* acc = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)words);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      memset(acc, 0, sizeof(uint64_t) * (size_t)words);
      for (int d = 0; d < diagonals; ++d) {
        int sum = d + 2;
        int lo = imax(1, sum - sb), hi = imin(sa, sum - 1);
        i128 sd = 0;
        for (int l = lo; l <= hi; ++l) {
          int h = sum - l;
          const int64_t* ar = sla + (int64_t)(l - 1) * m * k + i * k;
          const int64_t* bc = slb + (int64_t)(h - 1) * k * n + j;
          int64_t e = 0;
          for (int64_t r = 0; r < k; ++r) e += ar[r] * bc[r * n];
          sd += e;
        }
        words_add_shifted(acc, words, sd, (diagonals - 1 - d) * width);
      }
      /* weight of the least significant diagonal: scheme.cpp:252-254 */
      long w_last = -(long)(diagonals + 1) * width + (mode == 1 ? 2 : 0);
      c[i * n + j] = ozo_round_words(acc, words, (long)qa[i] + qb[j] + w_last);
    }
  free(acc), free(sla), free(slb), free(qa), free(qb);
  return 0;
}

/* --------------------------------------------------------------- analysis */

/* proj/src/analysis.cpp:25-47 (block_ratios) + :58-68 (scaling_profile) */
static double worst_ratio(int64_t rows, int64_t cols, const double* x, int orientation,
                          int* has_zero) {
  int64_t blocks = orientation == 0 ? rows : cols;
  int64_t len = orientation == 0 ? cols : rows;
  double worst = 1.0;
  *has_zero = 0;
  for (int64_t b = 0; b < blocks; ++b) {
    double mx = 0.0, mn = INFINITY;
    for (int64_t j = 0; j < len; ++j) {
      double v = fabs(orientation == 0 ? x[b * cols + j] : x[j * cols + b]);
      if (v == 0.0) continue;
      if (v > mx) mx = v;
      if (v < mn) mn = v;
    }
    if (mx == 0.0) {
      *has_zero = 1;
      continue;
    }
    double r = mx / mn;
    if (r > worst) worst = r;
  }
  return worst;
}

void ozo_scaling_profile(int64_t m, int64_t k, int64_t n, const double* a, const double* b,
                         double* kappa_a, double* kappa_b, int* a_zero, int* b_zero) {
  *kappa_a = 2.0 * worst_ratio(m, k, a, 0, a_zero);
  *kappa_b = 2.0 * worst_ratio(k, n, b, 1, b_zero);
}

/* proj/src/analysis.cpp:79-84 */
static double gamma_factor(int64_t n, double u) {
  double nu = (double)n * u;
  return nu / (1.0 - nu);
}

/* proj/src/analysis.cpp:142-207 */
int ozo_select_slices(double kappa_a, double kappa_b, int width, double u, int s_max,
                      int has_target, double target, int schedule, int strategy,
                      int acc_bits_used, int precision, int* sa_out, int* sb_out, double* lhs_out,
                      double* target_out, int64_t* products, double* gap) {
  if (width < 1 || s_max < 1 || s_max > 64 || !(u > 0.0) || !(u < 1.0)) return 1;
  if (!(kappa_a > 0.0) || !(kappa_b > 0.0)) return 1;
  int found = 0, bsa = 0, bsb = 0;
  double blhs = 0, btarget = 0;
  int64_t bcost = 0;
  double best_lhs_any = INFINITY, target_at_best = 0.0;
  for (int sa = 1; sa <= s_max; ++sa)
    for (int sb = 1; sb <= s_max; ++sb) {
      double lhs = ldexp(kappa_a, -sa * width) + ldexp(kappa_b, -sb * width);
      double tgt;
      if (has_target) {
        tgt = target;
      } else {
        int diagonals = schedule == 0 ? sa + sb - 1 : imax(sa, sb);
        int64_t psi;
        if (strategy == 2)
          psi = ozo_plan_levels(precision, width, acc_bits_used, diagonals, NULL, 0) - 1;
        else if (strategy == 1)
          psi = diagonals - 1;
        else
          psi = (schedule == 0 ? (int64_t)sa * sb : ozo_chi(sa, sb)) - 1;
        if (psi < 0) psi = 0; /* plan_levels' inexact_adds for an empty plan is 0 */
        tgt = gamma_factor(psi > 1 ? psi : 1, u);
      }
      if (lhs < best_lhs_any) {
        best_lhs_any = lhs;
        target_at_best = tgt;
      }
      if (lhs > tgt) continue;
      int64_t cost = ozo_chi(sa, sb);
      int better;
      if (!found)
        better = 1;
      else if (cost != bcost)
        better = cost < bcost;
      else if (imax(sa, sb) != imax(bsa, bsb))
        better = imax(sa, sb) < imax(bsa, bsb);
      else
        better = sa < bsa;
      if (better) {
        found = 1;
        bsa = sa, bsb = sb, blhs = lhs, btarget = tgt, bcost = cost;
      }
    }
  if (!found) {
    double den = target_at_best > 2.2250738585072014e-308 ? target_at_best : 2.2250738585072014e-308;
    if (gap) *gap = best_lhs_any / den;
    *lhs_out = best_lhs_any;
    *target_out = target_at_best;
    return 4;
  }
  *sa_out = bsa, *sb_out = bsb, *lhs_out = blhs, *target_out = btarget, *products = bcost;
  return 0;
}

/* ------------------------------------------------------------- generators */

/* std::mt19937_64 (the standard's parameters) */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = UINT64_C(6364136223846793005) * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & UINT64_C(0xFFFFFFFF80000000)) |
                   (g->mt[(i + 1) % 312] & UINT64_C(0x7FFFFFFF));
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= UINT64_C(0xB5026F5AA96619E9);
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & UINT64_C(0x5555555555555555);
  y ^= (y << 17) & UINT64_C(0x71D67FFFEDA60000);
  y ^= (y << 37) & UINT64_C(0xFFF7EEE000000000);
  y ^= y >> 43;
  return y;
}

/* proj/src/generators.cpp:25-31 */
static uint64_t splitmix64(uint64_t x) {
  x += UINT64_C(0x9e3779b97f4a7c15);
  x = (x ^ (x >> 30)) * UINT64_C(0xbf58476d1ce4e5b9);
  x = (x ^ (x >> 27)) * UINT64_C(0x94d049bb133111eb);
  return x ^ (x >> 31);
}

/* proj/src/generators.cpp:43-49 */
static double uniform01(mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1p-53; }

/* proj/src/generators.cpp:176-182 (RandomStream(seed) = stream 0) */
void ozo_random_uniform(int64_t m, int64_t n, uint64_t seed, double lo, double hi,
                        double* out) {
  mt64* g = (mt64*)malloc(sizeof(mt64));
  mt64_seed(g, splitmix64(seed + 0));
  for (int64_t i = 0; i < m * n; ++i) out[i] = lo + uniform01(g) * (hi - lo);
  free(g);
}

/* proj/src/generators.cpp:103-140 */
void ozo_gen_kappa_d(int64_t n, double kappa_d, uint64_t seed, int rotate, double* a,
                     double* b) {
  mt64* ga = (mt64*)malloc(sizeof(mt64));
  mt64* gb = (mt64*)malloc(sizeof(mt64));
  mt64_seed(ga, splitmix64(seed + 1));
  mt64_seed(gb, splitmix64(seed + 2));
  for (int64_t i = 0; i < n * n; ++i) a[i] = 1.0 + uniform01(ga) * (2.0 - 1.0);
  for (int64_t i = 0; i < n * n; ++i) b[i] = 1.0 + uniform01(gb) * (2.0 - 1.0);
  free(ga), free(gb);
  double* d = (double*)malloc(sizeof(double) * (size_t)n);
  double log_kd = log(kappa_d);
  for (int64_t i = 0; i < n; ++i) {
    double frac = n > 1 ? (double)i / (double)(n - 1) : 0.5;
    d[i] = exp(log_kd * (frac - 0.5));
  }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      a[i * n + j] *= d[j];
      b[i * n + j] /= d[i];
    }
  free(d);
  if (rotate) {
    double* ra = (double*)malloc(sizeof(double) * (size_t)(n * n));
    double* rb = (double*)malloc(sizeof(double) * (size_t)(n * n));
    for (int64_t i = 0; i < n; ++i) {
      int64_t shift = (i + 1) % n;
      for (int64_t j = 0; j < n; ++j) {
        ra[i * n + (j + shift) % n] = a[i * n + j];
        rb[((j + shift) % n) * n + i] = b[j * n + i];
      }
    }
    memcpy(a, ra, sizeof(double) * (size_t)(n * n));
    memcpy(b, rb, sizeof(double) * (size_t)(n * n));
    free(ra), free(rb);
  }
}
