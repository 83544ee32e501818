// Host-side plan logic of the Ozaki-I scheme, restated from the reference's
// specification (O(s^2) scalar code that stays on the host).  Each function
// cites the reference definition it mirrors; errors are thrown as the same
// std exception classes with the reference's messages, and converted to
// ozgpu error codes at the C-ABI boundary.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "ozgpu.h"

namespace ozgpu {

struct SelectionInfeasibleError : std::runtime_error {
  SelectionInfeasibleError(const std::string& msg, double g, double l, double t)
      : std::runtime_error(msg), gap(g), best_lhs(l), target(t) {}
  double gap, best_lhs, target;
};
struct OverflowError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ceil(log2 k), k >= 1 (mma_sim.cpp:27-30 / scheme.cpp:27-29)
inline int ceil_log2(int64_t k) {
  uint64_t u = static_cast<uint64_t>(k) - 1;
  int w = 0;
  while (u) {
    ++w;
    u >>= 1;
  }
  return w;
}

// MmaConfig::validate, mma_sim.cpp:34-41
inline void validate_cfg(const ozgpu_mma_config& c) {
  if (c.input_width < 1) throw std::invalid_argument("MmaConfig: input width must be >= 1");
  if (c.acc_width > 62)
    throw std::invalid_argument("MmaConfig: accumulator width above 62 is not modeled");
  if (c.acc_width < 2 * c.input_width + 1)
    throw std::invalid_argument("MmaConfig: accumulator cannot hold even a single product");
}

// mma_sim.cpp:50-59
inline int optimal_slice_width(const ozgpu_mma_config& c, int64_t k) {
  validate_cfg(c);
  if (k < 1) throw std::invalid_argument("optimal_slice_width: k must be >= 1");
  int t = std::min(c.input_width, (c.acc_width - ceil_log2(k)) / 2);
  if (t < 1)
    throw std::domain_error("optimal_slice_width: inner dimension " + std::to_string(k) +
                            " exceeds what I_" + std::to_string(c.acc_width) +
                            " accumulation supports");
  return t;
}

// mma_sim.cpp:66-72
inline int64_t max_inner_dim(const ozgpu_mma_config& c) {
  validate_cfg(c);
  int headroom = c.acc_width + 1 - 2 * (c.input_width + 1);
  if (headroom < 0)
    throw std::domain_error("max_inner_dim: accumulator too narrow for the input width");
  return int64_t{1} << headroom;
}

// scheme.cpp:46-52
inline int64_t chi(int sa, int sb) {
  if (sa < 1 || sb < 1) throw std::invalid_argument("chi: slice counts must be >= 1");
  int64_t lo = std::min(sa, sb), hi = std::max(sa, sb);
  return lo * (2 * hi - lo + 1) / 2;
}

// scheme.cpp:54-62
inline int64_t spare_carries(int first, int last, int width) {
  if (first < 1 || last < first || width < 1 || width > 61)
    throw std::invalid_argument("spare_carries: bad arguments");
  __int128 span = last - first + 1;
  __int128 v = span * ((static_cast<__int128>(1) << (width + 1)) - last - first) / 2;
  if (v > INT64_MAX || v < INT64_MIN)
    throw std::overflow_error("spare_carries: result out of range");
  return static_cast<int64_t>(v);
}

struct Levels {
  std::vector<std::pair<int, int>> levels;
  long long inexact_adds = 0;
};

// scheme.cpp:64-95
inline Levels plan_levels(int precision, int width, int acc_bits_used, int diagonals) {
  if (width < 1) throw std::invalid_argument("plan_levels: width must be >= 1");
  Levels out;
  if (diagonals < 1) return out;
  int extra = 0;
  if (diagonals >= 2) {
    int64_t eta = spare_carries(1, diagonals - 1, width);
    if (eta < 0) extra = ceil_log2(-eta);
  }
  int headroom = precision - acc_bits_used - 1 - extra;
  int per_level = headroom >= 0 ? headroom / width : 0;
  int first = 0;
  bool initial = true;
  while (first < diagonals) {
    int size = initial ? per_level + 1 : std::max(per_level, 1);
    int last = std::min(first + size - 1, diagonals - 1);
    out.levels.emplace_back(first, last);
    first = last + 1;
    initial = false;
  }
  out.inexact_adds = static_cast<long long>(out.levels.size()) - 1;
  return out;
}

// scheme.cpp:97-106
inline int64_t diagonal_flush_threshold(const ozgpu_mma_config& c, int width, int64_t k) {
  validate_cfg(c);
  if (width < 1 || k < 1) throw std::invalid_argument("diagonal_flush_threshold: bad arguments");
  int headroom = c.acc_width - 2 * width - ceil_log2(k);
  if (headroom < 0)
    throw std::domain_error("diagonal_flush_threshold: accumulator cannot hold one product sum");
  return int64_t{1} << std::min(headroom, 62);
}

// Schedule::max_diag_sum, scheme.cpp:39-44
inline int max_diag_sum(const ozgpu_plan& p) {
  int base = p.schedule == 0 ? p.slices_a + p.slices_b : std::max(p.slices_a, p.slices_b) + 1;
  if (p.diag_sum_limit > 0) base = std::min(base, p.diag_sum_limit);
  return std::max(base, 2);
}

// Pairs on diagonal d (0-based, l + h = d + 2), scheme.cpp:111-116,255-262
inline int diagonal_width(int d, int sa, int sb) {
  int sum = d + 2;
  int lo = std::max(1, sum - sb), hi = std::min(sa, sum - 1);
  return std::max(0, hi - lo + 1);
}
inline int diagonal_first_l(int d, int sb) { return std::max(1, d + 2 - sb); }

inline void set_levels(ozgpu_plan& p, const Levels& lv) {
  p.num_levels = static_cast<int>(lv.levels.size());
  for (int i = 0; i < p.num_levels && i < OZGPU_MAX_LEVELS; ++i) {
    p.levels[2 * i] = lv.levels[i].first;
    p.levels[2 * i + 1] = lv.levels[i].second;
  }
  p.level_inexact_adds = lv.inexact_adds;
}

// scheme.cpp:127-168
inline ozgpu_plan make_plan(const ozgpu_mma_config& c, int64_t k, int sa, int sb, int schedule,
                            int strategy, int mode, int precision) {
  if (sa < 1 || sb < 1) throw std::invalid_argument("make_plan: slice counts must be >= 1");
  ozgpu_plan p{};
  p.slices_a = sa;
  p.slices_b = sb;
  p.schedule = schedule;
  p.diag_sum_limit = 0;
  p.strategy = strategy;
  p.mode = mode;
  p.precision = precision;
  p.width = optimal_slice_width(c, k);
  p.acc_bits_used = 2 * p.width + ceil_log2(k);
  int diagonals = max_diag_sum(p) - 1;
  Levels lv = plan_levels(precision, p.width, p.acc_bits_used, diagonals);
  if (lv.levels.size() > OZGPU_MAX_LEVELS)
    throw std::invalid_argument("make_plan: more than 128 levels");
  set_levels(p, lv);
  switch (strategy) {
    case 0: {
      int64_t total = 0;
      for (int d = 0; d < diagonals; ++d) total += diagonal_width(d, sa, sb);
      p.psi = total - 1;
      break;
    }
    case 2:
      p.psi = lv.inexact_adds;
      break;
    case 1: {
      int64_t flush = diagonal_flush_threshold(c, p.width, k);
      if (p.precision < c.acc_width)
        flush = std::min(flush, int64_t{1} << std::max(0, p.precision - p.acc_bits_used));
      int64_t chunks = 0;
      for (int d = 0; d < diagonals; ++d) {
        int w = diagonal_width(d, sa, sb);
        if (w > 0) chunks += (w + flush - 1) / flush;
      }
      p.psi = chunks - 1;
      break;
    }
    default:
      throw std::invalid_argument("make_plan: unknown accumulation strategy");
  }
  p.psi = std::max(p.psi, 0LL);
  return p;
}

// analysis.cpp:79-84
inline double gamma_factor(int64_t n, double u) {
  if (n < 0) throw std::invalid_argument("gamma_factor: n must be >= 0");
  double nu = static_cast<double>(n) * u;
  if (nu >= 1.0) throw std::domain_error("gamma_factor: n*u >= 1, bound is meaningless");
  return nu / (1.0 - nu);
}

// analysis.cpp:142-207
ozgpu_selection select_slices(double kappa_a, double kappa_b, int width, double u, int s_max,
                              bool has_target, double target, int schedule, int strategy,
                              int acc_bits_used, int precision);

}  // namespace ozgpu
