// C-ABI wrapper over the UNMODIFIED reference library (arxiv/paper_2506_11277,
// /root/reference/proj), compiled from the reference's own sources by
// oracle/Makefile into oracle/_ref/libozref.so.
//
// TEST INFRASTRUCTURE ONLY: this is the parity checker and the CPU baseline
// (bench.py --impl reference / cpu_baseline).  The product never links it.
//
// Each function forwards to the reference symbol cited beside it and maps
// the reference's exceptions to integer codes:
//   0 ok, 1 std::invalid_argument, 2 std::domain_error, 3 other std::exception,
//   4 SelectionInfeasible, 5 MmaOverflowError.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "ozmul/analysis.hpp"
#include "ozmul/generators.hpp"
#include "ozmul/mma_sim.hpp"
#include "ozmul/oracle.hpp"
#include "ozmul/scheme.hpp"
#include "ozmul/slicing.hpp"

using namespace ozmul;

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return 0;
  } catch (const SelectionInfeasible& e) {
    g_last_error = e.what();
    return 4;
  } catch (const MmaOverflowError& e) {
    g_last_error = e.what();
    return 5;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return 1;
  } catch (const std::domain_error& e) {
    g_last_error = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return 3;
  }
}

Matrix to_matrix(std::int64_t rows, std::int64_t cols, const double* p) {
  Matrix m(rows, cols);
  if (rows * cols) std::memcpy(m.data(), p, sizeof(double) * rows * cols);
  return m;
}

MultiplyPlan plan_from(const MmaConfig& cfg, std::int64_t k, int sa, int sb, int schedule,
                       int strategy, int mode, int precision, int diag_sum_limit) {
  // make_plan: proj/src/scheme.cpp:127-168
  MultiplyPlan plan = make_plan(cfg, k, sa, sb, static_cast<ScheduleKind>(schedule),
                                static_cast<Accumulation>(strategy),
                                static_cast<SliceMode>(mode), precision);
  if (diag_sum_limit > 0) plan.schedule.diag_sum_limit = diag_sum_limit;
  return plan;
}

void fill_diag(const Diagnostics& d, std::int64_t* out) {
  if (!out) return;
  out[0] = d.products;
  out[1] = d.integer_adds;
  out[2] = d.float_adds;
  out[3] = d.flushes;
  out[4] = d.realized_psi;
  out[5] = d.planned_psi;
  out[6] = d.width;
  out[7] = d.acc_bits_used;
}

}  // namespace

extern "C" {

const char* ozref_last_error() { return g_last_error.c_str(); }

// proj/src/scheme.cpp:219-361 (multiply); enums follow scheme.hpp:30-49 and
// slicing.hpp (ScheduleKind kFull=0/kReduced=1, Accumulation
// kFloatPerProduct=0/kDiagonalInteger=1/kLevelledExact=2, SliceMode
// kTruncate=0/kNearest=1).
int ozref_multiply(std::int64_t m, std::int64_t n, std::int64_t k, const double* a,
                   const double* b, double* c, int sa, int sb, int schedule, int strategy,
                   int mode, int precision, int diag_sum_limit, int t_in, int t_acc,
                   std::int64_t* diag_out) {
  return guarded([&] {
    MmaConfig cfg{t_in, t_acc};
    Matrix A = to_matrix(m, k, a), B = to_matrix(k, n, b);
    MultiplyPlan plan =
        plan_from(cfg, k, sa, sb, schedule, strategy, mode, precision, diag_sum_limit);
    MultiplyResult r = multiply(A, B, cfg, plan);
    std::memcpy(c, r.c.data(), sizeof(double) * m * n);
    fill_diag(r.diagnostics, diag_out);
  });
}

// multiply() forged with an explicit slice width (scheme_test.cpp:294-302
// forges plan.width to provoke the capacity error).
int ozref_multiply_width(std::int64_t m, std::int64_t n, std::int64_t k, const double* a,
                         const double* b, double* c, int sa, int sb, int width) {
  return guarded([&] {
    MmaConfig cfg = MmaConfig::int8_int32();
    Matrix A = to_matrix(m, k, a), B = to_matrix(k, n, b);
    MultiplyPlan plan = make_plan(cfg, k, sa, sb);
    plan.width = width;
    MultiplyResult r = multiply(A, B, cfg, plan);
    std::memcpy(c, r.c.data(), sizeof(double) * m * n);
  });
}

// The CPU baseline: reference multiply() over `nblocks` C blocks, each
// (i0, i1, j0, j1) with the full inner dimension, one std::thread per block
// up to `threads` at a time.  2-D C blocking is bit-identical to a monolithic
// call because scales are per full row of A / column of B.
// Writes block results into c (m x n, row-major) and returns wall seconds
// in *seconds.
int ozref_multiply_blocks(std::int64_t m, std::int64_t n, std::int64_t k, const double* a,
                          const double* b, double* c, int sa, int sb, int schedule,
                          int strategy, int mode, int precision, int nblocks,
                          const std::int64_t* blocks, int threads, double* seconds) {
  return guarded([&] {
    MmaConfig cfg = MmaConfig::int8_int32();
    MultiplyPlan plan = plan_from(cfg, k, sa, sb, schedule, strategy, mode, precision, 0);
    std::vector<std::string> errors(nblocks);
    auto work = [&](int idx) {
      std::int64_t i0 = blocks[4 * idx], i1 = blocks[4 * idx + 1];
      std::int64_t j0 = blocks[4 * idx + 2], j1 = blocks[4 * idx + 3];
      Matrix A(i1 - i0, k), B(k, j1 - j0);
      for (std::int64_t i = i0; i < i1; ++i)
        std::memcpy(&A(i - i0, 0), a + i * k, sizeof(double) * k);
      for (std::int64_t r = 0; r < k; ++r)
        for (std::int64_t j = j0; j < j1; ++j) B(r, j - j0) = b[r * n + j];
      try {
        MultiplyResult res = multiply(A, B, cfg, plan);
        for (std::int64_t i = i0; i < i1; ++i)
          for (std::int64_t j = j0; j < j1; ++j) c[i * n + j] = res.c(i - i0, j - j0);
      } catch (const std::exception& e) {
        errors[idx] = e.what();
      }
    };
    auto t0 = std::chrono::steady_clock::now();
    int next = 0;
    if (threads < 1) threads = 1;
    while (next < nblocks) {
      std::vector<std::thread> pool;
      for (int t = 0; t < threads && next < nblocks; ++t) pool.emplace_back(work, next++);
      for (auto& th : pool) th.join();
    }
    auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    for (auto& e : errors)
      if (!e.empty()) throw std::runtime_error(e);
  });
}

// proj/src/slicing.cpp:67-132 (split_rows / split_cols).  slices_out is
// [count][rows][cols] int64; scales_out has rows (orientation 0) or cols (1).
int ozref_split(int orientation, std::int64_t rows, std::int64_t cols, const double* x,
                int width, int count, int mode, std::int64_t* slices_out, int* scales_out) {
  return guarded([&] {
    Matrix M = to_matrix(rows, cols, x);
    SlicedMatrix s = orientation == 0 ? split_rows(M, width, count, static_cast<SliceMode>(mode))
                                      : split_cols(M, width, count, static_cast<SliceMode>(mode));
    for (int l = 0; l < count; ++l)
      std::memcpy(slices_out + l * rows * cols, s.slices[l].data(),
                  sizeof(std::int64_t) * rows * cols);
    for (std::size_t b = 0; b < s.scale_exponents.size(); ++b) scales_out[b] = s.scale_exponents[b];
  });
}

// proj/src/slicing.cpp:164-204 (reconstruct) from a split of x.
int ozref_reconstruct(int orientation, std::int64_t rows, std::int64_t cols, const double* x,
                      int width, int count, int mode, double* out) {
  return guarded([&] {
    Matrix M = to_matrix(rows, cols, x);
    SlicedMatrix s = orientation == 0 ? split_rows(M, width, count, static_cast<SliceMode>(mode))
                                      : split_cols(M, width, count, static_cast<SliceMode>(mode));
    Matrix r = reconstruct(s);
    std::memcpy(out, r.data(), sizeof(double) * rows * cols);
  });
}

// proj/src/slicing.cpp:212-249
int ozref_min_exact_slices(int orientation, std::int64_t rows, std::int64_t cols,
                           const double* x, int width, int mode, int* out) {
  return guarded([&] {
    Matrix M = to_matrix(rows, cols, x);
    *out = min_exact_slices(M,
                            width, orientation == 0 ? BlockOrientation::kRows
                                                    : BlockOrientation::kColumns,
                            static_cast<SliceMode>(mode));
  });
}

// proj/src/mma_sim.cpp:76-125 (integer_gemm, no C input)
int ozref_integer_gemm(std::int64_t m, std::int64_t k, std::int64_t n, const std::int64_t* x,
                       const std::int64_t* y, std::int64_t* out, int t_in, int t_acc) {
  return guarded([&] {
    IntMatrix X(m, k), Y(k, n);
    std::memcpy(X.data(), x, sizeof(std::int64_t) * m * k);
    std::memcpy(Y.data(), y, sizeof(std::int64_t) * k * n);
    IntMatrix E = integer_gemm(X, Y, MmaConfig{t_in, t_acc});
    std::memcpy(out, E.data(), sizeof(std::int64_t) * m * n);
  });
}

// proj/src/scheme.cpp:127-168 (make_plan).  levels_out holds 2*max_levels ints.
int ozref_make_plan(std::int64_t k, int sa, int sb, int schedule, int strategy, int mode,
                    int precision, int t_in, int t_acc, int* width, int* acc_bits_used,
                    long long* psi, int* nlevels, int* levels_out, int max_levels) {
  return guarded([&] {
    MultiplyPlan p = plan_from(MmaConfig{t_in, t_acc}, k, sa, sb, schedule, strategy, mode,
                               precision, 0);
    *width = p.width;
    *acc_bits_used = p.acc_bits_used;
    *psi = p.psi;
    *nlevels = static_cast<int>(p.levels.levels.size());
    for (int i = 0; i < *nlevels && i < max_levels; ++i) {
      levels_out[2 * i] = p.levels.levels[i].first;
      levels_out[2 * i + 1] = p.levels.levels[i].second;
    }
  });
}

// proj/src/scheme.cpp:64-95
int ozref_plan_levels(int precision, int width, int acc_bits_used, int diagonals,
                      int* nlevels, int* levels_out, int max_levels) {
  return guarded([&] {
    LevelPlan p = plan_levels(precision, width, acc_bits_used, diagonals);
    *nlevels = static_cast<int>(p.levels.size());
    for (int i = 0; i < *nlevels && i < max_levels; ++i) {
      levels_out[2 * i] = p.levels[i].first;
      levels_out[2 * i + 1] = p.levels[i].second;
    }
  });
}

long long ozref_chi(int sa, int sb) { return chi(sa, sb); }

// proj/src/analysis.cpp:142-207
int ozref_select_slices(double kappa_a, double kappa_b, int width, double u, int s_max,
                        int has_target, double target, int schedule, int strategy,
                        int acc_bits_used, int precision, int* sa, int* sb, double* lhs,
                        double* target_out, long long* products, double* gap) {
  return guarded([&] {
    SelectOptions o;
    if (has_target) o.target = target;
    o.schedule = static_cast<ScheduleKind>(schedule);
    o.strategy = static_cast<Accumulation>(strategy);
    o.acc_bits_used = acc_bits_used;
    o.precision = precision;
    try {
      SliceSelection s = select_slices(kappa_a, kappa_b, width, u, s_max, o);
      *sa = s.slices_a;
      *sb = s.slices_b;
      *lhs = s.lhs;
      *target_out = s.target;
      *products = s.products;
    } catch (const SelectionInfeasible& e) {
      if (gap) *gap = e.gap;
      *lhs = e.best_lhs;
      *target_out = e.target;
      throw;
    }
  });
}

// proj/src/analysis.cpp:58-68
int ozref_scaling_profile(std::int64_t m, std::int64_t k, std::int64_t n, const double* a,
                          const double* b, double* kappa_a, double* kappa_b, int* a_zero,
                          int* b_zero) {
  return guarded([&] {
    ScalingProfile p = scaling_profile(to_matrix(m, k, a), to_matrix(k, n, b));
    *kappa_a = p.kappa_a;
    *kappa_b = p.kappa_b;
    *a_zero = p.a_has_zero_block;
    *b_zero = p.b_has_zero_block;
  });
}

// proj/src/analysis.cpp:86-131; bound_out may be null.
int ozref_error_bound(std::int64_t m, std::int64_t k, std::int64_t n, const double* a,
                      const double* b, int sa, int sb, int schedule, int strategy, int mode,
                      int precision, double* coefficient, double* bound_out) {
  return guarded([&] {
    MultiplyPlan p = plan_from(MmaConfig::int8_int32(), k, sa, sb, schedule, strategy, mode,
                               precision, 0);
    ErrorReport r = error_bound(to_matrix(m, k, a), to_matrix(k, n, b), p);
    *coefficient = r.coefficient;
    if (bound_out) std::memcpy(bound_out, r.bound.data(), sizeof(double) * m * n);
  });
}

// proj/src/oracle.cpp:223-232 + ExactProduct::to_matrix (RN of the exact AB)
int ozref_exact_gemm(std::int64_t m, std::int64_t k, std::int64_t n, const double* a,
                     const double* b, double* out) {
  return guarded([&] {
    Matrix r = exact_gemm(to_matrix(m, k, a), to_matrix(k, n, b)).to_matrix();
    std::memcpy(out, r.data(), sizeof(double) * m * n);
  });
}

// proj/src/matrix.cpp:31-54 (abs_product, gemm_reference)
int ozref_fp64_gemm(int absolute, std::int64_t m, std::int64_t k, std::int64_t n,
                    const double* a, const double* b, double* out) {
  return guarded([&] {
    Matrix ma = to_matrix(m, k, a), mb = to_matrix(k, n, b);
    Matrix r = absolute ? abs_product(ma, mb) : gemm_reference(ma, mb);
    std::memcpy(out, r.data(), sizeof(double) * m * n);
  });
}

// proj/src/oracle.cpp:263-271 and 273-292: the metrics of `computed` against
// exact_gemm(a, b) (beta = 0, c = 0 for the normwise one unless given)
int ozref_error_metrics(std::int64_t m, std::int64_t k, std::int64_t n, const double* a,
                        const double* b, const double* computed, double* max_elementwise,
                        double* normwise) {
  return guarded([&] {
    Matrix ma = to_matrix(m, k, a), mb = to_matrix(k, n, b), mc = to_matrix(m, n, computed);
    ExactProduct e = exact_gemm(ma, mb);
    *max_elementwise = max_elementwise_error(mc, e);
    Matrix zero(m, n);
    *normwise = normwise_gemm_error(mc, e, ma, mb, zero, 1.0, 0.0);
  });
}

// proj/src/oracle.cpp:234-251 (exact alpha*AB + beta*C, rounded once)
int ozref_exact_gemm_axpby(std::int64_t m, std::int64_t k, std::int64_t n, double alpha,
                           const double* a, const double* b, double beta, const double* c,
                           double* out) {
  return guarded([&] {
    Matrix r = exact_gemm_axpby(alpha, to_matrix(m, k, a), to_matrix(k, n, b), beta,
                                to_matrix(m, n, c))
                   .to_matrix();
    std::memcpy(out, r.data(), sizeof(double) * m * n);
  });
}

// proj/src/scheme.cpp:363-372
int ozref_multiply_axpby(std::int64_t m, std::int64_t n, std::int64_t k, double alpha,
                         const double* a, const double* b, double beta, const double* c,
                         double* out, int sa, int sb, int schedule, int strategy, int mode,
                         int precision) {
  return guarded([&] {
    MmaConfig cfg = MmaConfig::int8_int32();
    MultiplyPlan p = plan_from(cfg, k, sa, sb, schedule, strategy, mode, precision, 0);
    MultiplyResult r = multiply_axpby(alpha, to_matrix(m, k, a), to_matrix(k, n, b), beta,
                                      to_matrix(m, n, c), cfg, p);
    std::memcpy(out, r.c.data(), sizeof(double) * m * n);
  });
}

// proj/src/generators.cpp:176-182
void ozref_random_uniform(std::int64_t m, std::int64_t n, std::uint64_t seed, double lo,
                          double hi, double* out) {
  Matrix r = random_uniform(m, n, seed, lo, hi);
  std::memcpy(out, r.data(), sizeof(double) * m * n);
}

// proj/src/generators.cpp:103-140
int ozref_gen_kappa_d(std::int64_t n, double kappa_d, std::uint64_t seed, int rotate,
                      double* a_out, double* b_out) {
  return guarded([&] {
    auto [a, b] = gen_kappa_d(n, kappa_d, seed, rotate != 0);
    std::memcpy(a_out, a.data(), sizeof(double) * n * n);
    std::memcpy(b_out, b.data(), sizeof(double) * n * n);
  });
}

// proj/src/generators.cpp:86-101
int ozref_gen_lognormal(std::int64_t m, std::int64_t k, std::int64_t n, double phi,
                        std::uint64_t seed, double* a_out, double* b_out) {
  return guarded([&] {
    auto [a, b] = gen_lognormal(m, k, n, phi, seed);
    std::memcpy(a_out, a.data(), sizeof(double) * m * k);
    std::memcpy(b_out, b.data(), sizeof(double) * k * n);
  });
}

}  // extern "C"
