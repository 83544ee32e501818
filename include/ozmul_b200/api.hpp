// C++ drop-in API of the B200-native Ozaki-I FP64 GEMM.
//
// Source-compatible with the reference library's public headers
// (proj/include/ozmul/{matrix,fpcore,mma_sim,slicing,scheme,analysis}.hpp):
// a program written against `namespace ozmul` recompiles against
// include/ozmul/*.hpp (which forward here) and links libozgpu.so instead of
// the reference.  The GEMM path -- multiply, multiply_axpby, split_rows /
// split_cols, integer_gemm, scaling_profile, error_bound's |A||B| -- runs on
// the GPU through the C-ABI in include/ozgpu.h; the scalar plan / estimator /
// fpcore helpers are host code.  Exceptions are the reference's classes with
// its messages.
//
// Declarations are grouped by subsystem; each cites the reference declaration
// it matches.
#ifndef OZMUL_B200_API_HPP
#define OZMUL_B200_API_HPP

#include <cstddef>
#include <cstdint>
#include <functional>
#include <optional>
#include <span>
#include <stdexcept>
#include <utility>
#include <vector>

namespace ozmul {

// ===================================================== dense matrices
// matrix.hpp:26-96

class Matrix {
 public:
  Matrix() = default;
  Matrix(std::size_t rows, std::size_t cols, double fill = 0.0)
      : rows_(rows), cols_(cols), data_(rows * cols, fill) {}
  static Matrix identity(std::size_t n) {
    Matrix id(n, n);
    for (std::size_t i = 0; i < n; ++i) id(i, i) = 1.0;
    return id;
  }
  std::size_t rows() const { return rows_; }
  std::size_t cols() const { return cols_; }
  std::size_t size() const { return data_.size(); }
  double& operator()(std::size_t i, std::size_t j) { return data_[i * cols_ + j]; }
  double operator()(std::size_t i, std::size_t j) const { return data_[i * cols_ + j]; }
  std::span<double> row(std::size_t i) { return {data_.data() + i * cols_, cols_}; }
  std::span<const double> row(std::size_t i) const { return {data_.data() + i * cols_, cols_}; }
  double* data() { return data_.data(); }
  const double* data() const { return data_.data(); }
  bool operator==(const Matrix&) const = default;

 private:
  std::size_t rows_ = 0, cols_ = 0;
  std::vector<double> data_;
};

class IntMatrix {
 public:
  IntMatrix() = default;
  IntMatrix(std::size_t rows, std::size_t cols, std::int64_t fill = 0)
      : rows_(rows), cols_(cols), data_(rows * cols, fill) {}
  std::size_t rows() const { return rows_; }
  std::size_t cols() const { return cols_; }
  std::int64_t& operator()(std::size_t i, std::size_t j) { return data_[i * cols_ + j]; }
  std::int64_t operator()(std::size_t i, std::size_t j) const { return data_[i * cols_ + j]; }
  std::int64_t* data() { return data_.data(); }
  const std::int64_t* data() const { return data_.data(); }
  std::size_t size() const { return data_.size(); }
  bool operator==(const IntMatrix&) const = default;

 private:
  std::size_t rows_ = 0, cols_ = 0;
  std::vector<std::int64_t> data_;
};

bool is_clean_input(const Matrix& m);                       // finite, no -0 (host scan)
Matrix abs_product(const Matrix& a, const Matrix& b);       // |A||B| in binary64 (GPU)
Matrix gemm_reference(const Matrix& a, const Matrix& b);    // plain binary64 product (GPU)

// ========================================================== fp core
// fpcore.hpp:25-83

struct FloatFormat {
  int precision;
  int e_max;
  int e_min() const { return 1 - e_max; }
  double unit_roundoff() const;
  double max_value() const;
  static constexpr FloatFormat binary64() { return {53, 1023}; }
  void validate() const;
};

struct IntFormat {
  int width;
  std::int64_t min_value() const { return -(std::int64_t{1} << width); }
  std::int64_t max_value() const { return (std::int64_t{1} << width) - 1; }
  bool contains(std::int64_t v) const { return v >= min_value() && v <= max_value(); }
};

double round_nearest(double x, const FloatFormat& fmt);

struct SignificandView {
  std::uint64_t significand = 0;
  int exponent = 0;
  bool negative = false;
};
SignificandView significand_view(double x);
int scale_exponent(std::span<const double> values);
int scale_exponent_direct(double m);
int scale_exponent_fl_trick(double m);
int scale_exponent_bit_trick(double m);

// ======================================================= MMA unit model
// mma_sim.hpp:27-66

struct MmaConfig {
  int input_width;  // t'
  int acc_width;    // T
  static constexpr MmaConfig int8_int32() { return {7, 31}; }
  static constexpr MmaConfig int4_int32() { return {3, 31}; }
  void validate() const;
};

class MmaOverflowError : public std::runtime_error {
 public:
  MmaOverflowError(std::size_t row, std::size_t col, int acc_width);
  std::size_t row;
  std::size_t col;
};

int optimal_slice_width(const MmaConfig& cfg, std::int64_t k);
int optimal_slice_width_diagonal(const MmaConfig& cfg, std::int64_t k, int s);
std::int64_t max_inner_dim(const MmaConfig& cfg);
IntMatrix integer_gemm(const IntMatrix& x, const IntMatrix& y, const MmaConfig& cfg);
IntMatrix integer_gemm(const IntMatrix& x, const IntMatrix& y, const IntMatrix& c,
                       const MmaConfig& cfg);

// ============================================================= slicing
// slicing.hpp:27-86

enum class SliceMode { kTruncate, kNearest };
enum class BlockOrientation { kRows, kColumns };

struct SlicedMatrix {
  BlockOrientation orientation;
  SliceMode mode;
  int width;
  std::size_t rows = 0;
  std::size_t cols = 0;
  std::vector<int> scale_exponents;
  std::vector<IntMatrix> slices;
  int slice_count() const { return static_cast<int>(slices.size()); }
  int end_bit(int index) const {
    const int last = (index + 1) * width;
    return mode == SliceMode::kNearest ? last - 1 : last;
  }
};

SlicedMatrix split_rows(const Matrix& a, int width, int count,
                        SliceMode mode = SliceMode::kTruncate);
SlicedMatrix split_cols(const Matrix& b, int width, int count,
                        SliceMode mode = SliceMode::kTruncate);
Matrix reconstruct(const SlicedMatrix& s);
int bit_spread(double x);
int min_exact_slices(const Matrix& m, int width, BlockOrientation orientation,
                     SliceMode mode = SliceMode::kTruncate);

// ============================================================== scheme
// scheme.hpp:30-123

enum class ScheduleKind { kFull, kReduced };

struct Schedule {
  ScheduleKind kind = ScheduleKind::kReduced;
  std::optional<int> diag_sum_limit;
  bool contains(int l, int h, int slices_a, int slices_b) const;
  int max_diag_sum(int slices_a, int slices_b) const;
};

enum class Accumulation { kFloatPerProduct, kDiagonalInteger, kLevelledExact };

struct LevelPlan {
  std::vector<std::pair<int, int>> levels;
  long long inexact_adds = 0;
};

std::int64_t chi(int slices_a, int slices_b);
std::int64_t spare_carries(int first_diag, int last_diag, int width);
LevelPlan plan_levels(int precision, int width, int acc_bits_used, int num_diagonals);
std::int64_t diagonal_flush_threshold(const MmaConfig& cfg, int width, std::int64_t k);

struct MultiplyPlan {
  int slices_a = 1;
  int slices_b = 1;
  int width = 7;
  Schedule schedule;
  Accumulation strategy = Accumulation::kLevelledExact;
  SliceMode mode = SliceMode::kTruncate;
  int precision = 53;
  int acc_bits_used = 0;
  LevelPlan levels;
  long long psi = 0;
};

MultiplyPlan make_plan(const MmaConfig& cfg, std::int64_t k, int slices_a, int slices_b,
                       ScheduleKind schedule = ScheduleKind::kReduced,
                       Accumulation strategy = Accumulation::kLevelledExact,
                       SliceMode mode = SliceMode::kTruncate, int precision = 53);

struct Diagnostics {
  std::int64_t products = 0;
  std::int64_t integer_adds = 0;
  std::int64_t float_adds = 0;
  std::int64_t flushes = 0;
  long long realized_psi = 0;
  long long planned_psi = 0;
  int width = 0;
  int acc_bits_used = 0;
};

struct MultiplyResult {
  Matrix c;
  Diagnostics diagnostics;
};

MultiplyResult multiply(const Matrix& a, const Matrix& b, const MmaConfig& cfg,
                        const MultiplyPlan& plan);
MultiplyResult multiply_axpby(double alpha, const Matrix& a, const Matrix& b, double beta,
                              const Matrix& c, const MmaConfig& cfg, const MultiplyPlan& plan);

// The operator hook callers plug the emulated product into
// (`GemmFn`, oracle.hpp:117; consumed by block_lu_solve, oracle.cpp:371):
// the callable the reference's callers build by hand (main.cpp:578-582,
// acceptance_test.cpp:278-282) -- a plan made per call for the operands'
// inner dimension, then the GPU multiply.  The alias is the reference's own
// type, so the two may be declared together.
using GemmFn = std::function<Matrix(const Matrix&, const Matrix&)>;
inline GemmFn make_gemm_fn(const MmaConfig& cfg, int slices_a, int slices_b,
                           ScheduleKind schedule = ScheduleKind::kReduced,
                           Accumulation strategy = Accumulation::kLevelledExact,
                           SliceMode mode = SliceMode::kTruncate, int precision = 53) {
  return [=](const Matrix& x, const Matrix& y) {
    const MultiplyPlan plan = make_plan(cfg, static_cast<std::int64_t>(x.cols()), slices_a,
                                        slices_b, schedule, strategy, mode, precision);
    return multiply(x, y, cfg, plan).c;
  };
}

// ============================================================ analysis
// analysis.hpp:30-107

struct ScalingProfile {
  double kappa_a = 2.0;
  double kappa_b = 2.0;
  std::vector<double> row_ratios_a;
  std::vector<double> col_ratios_b;
  bool a_has_zero_block = false;
  bool b_has_zero_block = false;
};

double kappa(const Matrix& m, BlockOrientation orientation);
ScalingProfile scaling_profile(const Matrix& a, const Matrix& b);
double zeta(double kappa_a, double kappa_b, int slices_a, int slices_b, int width);
double gamma_factor(std::int64_t n, double u);

enum class BoundKind { kFull, kReducedALeB, kReducedAGtB };

struct ErrorReport {
  double kappa_a = 0.0;
  double kappa_b = 0.0;
  double zeta_ab = 0.0;
  double gamma_psi = 0.0;
  double coefficient = 0.0;
  double first_order_coefficient = 0.0;
  BoundKind kind = BoundKind::kFull;
  Matrix bound;
  bool a_has_zero_block = false;
  bool b_has_zero_block = false;
};

ErrorReport error_bound(const Matrix& a, const Matrix& b, const MultiplyPlan& plan,
                        double u = 0x1p-53);

class SelectionInfeasible : public std::runtime_error {
 public:
  SelectionInfeasible(double gap, double best_lhs, double target, int s_max);
  double gap;
  double best_lhs;
  double target;
};

struct SliceSelection {
  int slices_a = 1;
  int slices_b = 1;
  double lhs = 0.0;
  double target = 0.0;
  std::int64_t products = 0;
};

struct SelectOptions {
  std::optional<double> target;
  ScheduleKind schedule = ScheduleKind::kReduced;
  Accumulation strategy = Accumulation::kLevelledExact;
  int acc_bits_used = 31;
  int precision = 53;
};

SliceSelection select_slices(double kappa_a, double kappa_b, int width, double u, int s_max,
                             const SelectOptions& options = {});

}  // namespace ozmul

#endif  // OZMUL_B200_API_HPP
