// C++ drop-in API (include/ozmul_b200/api.hpp) over the C-ABI.
//
// GPU work goes through include/ozgpu.h on the process-wide default context
// of device $OZGPU_DEVICE (0 by default); C-ABI error codes are rethrown as
// the reference's exception classes with its messages.  Scalar helpers
// (fpcore, plan validation, reconstruct) are host code restated from the
// reference's specification; each cites the definition it follows.
#include <bit>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "ozgpu.h"
#include "ozgpu_numeric.h"
#include "ozmul_b200/api.hpp"

namespace ozmul {
namespace {

ozgpu_ctx* ctx() {
  const char* env = std::getenv("OZGPU_DEVICE");
  ozgpu_ctx* c = ozgpu_default_context(env ? std::atoi(env) : 0);
  if (!c) throw std::runtime_error(ozgpu_last_error());
  return c;
}

// $OZGPU_DEVICES (e.g. "0,1,2,3"): the device slots multiply() shards C over
// (ozgpu_dgemm_multi); empty when unset or a single slot.
std::vector<ozgpu_ctx*> shard_contexts() {
  std::vector<ozgpu_ctx*> out;
  const char* env = std::getenv("OZGPU_DEVICES");
  if (!env || !*env) return out;
  std::vector<int> devs;
  for (const char* p = env; *p;) {
    char* end = nullptr;
    const long v = std::strtol(p, &end, 10);
    if (end == p) throw std::invalid_argument("OZGPU_DEVICES: expected a comma-separated device list");
    devs.push_back(static_cast<int>(v));
    p = *end == ',' ? end + 1 : end;
  }
  if (devs.size() < 2) return out;
  out.resize(devs.size());
  if (ozgpu_device_contexts(devs.data(), static_cast<int>(devs.size()), out.data()) != OZGPU_OK)
    throw std::runtime_error(ozgpu_last_error());
  return out;
}

[[noreturn]] void rethrow(int rc, int acc_width = 31) {
  const std::string msg = ozgpu_last_error();
  switch (rc) {
    case OZGPU_INVALID_ARGUMENT:
      throw std::invalid_argument(msg);
    case OZGPU_DOMAIN_ERROR:
      throw std::domain_error(msg);
    case OZGPU_OVERFLOW: {
      unsigned long long r = 0, c = 0;
      std::sscanf(msg.c_str(), "integer accumulator overflow at (%llu, %llu)", &r, &c);
      throw MmaOverflowError(r, c, acc_width);
    }
    default:
      throw std::runtime_error(msg);
  }
}

inline void check(int rc) {
  if (rc != OZGPU_OK) rethrow(rc);
}

ozgpu_mma_config to_c(const MmaConfig& c) { return {c.input_width, c.acc_width}; }

ozgpu_plan to_c(const MultiplyPlan& p) {
  ozgpu_plan out{};
  out.slices_a = p.slices_a;
  out.slices_b = p.slices_b;
  out.width = p.width;
  out.schedule = p.schedule.kind == ScheduleKind::kFull ? 0 : 1;
  // an explicit limit <= 2 behaves as 2 (max_diag_sum clamps, scheme.cpp:39-44)
  out.diag_sum_limit = p.schedule.diag_sum_limit ? std::max(*p.schedule.diag_sum_limit, 2) : 0;
  out.strategy = static_cast<int>(p.strategy);
  out.mode = p.mode == SliceMode::kNearest ? 1 : 0;
  out.precision = p.precision;
  out.acc_bits_used = p.acc_bits_used;
  if (p.levels.levels.size() > OZGPU_MAX_LEVELS)
    throw std::invalid_argument("multiply: more than 128 levels in the plan");
  out.num_levels = static_cast<int>(p.levels.levels.size());
  for (int i = 0; i < out.num_levels; ++i) {
    out.levels[2 * i] = p.levels.levels[i].first;
    out.levels[2 * i + 1] = p.levels.levels[i].second;
  }
  out.level_inexact_adds = p.levels.inexact_adds;
  out.psi = p.psi;
  return out;
}

Diagnostics from_c(const ozgpu_diag& d) {
  Diagnostics o;
  o.products = d.products;
  o.integer_adds = d.integer_adds;
  o.float_adds = d.float_adds;
  o.flushes = d.flushes;
  o.realized_psi = d.realized_psi;
  o.planned_psi = d.planned_psi;
  o.width = d.width;
  o.acc_bits_used = d.acc_bits_used;
  return o;
}

int ceil_log2(std::int64_t k) { return std::bit_width(static_cast<std::uint64_t>(k) - 1); }

}  // namespace

// ------------------------------------------------------------------ matrix

bool is_clean_input(const Matrix& m) {  // matrix.cpp:22-29
  for (std::size_t i = 0; i < m.size(); ++i) {
    const double v = m.data()[i];
    if (!std::isfinite(v) || (v == 0.0 && std::signbit(v))) return false;
  }
  return true;
}

static Matrix fp64_product(const Matrix& a, const Matrix& b, int absolute, const char* who) {
  if (a.cols() != b.rows()) throw std::invalid_argument(std::string(who) + ": shape mismatch");
  Matrix out(a.rows(), b.cols());
  check(ozgpu_fp64_gemm(ctx(), absolute, static_cast<int64_t>(a.rows()),
                        static_cast<int64_t>(a.cols()), static_cast<int64_t>(b.cols()), a.data(),
                        static_cast<int64_t>(a.cols()), b.data(), static_cast<int64_t>(b.cols()),
                        out.data(), static_cast<int64_t>(b.cols())));
  return out;
}

Matrix abs_product(const Matrix& a, const Matrix& b) { return fp64_product(a, b, 1, "abs_product"); }
Matrix gemm_reference(const Matrix& a, const Matrix& b) {
  return fp64_product(a, b, 0, "gemm_reference");
}

// ------------------------------------------------------------------ fpcore

double FloatFormat::unit_roundoff() const { return std::ldexp(1.0, -precision); }  // fpcore.cpp:24
double FloatFormat::max_value() const {  // fpcore.cpp:26-28
  return std::ldexp(2.0 - std::ldexp(1.0, 1 - precision), e_max);
}
void FloatFormat::validate() const {  // fpcore.cpp:30-35
  if (precision < 2 || precision > 53)
    throw std::invalid_argument("FloatFormat: precision must be in [2, 53]");
  if (e_max < 1 || e_max > 1023)
    throw std::invalid_argument("FloatFormat: e_max must be in [1, 1023]");
}

double round_nearest(double x, const FloatFormat& fmt) {  // fpcore.cpp:37-56
  fmt.validate();
  if (!std::isfinite(x)) throw std::invalid_argument("round_nearest: non-finite input");
  if (x == 0.0) return 0.0;
  const int quantum = std::max(std::ilogb(x), fmt.e_min()) - fmt.precision + 1;
  const double r = std::ldexp(std::nearbyint(std::ldexp(x, -quantum)), quantum);
  if (std::abs(r) > fmt.max_value())
    throw std::overflow_error("round_nearest: value exceeds format range");
  return r;
}

SignificandView significand_view(double x) {  // fpcore.cpp:58-74
  if (!std::isfinite(x)) throw std::invalid_argument("significand_view: non-finite input");
  SignificandView v;
  v.negative = std::signbit(x);
  const std::uint64_t bits = std::bit_cast<std::uint64_t>(std::abs(x));
  const std::uint64_t biased = bits >> 52, frac = bits & ((std::uint64_t{1} << 52) - 1);
  v.significand = biased ? (frac | (std::uint64_t{1} << 52)) : frac;
  v.exponent = biased ? static_cast<int>(biased) - 1023 : -1022;
  return v;
}

int scale_exponent_direct(double m) {  // fpcore.cpp:83-87
  if (!(m > 0.0) || !std::isfinite(m))
    throw std::invalid_argument("scale_exponent_direct: need finite m > 0");
  return std::ilogb(m) + 1;
}

int scale_exponent(std::span<const double> values) {  // fpcore.cpp:76-81
  double mx = 0.0;
  for (double v : values) mx = std::max(mx, std::abs(v));
  return mx == 0.0 ? 0 : scale_exponent_direct(mx);
}

int scale_exponent_fl_trick(double m) {  // fpcore.cpp:89-101
  if (!(m > 0.0) || !std::isfinite(m))
    throw std::invalid_argument("scale_exponent_fl_trick: need finite m > 0");
  if (m < 0x1p-1022 || m >= 0x1p970) return scale_exponent_direct(m);
  const double u_inv = 0x1p53;
  double alpha = u_inv * m + (1.0 - u_inv) * m;
  if (alpha <= m) alpha *= 2.0;
  return std::ilogb(alpha);
}

int scale_exponent_bit_trick(double m) {  // fpcore.cpp:103-114
  if (!(m > 0.0) || !std::isfinite(m))
    throw std::invalid_argument("scale_exponent_bit_trick: need finite m > 0");
  const std::uint64_t bits = std::bit_cast<std::uint64_t>(m);
  const std::uint64_t field = bits & ~((std::uint64_t{1} << 52) - 1);
  if (field == 0 || (field >> 52) >= 2046) return scale_exponent_direct(m);
  return std::ilogb(std::bit_cast<double>(field + (std::uint64_t{1} << 52)));
}

// ----------------------------------------------------------------- MMA unit

void MmaConfig::validate() const {  // mma_sim.cpp:34-41
  if (input_width < 1) throw std::invalid_argument("MmaConfig: input width must be >= 1");
  if (acc_width > 62)
    throw std::invalid_argument("MmaConfig: accumulator width above 62 is not modeled");
  if (acc_width < 2 * input_width + 1)
    throw std::invalid_argument("MmaConfig: accumulator cannot hold even a single product");
}

MmaOverflowError::MmaOverflowError(std::size_t row_, std::size_t col_, int acc_width)
    : std::runtime_error("integer accumulator overflow at (" + std::to_string(row_) + ", " +
                         std::to_string(col_) + "): value left I_" + std::to_string(acc_width)),
      row(row_),
      col(col_) {}

int optimal_slice_width(const MmaConfig& cfg, std::int64_t k) {
  int out = 0;
  check(ozgpu_optimal_slice_width(to_c(cfg), k, &out));
  return out;
}

int optimal_slice_width_diagonal(const MmaConfig& cfg, std::int64_t k, int s) {  // mma_sim.cpp:61-64
  if (s < 1) throw std::invalid_argument("optimal_slice_width_diagonal: s must be >= 1");
  return optimal_slice_width(cfg, k + s - 1);
}

std::int64_t max_inner_dim(const MmaConfig& cfg) {
  int64_t out = 0;
  check(ozgpu_max_inner_dim(to_c(cfg), &out));
  return out;
}

static IntMatrix int_gemm(const IntMatrix& x, const IntMatrix& y, const IntMatrix* c,
                          const MmaConfig& cfg) {
  cfg.validate();
  if (x.cols() != y.rows()) throw std::invalid_argument("integer_gemm: shape mismatch");
  if (c && (c->rows() != x.rows() || c->cols() != y.cols()))
    throw std::invalid_argument("integer_gemm: accumulator shape mismatch");
  IntMatrix out(x.rows(), y.cols());
  const int rc = ozgpu_integer_gemm(ctx(), static_cast<int64_t>(x.rows()),
                                    static_cast<int64_t>(x.cols()), static_cast<int64_t>(y.cols()),
                                    x.data(), y.data(), c ? c->data() : nullptr, out.data(),
                                    to_c(cfg));
  if (rc != OZGPU_OK) rethrow(rc, cfg.acc_width);
  return out;
}

IntMatrix integer_gemm(const IntMatrix& x, const IntMatrix& y, const MmaConfig& cfg) {
  return int_gemm(x, y, nullptr, cfg);
}
IntMatrix integer_gemm(const IntMatrix& x, const IntMatrix& y, const IntMatrix& c,
                       const MmaConfig& cfg) {
  return int_gemm(x, y, &c, cfg);
}

// ------------------------------------------------------------------ slicing

static SlicedMatrix gpu_split(const Matrix& m, int width, int count, SliceMode mode,
                              BlockOrientation o) {
  SlicedMatrix s;
  s.orientation = o;
  s.mode = mode;
  s.width = width;
  s.rows = m.rows();
  s.cols = m.cols();
  const int orient = o == BlockOrientation::kRows ? 0 : 1;
  std::vector<std::int64_t> flat(static_cast<std::size_t>(std::max(count, 0)) * m.size());
  s.scale_exponents.assign(orient == 0 ? m.rows() : m.cols(), 0);
  check(ozgpu_split(ctx(), orient, static_cast<int64_t>(m.rows()), static_cast<int64_t>(m.cols()),
                    m.data(), static_cast<int64_t>(m.cols()), width, count,
                    mode == SliceMode::kNearest ? 1 : 0, flat.data(), s.scale_exponents.data()));
  s.slices.assign(count, IntMatrix(m.rows(), m.cols()));
  for (int l = 0; l < count; ++l)
    if (m.size())
      std::memcpy(s.slices[l].data(), flat.data() + static_cast<std::size_t>(l) * m.size(),
                  sizeof(std::int64_t) * m.size());
  return s;
}

SlicedMatrix split_rows(const Matrix& a, int width, int count, SliceMode mode) {
  return gpu_split(a, width, count, mode, BlockOrientation::kRows);
}
SlicedMatrix split_cols(const Matrix& b, int width, int count, SliceMode mode) {
  return gpu_split(b, width, count, mode, BlockOrientation::kColumns);
}

Matrix reconstruct(const SlicedMatrix& s) {  // slicing.cpp:164-204
  Matrix out(s.rows, s.cols);
  for (std::size_t i = 0; i < s.rows; ++i)
    for (std::size_t j = 0; j < s.cols; ++j) {
      const std::size_t blk = s.orientation == BlockOrientation::kRows ? i : j;
      const int q = s.scale_exponents.empty() ? 0 : s.scale_exponents[blk];
      __int128 acc = 0;
      int acc_end = 0;
      bool sticky = false;
      for (int l = 0; l < s.slice_count(); ++l) {
        const std::int64_t v = s.slices[l](i, j);
        if (v == 0) continue;
        if (acc == 0) {
          acc = v;
          acc_end = s.end_bit(l);
          continue;
        }
        const int gap = s.end_bit(l) - acc_end;
        const unsigned __int128 mag =
            acc < 0 ? -static_cast<unsigned __int128>(acc) : static_cast<unsigned __int128>(acc);
        const std::uint64_t mh = static_cast<std::uint64_t>(mag >> 64);
        const int used = mh ? 128 - std::countl_zero(mh)
                            : 64 - std::countl_zero(static_cast<std::uint64_t>(mag));
        if (used + gap > 126) {
          sticky = true;
          continue;
        }
        acc = (acc << gap) + v;
        acc_end = s.end_bit(l);
      }
      if (acc == 0) continue;
      const bool neg = acc < 0;
      const unsigned __int128 mag =
          neg ? -static_cast<unsigned __int128>(acc) : static_cast<unsigned __int128>(acc);
      // slicing.cpp:134-157 rounds through a 55-bit window with the dropped
      // slices as an extra sticky bit: the same RN-to-odd-at-55-bits as the
      // exact combine's round_i128 once that sticky is ORed into bit 0
      const double v = ozgpu::round_i128(mag | (sticky ? 1u : 0u), q - acc_end);
      out(i, j) = neg ? -v : v;
    }
  return out;
}

int bit_spread(double x) {  // slicing.cpp:206-210
  const SignificandView d = significand_view(x);
  if (d.significand == 0) return 0;
  return std::bit_width(d.significand) - std::countr_zero(d.significand);
}

int min_exact_slices(const Matrix& m, int width, BlockOrientation o, SliceMode mode) {
  // slicing.cpp:212-249 on the GPU (ozgpu_min_exact_slices): the deepest set
  // fraction bit over the blocks fixes the count exactly, so the reference's
  // closing round-trip check (split + reconstruct) cannot fail and is skipped
  int out = 0;
  check(ozgpu_min_exact_slices(ctx(), o == BlockOrientation::kRows ? 0 : 1,
                               static_cast<int64_t>(m.rows()), static_cast<int64_t>(m.cols()),
                               m.data(), static_cast<int64_t>(m.cols()), width,
                               mode == SliceMode::kNearest ? 1 : 0, &out));
  return out;
}

// ------------------------------------------------------------------- scheme

int Schedule::max_diag_sum(int slices_a, int slices_b) const {  // scheme.cpp:39-44
  int base = kind == ScheduleKind::kFull ? slices_a + slices_b : std::max(slices_a, slices_b) + 1;
  if (diag_sum_limit) base = std::min(base, *diag_sum_limit);
  return std::max(base, 2);
}

bool Schedule::contains(int l, int h, int slices_a, int slices_b) const {  // scheme.cpp:34-37
  if (l < 1 || l > slices_a || h < 1 || h > slices_b) return false;
  return l + h <= max_diag_sum(slices_a, slices_b);
}

std::int64_t chi(int slices_a, int slices_b) {
  int64_t out = 0;
  check(ozgpu_chi(slices_a, slices_b, &out));
  return out;
}

std::int64_t spare_carries(int first_diag, int last_diag, int width) {
  int64_t out = 0;
  check(ozgpu_spare_carries(first_diag, last_diag, width, &out));
  return out;
}

LevelPlan plan_levels(int precision, int width, int acc_bits_used, int num_diagonals) {
  ozgpu_plan p{};
  check(ozgpu_plan_levels(precision, width, acc_bits_used, num_diagonals, &p));
  LevelPlan out;
  for (int i = 0; i < p.num_levels; ++i) out.levels.emplace_back(p.levels[2 * i], p.levels[2 * i + 1]);
  out.inexact_adds = p.level_inexact_adds;
  return out;
}

std::int64_t diagonal_flush_threshold(const MmaConfig& cfg, int width, std::int64_t k) {
  int64_t out = 0;
  check(ozgpu_diagonal_flush_threshold(to_c(cfg), width, k, &out));
  return out;
}

MultiplyPlan make_plan(const MmaConfig& cfg, std::int64_t k, int slices_a, int slices_b,
                       ScheduleKind schedule, Accumulation strategy, SliceMode mode,
                       int precision) {
  ozgpu_plan p{};
  check(ozgpu_make_plan(to_c(cfg), k, slices_a, slices_b, schedule == ScheduleKind::kFull ? 0 : 1,
                        static_cast<int>(strategy), mode == SliceMode::kNearest ? 1 : 0,
                        precision, &p));
  MultiplyPlan out;
  out.slices_a = p.slices_a;
  out.slices_b = p.slices_b;
  out.width = p.width;
  out.schedule.kind = schedule;
  out.strategy = strategy;
  out.mode = mode;
  out.precision = p.precision;
  out.acc_bits_used = p.acc_bits_used;
  for (int i = 0; i < p.num_levels; ++i)
    out.levels.levels.emplace_back(p.levels[2 * i], p.levels[2 * i + 1]);
  out.levels.inexact_adds = p.level_inexact_adds;
  out.psi = p.psi;
  return out;
}

MultiplyResult multiply(const Matrix& a, const Matrix& b, const MmaConfig& cfg,
                        const MultiplyPlan& plan) {
  cfg.validate();  // scheme.cpp:221-222 order: config, shape, then the GPU-side checks
  if (a.cols() != b.rows()) throw std::invalid_argument("multiply: shape mismatch");
  MultiplyResult r{Matrix(a.rows(), b.cols()), {}};
  ozgpu_plan p = to_c(plan);
  ozgpu_diag d{};
  const std::vector<ozgpu_ctx*> slots = shard_contexts();
  if (!slots.empty()) {  // 2-D C tiles over the listed GPUs (bit-identical)
    check(ozgpu_dgemm_multi(slots.data(), static_cast<int>(slots.size()),
                            static_cast<int64_t>(a.rows()), static_cast<int64_t>(b.cols()),
                            static_cast<int64_t>(a.cols()), a.data(),
                            static_cast<int64_t>(a.cols()), b.data(),
                            static_cast<int64_t>(b.cols()), r.c.data(),
                            static_cast<int64_t>(b.cols()), to_c(cfg), &p, &d));
    r.diagnostics = from_c(d);
    return r;
  }
  check(ozgpu_dgemm(ctx(), static_cast<int64_t>(a.rows()), static_cast<int64_t>(b.cols()),
                    static_cast<int64_t>(a.cols()), a.data(), static_cast<int64_t>(a.cols()),
                    b.data(), static_cast<int64_t>(b.cols()), r.c.data(),
                    static_cast<int64_t>(b.cols()), to_c(cfg), &p, &d));
  r.diagnostics = from_c(d);
  return r;
}

MultiplyResult multiply_axpby(double alpha, const Matrix& a, const Matrix& b, double beta,
                              const Matrix& c, const MmaConfig& cfg, const MultiplyPlan& plan) {
  if (c.rows() != a.rows() || c.cols() != b.cols())  // scheme.cpp:366-367
    throw std::invalid_argument("multiply_axpby: shape mismatch");
  cfg.validate();
  if (a.cols() != b.rows()) throw std::invalid_argument("multiply: shape mismatch");
  MultiplyResult r{Matrix(a.rows(), b.cols()), {}};
  ozgpu_plan p = to_c(plan);
  ozgpu_diag d{};
  const int64_t n = static_cast<int64_t>(b.cols());
  check(ozgpu_dgemm_axpby(ctx(), static_cast<int64_t>(a.rows()), n,
                          static_cast<int64_t>(a.cols()), alpha, a.data(),
                          static_cast<int64_t>(a.cols()), b.data(), n, beta, c.data(), n,
                          r.c.data(), n, to_c(cfg), &p, &d));
  r.diagnostics = from_c(d);
  return r;
}

// ----------------------------------------------------------------- analysis

static std::vector<double> gpu_ratios(const Matrix& m, BlockOrientation o, bool* has_zero) {
  const int orient = o == BlockOrientation::kRows ? 0 : 1;
  std::vector<double> r(orient == 0 ? m.rows() : m.cols(), 1.0);
  int z = 0;
  check(ozgpu_block_ratios(ctx(), orient, static_cast<int64_t>(m.rows()),
                           static_cast<int64_t>(m.cols()), m.data(),
                           static_cast<int64_t>(m.cols()), r.data(), &z));
  if (has_zero) *has_zero = z != 0;
  return r;
}

double kappa(const Matrix& m, BlockOrientation orientation) {  // analysis.cpp:51-56
  double worst = 1.0;
  for (double r : gpu_ratios(m, orientation, nullptr)) worst = std::max(worst, r);
  return 2.0 * worst;
}

ScalingProfile scaling_profile(const Matrix& a, const Matrix& b) {  // analysis.cpp:58-68
  ScalingProfile p;
  p.row_ratios_a = gpu_ratios(a, BlockOrientation::kRows, &p.a_has_zero_block);
  p.col_ratios_b = gpu_ratios(b, BlockOrientation::kColumns, &p.b_has_zero_block);
  double wa = 1.0, wb = 1.0;
  for (double r : p.row_ratios_a) wa = std::max(wa, r);
  for (double r : p.col_ratios_b) wb = std::max(wb, r);
  p.kappa_a = 2.0 * wa;
  p.kappa_b = 2.0 * wb;
  return p;
}

double zeta(double kappa_a, double kappa_b, int slices_a, int slices_b, int width) {
  // analysis.cpp:70-77
  if (!(kappa_a > 0.0) || !(kappa_b > 0.0))
    throw std::invalid_argument("zeta: kappas must be positive");
  return std::ldexp(kappa_a, -slices_a * width) + std::ldexp(kappa_b, -slices_b * width) +
         std::ldexp(kappa_a * kappa_b, -(slices_a + slices_b) * width);
}

double gamma_factor(std::int64_t n, double u) {  // analysis.cpp:79-84
  if (n < 0) throw std::invalid_argument("gamma_factor: n must be >= 0");
  const double nu = static_cast<double>(n) * u;
  if (nu >= 1.0) throw std::domain_error("gamma_factor: n*u >= 1, bound is meaningless");
  return nu / (1.0 - nu);
}

ErrorReport error_bound(const Matrix& a, const Matrix& b, const MultiplyPlan& plan, double u) {
  // analysis.cpp:86-131; |A||B| on the GPU in the reference's rounding order
  ErrorReport rep;
  const ScalingProfile prof = scaling_profile(a, b);
  rep.kappa_a = prof.kappa_a;
  rep.kappa_b = prof.kappa_b;
  rep.a_has_zero_block = prof.a_has_zero_block;
  rep.b_has_zero_block = prof.b_has_zero_block;
  const int t = plan.width, sa = plan.slices_a, sb = plan.slices_b;
  rep.zeta_ab = zeta(rep.kappa_a, rep.kappa_b, sa, sb, t);
  rep.gamma_psi = gamma_factor(plan.psi, u);
  if (plan.schedule.kind == ScheduleKind::kFull) {
    rep.kind = BoundKind::kFull;
    rep.coefficient = rep.zeta_ab + rep.gamma_psi * (1.0 + rep.zeta_ab);
  } else {
    double cut;
    if (sa <= sb) {
      rep.kind = BoundKind::kReducedALeB;
      cut = std::ldexp(static_cast<double>(sa) * rep.kappa_a * rep.kappa_b, -sb * t);
    } else {
      rep.kind = BoundKind::kReducedAGtB;
      cut = std::ldexp(static_cast<double>(sb) * rep.kappa_a * rep.kappa_b, -sa * t);
    }
    const double gamma_next = gamma_factor(plan.psi + 1, u);
    rep.coefficient = rep.zeta_ab + cut + gamma_next * (1.0 + rep.zeta_ab + cut);
  }
  rep.first_order_coefficient = std::ldexp(rep.kappa_a, -sa * t) +
                                std::ldexp(rep.kappa_b, -sb * t) +
                                static_cast<double>(plan.psi) * u;
  Matrix prod = abs_product(a, b);
  const double inflated = rep.coefficient * (1.0 + 8.0 * u);
  for (std::size_t i = 0; i < prod.size(); ++i) prod.data()[i] *= inflated;
  rep.bound = std::move(prod);
  return rep;
}

SelectionInfeasible::SelectionInfeasible(double gap_, double best_lhs_, double target_, int s_max)
    : std::runtime_error("select_slices: no feasible pair within s_max = " +
                         std::to_string(s_max) +
                         "; best achievable term exceeds the target by a factor " +
                         std::to_string(gap_)),
      gap(gap_),
      best_lhs(best_lhs_),
      target(target_) {}

SliceSelection select_slices(double kappa_a, double kappa_b, int width, double u, int s_max,
                             const SelectOptions& o) {
  ozgpu_selection s{};
  const int rc = ozgpu_select_slices(
      kappa_a, kappa_b, width, u, s_max, o.target ? 1 : 0, o.target ? *o.target : 0.0,
      o.schedule == ScheduleKind::kFull ? 0 : 1, static_cast<int>(o.strategy), o.acc_bits_used,
      o.precision, &s);
  if (rc == OZGPU_INFEASIBLE) throw SelectionInfeasible(s.gap, s.lhs, s.target, s_max);
  check(rc);
  SliceSelection out;
  out.slices_a = s.slices_a;
  out.slices_b = s.slices_b;
  out.lhs = s.lhs;
  out.target = s.target;
  out.products = s.products;
  return out;
}

}  // namespace ozmul
