// The GemmFn operator hook (oracle.hpp:117) of the C++ drop-in:
// ozmul::make_gemm_fn (include/ozmul_b200/api.hpp) against the lambda the
// reference's callers build by hand (main.cpp:578-582,
// acceptance_test.cpp:278-282), bitwise, over the shapes a block-LU Schur
// update feeds it; then a right-looking block LU whose Schur updates all go
// through the adaptor (the block_lu_solve pattern, oracle.cpp:313-380).
// Built and run by tests/test_gpu_contract.py.
#include <ozmul/scheme.hpp>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

using namespace ozmul;

static Matrix random_matrix(std::size_t r, std::size_t c, std::uint64_t seed) {
  Matrix m(r, c);
  std::uint64_t s = seed * 0x9E3779B97F4A7C15ull + 1;
  for (std::size_t i = 0; i < r; ++i)
    for (std::size_t j = 0; j < c; ++j) {
      s = s * 6364136223846793005ull + 1442695040888963407ull;
      m(i, j) = static_cast<double>(static_cast<std::int64_t>(s >> 11) - (1ll << 52)) / (1ll << 52);
    }
  return m;
}

static bool same_bits(const Matrix& x, const Matrix& y) {
  if (x.rows() != y.rows() || x.cols() != y.cols()) return false;
  for (std::size_t i = 0; i < x.rows(); ++i)
    for (std::size_t j = 0; j < x.cols(); ++j) {
      double a = x(i, j), b = y(i, j);
      if (std::memcmp(&a, &b, sizeof a) != 0) return false;
    }
  return true;
}

int main() {
  const MmaConfig cfg = MmaConfig::int8_int32();
  const GemmFn fn = make_gemm_fn(cfg, 8, 8);
  auto manual = [&](const Matrix& x, const Matrix& y) {
    const MultiplyPlan plan = make_plan(cfg, static_cast<std::int64_t>(x.cols()), 8, 8,
                                        ScheduleKind::kReduced, Accumulation::kLevelledExact);
    return multiply(x, y, cfg, plan).c;
  };
  const std::size_t shapes[][3] = {{300, 16, 290}, {284, 16, 274}, {128, 64, 96}, {1, 1, 1},
                                    {700, 333, 650}};
  for (const auto& s : shapes) {
    const Matrix x = random_matrix(s[0], s[1], s[0] + 7), y = random_matrix(s[1], s[2], s[2] + 11);
    if (!same_bits(fn(x, y), manual(x, y))) {
      std::printf("FAIL: adaptor differs from the hand-built lambda at %zux%zux%zu\n", s[0], s[1],
                  s[2]);
      return 1;
    }
  }
  // right-looking block LU (no pivoting; diagonally dominant system), the
  // Schur update A22 -= L21 U12 through the hook
  const std::size_t n = 256, nb = 32;
  Matrix a = random_matrix(n, n, 5);
  for (std::size_t i = 0; i < n; ++i) a(i, i) += static_cast<double>(n);
  Matrix lu = a;
  for (std::size_t k0 = 0; k0 < n; k0 += nb) {
    const std::size_t k1 = k0 + nb;
    for (std::size_t c = k0; c < k1; ++c)
      for (std::size_t r = c + 1; r < n; ++r) {
        lu(r, c) /= lu(c, c);
        for (std::size_t j = c + 1; j < k1; ++j) lu(r, j) -= lu(r, c) * lu(c, j);
      }
    if (k1 >= n) break;
    for (std::size_t r = k0 + 1; r < k1; ++r)
      for (std::size_t r2 = k0; r2 < r; ++r2)
        for (std::size_t j = k1; j < n; ++j) lu(r, j) -= lu(r, r2) * lu(r2, j);
    Matrix l21(n - k1, nb), u12(nb, n - k1);
    for (std::size_t i = 0; i < n - k1; ++i)
      for (std::size_t j = 0; j < nb; ++j) l21(i, j) = lu(k1 + i, k0 + j);
    for (std::size_t i = 0; i < nb; ++i)
      for (std::size_t j = 0; j < n - k1; ++j) u12(i, j) = lu(k0 + i, k1 + j);
    const Matrix prod = fn(l21, u12);
    for (std::size_t i = 0; i < n - k1; ++i)
      for (std::size_t j = 0; j < n - k1; ++j) lu(k1 + i, k1 + j) -= prod(i, j);
  }
  // solve LU x = b for b = A * ones and compare x with ones
  std::vector<double> b(n, 0.0), x(n);
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j < n; ++j) b[i] += a(i, j);
  for (std::size_t i = 0; i < n; ++i) {
    double v = b[i];
    for (std::size_t j = 0; j < i; ++j) v -= lu(i, j) * x[j];
    x[i] = v;
  }
  for (std::size_t i = n; i-- > 0;) {
    double v = x[i];
    for (std::size_t j = i + 1; j < n; ++j) v -= lu(i, j) * x[j];
    x[i] = v / lu(i, i);
  }
  double err = 0.0;
  for (double v : x) err = std::fmax(err, std::fabs(v - 1.0));
  if (!(err < 1e-12)) {
    std::printf("FAIL: block LU through the hook, max |x - 1| = %g\n", err);
    return 1;
  }
  std::printf("ok: make_gemm_fn bitwise == hand-built lambda; block LU max |x-1| = %g\n", err);
  return 0;
}
