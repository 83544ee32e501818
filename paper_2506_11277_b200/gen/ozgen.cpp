// Synthetic inputs for the benchmarks and tests (libozgen.so, include/ozgen.h):
// the reference's random_uniform and gen_kappa_d restated with identical
// bytes.  Kept out of libozgpu.so: input generation is not the GEMM path.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <vector>

#include "ozgen.h"

extern "C" {

// generators.cpp:25-49,176-182 -- std::mt19937_64 is the identical engine.
static uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

void ozgen_random_uniform(int64_t m, int64_t n, uint64_t seed, double lo, double hi, double* out) {
  std::mt19937_64 eng(splitmix64(seed));
  const int64_t total = m * n;
  for (int64_t i = 0; i < total; ++i)
    out[i] = lo + static_cast<double>(eng() >> 11) * 0x1p-53 * (hi - lo);
}

void ozgen_gen_kappa_d(int64_t n, double kappa_d, uint64_t seed, int rotate, double* a,
                       double* b) {
  std::mt19937_64 ea(splitmix64(seed + 1)), eb(splitmix64(seed + 2));
  for (int64_t i = 0; i < n * n; ++i) a[i] = 1.0 + static_cast<double>(ea() >> 11) * 0x1p-53 * 1.0;
  for (int64_t i = 0; i < n * n; ++i) b[i] = 1.0 + static_cast<double>(eb() >> 11) * 0x1p-53 * 1.0;
  std::vector<double> d(n);
  double log_kd = std::log(kappa_d);
  for (int64_t i = 0; i < n; ++i) {
    double frac = n > 1 ? static_cast<double>(i) / static_cast<double>(n - 1) : 0.5;
    d[i] = std::exp(log_kd * (frac - 0.5));
  }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      a[i * n + j] *= d[j];
      b[i * n + j] /= d[i];
    }
  if (rotate) {
    std::vector<double> ra(n * n), rb(n * n);
    for (int64_t i = 0; i < n; ++i) {
      int64_t shift = (i + 1) % n;
      for (int64_t j = 0; j < n; ++j) {
        ra[i * n + (j + shift) % n] = a[i * n + j];
        rb[((j + shift) % n) * n + i] = b[j * n + i];
      }
    }
    std::memcpy(a, ra.data(), sizeof(double) * n * n);
    std::memcpy(b, rb.data(), sizeof(double) * n * n);
  }
}

}  // extern "C"
