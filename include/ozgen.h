/* ozgen.h -- synthetic inputs for the benchmarks and tests (libozgen.so).
 * Not part of the GEMM path: the reference's two input families the
 * BASELINE configs are quoted on, with bytes identical to its generators
 * (proj/src/generators.cpp), so the GPU run and the reference CPU run see
 * the same matrices.  Host code only. */
#ifndef OZGEN_H
#define OZGEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* random_uniform, proj/src/generators.cpp:25-49,176-182: mt19937_64 seeded
 * through splitmix64; m x n row-major. */
void ozgen_random_uniform(int64_t m, int64_t n, uint64_t seed, double lo, double hi,
                          double* out);
/* gen_kappa_d, proj/src/generators.cpp:103-140 (n x n factors). */
void ozgen_gen_kappa_d(int64_t n, double kappa_d, uint64_t seed, int rotate, double* a_out,
                       double* b_out);

#ifdef __cplusplus
}
#endif
#endif /* OZGEN_H */
