/* ozoracle -- plain-C CPU restatement of the reference's Ozaki-I hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may load this library, and only as the
 * checker: it is never the thing measured or shipped.
 *
 * Parity is pinned: tests/test_oracle.py checks every function below against
 * the reference's golden vectors (proj/tests/ *_test.cpp) and against the
 * unmodified reference compiled from its own sources (oracle/_ref/libozref.so,
 * see oracle/Makefile).
 *
 * Enumerations follow the reference headers:
 *   orientation 0 = rows (left factor), 1 = columns (right factor)
 *   mode        0 = truncate, 1 = nearest       (slicing.hpp SliceMode)
 *   schedule    0 = full, 1 = reduced           (scheme.hpp ScheduleKind)
 *   strategy    0 = float-per-product, 1 = diagonal-integer, 2 = levelled-exact
 */
#ifndef OZ_ORACLE_H
#define OZ_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* proj/src/mma_sim.cpp:50-59 */
int ozo_optimal_slice_width(int t_in, int t_acc, int64_t k);
/* proj/src/scheme.cpp:46-52 */
int64_t ozo_chi(int sa, int sb);
/* proj/src/scheme.cpp:54-62 */
int64_t ozo_spare_carries(int first, int last, int width);
/* proj/src/scheme.cpp:64-95; returns the level count, writes [first,last] pairs */
int ozo_plan_levels(int precision, int width, int acc_bits_used, int diagonals,
                    int* levels_out, int max_levels);
/* proj/src/scheme.cpp:39-44 (Schedule::max_diag_sum); diag_sum_limit <= 0 = none */
int ozo_max_diag_sum(int schedule, int diag_sum_limit, int sa, int sb);

/* proj/src/slicing.cpp:67-132 -- slices_out is [count][rows][cols] int64,
 * scales_out has one entry per block.  Returns 0, or 1 on bad arguments /
 * non-finite input (the reference's std::invalid_argument). */
int ozo_split(int orientation, int64_t rows, int64_t cols, const double* x, int width,
              int count, int mode, int64_t* slices_out, int* scales_out);

/* proj/src/mma_sim.cpp:76-114 -- exact X*Y; returns 0, or 5 when a running
 * sum leaves I_T (MmaOverflowError), 2 when an input leaves I_t'. */
int ozo_integer_gemm(int64_t m, int64_t k, int64_t n, const int64_t* x, const int64_t* y,
                     int64_t* out, int t_in, int t_acc);

/* proj/src/oracle.cpp:157-180 (ExactValue::to_double) applied to the signed
 * multi-word two's-complement integer v[0..words) (little-endian words)
 * times 2^exp. */
double ozo_round_words(const uint64_t* v, int words, long exp);

/* The default levelled-exact multiply (proj/src/scheme.cpp:219-361 with
 * kLevelledExact), restated as one rounding of the exact scheduled sum:
 *   C_ij = RN( sum_{(l,h) in S} 2^(qa_i + qb_j + w(l+h-2)) * E_lh[i,j] )
 * where w(d) = -(d+2)t (+2 in nearest mode).  Returns 0 / 1 / 2 with the
 * reference's validation order (scheme.cpp:221-239). */
int ozo_multiply_exact(int64_t m, int64_t n, int64_t k, const double* a, const double* b,
                       double* c, int sa, int sb, int schedule, int diag_sum_limit, int mode,
                       int width);

/* proj/src/analysis.cpp:25-68 */
void ozo_scaling_profile(int64_t m, int64_t k, int64_t n, const double* a, const double* b,
                         double* kappa_a, double* kappa_b, int* a_zero, int* b_zero);

/* proj/src/analysis.cpp:142-207.  Returns 0 ok, 1 bad arguments,
 * 4 infeasible (gap/best_lhs/target written). */
int ozo_select_slices(double kappa_a, double kappa_b, int width, double u, int s_max,
                      int has_target, double target, int schedule, int strategy,
                      int acc_bits_used, int precision, int* sa, int* sb, double* lhs,
                      double* target_out, int64_t* products, double* gap);

/* proj/src/generators.cpp:25-49,176-182: mt19937_64 seeded by splitmix64 */
void ozo_random_uniform(int64_t m, int64_t n, uint64_t seed, double lo, double hi,
                        double* out);
/* proj/src/generators.cpp:103-140 */
void ozo_gen_kappa_d(int64_t n, double kappa_d, uint64_t seed, int rotate, double* a_out,
                     double* b_out);

#ifdef __cplusplus
}
#endif
#endif /* OZ_ORACLE_H */
