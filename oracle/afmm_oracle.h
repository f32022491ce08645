/*
 * afmm_oracle.h -- CPU restatement of the reference AFMM hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the parity checker for the sm_100a
 * product in paper_1308_2400_b200/. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it. The product
 * path never links, calls or falls back to it.
 *
 * Every function restates a function of the reference (paths relative to
 * /root/reference):
 *   oracle_case_{a,b}_*      proj/include/afmm/kernels.hpp:113-136 / :142-165
 *   (add-repeated core)      proj/include/afmm/kernels.hpp:95-104
 *   (rep-operand validation) proj/include/afmm/kernels.hpp:25-43
 *   oracle_mt64_*            std::mt19937_64 as used by proj/include/afmm/random.hpp:113
 *   oracle_uniform01 / _below proj/include/afmm/random.hpp:92-104
 *   oracle_splitmix64        proj/include/afmm/random.hpp:84-89
 *   oracle_generate          proj/include/afmm/random.hpp:111-129
 *   oracle_random_integer_matrix  proj/tests/test_kernels.cpp:16-24
 *
 * Parity pin: tests/test_oracle.py checks this restatement bit-for-bit against
 * (1) the golden vectors in tests/golden/ produced by the unmodified reference
 * (oracle/_ref, built from /root/reference by oracle/Makefile), and (2) the
 * live oracle/_ref library whenever it is present.
 */
#ifndef AFMM_ORACLE_H
#define AFMM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint64_t additions;
  uint64_t multiplications;
  uint64_t zero_skips;
} oracle_counts;

/* kind: 0 = ok, 1 = "is not integer-valued", 2 = "exceeds the exact integer
 * range" (kernels.hpp:31-40). row/col is the first offender in row-major
 * order, value its (widened) value. */
typedef struct {
  int kind;
  uint64_t row;
  uint64_t col;
  double value;
} oracle_error;

/* Product rows [row_begin, row_end) of Z = lhs * rhs (n x n, row-major).
 * `out` receives (row_end - row_begin) x n values. When `validate` is nonzero
 * the whole rep operand is checked first, exactly as the reference does, and
 * nothing is computed on failure (return value 1). Counts cover the computed
 * rows only. */
int oracle_case_a_f64(const double* lhs, const double* rhs, double* out, uint64_t n,
                      uint64_t row_begin, uint64_t row_end, int validate,
                      oracle_counts* counts, oracle_error* err);
int oracle_case_b_f64(const double* lhs, const double* rhs, double* out, uint64_t n,
                      uint64_t row_begin, uint64_t row_end, int validate,
                      oracle_counts* counts, oracle_error* err);
/* fp32 restatement: identical control flow, float accumulator and float
 * step (the reference is fp64-only, proj/README.md:91). Rep validation and
 * llround run on the exactly widened double value, as the reference would
 * see it. */
int oracle_case_a_f32(const float* lhs, const float* rhs, float* out, uint64_t n,
                      uint64_t row_begin, uint64_t row_end, int validate,
                      oracle_counts* counts, oracle_error* err);
int oracle_case_b_f32(const float* lhs, const float* rhs, float* out, uint64_t n,
                      uint64_t row_begin, uint64_t row_end, int validate,
                      oracle_counts* counts, oracle_error* err);

/* Row-parallel variants (pthreads, `threads` workers over disjoint row
 * blocks; rows are independent, kernels.hpp:119/148, so results are
 * bit-identical to the single-thread call). No validation. Used only as the
 * CPU baseline in bench.py. */
int oracle_case_a_f64_mt(const double* lhs, const double* rhs, double* out, uint64_t n,
                         uint64_t row_begin, uint64_t row_end, int threads,
                         oracle_counts* counts);
int oracle_case_b_f64_mt(const double* lhs, const double* rhs, double* out, uint64_t n,
                         uint64_t row_begin, uint64_t row_end, int threads,
                         oracle_counts* counts);
int oracle_case_a_f32_mt(const float* lhs, const float* rhs, float* out, uint64_t n,
                         uint64_t row_begin, uint64_t row_end, int threads,
                         oracle_counts* counts);
int oracle_case_b_f32_mt(const float* lhs, const float* rhs, float* out, uint64_t n,
                         uint64_t row_begin, uint64_t row_end, int threads,
                         oracle_counts* counts);

/* Classical i-j-k product (kernels.hpp:50-66), the reference tests' product
 * oracle on integer inputs (test_kernels.cpp:143,203). */
void oracle_multiply_ijk_f64(const double* lhs, const double* rhs, double* out, uint64_t n);

/* Seeded generation, restated from random.hpp / test_kernels.cpp. */
uint64_t oracle_splitmix64(uint64_t x);
void oracle_random_integer_matrix(uint64_t n, int low, int high, uint64_t seed, double* out);
/* role: 0 = RealValued [low, high], 1 = IntegerValued {1..2mu-1}. Returns 0,
 * or -1 on an invalid spec (random.hpp:60-79). */
int oracle_generate(uint64_t n, double density, double mu_prime, int role, double low,
                    double high, uint64_t seed, double* out);

#ifdef __cplusplus
}
#endif

#endif
