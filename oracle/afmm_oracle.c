/*
 * afmm_oracle.c -- CPU restatement of the reference AFMM hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see afmm_oracle.h): the checker for the sm_100a
 * product, never part of it. Compiled with -O2 -ffp-contract=off, the
 * reference's own FP flag (proj/CMakeLists.txt:14-16), so every `acc += step`
 * below is one IEEE add in program order.
 */
#include "afmm_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* kernels.hpp:25-43: |v - round(v)| > 1e-9 -> not integer-valued, then
 * |v| > 2^53 -> exceeds the exact integer range; first offender in row-major
 * order wins, and the first failing test at that element names the kind. */
static int validate_rep_operand_f64(const double* m, uint64_t n, oracle_error* err) {
  for (uint64_t i = 0; i < n; ++i) {
    for (uint64_t j = 0; j < n; ++j) {
      const double v = m[i * n + j];
      int kind = 0;
      if (fabs(v - round(v)) > 1e-9) kind = 1;
      else if (fabs(v) > 9007199254740992.0) kind = 2;
      if (kind) {
        if (err) { err->kind = kind; err->row = i; err->col = j; err->value = v; }
        return 1;
      }
    }
  }
  if (err) { err->kind = 0; err->row = 0; err->col = 0; err->value = 0.0; }
  return 0;
}

static int validate_rep_operand_f32(const float* m, uint64_t n, oracle_error* err) {
  for (uint64_t i = 0; i < n; ++i) {
    for (uint64_t j = 0; j < n; ++j) {
      const double v = (double)m[i * n + j];
      int kind = 0;
      if (fabs(v - round(v)) > 1e-9) kind = 1;
      else if (fabs(v) > 9007199254740992.0) kind = 2;
      if (kind) {
        if (err) { err->kind = kind; err->row = i; err->col = j; err->value = v; }
        return 1;
      }
    }
  }
  if (err) { err->kind = 0; err->row = 0; err->col = 0; err->value = 0.0; }
  return 0;
}

/* The body of both cases, instantiated for T = double and T = float.
 * Case A (kernels.hpp:113-136): base = lhs(i,k); zero base -> ++zero_skips;
 *   rep = rhs(k,j); rep == 0.0 or llround(rep) == 0 -> skip, not tallied.
 * Case B (kernels.hpp:142-165): rep = lhs(i,k); rep == 0.0 or llround == 0 ->
 *   skip the j loop, not tallied; base = rhs(k,j); zero base -> ++zero_skips.
 * add_repeated (kernels.hpp:95-104): step = reps >= 0 ? base : -base, then
 *   |reps| sequential `acc += step`, additions += |reps|. */
#define DEFINE_CASES(SUF, T)                                                                  \
  static void case_a_rows_##SUF(const T* lhs, const T* rhs, T* out, uint64_t n, uint64_t r0,  \
                                uint64_t r1, oracle_counts* c) {                              \
    memset(out, 0, sizeof(T) * (r1 - r0) * n);                                                \
    for (uint64_t i = r0; i < r1; ++i) {                                                      \
      T* zrow = out + (i - r0) * n;                                                           \
      for (uint64_t k = 0; k < n; ++k) {                                                      \
        const T base = lhs[i * n + k];                                                        \
        if (base == (T)0) { ++c->zero_skips; continue; }                                      \
        for (uint64_t j = 0; j < n; ++j) {                                                    \
          const T rep_value = rhs[k * n + j];                                                 \
          if (rep_value == (T)0) continue;                                                    \
          const long long reps = llround((double)rep_value);                                  \
          if (reps == 0) continue;                                                            \
          const T step = reps >= 0 ? base : -base;                                            \
          const uint64_t times = reps >= 0 ? (uint64_t)reps : (uint64_t)(-reps);              \
          T acc = zrow[j];                                                                    \
          for (uint64_t t = 0; t < times; ++t) acc += step;                                   \
          zrow[j] = acc;                                                                      \
          c->additions += times;                                                              \
        }                                                                                     \
      }                                                                                       \
    }                                                                                         \
  }                                                                                           \
  static void case_b_rows_##SUF(const T* lhs, const T* rhs, T* out, uint64_t n, uint64_t r0,  \
                                uint64_t r1, oracle_counts* c) {                              \
    memset(out, 0, sizeof(T) * (r1 - r0) * n);                                                \
    for (uint64_t i = r0; i < r1; ++i) {                                                      \
      T* zrow = out + (i - r0) * n;                                                           \
      for (uint64_t k = 0; k < n; ++k) {                                                      \
        const T rep_value = lhs[i * n + k];                                                   \
        if (rep_value == (T)0) continue;                                                      \
        const long long reps = llround((double)rep_value);                                    \
        if (reps == 0) continue;                                                              \
        const uint64_t times = reps >= 0 ? (uint64_t)reps : (uint64_t)(-reps);                \
        for (uint64_t j = 0; j < n; ++j) {                                                    \
          const T base = rhs[k * n + j];                                                      \
          if (base == (T)0) { ++c->zero_skips; continue; }                                    \
          const T step = reps >= 0 ? base : -base;                                            \
          T acc = zrow[j];                                                                    \
          for (uint64_t t = 0; t < times; ++t) acc += step;                                   \
          zrow[j] = acc;                                                                      \
          c->additions += times;                                                              \
        }                                                                                     \
      }                                                                                       \
    }                                                                                         \
  }                                                                                           \
  int oracle_case_a_##SUF(const T* lhs, const T* rhs, T* out, uint64_t n, uint64_t r0,        \
                          uint64_t r1, int validate, oracle_counts* counts,                   \
                          oracle_error* err) {                                                \
    oracle_counts c = {0, 0, 0};                                                              \
    if (validate && validate_rep_operand_##SUF(rhs, n, err)) return 1;                        \
    case_a_rows_##SUF(lhs, rhs, out, n, r0, r1, &c);                                          \
    if (counts) *counts = c;                                                                  \
    return 0;                                                                                 \
  }                                                                                           \
  int oracle_case_b_##SUF(const T* lhs, const T* rhs, T* out, uint64_t n, uint64_t r0,        \
                          uint64_t r1, int validate, oracle_counts* counts,                   \
                          oracle_error* err) {                                                \
    oracle_counts c = {0, 0, 0};                                                              \
    if (validate && validate_rep_operand_##SUF(lhs, n, err)) return 1;                        \
    case_b_rows_##SUF(lhs, rhs, out, n, r0, r1, &c);                                          \
    if (counts) *counts = c;                                                                  \
    return 0;                                                                                 \
  }

DEFINE_CASES(f64, double)
DEFINE_CASES(f32, float)

/* ---- row-parallel CPU baseline ------------------------------------------ */

typedef struct {
  int which; /* 0 a64, 1 b64, 2 a32, 3 b32 */
  const void* lhs;
  const void* rhs;
  void* out;
  uint64_t n, r0, r1, base_row;
  oracle_counts counts;
} mt_job;

static void* mt_worker(void* arg) {
  mt_job* j = (mt_job*)arg;
  memset(&j->counts, 0, sizeof j->counts);
  if (j->r0 >= j->r1) return NULL;
  const uint64_t off = (j->r0 - j->base_row) * j->n;
  switch (j->which) {
    case 0: case_a_rows_f64((const double*)j->lhs, (const double*)j->rhs,
                            (double*)j->out + off, j->n, j->r0, j->r1, &j->counts); break;
    case 1: case_b_rows_f64((const double*)j->lhs, (const double*)j->rhs,
                            (double*)j->out + off, j->n, j->r0, j->r1, &j->counts); break;
    case 2: case_a_rows_f32((const float*)j->lhs, (const float*)j->rhs,
                            (float*)j->out + off, j->n, j->r0, j->r1, &j->counts); break;
    default: case_b_rows_f32((const float*)j->lhs, (const float*)j->rhs,
                             (float*)j->out + off, j->n, j->r0, j->r1, &j->counts); break;
  }
  return NULL;
}

static int run_mt(int which, const void* lhs, const void* rhs, void* out, uint64_t n,
                  uint64_t r0, uint64_t r1, int threads, oracle_counts* counts) {
  if (threads < 1) threads = 1;
  const uint64_t rows = r1 > r0 ? r1 - r0 : 0;
  if ((uint64_t)threads > rows && rows > 0) threads = (int)rows;
  mt_job* jobs = (mt_job*)calloc((size_t)threads, sizeof(mt_job));
  pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  if (!jobs || !tids) { free(jobs); free(tids); return -1; }
  for (int t = 0; t < threads; ++t) {
    jobs[t].which = which; jobs[t].lhs = lhs; jobs[t].rhs = rhs; jobs[t].out = out;
    jobs[t].n = n; jobs[t].base_row = r0;
    /* interleaved row blocks of 1 row keep heavy rows spread over workers */
    jobs[t].r0 = r0 + rows * (uint64_t)t / (uint64_t)threads;
    jobs[t].r1 = r0 + rows * (uint64_t)(t + 1) / (uint64_t)threads;
    pthread_create(&tids[t], NULL, mt_worker, &jobs[t]);
  }
  oracle_counts c = {0, 0, 0};
  for (int t = 0; t < threads; ++t) {
    pthread_join(tids[t], NULL);
    c.additions += jobs[t].counts.additions;
    c.zero_skips += jobs[t].counts.zero_skips;
  }
  if (counts) *counts = c;
  free(jobs);
  free(tids);
  return 0;
}

int oracle_case_a_f64_mt(const double* l, const double* r, double* o, uint64_t n, uint64_t r0,
                         uint64_t r1, int th, oracle_counts* c) {
  return run_mt(0, l, r, o, n, r0, r1, th, c);
}
int oracle_case_b_f64_mt(const double* l, const double* r, double* o, uint64_t n, uint64_t r0,
                         uint64_t r1, int th, oracle_counts* c) {
  return run_mt(1, l, r, o, n, r0, r1, th, c);
}
int oracle_case_a_f32_mt(const float* l, const float* r, float* o, uint64_t n, uint64_t r0,
                         uint64_t r1, int th, oracle_counts* c) {
  return run_mt(2, l, r, o, n, r0, r1, th, c);
}
int oracle_case_b_f32_mt(const float* l, const float* r, float* o, uint64_t n, uint64_t r0,
                         uint64_t r1, int th, oracle_counts* c) {
  return run_mt(3, l, r, o, n, r0, r1, th, c);
}

/* kernels.hpp:50-66 */
void oracle_multiply_ijk_f64(const double* lhs, const double* rhs, double* out, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i)
    for (uint64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (uint64_t k = 0; k < n; ++k) acc += lhs[i * n + k] * rhs[k * n + j];
      out[i * n + j] = acc;
    }
}

/* ---- seeded generation --------------------------------------------------- */

/* std::mt19937_64 (the published MT19937-64 parameters). */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ull) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFull);
      uint64_t xa = x >> 1;
      if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

/* random.hpp:84-89 */
uint64_t oracle_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* random.hpp:92-94 */
static double uniform01(mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; }

/* random.hpp:97-104 */
static uint64_t uniform_below(mt64* g, uint64_t range) {
  const uint64_t limit = UINT64_MAX - UINT64_MAX % range;
  uint64_t x = mt64_next(g);
  while (x >= limit) x = mt64_next(g);
  return x % range;
}

/* test_kernels.cpp:16-24 (also acceptance.hpp:72-82) */
void oracle_random_integer_matrix(uint64_t n, int low, int high, uint64_t seed, double* out) {
  mt64 g;
  mt64_seed(&g, seed);
  const uint64_t range = (uint64_t)(high - low + 1);
  for (uint64_t idx = 0; idx < n * n; ++idx)
    out[idx] = (double)(low + (long long)uniform_below(&g, range));
}

/* random.hpp:60-79 (validate) and :111-129 (generate) */
int oracle_generate(uint64_t n, double density, double mu_prime, int role, double low,
                    double high, uint64_t seed, double* out) {
  if (n == 0 || !(density >= 0.0 && density <= 1.0) || !(mu_prime > 0.0)) return -1;
  if (role == 1) {
    if (fabs(mu_prime - round(mu_prime)) > 1e-9 || mu_prime < 1.0) return -1;
  } else if (!(isfinite(low) && isfinite(high)) || low > high) {
    return -1;
  }
  mt64 g;
  mt64_seed(&g, seed);
  memset(out, 0, sizeof(double) * n * n);
  const uint64_t value_range = role == 1 ? 2 * (uint64_t)llround(mu_prime) - 1 : 0;
  for (uint64_t idx = 0; idx < n * n; ++idx) {
    if (uniform01(&g) >= density) continue;
    if (role == 1) out[idx] = (double)(1 + uniform_below(&g, value_range));
    else out[idx] = low + (high - low) * uniform01(&g);
  }
  return 0;
}
