/*
 * fast_check.c -- a vectorised CPU checker for FULL-SIZE parity runs.
 *
 * TEST INFRASTRUCTURE ONLY (like afmm_oracle.c): it exists so the GPU product
 * can be checked on EVERY row at the BASELINE sizes (cfg5: 4.3e13 additions),
 * which the scalar restatement (afmm_oracle.c, ~1e9 adds/s per core) cannot
 * do in test time. It computes Case B rows (kernels.hpp:142-165) with the
 * reference's per-element order -- for every element Z[i][j] the terms arrive
 * in increasing k, each as |rep| sequential `acc += step` (kernels.hpp:95-104)
 * -- but vectorised ACROSS j: the loop over an element's adds is unchanged,
 * only independent elements run side by side. Two deliberate differences from
 * the reference, both bit-neutral and both pinned by tests/test_oracle.py
 * against the scalar oracle and the unmodified reference:
 *   - zero bases are added (as +0 / -0) instead of skipped: the accumulator
 *     starts at +0 and a round-to-nearest sum is -0 only if both addends are
 *     -0, so adding a zero never changes it;
 *   - a negative rep subtracts the base (acc - b == acc + (-b) in IEEE 754).
 * Case A is checked through the identity afmm_case_a(X, Y) ==
 * afmm_case_b(Y^T, X^T)^T (same per-element add sequence; verified bit for bit
 * against the reference in tests/test_oracle.py), so the caller passes the
 * transposed operands and gets Z^T rows.
 *
 * Compiled with -O3 -ffp-contract=off (no FMA contraction) and without
 * -ffast-math: every vector add is an IEEE round-to-nearest add per lane.
 * target_clones picks AVX-512 / AVX2 / SSE2 at run time (the GPU box's host).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define RB 32 /* output rows per tile: one pass over Y serves RB rows */
#define NV 16 /* vectors per column chunk (1 KB of a row) */

typedef float vf32 __attribute__((vector_size(64)));
typedef double vf64 __attribute__((vector_size(64)));

/* Rows [i0, i0 + rb) x columns [j0, j0 + NV * W) of Z = caseB(x, y), tile
 * accumulators in z (row stride n). reps[q * n + k] = the term count of row
 * i0 + q at k (0 = no term). For every k the chunk of Y row k is loaded once
 * and serves all rb rows; each row's chunk is held in registers for its
 * |rep| steps of `z += y` (or `z -= y`, a negative rep). */
#define DEFINE_TILE(SUF, T, V)                                                                \
  __attribute__((target_clones("avx512f", "avx2", "default"))) static void tile_##SUF(        \
      T* __restrict z, const T* __restrict y, uint64_t n, uint64_t j0, uint64_t rb,            \
      const int64_t* __restrict reps) {                                                       \
    enum { W = sizeof(V) / sizeof(T) };                                                       \
    for (uint64_t k = 0; k < n; ++k) {                                                        \
      V yv[NV];                                                                               \
      int loaded = 0;                                                                         \
      for (uint64_t q = 0; q < rb; ++q) {                                                     \
        const int64_t r = reps[q * n + k];                                                    \
        if (r == 0) continue;                                                                 \
        if (!loaded) {                                                                        \
          memcpy(yv, y + k * n + j0, sizeof yv);                                              \
          loaded = 1;                                                                         \
        }                                                                                     \
        T* zq = z + q * n + j0;                                                               \
        V zv[NV];                                                                             \
        memcpy(zv, zq, sizeof zv);                                                            \
        const uint64_t a = r < 0 ? (uint64_t)0 - (uint64_t)r : (uint64_t)r;                  \
        if (r > 0) {                                                                          \
          for (uint64_t s = 0; s < a; ++s)                                                    \
            for (int v = 0; v < NV; ++v) zv[v] += yv[v];                                      \
        } else {                                                                              \
          for (uint64_t s = 0; s < a; ++s)                                                    \
            for (int v = 0; v < NV; ++v) zv[v] -= yv[v];                                      \
        }                                                                                     \
        memcpy(zq, zv, sizeof zv);                                                            \
      }                                                                                       \
    }                                                                                         \
  }                                                                                           \
  /* the columns past the last whole chunk, element by element (same order) */               \
  static void tail_##SUF(T* z, const T* y, uint64_t n, uint64_t j0, uint64_t rb,              \
                         const int64_t* reps) {                                               \
    for (uint64_t k = 0; k < n; ++k)                                                          \
      for (uint64_t q = 0; q < rb; ++q) {                                                     \
        const int64_t r = reps[q * n + k];                                                    \
        if (r == 0) continue;                                                                 \
        const uint64_t a = r < 0 ? (uint64_t)0 - (uint64_t)r : (uint64_t)r;                  \
        for (uint64_t j = j0; j < n; ++j) {                                                   \
          T acc = z[q * n + j];                                                               \
          const T b = y[k * n + j];                                                           \
          if (r > 0)                                                                          \
            for (uint64_t s = 0; s < a; ++s) acc += b;                                        \
          else                                                                                \
            for (uint64_t s = 0; s < a; ++s) acc -= b;                                        \
          z[q * n + j] = acc;                                                                 \
        }                                                                                     \
      }                                                                                       \
  }                                                                                           \
  /* rows idx[0 .. cnt) of Z = caseB(x, y) into z (list position p at z[p * n]) */          \
  static void rows_##SUF(const T* x, const T* y, uint64_t n, const uint64_t* idx,             \
                         uint64_t cnt, T* z, int64_t* reps) {                                 \
    enum { W = sizeof(V) / sizeof(T), CW = NV * W };                                          \
    for (uint64_t p = 0; p < cnt; p += RB) {                                                  \
      const uint64_t rb = p + RB <= cnt ? RB : cnt - p;                                       \
      for (uint64_t q = 0; q < rb; ++q) {                                                     \
        const T* xr = x + idx[p + q] * n;                                                     \
        for (uint64_t k = 0; k < n; ++k) {                                                    \
          const double v = (double)xr[k];                                                     \
          reps[q * n + k] = v == 0.0 ? 0 : llround(v);                                        \
        }                                                                                     \
        memset(z + (p + q) * n, 0, n * sizeof(T));                                            \
      }                                                                                       \
      uint64_t j0 = 0;                                                                        \
      for (; j0 + CW <= n; j0 += CW) tile_##SUF(z + p * n, y, n, j0, rb, reps);               \
      if (j0 < n) tail_##SUF(z + p * n, y, n, j0, rb, reps);                                  \
    }                                                                                         \
  }

DEFINE_TILE(f32, float, vf32)
DEFINE_TILE(f64, double, vf64)

typedef struct {
  int dtype;
  const void* x;
  const void* y;
  uint64_t n;
  const uint64_t* idx;
  uint64_t cnt;
  void* z;
} job;

static void* worker(void* p) {
  job* j = (job*)p;
  int64_t* scratch = (int64_t*)malloc(sizeof(int64_t) * RB * (j->n ? j->n : 1));
  if (!scratch) return (void*)1;
  if (j->dtype == 0)
    rows_f64((const double*)j->x, (const double*)j->y, j->n, j->idx, j->cnt, (double*)j->z,
             scratch);
  else
    rows_f32((const float*)j->x, (const float*)j->y, j->n, j->idx, j->cnt, (float*)j->z, scratch);
  free(scratch);
  return NULL;
}

/* Rows rows[0 .. count) of afmm_case_b(x, y) (x = integer-valued reps, y =
 * bases, both row-major n x n, dtype 0 = f64, 1 = f32) into z (count x n,
 * position p = row rows[p]), on `threads` threads. The inputs must already be
 * valid (finite, integer reps): the checker does not validate. Returns 0 on
 * success. */
int fast_case_b_rows(int dtype, const void* x, const void* y, uint64_t n, const uint64_t* rows,
                     uint64_t count, void* z, int threads) {
  if (threads < 1) threads = 1;
  const uint64_t tiles = (count + RB - 1) / RB;
  if ((uint64_t)threads > tiles) threads = (int)tiles;
  if (threads < 1) return 0;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  job* jobs = (job*)malloc(sizeof(job) * threads);
  if (!th || !jobs) {
    free(th);
    free(jobs);
    return 1;
  }
  const size_t es = dtype == 0 ? 8 : 4;
  /* contiguous shares of whole RB-row tiles of the list */
  const uint64_t per = (tiles + (uint64_t)threads - 1) / (uint64_t)threads;
  int nt = 0;
  for (uint64_t t = 0; t < tiles; t += per, ++nt) {
    const uint64_t lo = t * RB, hi = (t + per) * RB < count ? (t + per) * RB : count;
    jobs[nt].dtype = dtype;
    jobs[nt].x = x;
    jobs[nt].y = y;
    jobs[nt].n = n;
    jobs[nt].idx = rows + lo;
    jobs[nt].cnt = hi - lo;
    jobs[nt].z = (char*)z + lo * n * es;
  }
  int rc = 0, started = 0;
  for (int t = 0; t < nt; ++t) {
    if (pthread_create(&th[t], NULL, worker, &jobs[t]) != 0) {
      rc = 1;
      break;
    }
    ++started;
  }
  for (int t = 0; t < started; ++t) {
    void* ret = NULL;
    pthread_join(th[t], &ret);
    if (ret) rc = 1;
  }
  free(th);
  free(jobs);
  return rc;
}
