// costmodel.h -- the Case A kernel-time model (host and device).
//
// Case A can run in two orientations (bform.cu): the B-form (Case B on
// transposed operands; its cost per 1024/512-row tile of the slab does not
// depend on X's density, every zero base still issues an add) and the A-form
// (the reference's own orientation, kernels.hpp:118-135; a warp per Z row
// skips zero bases, so a row costs in proportion to its nonzero bases). The
// model estimates both in SM sub-partition cycles from prepass statistics and
// picks the cheapest of: pure B-form, pure A-form, or "the m sparsest rows
// A-form, the rest B-form in whole tiles". It is evaluated on the device
// (k_choose in prepass.cu: no host round trip, so Case A calls stay
// asynchronous and graph-capturable) and on the host (the multi-GPU row
// partition predicts per-row time with the same constants).
//
// Constants fitted on B200:
//   A-form: ~75 cycles per (nonzero base, column tile) entry + ~54 (fp32) /
//           ~45 (fp64) per predicated iteration; an entry's trip count is its
//           tile's max |rep| at its k (mean R = trip_sum / (n x tiles)).
//   B-form: per B tile, b_step cycles per rep step per list entry + an entry
//           overhead (larger when the mean rep is below 3: the smem-bound
//           regime), over all of Y's nonzero reps; in group mode (k_bgroup,
//           reps <= 2) 16 cycles per rep step and row + 78 per nonempty
//           (group of 5 rows, k), per 512-row tile (fitted on constant reps 1
//           and 2 at n = 4096: 3.59 and 5.37 ms).
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define AFMM_HD __host__ __device__ __forceinline__
#else
#define AFMM_HD inline
#endif

namespace afmm_dev {

struct CaseAModel {
  // inputs
  uint32_t elem = 4;        // sizeof(T)
  uint64_t n = 0;           // problem size (k range and B-form rows)
  uint32_t sms = 148;
  uint64_t nnz_y = 0;       // nonzero reps of Y
  uint64_t trip_sum = 0;    // sum over (k, A tile) of the tile's max |rep|
  uint64_t rep_sum = 0;     // sum of |rep| over Y
  // B-form launch geometry (the shape the runtime picks for the B part)
  uint32_t b_tile = 1024;       // slab rows per B-form tile (TILE_N)
  uint32_t b_warps_per_cta = 16; // B-form rows (consumer warps) per CTA
  uint32_t b_ctas_per_sm = 1;
  double b_step = 32.0;         // cycles per rep step per list entry and tile
  double b_entry = 56.0;        // cycles per list entry and tile (mean rep >= 3)
  double b_entry_small = 100.0; // the same when the mean rep is below 3
  // Group kernel (k_bgroup: every |rep| <= 2, none negative, fp32): the B part
  // runs 5 B-form rows per warp over 512-column tiles. group_allow is the
  // host's half of the decision, group the device's (group_mode in k_choose,
  // or the merged status of a multi-device call).
  int group_allow = 0;
  bool group = false;
  uint32_t g_tile = 512;       // slab rows per k_bgroup tile
  uint32_t g_warps_per_cta = 15;
  double g_step = 16.0;        // cycles per rep step per B-form row and tile (8 FADD2)
  double g_entry = 78.0;       // cycles per nonempty (group, k) and tile
  // A-form launch geometry
  uint32_t a_tile = 1024;   // columns per A-form CTA (aform_tile_cols)
  uint32_t a_rows_per_cta = 16;
  uint32_t a_ctas_per_sm = 1;

  AFMM_HD double a_tiles() const { return (double)((n + a_tile - 1) / a_tile); }
  // A-form cycles per nonzero base of a row
  AFMM_HD double per_base() const {
    const double tiles = a_tiles();
    const double rmean = (double)trip_sum / ((double)n * tiles);
    const double it = elem == 4 ? 54.0 : 45.0;
    return tiles * (75.0 + it * rmean);
  }
  // B-form slab rows per tile
  AFMM_HD uint64_t tile_rows() const { return group ? g_tile : b_tile; }
  // B-form cycles per tile of slab rows
  AFMM_HD double per_tile() const {
    if (nnz_y == 0) return 0.0;
    if (group) {
      // nonempty (group, k): a group of 5 rows is empty at k with
      // probability (1 - d)^5, d = the density of nonzero reps
      const double d = (double)nnz_y / ((double)n * (double)n);
      const double e1 = 1.0 - d, e5 = e1 * e1 * e1 * e1 * e1;
      const double entries = (double)((n + 4) / 5) * (double)n * (1.0 - e5);
      return g_step * (double)rep_sum + g_entry * entries;
    }
    const double rbar = (double)rep_sum / (double)nnz_y;
    return b_step * (double)rep_sum + (rbar < 3.0 ? b_entry_small : b_entry) * (double)nnz_y;
  }
  // Busy fraction of the GPU's warp slots for `rows` rows (warps) of `tiles`
  // column tiles in CTAs of at most cw rows, `per_sm` CTAs per SM: the
  // launchers trim the rows per CTA (balanced_rows in bform.cu) to the r in
  // [cw/2, cw] minimising waves x r, i.e. the busiest SM's share of rows.
  AFMM_HD double wave_eff(uint64_t rows, uint64_t tiles, uint32_t cw, uint32_t per_sm) const {
    if (rows == 0 || tiles == 0) return 1.0;
    const uint64_t slots = (uint64_t)per_sm * sms;
    uint64_t best = 0;
    for (uint32_t r = cw; r >= 1 && 2 * r >= cw; --r) {
      const uint64_t ctas = (rows + r - 1) / r * tiles;
      const uint64_t c = (ctas + slots - 1) / slots * r;
      if (best == 0 || c * 100 < best * 97) best = c;
    }
    return (double)rows * (double)tiles / ((double)slots * (double)best);
  }
  // B part of tiles_b whole tiles (n B-form rows), charged its wave quantisation
  AFMM_HD double cost_b(uint64_t tiles_b) const {
    if (tiles_b == 0) return 0.0;
    if (group)
      return (double)tiles_b * per_tile() / wave_eff((n + 4) / 5, tiles_b, g_warps_per_cta, 1);
    return (double)tiles_b * per_tile() / wave_eff(n, tiles_b, b_warps_per_cta, b_ctas_per_sm);
  }
  // A part of m rows holding `bases` nonzero bases in total
  AFMM_HD double cost_a(uint64_t m, double bases) const {
    if (m == 0) return 0.0;
    return per_base() * bases / wave_eff(m, (uint64_t)a_tiles(), a_rows_per_cta, a_ctas_per_sm);
  }
};

// Variants of the choice: 0 = by cost (a full switch to the A-form needs a
// 15% margin over the pure B-form, a split 10%), 1 = A-form forced, 2 = the
// best split forced (tests).
constexpr int kChooseAuto = 0;
constexpr int kChooseAForm = 1;
constexpr int kChooseSplit = 2;

// The number m of slab rows to run in the A-form (the m sparsest rows; 0 =
// pure B-form, rows = pure A-form). pre(m) = total nonzero bases of the m
// sparsest rows. Splits keep the B part a whole number of tiles. *time (if
// given) receives the modeled cycles of the choice. split_cost (optional):
// split_cost[j] = the cost of the split with j B tiles, precomputed (k_choose
// prices the candidates in parallel; the same expression).
// (host instantiations pass host lambdas; the device one a device functor)
#pragma nv_exec_check_disable
template <class Pre>
AFMM_HD uint64_t choose_aform_rows(const CaseAModel& md, uint64_t rows, int variant, Pre pre,
                                   double* time = nullptr, const double* split_cost = nullptr) {
  if (rows == 0 || md.nnz_y == 0) {
    if (time) *time = 0.0;
    return variant == kChooseAForm ? rows : 0;
  }
  const uint64_t tb = md.tile_rows(), tiles_all = (rows + tb - 1) / tb;
  const double pure_b = md.cost_b(tiles_all);
  const double pure_a = md.cost_a(rows, pre(rows));
  if (variant == kChooseAForm) {
    if (time) *time = pure_a;
    return rows;
  }
  double best_split = 0.0;
  uint64_t m_split = 0;
  for (uint64_t j = 1; j * tb < rows; ++j) {
    const uint64_t m = rows - j * tb;
    const double c = split_cost ? split_cost[j] : md.cost_a(m, pre(m)) + md.cost_b(j);
    if (m_split == 0 || c < best_split) {
      best_split = c;
      m_split = m;
    }
  }
  if (variant == kChooseSplit) {
    if (time) *time = m_split ? best_split : pure_b;
    return m_split;
  }
  double best = pure_b;
  uint64_t best_m = 0;
  if (pure_a < 0.85 * pure_b) {
    best = pure_a;
    best_m = rows;
  }
  if (m_split && best_split < 0.90 * pure_b && best_split < best) {
    best = best_split;
    best_m = m_split;
  }
  if (time) *time = best;
  return best_m;
}

}  // namespace afmm_dev
