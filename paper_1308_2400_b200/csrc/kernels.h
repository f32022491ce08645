// kernels.h -- internal launch interface between the host runtime and the
// sm_100a kernels (not part of the public C ABI).
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "costmodel.h"

namespace afmm_dev {

void note_launch();  // counts library kernel launches, records launch errors (runtime.cu)
cudaError_t take_launch_error();  // first launch error of this host thread since the last call

// Rows [l0, l1) of lhs and [q0, q1) of rhs: finite check (check_finite; a
// NaN rep is recorded either way), rep validation
// (into st, global row-major indices), and the per-k vector of the rhs rows
// (Case B: nnz[k] of rhs rows; Case A: rsum[k] of rhs rows). which_case: 0 = A, 1 = B.
// fstats (Case A, optional): the cost-model statistics of the rhs rows
// (launch_counts_f16's four sums), accumulated.
template <class T>
void launch_scan_stats(const T* lhs, const T* rhs, uint64_t ld, uint32_t n, int which_case,
                       uint32_t l0, uint32_t l1, uint32_t q0, uint32_t q1, DevStatus* st,
                       uint32_t* nnz, unsigned long long* rsum, cudaStream_t s,
                       int check_finite = 1, unsigned long long* fstats = nullptr);
// Rows [a0, a1) of X: work[i] (if work != nullptr); slab rows [r0, r1) add
// OpCounts to st and, for Case B with lists != nullptr, get their compacted
// int2 (k, rep) lists; nnz_row (optional, Case A): nonzero bases of each slab row.
template <class T>
void launch_rows(const T* x, uint64_t ld, uint32_t n, int which_case, const uint32_t* nnz,
                 const unsigned long long* rsum, uint32_t a0, uint32_t a1, uint32_t r0,
                 uint32_t r1, int2* lists, uint64_t cap, uint32_t* counts,
                 unsigned long long* work, DevStatus* st, cudaStream_t s,
                 uint32_t* nnz_row = nullptr, int group_allow = 0);
// Case A rep lists: list j = compacted column j of Y. skip (optional): no-op
// when *skip == 0; also a no-op in group mode (group_mode(st, group_allow)).
template <class T>
void launch_transpose_compact(const T* y, uint64_t ld, uint32_t n, int2* lists, uint64_t cap,
                              uint32_t* counts, DevStatus* st, const uint32_t* skip,
                              cudaStream_t s, int group_allow = 0);
// Dense group index of k_bgroup (gidx[g][k], g < ceil(B-form rows / 5), k <
// ldg, ldg % 8 == 0): Case B (which_case 1) from slab rows [r0, r0 + rows) of
// X, Case A from the columns of Y. A no-op unless group_mode(st, allow), and
// (Case A) when skip is given and *skip == 0 (no B-form rows).
template <class T>
void launch_group_idx(const T* rep, uint64_t ld, uint32_t n, int which_case, uint32_t r0,
                      uint32_t rows, uint16_t* gidx, uint64_t ldg, const DevStatus* st, int allow,
                      cudaStream_t s, const uint32_t* skip = nullptr);
// out[oc][r] = in[ir][c] with optional row maps ir = in_rows[r], oc = out_rows[c];
// with a status, nothing is written after a failed validation. plan/dyn: the
// device-side Case A choice (1: rows = plan[1], in_rows += plan[0]; 2: cols =
// plan[1], out_rows += plan[0]).
template <class T>
void launch_transpose(const T* in, uint64_t ld_in, uint32_t rows, uint32_t cols, T* out,
                      uint64_t ld_out, cudaStream_t s, const uint32_t* in_rows = nullptr,
                      const uint32_t* out_rows = nullptr, const DevStatus* st = nullptr,
                      const uint32_t* plan = nullptr, int dyn = 0);

// ---- A-form (Case A, base uniform per warp; aform in bform.cu) ----
// fp16 rep counts of Y (|rep| <= 2048) + per (k, tile) max |rep| | neg flag.
// fstats (4 x u64, accumulated; optional): nonzero reps, sum of trip counts,
// reps beyond 2048, sum of |rep|. need (optional): a no-op when *need == 0
// (run after k_choose with need = the A-form row count).
template <class T>
void launch_counts_f16(const T* y, uint64_t ld, uint32_t n, uint32_t tile_cols, __half* cnt,
                       uint64_t ldc, uint16_t* rmax, unsigned long long* fstats, cudaStream_t s,
                       const uint32_t* need = nullptr);
// Device-side Case A choice (costmodel.h): plan[0] = A-form rows, plan[1] =
// B-form rows, ridx = the slab row order (A rows first), st->a_rows.
size_t choose_scratch_bytes(uint64_t n);
cudaError_t launch_choose(const CaseAModel& md, uint32_t rows, int variant, const uint32_t* nnz_row,
                   const unsigned long long* fstats, uint32_t* scratch, uint32_t* plan,
                   uint32_t* ridx, DevStatus* st, cudaStream_t s);
// Compacted nonzero bases (k, X[r0 + q, k]) of slab rows q = rows_idx[t]
// (or t), t < ntask (or *dyn_ntask), into lists row q / counts[q].
template <class T>
void launch_acompact(const T* x, uint64_t ld, uint32_t n, uint32_t r0, uint32_t ntask,
                     const uint32_t* dyn_ntask, const uint32_t* rows_idx,
                     typename AEntry<T>::type* lists, uint64_t cap, uint32_t* counts,
                     cudaStream_t s);
// Columns per A-form CTA tile (also the rmax tile width).
template <class T>
constexpr uint32_t aform_tile_cols() { return sizeof(T) == 4 ? 1024u : 512u; }
constexpr int kAformRows = 16;      // A-form CTA: 16 consumer warps + 1 TMA warp,
constexpr int kAformCtasPerSm = 1;  // 12-stage fp16 count ring (192 KB), 1 CTA per SM  // rows (warps) per A-form CTA
constexpr uint32_t kAformMaxRep = 2048;  // fp16 counts are exact up to here
// Warp b computes Z row q = row_idx ? row_idx[b] : b (its list is lists row q,
// its output out row q), b < nrows; cmap = fp16 count tensor map (box 256 x KB).
// dyn_nrows (optional): nrows decided on the device (grid sized for nrows).
template <class T>
cudaError_t launch_aform(const CUtensorMap* cmap, const typename AEntry<T>::type* lists,
                         uint64_t cap, const uint32_t* counts, uint32_t nrows,
                         const uint32_t* dyn_nrows, uint32_t ncols, uint32_t nk,
                         const uint16_t* rmax, T* out, uint64_t ld_out, const uint32_t* row_idx,
                         const DevStatus* st, cudaStream_t s);

// TMA geometry shared by the ring kernels: boxes of bform_kb() rows x
// bform_box_bytes() bytes.
int bform_kb();
int bform_box_bytes();
int aform_kb();  // k rows per A-form stage (the fp16 count map's box height)

// k_bform tile shapes: narrow = 512 fp32 / 256 fp64 columns, 2 CTAs per SM;
// wide = 1024 / 512 columns, 1 CTA per SM; small = 256 / 128 columns x 4 rows
// for problems too small to fill the GPU with the larger tiles; fast = the
// reassociated mode's kernel (narrow tile, 1 CTA per SM, blocked fp64 totals).
constexpr int kShapeNarrow = 0;
constexpr int kShapeWide = 1;
constexpr int kShapeSmall = 2;
constexpr int kShapeFast = 4;
constexpr int kWideRows = 16;      // rows per wide CTA (16 consumer warps + 1 TMA warp)
constexpr int kWideCtasPerSm = 1;  // wide CTAs resident per SM (6-stage ring, 192 KB smem)

struct BformLaunch {
  int shape = kShapeNarrow;
  const CUtensorMap* tmap = nullptr;  // base matrix, box bform_kb() x bform_box_bytes()
  const int2* lists = nullptr;  // {k, rep} per row
  uint64_t cap = 0;             // entries per list
  const uint32_t* counts = nullptr;  // entries of each list
  uint32_t nrows = 0;           // B-form rows
  int32_t col0 = 0, ncols = 0;  // base columns [col0, col0 + ncols)
  const uint32_t* dyn_ncols = nullptr;  // optional: ncols decided on the device
  uint32_t nk = 0;              // k range
  uint32_t splits = 1;          // k slices: requested in, launched out (1 = order-preserving)
  uint64_t slice_stride = 0;    // slice z writes to out + z * slice_stride
  uint64_t ld_out = 0;
  const DevStatus* st = nullptr;
  int group_allow = 0;          // exit when the device chose the group kernel (group_mode)
  int ladder = 0;               // fast shape only: each term as a doubling ladder
};
template <class T>
cudaError_t launch_bform(BformLaunch& a, T* out, cudaStream_t s);

// The small-rep group kernel (fp32, order-preserving): B-form rows [0, nrows)
// in groups of kGroupRows over the dense group index gidx (ldg >= nk rounded
// up to bform_kb()), base columns [0, ncols) of the map's matrix (box
// bform_kb() x bform_box_bytes()). Exits unless group_mode(st, allow).
constexpr int kGroupWarps = 15;  // groups (consumer warps) per k_bgroup CTA
cudaError_t launch_bgroup(const CUtensorMap* tmap, const uint16_t* gidx, uint64_t ldg,
                          uint32_t nrows, int32_t ncols, const uint32_t* dyn_ncols, uint32_t nk,
                          float* out, uint64_t ld_out, const DevStatus* st, int allow,
                          cudaStream_t s);

// out[r*ld_out + c] = sum over z (ascending) of part[z*stride + r*ld_part + c]
template <class T>
void launch_reduce_slices(const T* part, uint64_t stride, uint64_t ld_part, uint32_t splits,
                          uint32_t rows, uint32_t cols, T* out, uint64_t ld_out,
                          const DevStatus* st, const uint32_t* dyn_cols, cudaStream_t s);

// ---- device-side seeded generation (generate.cu; random.hpp:111-129) ----
struct GenSpecDev {
  uint64_t n = 0;
  double density = 0.0, low = 0.0, high = 0.0;
  uint64_t range = 0, limit = 0;  // IntegerValued: 2 mu' - 1 and the rejection limit
  int integer = 0;
};
size_t gen_block_count(uint64_t ndraws);
size_t gen_scratch_bytes(uint64_t ndraws);  // per chunk of ndraws draws
size_t gen_carry_bytes();                   // the device carry record
// One chunk: `ctas` stretches of twists x 312 draws of the MT19937-64
// stream, the first starting at the window windows[0] (mt64jump.h's window
// convention); windows[1 .. ctas) are filled by the jump tree (polys: per
// level of stride 4^l, the 3 x 312-word polynomials x^(a 4^l twists 312) mod
// phi, a = 1..3), the window after the chunk goes to end_window; then the
// entries the draws complete are written to out (row-major, leading dimension
// ld; out zeroed beforehand). carry: device record {state, entries started},
// updated (zero = the start of a matrix). scratch: gen_scratch_bytes(draws).
constexpr uint32_t kGenTwistsPerCta = 2048;  // the stretch L = 2048 x 312 draws
constexpr uint32_t kGenMaxCtas = 512;        // 4.5 tree levels; 2.6 GB of draws
constexpr uint32_t kGenLevels = 5;
template <class T>
cudaError_t launch_generate_chunk(const GenSpecDev& spec, uint64_t* windows,
                                  const uint64_t* polys, uint32_t ctas, uint32_t twists,
                                  uint64_t* end_window, uint64_t* draws, void* scratch, void* carry,
                                  T* out, uint64_t ld, cudaStream_t s);

// FP-add peak microbenchmark (peak.cu)
cudaError_t run_peak(int dtype, double* adds_per_second, double* sm_mhz);

}  // namespace afmm_dev
