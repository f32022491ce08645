// kernels.h -- internal launch interface between the host runtime and the
// sm_100a kernels (not part of the public C ABI).
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace afmm_dev {

void note_launch();  // counts library kernel launches (runtime.cu)

// Both operands: finite check, rep validation (into st), and the per-k vector
// (Case B: nnz[k] of rhs rows; Case A: rsum[k] of rhs rows). which_case: 0 = A, 1 = B.
template <class T>
void launch_scan_stats(const T* lhs, const T* rhs, uint64_t ld, uint32_t n, int which_case,
                       DevStatus* st, uint32_t* nnz, unsigned long long* rsum, cudaStream_t s);
// Rows of X: work[i] for all rows; slab [r0, r1) adds OpCounts to st and, for
// Case B with lists != nullptr, gets its compacted (k, rep) lists.
// nnz_row (optional, Case A): nonzero bases of each slab row.
template <class T>
void launch_rows(const T* x, uint64_t ld, uint32_t n, int which_case, const uint32_t* nnz,
                 const unsigned long long* rsum, uint32_t r0, uint32_t r1, int2* lists,
                 uint64_t cap, uint32_t* counts, unsigned long long* work, DevStatus* st,
                 cudaStream_t s, uint32_t* nnz_row = nullptr);
// Case A rep lists: list j = compacted column j of Y.
template <class T>
void launch_transpose_compact(const T* y, uint64_t ld, uint32_t n, int2* lists, uint64_t cap,
                              uint32_t* counts, cudaStream_t s);
// out[oc][r] = in[ir][c] with optional row maps ir = in_rows[r], oc = out_rows[c];
// with a status, nothing is written after a failed validation.
template <class T>
void launch_transpose(const T* in, uint64_t ld_in, uint32_t rows, uint32_t cols, T* out,
                      uint64_t ld_out, cudaStream_t s, const uint32_t* in_rows = nullptr,
                      const uint32_t* out_rows = nullptr, const DevStatus* st = nullptr);

// ---- A-form (Case A, base uniform per warp; aform in bform.cu) ----
// fp16 rep counts of Y (|rep| <= 2048) + per (k, tile) max |rep| | neg flag.
// fstats (optional, 4 x u64, accumulated): nonzero reps, sum of trip counts,
// reps beyond 2048, sum of |rep|.
template <class T>
void launch_counts_f16(const T* y, uint64_t ld, uint32_t n, uint32_t tile_cols, __half* cnt,
                       uint64_t ldc, uint16_t* rmax, unsigned long long* fstats, cudaStream_t s);
// Compacted nonzero bases (k, X[r0 + q, k]) of slab rows q = rows_idx[t]
// (or t), t < ntask, into lists row q / counts[q].
template <class T>
void launch_acompact(const T* x, uint64_t ld, uint32_t n, uint32_t r0, uint32_t ntask,
                     const uint32_t* rows_idx, typename AEntry<T>::type* lists, uint64_t cap,
                     uint32_t* counts, cudaStream_t s);
// Columns per A-form CTA tile (also the rmax tile width).
template <class T>
constexpr uint32_t aform_tile_cols() { return sizeof(T) == 4 ? 1024u : 512u; }
constexpr int kAformRows = 16;      // A-form CTA: 16 consumer warps + 1 TMA warp,
constexpr int kAformCtasPerSm = 1;  // 12-stage fp16 count ring (192 KB), 1 CTA per SM  // rows (warps) per A-form CTA
constexpr uint32_t kAformMaxRep = 2048;  // fp16 counts are exact up to here
// Warp b computes Z row q = row_idx ? row_idx[b] : b (its list is lists row q,
// its output out row q), b < nrows; cmap = fp16 count tensor map (box 256 x KB).
template <class T>
cudaError_t launch_aform(const CUtensorMap* cmap, const typename AEntry<T>::type* lists,
                         uint64_t cap, const uint32_t* counts, uint32_t nrows, uint32_t ncols,
                         uint32_t nk, const uint16_t* rmax, T* out, uint64_t ld_out,
                         const uint32_t* row_idx, const DevStatus* st, cudaStream_t s);

// TMA geometry shared by the ring kernels: boxes of bform_kb() rows x
// bform_box_bytes() bytes.
int bform_kb();
int bform_box_bytes();

// k_bform tile shapes: narrow = 512 fp32 / 256 fp64 columns per CTA, 2 CTAs
// per SM; wide = 1024 / 512 columns, 32 accumulators per lane, 1 CTA per SM.
// small = 256 / 128 columns x 4 rows per CTA, for problems too small to fill
// the GPU with the larger tiles.
constexpr int kShapeNarrow = 0;
constexpr int kShapeWide = 1;
constexpr int kShapeSmall = 2;
constexpr int kShapeTmem = 3;
constexpr int kWideRows = 16;      // rows per wide CTA (16 consumer warps + 1 TMA warp)
constexpr int kWideCtasPerSm = 1;  // wide CTAs resident per SM (6-stage ring, 192 KB smem)
constexpr int kTmemRows = 14; // rows per TMEM-fed CTA (14 + 2 warps: 128-register budget)
// *splits: requested k slices in, slices launched out (1 = order-preserving).
// Slice z writes its partial product to out + z * slice_stride.
template <class T>
cudaError_t launch_bform(int shape, const CUtensorMap* tmap, const int2* lists, uint64_t cap,
                         const uint32_t* counts, uint32_t nrows, int32_t col0, int32_t ncols,
                         uint32_t nk, uint32_t* splits, uint64_t slice_stride, T* out,
                         uint64_t ld_out, const DevStatus* st, cudaStream_t s);

// out[r*ld_out + c] = sum over z (ascending) of part[z*stride + r*ld_part + c]
template <class T>
void launch_reduce_slices(const T* part, uint64_t stride, uint64_t ld_part, uint32_t splits,
                          uint32_t rows, uint32_t cols, T* out, uint64_t ld_out,
                          const DevStatus* st, cudaStream_t s);

// Multi-row dense-rep kernel: rmap = int32 reps R'[k][row] (row inner),
// box bform_mr_rows() x bform_kb().
int bform_mr_rows();
template <class T>
cudaError_t launch_bform_mr(const CUtensorMap* tmap, const CUtensorMap* rmap, uint32_t nrows,
                            int32_t col0, int32_t ncols, uint32_t nk, T* out, uint64_t ld_out,
                            const DevStatus* st, cudaStream_t s);
// Dense int32 reps: dst[r * ld_dst + c] = llround(src[r][c]) (transpose = 0)
// or llround(src[c][r]) (transpose = 1) over an rows x cols destination.
template <class T>
void launch_reps_dense(const T* src, uint64_t ld_src, uint32_t rows, uint32_t cols,
                       int transpose, int32_t* dst, uint64_t ld_dst, cudaStream_t s);

// FP-add peak microbenchmark (peak.cu)
cudaError_t run_peak(int dtype, double* adds_per_second, double* sm_mhz);

}  // namespace afmm_dev
