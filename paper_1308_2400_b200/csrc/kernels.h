// kernels.h -- internal launch interface between the host runtime and the
// sm_100a kernels (not part of the public C ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace afmm_dev {

void note_launch();  // counts library kernel launches (runtime.cu)

template <class T>
void launch_scan_operand(const T* m, uint64_t ld, uint32_t n, int is_rep,
                         unsigned long long* nonfinite, unsigned long long* rep_bad,
                         unsigned long long* too_large, cudaStream_t s);
template <class T>
void launch_row_nnz(const T* m, uint64_t ld, uint32_t n, uint32_t* nnz, cudaStream_t s);
template <class T>
void launch_row_repsum(const T* m, uint64_t ld, uint32_t n, unsigned long long* rsum,
                       cudaStream_t s);
template <class T>
void launch_compact_reps(const T* m, uint64_t ld, uint32_t rows, uint32_t n, int2* lists,
                         uint64_t cap, uint32_t* counts, cudaStream_t s);
template <class T>
void launch_row_work(const T* x, uint64_t ld, uint32_t n, int which_case, const uint32_t* nnz_b,
                     const unsigned long long* rsum, unsigned long long* work,
                     unsigned long long* zs, cudaStream_t s);
void launch_sum_counts(const unsigned long long* work, const unsigned long long* zs, uint32_t r0,
                       uint32_t r1, DevStatus* st, cudaStream_t s);
template <class T>
void launch_transpose(const T* in, uint64_t ld_in, uint32_t rows, uint32_t cols, T* out,
                      uint64_t ld_out, cudaStream_t s);

// TMA geometry shared by the ring kernels: boxes of bform_kb() rows x
// bform_box_bytes() bytes.
int bform_kb();
int bform_box_bytes();

// k_bform tile shapes: narrow = 512 fp32 / 256 fp64 columns per CTA, 2 CTAs
// per SM; wide = 1024 / 512 columns, 32 accumulators per lane, 1 CTA per SM.
constexpr int kShapeNarrow = 0;
constexpr int kShapeWide = 1;
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
                          uint32_t rows, uint32_t cols, T* out, uint64_t ld_out, cudaStream_t s);

template <class T>
cudaError_t launch_bform_dyn(const CUtensorMap* tmap, const int2* lists, uint64_t cap,
                             const uint32_t* counts, uint32_t nrows, int32_t col0, int32_t ncols,
                             uint32_t nk, T* out, uint64_t ld_out, const DevStatus* st,
                             cudaStream_t s);
template <class T>
cudaError_t launch_bform_l1(const T* base, uint64_t ldb, const int2* lists, uint64_t cap,
                            const uint32_t* counts, uint32_t nrows, int32_t col0, int32_t ncols,
                            T* out, uint64_t ld_out, const DevStatus* st, cudaStream_t s);

// FP-add peak microbenchmark (peak.cu)
cudaError_t run_peak(int dtype, double* adds_per_second, double* sm_mhz);

}  // namespace afmm_dev
