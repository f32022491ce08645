// acceptance_gpu_shim.hpp -- TEST-ONLY: points the reference's own acceptance
// gate at the B200 kernels.
//
// The reference's verification suites (/root/reference/proj/include/afmm/
// acceptance.hpp) funnel every repeated-addition run through
// Context::case_a / case_b (acceptance.hpp:52-69), which call the unqualified
// afmm_case_a / afmm_case_b, and the timing criterion runs run_plan ->
// run_kernel (bench.hpp:103-113), which calls them too. Included BEFORE
// acceptance.hpp (and after kernels.hpp, whose CPU definitions stay intact),
// this header renames those calls to wrappers that run the drop-in
// afmm::gpu::afmm_case_{a,b} (include/afmm_b200/kernels.hpp), so the
// reference's unmodified criteria c01-c10 and c12 check the GPU path.
#pragma once

#include "afmm/kernels.hpp"
#include "afmm_b200/kernels.hpp"

namespace afmm {

inline std::uint64_t g_gpu_calls = 0;

inline MultiplyResult afmm_case_a_on_b200(const DenseMatrix& lhs, const DenseMatrix& rhs) {
  ++g_gpu_calls;
  return gpu::afmm_case_a(lhs, rhs);
}

inline MultiplyResult afmm_case_b_on_b200(const DenseMatrix& lhs, const DenseMatrix& rhs) {
  ++g_gpu_calls;
  return gpu::afmm_case_b(lhs, rhs);
}

}  // namespace afmm

#define afmm_case_a afmm_case_a_on_b200
#define afmm_case_b afmm_case_b_on_b200
