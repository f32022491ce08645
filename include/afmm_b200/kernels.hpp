// afmm_b200/kernels.hpp -- drop-in C++ front end of the B200 AFMM product.
//
// Header-only, namespace afmm::gpu, same signatures as the reference's hot path
// (/root/reference/proj/include/afmm/kernels.hpp):
//
//   afmm::afmm_case_a(const DenseMatrix&, const DenseMatrix&) -> MultiplyResult  (:113)
//   afmm::afmm_case_b(const DenseMatrix&, const DenseMatrix&) -> MultiplyResult  (:142)
//   afmm::generate(const GeneratorSpec&, Seed) -> DenseMatrix       (random.hpp:111)
//
// Include it next to the reference headers (it uses their DenseMatrix,
// MultiplyResult, OpCounts and shape_error) and link libafmm_b200.so. Errors
// are rethrown with the reference's exception types and message text:
// shape_error (kernels.hpp:15-21), std::domain_error (kernels.hpp:25-43,
// matrix.hpp:31-35), std::invalid_argument (matrix.hpp:54-57). The product is
// computed on the B200; there is no CPU fallback (a missing device throws
// std::runtime_error).
#pragma once

#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "afmm/errors.hpp"
#include "afmm/matrix.hpp"
#include "afmm/op_counts.hpp"
#include "afmm/random.hpp"
#include "afmm_b200.h"

namespace afmm::gpu {

enum class Mode {
  OrderPreserving = AFMM_MODE_ORDER_PRESERVING,
  Fast = AFMM_MODE_FAST,
  FastLadder = AFMM_MODE_FAST_LADDER
};

enum class Partition { Work = AFMM_PARTITION_WORK, Rows = AFMM_PARTITION_ROWS };

struct Options {
  Mode mode = Mode::OrderPreserving;
  int device = -1;           // -1: the calling thread's current CUDA device
  std::vector<int> devices;  // > 1 entries: Z rows sharded over these devices (may repeat)
  Partition partition = Partition::Work;  // row cuts: predicted time, or equal rows
  int split_k = 0;           // fast mode: upper bound on k slices (0 = automatic)
  afmm_timing* timing = nullptr;  // optional out: device-measured phases of the call
};

/// fp32 storage for BASELINE configs 3-5 (the reference has no fp32 type,
/// proj/README.md:91). Row-major n x n like DenseMatrix (matrix.hpp:41-46).
struct DenseMatrixF32 {
  std::size_t n = 0;
  std::vector<float> values;
  DenseMatrixF32() = default;
  explicit DenseMatrixF32(std::size_t dim) : n(dim), values(dim * dim, 0.0f) {
    if (dim == 0) throw std::invalid_argument("DenseMatrix: dimension must be >= 1");
  }
  std::size_t dim() const noexcept { return n; }
  float operator()(std::size_t i, std::size_t j) const noexcept { return values[i * n + j]; }
  float& operator()(std::size_t i, std::size_t j) noexcept { return values[i * n + j]; }
};

struct MultiplyResultF32 {
  DenseMatrixF32 product;
  OpCounts counts;
};

namespace detail {

inline void throw_for(afmm_status status, const afmm_error& err) {
  const std::string msg = err.message;
  switch (status) {
    case AFMM_OK: return;
    case AFMM_ERR_SHAPE: throw shape_error(msg);
    case AFMM_ERR_DOMAIN: throw std::domain_error(msg);
    // n beyond the device index range, or a NaN rep (the reference would not finish)
    case AFMM_ERR_UNSUPPORTED: throw std::length_error(msg);
    case AFMM_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case AFMM_ERR_OUT_OF_MEMORY: throw std::bad_alloc();
    default: throw std::runtime_error(msg.empty() ? "afmm: CUDA failure" : msg);
  }
}

static_assert(sizeof(int) == sizeof(int32_t), "device ordinals are passed as int32_t");

// (the returned struct points into o.devices: keep `o` alive for the call)
inline afmm_options to_c(const Options& o) {
  afmm_options c{};
  c.mode = static_cast<int32_t>(o.mode);
  c.device = o.device;
  c.split_k = o.split_k;
  c.partition = static_cast<int32_t>(o.partition);
  c.timing = o.timing;
  // the arguments are constructed matrices: the kernel's checks only
  // (non-finite bases are computed, an infinite rep is out of range)
  c.flags = AFMM_FLAG_KERNEL_SEMANTICS;
  if (!o.devices.empty()) {
    c.num_devices = static_cast<int32_t>(o.devices.size());
    c.devices = reinterpret_cast<const int32_t*>(o.devices.data());
  }
  return c;
}

inline OpCounts to_counts(const afmm_op_counts& c) {
  OpCounts out;
  out.additions = c.additions;
  out.multiplications = c.multiplications;
  out.zero_skips = c.zero_skips;
  return out;
}

using FnF64 = afmm_status (*)(const double*, uint64_t, const double*, uint64_t, double*,
                              const afmm_options*, afmm_op_counts*, afmm_error*);
using FnF32 = afmm_status (*)(const float*, uint64_t, const float*, uint64_t, float*,
                              const afmm_options*, afmm_op_counts*, afmm_error*);

inline MultiplyResult run_f64(FnF64 fn, const DenseMatrix& lhs, const DenseMatrix& rhs,
                              const Options& opt) {
  // The result buffer is allocated only once the dimensions are known to be
  // valid, so a mismatch reports shape_error exactly like kernels.hpp:114/143.
  // The C ABI checks dimensions before touching `out`, so an invalid call
  // passes nullptr and reports the reference's own error.
  const bool valid = lhs.dim() == rhs.dim() && lhs.dim() > 0;
  MultiplyResult result{valid ? DenseMatrix(lhs.dim()) : DenseMatrix(), {}};
  afmm_op_counts counts{};
  afmm_error err{};
  const afmm_options c = to_c(opt);
  throw_for(fn(lhs.data().data(), lhs.dim(), rhs.data().data(), rhs.dim(),
               valid ? result.product.data().data() : nullptr, &c, &counts, &err),
            err);
  result.counts = to_counts(counts);
  return result;
}

inline MultiplyResultF32 run_f32(FnF32 fn, const DenseMatrixF32& lhs, const DenseMatrixF32& rhs,
                                 const Options& opt) {
  const bool valid = lhs.dim() == rhs.dim() && lhs.dim() > 0;
  MultiplyResultF32 r;
  if (valid) r.product = DenseMatrixF32(lhs.dim());
  afmm_op_counts counts{};
  afmm_error err{};
  const afmm_options c = to_c(opt);
  throw_for(fn(lhs.values.data(), lhs.dim(), rhs.values.data(), rhs.dim(),
               valid ? r.product.values.data() : nullptr, &c, &counts, &err),
            err);
  r.counts = to_counts(counts);
  return r;
}

}  // namespace detail

/// AFMM Case A on the B200 (kernels.hpp:113-136): real lhs bases, integer rhs reps.
inline MultiplyResult afmm_case_a(const DenseMatrix& lhs, const DenseMatrix& rhs,
                                  Options opt = {}) {
  return detail::run_f64(&::afmm_case_a_f64, lhs, rhs, opt);
}

/// AFMM Case B on the B200 (kernels.hpp:142-165): integer lhs reps, real rhs bases.
inline MultiplyResult afmm_case_b(const DenseMatrix& lhs, const DenseMatrix& rhs,
                                  Options opt = {}) {
  return detail::run_f64(&::afmm_case_b_f64, lhs, rhs, opt);
}

inline MultiplyResultF32 afmm_case_a(const DenseMatrixF32& lhs, const DenseMatrixF32& rhs,
                                     Options opt = {}) {
  return detail::run_f32(&::afmm_case_a_f32, lhs, rhs, opt);
}

inline MultiplyResultF32 afmm_case_b(const DenseMatrixF32& lhs, const DenseMatrixF32& rhs,
                                     Options opt = {}) {
  return detail::run_f32(&::afmm_case_b_f32, lhs, rhs, opt);
}

// ---- kernel registry extension (op_counts.hpp:35-59, bench.hpp:103-113) ----

enum class KernelId { AFMM_A_GPU, AFMM_B_GPU };

inline std::string_view kernel_name(KernelId id) {
  return id == KernelId::AFMM_A_GPU ? "afmm-a-gpu" : "afmm-b-gpu";
}

inline std::optional<KernelId> parse_kernel(std::string_view name) {
  if (name == "afmm-a-gpu") return KernelId::AFMM_A_GPU;
  if (name == "afmm-b-gpu") return KernelId::AFMM_B_GPU;
  return std::nullopt;
}

/// afmm::generate(spec, seed) (random.hpp:111-129) on the GPU: the same
/// matrix, bit for bit; an invalid spec throws std::invalid_argument with
/// validate()'s text (random.hpp:60-79). opt.device selects the GPU.
inline DenseMatrix generate(const GeneratorSpec& spec, Seed seed, Options opt = {}) {
  afmm_generator_spec c{};
  c.n = spec.n;
  c.density = spec.density;
  c.mu_prime = spec.mu_prime;
  c.role = spec.role == ValueRole::IntegerValued ? AFMM_ROLE_INTEGER : AFMM_ROLE_REAL;
  c.value_low = spec.value_low;
  c.value_high = spec.value_high;
  // the spec is validated before `out` is touched, so an invalid one reports
  // the reference's error rather than DenseMatrix's
  DenseMatrix m = spec.n > 0 ? DenseMatrix(spec.n) : DenseMatrix();
  afmm_error err{};
  const afmm_options o = detail::to_c(opt);
  detail::throw_for(afmm_generate_f64(&c, seed.value, spec.n > 0 ? m.data().data() : nullptr, &o,
                                      &err),
                    err);
  return m;
}

/// The GPU arm of afmm::run_kernel (bench.hpp:103-113).
inline MultiplyResult run_kernel(KernelId id, const DenseMatrix& lhs, const DenseMatrix& rhs,
                                 Options opt = {}) {
  return id == KernelId::AFMM_A_GPU ? afmm_case_a(lhs, rhs, opt) : afmm_case_b(lhs, rhs, opt);
}

}  // namespace afmm::gpu
