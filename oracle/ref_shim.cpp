// ref_shim.cpp -- C-ABI shim over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY. oracle/Makefile compiles this file against
// /root/reference/proj/include (the reference's sources where they lie; no
// copy) with the reference's Release flags (-O3 -ffp-contract=off,
// proj/CMakeLists.txt:8-16) into oracle/_ref/libafmm_ref.so. It exists so the
// tests and the golden-vector script can call the real reference kernels
// (proj/include/afmm/kernels.hpp:113,142), the reference generator
// (random.hpp:111) and the reference tests' integer generator
// (test_kernels.cpp:16-24, restated here on top of detail::uniform_below).

#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "afmm/bench.hpp"
#include "afmm/errors.hpp"
#include "afmm/kernels.hpp"
#include "afmm/matrix.hpp"
#include "afmm/random.hpp"
#include "afmm/report.hpp"

namespace {

struct RefCounts {
  std::uint64_t additions, multiplications, zero_skips;
};

// Status: 0 ok, 1 shape_error, 2 domain_error, 3 invalid_argument, 4 other.
int classify_and_copy(const std::exception& e, int code, char* msg, std::size_t cap) {
  if (msg && cap) {
    std::strncpy(msg, e.what(), cap - 1);
    msg[cap - 1] = '\0';
  }
  return code;
}

template <class Fn>
int guarded(Fn&& fn, char* msg, std::size_t cap) {
  try {
    fn();
    if (msg && cap) msg[0] = '\0';
    return 0;
  } catch (const afmm::shape_error& e) {
    return classify_and_copy(e, 1, msg, cap);
  } catch (const std::domain_error& e) {
    return classify_and_copy(e, 2, msg, cap);
  } catch (const std::invalid_argument& e) {
    return classify_and_copy(e, 3, msg, cap);
  } catch (const std::exception& e) {
    return classify_and_copy(e, 4, msg, cap);
  }
}

afmm::DenseMatrix wrap(const double* p, std::uint64_t n) {
  return afmm::DenseMatrix(n, std::vector<double>(p, p + n * n));
}

template <class Kernel>
int run(Kernel kernel, const double* lhs, std::uint64_t n_lhs, const double* rhs,
        std::uint64_t n_rhs, double* out, RefCounts* counts, char* msg, std::size_t cap) {
  return guarded(
      [&] {
        const auto l = wrap(lhs, n_lhs);
        const auto r = wrap(rhs, n_rhs);
        const afmm::MultiplyResult res = kernel(l, r);
        const auto d = res.product.data();
        std::memcpy(out, d.data(), d.size() * sizeof(double));
        if (counts) {
          counts->additions = res.counts.additions;
          counts->multiplications = res.counts.multiplications;
          counts->zero_skips = res.counts.zero_skips;
        }
      },
      msg, cap);
}

}  // namespace

extern "C" {

int ref_afmm_case_a(const double* lhs, std::uint64_t n_lhs, const double* rhs,
                    std::uint64_t n_rhs, double* out, RefCounts* counts, char* msg,
                    std::size_t cap) {
  return run([](const auto& l, const auto& r) { return afmm::afmm_case_a(l, r); }, lhs, n_lhs,
             rhs, n_rhs, out, counts, msg, cap);
}

int ref_afmm_case_b(const double* lhs, std::uint64_t n_lhs, const double* rhs,
                    std::uint64_t n_rhs, double* out, RefCounts* counts, char* msg,
                    std::size_t cap) {
  return run([](const auto& l, const auto& r) { return afmm::afmm_case_b(l, r); }, lhs, n_lhs,
             rhs, n_rhs, out, counts, msg, cap);
}

int ref_multiply_ijk(const double* lhs, const double* rhs, std::uint64_t n, double* out,
                     RefCounts* counts, char* msg, std::size_t cap) {
  return run([](const auto& l, const auto& r) { return afmm::multiply_ijk(l, r); }, lhs, n, rhs,
             n, out, counts, msg, cap);
}

// DenseMatrix(n) with n == 0 -> std::invalid_argument (matrix.hpp:54-57).
int ref_make_matrix(std::uint64_t n, char* msg, std::size_t cap) {
  return guarded([&] { afmm::DenseMatrix m(n); (void)m; }, msg, cap);
}

// DenseMatrix(n, values) finite-only constructor (matrix.hpp:25-36).
int ref_make_matrix_from(const double* p, std::uint64_t n, char* msg, std::size_t cap) {
  return guarded([&] { (void)wrap(p, n); }, msg, cap);
}

std::uint64_t ref_splitmix64(std::uint64_t x) { return afmm::detail::splitmix64(x); }

// test_kernels.cpp:16-24 / acceptance.hpp:72-82, on the reference's own
// detail::uniform_below.
void ref_random_integer_matrix(std::uint64_t n, int low, int high, std::uint64_t seed,
                               double* out) {
  std::mt19937_64 rng(seed);
  const auto range = static_cast<std::uint64_t>(high - low + 1);
  for (std::uint64_t idx = 0; idx < n * n; ++idx) {
    out[idx] = static_cast<double>(
        low + static_cast<long long>(afmm::detail::uniform_below(rng, range)));
  }
}

int ref_generate(std::uint64_t n, double density, double mu_prime, int role, double low,
                 double high, std::uint64_t seed, double* out, char* msg, std::size_t cap) {
  return guarded(
      [&] {
        afmm::GeneratorSpec spec =
            role == 1 ? afmm::GeneratorSpec::integer_valued(n, density, mu_prime)
                      : afmm::GeneratorSpec::real_valued(n, density, low, high);
        const auto m = afmm::generate(spec, afmm::Seed{seed});
        const auto d = m.data();
        std::memcpy(out, d.data(), d.size() * sizeof(double));
      },
      msg, cap);
}

// bench.hpp:82-85 and :90-101 (AFMM_A when case_b == 0, AFMM_B otherwise).
std::uint64_t ref_cell_seed(std::uint64_t base, std::uint64_t n, std::uint64_t rep) {
  return afmm::cell_seed(afmm::Seed{base}, n, rep);
}

void ref_make_factor_pair(int case_b, std::uint64_t n, double d1, double d2, double mu_prime,
                          std::uint64_t seed, double* lhs, double* rhs) {
  const auto pair = afmm::make_factor_pair(case_b ? afmm::KernelId::AFMM_B : afmm::KernelId::AFMM_A,
                                           n, d1, d2, mu_prime, seed);
  std::memcpy(lhs, pair.first.data().data(), n * n * sizeof(double));
  std::memcpy(rhs, pair.second.data().data(), n * n * sizeof(double));
}

// The reference's own benchmark flow: run_plan (bench.hpp:120-154) for an
// afmm kernel id, rendered by emit_csv (report.hpp:27-39) into `out`. Returns
// 0, or -1 when `out` is too small (the needed size in *needed).
int ref_run_plan_csv(int case_b, const std::uint64_t* sizes, std::size_t nsizes, double d1,
                     double d2, double mu_prime, std::uint64_t reps, std::uint64_t warmups,
                     std::uint64_t seed, char* out, std::size_t cap, std::size_t* needed,
                     char* msg, std::size_t msg_cap) {
  int fit = 0;
  const int rc = guarded(
      [&] {
        afmm::ExperimentPlan plan;
        plan.kernel = case_b ? afmm::KernelId::AFMM_B : afmm::KernelId::AFMM_A;
        plan.sizes.assign(sizes, sizes + nsizes);
        plan.d1 = d1;
        plan.d2 = d2;
        plan.mu_prime = mu_prime;
        plan.replications = reps;
        plan.warmups = warmups;
        plan.base_seed = afmm::Seed{seed};
        std::ostringstream csv;
        afmm::emit_csv(afmm::run_plan(plan, nullptr), csv);
        const std::string s = csv.str();
        *needed = s.size() + 1;
        if (s.size() + 1 > cap) {
          fit = -1;
          return;
        }
        std::memcpy(out, s.c_str(), s.size() + 1);
      },
      msg, msg_cap);
  return rc != 0 ? rc : fit;
}

// The reference's report flow: parse_csv (report.hpp:74-124) + emit_table
// (report.hpp:265-267) of the record CSV text `csv`, into `out`. Returns 0,
// -1 when `out` is too small (the needed size in *needed), or the status of
// the reference's exception (its message in msg).
int ref_emit_table(const char* csv, char* out, std::size_t cap, std::size_t* needed, char* msg,
                   std::size_t msg_cap) {
  int fit = 0;
  const int rc = guarded(
      [&] {
        std::istringstream in(csv);
        const std::string s = afmm::emit_table(afmm::parse_csv(in));
        *needed = s.size() + 1;
        if (s.size() + 1 > cap) {
          fit = -1;
          return;
        }
        std::memcpy(out, s.c_str(), s.size() + 1);
      },
      msg, msg_cap);
  return rc != 0 ? rc : fit;
}

// ---- row-block entry for the CPU baseline (bench.py) ----
// A DenseMatrix held across calls (the shared rhs of a timing batch).
void* ref_hold_matrix(const double* p, std::uint64_t n, char* msg, std::size_t cap) {
  afmm::DenseMatrix* m = nullptr;
  const int rc = guarded([&] { m = new afmm::DenseMatrix(wrap(p, n)); }, msg, cap);
  return rc == 0 ? m : nullptr;
}

void ref_release_matrix(void* h) { delete static_cast<afmm::DenseMatrix*>(h); }

// The unmodified afmm_case_{a,b} on (lhs with only rows [r0, r1) kept, the
// other rows zero) x rhs. Rows are independent (kernels.hpp:119,148), so rows
// [r0, r1) of the product are the reference's result for those rows; the zero
// rows cost only the per-call overhead (validation, Z allocation, zero-row
// scans), which the caller measures with r0 == r1 and subtracts. Several
// threads may call this concurrently with the same rhs handle.
int ref_case_rows(int case_b, const double* lhs, std::uint64_t n, std::uint64_t r0,
                  std::uint64_t r1, const void* rhs_h, double* out_rows, RefCounts* counts,
                  char* msg, std::size_t cap) {
  return guarded(
      [&] {
        afmm::DenseMatrix l(n);
        const auto ld = l.data();
        std::memcpy(ld.data() + r0 * n, lhs + r0 * n, (r1 - r0) * n * sizeof(double));
        const auto& r = *static_cast<const afmm::DenseMatrix*>(rhs_h);
        const afmm::MultiplyResult res = case_b ? afmm::afmm_case_b(l, r) : afmm::afmm_case_a(l, r);
        const auto d = res.product.data();
        if (out_rows) std::memcpy(out_rows, d.data() + r0 * n, (r1 - r0) * n * sizeof(double));
        if (counts) {
          counts->additions = res.counts.additions;
          counts->multiplications = res.counts.multiplications;
          counts->zero_skips = res.counts.zero_skips;
        }
      },
      msg, cap);
}

// test_kernels.cpp:208-217: the 16-bit-magnitude operands (|entries| <= 2^15),
// drawn from std::mt19937_64(0xB16) exactly as that test does.
void ref_b16_pair(double* lhs, double* rhs) {
  std::mt19937_64 rng(0xB16);
  for (int idx = 0; idx < 64; ++idx) {
    lhs[idx] = rng() % 3 == 0 ? static_cast<double>(static_cast<int>(rng() % 65536) - 32768) : 0.0;
  }
  for (int idx = 0; idx < 64; ++idx) {
    rhs[idx] = rng() % 3 == 0 ? static_cast<double>(static_cast<int>(rng() % 65536) - 32768) : 0.0;
  }
}

}  // extern "C"
