// The reference's own kernel tests (proj/tests/test_kernels.cpp:109-223),
// restated against the drop-in front end afmm::gpu::afmm_case_{a,b} and the
// reference's DenseMatrix / OpCounts / shape_error types. Each GPU result is
// also compared with the reference kernel itself on the same inputs.
//
// Built by `make cpptest` against /root/reference/proj/include (build
// container only); run on the B200 by tests/test_cpp_dropin.py.
#include <cmath>
#include <cstdio>
#include <limits>
#include <cstdlib>
#include <random>
#include <string>

#include "afmm/kernels.hpp"
#include "afmm/random.hpp"
#include "afmm_b200/kernels.hpp"

using namespace afmm;

static int g_failures = 0;
static int g_checks = 0;

#define CHECK(cond)                                                     \
  do {                                                                  \
    ++g_checks;                                                         \
    if (!(cond)) {                                                      \
      ++g_failures;                                                     \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                   \
  } while (0)

template <class Ex, class Fn>
static std::string expect_throw(Fn&& fn) {
  try {
    fn();
  } catch (const Ex& e) {
    return e.what();
  } catch (...) {
    return "<wrong exception type>";
  }
  return "<no exception>";
}

static DenseMatrix random_integer_matrix(std::size_t n, int low, int high, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  DenseMatrix m(n);
  const auto range = static_cast<std::uint64_t>(high - low + 1);
  for (double& v : m.data())
    v = static_cast<double>(low + static_cast<long long>(detail::uniform_below(rng, range)));
  return m;
}

static void same_as_reference_a(const DenseMatrix& l, const DenseMatrix& r) {
  const auto g = gpu::afmm_case_a(l, r);
  const auto c = afmm_case_a(l, r);
  CHECK(g.product == c.product);
  CHECK(g.counts == c.counts);
}

static void same_as_reference_b(const DenseMatrix& l, const DenseMatrix& r) {
  const auto g = gpu::afmm_case_b(l, r);
  const auto c = afmm_case_b(l, r);
  CHECK(g.product == c.product);
  CHECK(g.counts == c.counts);
}

int main() {
  // case A: hand trace (test_kernels.cpp:109-115)
  {
    const auto result = gpu::afmm_case_a(from_rows({{2, 0}, {0.5, 1}}), from_rows({{3, 1}, {0, 2}}));
    CHECK(result.product == from_rows({{6, 2}, {1.5, 2.5}}));
    CHECK(result.counts.additions == 10);
    CHECK(result.counts.multiplications == 0);
    CHECK(result.counts.zero_skips == 1);
  }
  // case A: degenerate inputs (:117-127)
  {
    const auto all_zero = gpu::afmm_case_a(zeros(3), from_rows({{1, 2, 3}, {4, 5, 6}, {7, 8, 9}}));
    CHECK(all_zero.product == zeros(3));
    CHECK(all_zero.counts.additions == 0);
    CHECK(all_zero.counts.zero_skips == 9);
    const auto y = from_rows({{1, -2, 0}, {3, 0, 4}, {0, 5, -6}});
    const auto via_identity = gpu::afmm_case_a(identity(3), y);
    CHECK(via_identity.product == y);
    CHECK(via_identity.counts.additions == 21);
  }
  // case A: errors (:129-136)
  {
    CHECK(expect_throw<shape_error>([] { gpu::afmm_case_a(zeros(2), zeros(3)); }) ==
          "afmm_case_a: dimension mismatch 2 vs 3");
    const std::string msg = expect_throw<std::domain_error>(
        [] { gpu::afmm_case_a(zeros(2), from_rows({{1, 0.5}, {0, 2}})); });
    CHECK(msg.find("[0][1]") != std::string::npos);
    const std::string ref_msg = expect_throw<std::domain_error>(
        [] { afmm_case_a(zeros(2), from_rows({{1, 0.5}, {0, 2}})); });
    CHECK(msg == ref_msg);
    const auto nearly = from_rows({{1 + 1e-12, 0}, {0, 2 - 1e-12}});
    bool ok = true;
    try {
      gpu::afmm_case_a(identity(2), nearly);
    } catch (...) {
      ok = false;
    }
    CHECK(ok);
  }
  // case A: integer exactness + counts (:138-147)
  for (std::uint64_t seed = 0; seed < 10; ++seed) {
    const auto lhs = random_integer_matrix(16, -9, 9, seed * 2 + 1);
    const auto rhs = random_integer_matrix(16, -9, 9, seed * 2 + 2);
    const auto result = gpu::afmm_case_a(lhs, rhs);
    CHECK(result.product == multiply_ijk(lhs, rhs).product);
    CHECK(result.counts.multiplications == 0);
    same_as_reference_a(lhs, rhs);
  }
  // case A: real x integer (:149-155), bit-exact vs the reference kernel
  for (std::uint64_t seed = 0; seed < 10; ++seed) {
    const auto lhs = generate(GeneratorSpec::real_valued(32, 0.9), Seed{seed});
    const auto rhs = generate(GeneratorSpec::integer_valued(32, 0.8, 21), Seed{seed + 31});
    CHECK(approx_equal(gpu::afmm_case_a(lhs, rhs).product, multiply_ijk(lhs, rhs).product, 1e-9));
    same_as_reference_a(lhs, rhs);
  }
  // case B: hand trace (:175-186)
  {
    const auto result = gpu::afmm_case_b(from_rows({{3, 0}, {1, 2}}), from_rows({{0.5, 0}, {1, 1}}));
    CHECK(result.product == from_rows({{1.5, 0}, {2.5, 2}}));
    CHECK(result.counts.additions == 8);
    CHECK(result.counts.multiplications == 0);
    CHECK(result.counts.zero_skips == 2);
  }
  // case B: degenerate and errors (:188-196)
  {
    const auto all_zero = gpu::afmm_case_b(zeros(3), from_rows({{1, 2, 3}, {4, 5, 6}, {7, 8, 9}}));
    CHECK(all_zero.product == zeros(3));
    CHECK(all_zero.counts.additions == 0);
    CHECK(expect_throw<shape_error>([] { gpu::afmm_case_b(zeros(2), zeros(3)); }) ==
          "afmm_case_b: dimension mismatch 2 vs 3");
    const std::string msg = expect_throw<std::domain_error>(
        [] { gpu::afmm_case_b(from_rows({{1, 0}, {0.25, 2}}), zeros(2)); });
    CHECK(msg.find("[1][0]") != std::string::npos);
  }
  // case B: integer exactness (:198-206)
  for (std::uint64_t seed = 0; seed < 10; ++seed) {
    const auto lhs = random_integer_matrix(16, -9, 9, seed * 3 + 1);
    const auto rhs = random_integer_matrix(16, -9, 9, seed * 3 + 2);
    CHECK(gpu::afmm_case_b(lhs, rhs).product == multiply_ijk(lhs, rhs).product);
    same_as_reference_b(lhs, rhs);
  }
  // 16-bit magnitudes (:208-223)
  {
    std::mt19937_64 rng(0xB16);
    DenseMatrix lhs(8), rhs(8);
    for (double& v : lhs.data())
      v = rng() % 3 == 0 ? static_cast<double>(static_cast<int>(rng() % 65536) - 32768) : 0.0;
    for (double& v : rhs.data())
      v = rng() % 3 == 0 ? static_cast<double>(static_cast<int>(rng() % 65536) - 32768) : 0.0;
    const auto reference = multiply_ijk(lhs, rhs).product;
    CHECK(gpu::afmm_case_a(lhs, rhs).product == reference);
    CHECK(gpu::afmm_case_b(lhs, rhs).product == reference);
  }
  // registry extension round trip (op_counts.hpp:35-59 style)
  for (const auto id : {gpu::KernelId::AFMM_A_GPU, gpu::KernelId::AFMM_B_GPU})
    CHECK(gpu::parse_kernel(gpu::kernel_name(id)) == id);
  {
    const auto x = from_rows({{2, 0}, {0.5, 1}});
    const auto y = from_rows({{3, 1}, {0, 2}});
    CHECK(gpu::run_kernel(gpu::KernelId::AFMM_A_GPU, x, y).product == afmm_case_a(x, y).product);
  }
  // fp32 overloads
  {
    gpu::DenseMatrixF32 x(2), y(2);
    x(0, 0) = 2; x(1, 0) = 0.5f; x(1, 1) = 1;
    y(0, 0) = 3; y(0, 1) = 1; y(1, 1) = 2;
    const auto r = gpu::afmm_case_a(x, y);
    CHECK(r.product(0, 0) == 6.f && r.product(0, 1) == 2.f && r.product(1, 0) == 1.5f &&
          r.product(1, 1) == 2.5f);
    CHECK(r.counts.additions == 10 && r.counts.zero_skips == 1);
  }
  // matrices built element by element may hold non-finite values: the drop-in
  // applies only the kernel's checks, like the reference (kernels.hpp:25-43)
  {
    DenseMatrix x(3), y(3);
    x(0, 1) = std::numeric_limits<double>::infinity();
    x(1, 2) = 2.5;
    x(2, 0) = -1.0;
    y(1, 0) = 3; y(2, 2) = -2; y(0, 1) = 1;
    same_as_reference_a(x, y);  // inf base: computed, Z gets inf
    CHECK(std::isinf(gpu::afmm_case_a(x, y).product(0, 0)));
    DenseMatrix bad(3);
    bad(2, 1) = std::numeric_limits<double>::infinity();
    const std::string ref_msg = expect_throw<std::domain_error>([&] { afmm_case_a(x, bad); });
    const std::string gpu_msg = expect_throw<std::domain_error>([&] { gpu::afmm_case_a(x, bad); });
    CHECK(ref_msg == gpu_msg);
    CHECK(gpu_msg.find("exceeds the exact integer range") != std::string::npos);
  }
  // a rep beyond int32: split into consecutive list entries, same bits
  {
    const auto x = from_rows({{0.5, -0.25}, {1e-3, 3.0}});
    const auto y = from_rows({{1, 2147483653.0}, {-2, 0}});
    same_as_reference_a(x, y);
  }
  // sharded over two contexts of one device (options.devices), same bits
  {
    gpu::Options o;
    o.devices = {0, 0};
    const auto x = random_integer_matrix(70, -9, 9, 5);
    const auto y = random_integer_matrix(70, -9, 9, 6);
    CHECK(gpu::afmm_case_a(x, y, o).product == afmm_case_a(x, y).product);
    CHECK(gpu::afmm_case_b(x, y, o).counts == afmm_case_b(x, y).counts);
  }
  // the reassociated modes on integer inputs: every partial sum is exact in
  // any association, so Fast and FastLadder (each term a doubling ladder)
  // must give the reference's product and its counts
  for (const auto mode : {gpu::Mode::Fast, gpu::Mode::FastLadder}) {
    gpu::Options o;
    o.mode = mode;
    const auto x = random_integer_matrix(90, -40, 40, 11);
    const auto y = random_integer_matrix(90, -40, 40, 12);
    CHECK(gpu::afmm_case_a(x, y, o).product == afmm_case_a(x, y).product);
    CHECK(gpu::afmm_case_b(x, y, o).product == afmm_case_b(x, y).product);
    CHECK(gpu::afmm_case_b(x, y, o).counts == afmm_case_b(x, y).counts);
  }
  // seeded generation on the GPU: the reference's generator, bit for bit
  // (random.hpp:111-129), both roles, edge densities, and validate()'s errors
  {
    const GeneratorSpec specs[] = {
        GeneratorSpec::integer_valued(1, 1.0, 1.0),   GeneratorSpec::integer_valued(33, 0.5, 21.0),
        GeneratorSpec::integer_valued(64, 1.0, 4.0),  GeneratorSpec::integer_valued(100, 0.0, 3.0),
        GeneratorSpec::real_valued(50, 0.9),          GeneratorSpec::real_valued(257, 0.3, -2.0, 5.0),
        GeneratorSpec::real_valued(16, 1.0, 1.0, 1.0)};
    for (const auto& sp : specs)
      for (std::uint64_t seed : {0ull, 7ull, 0xFFFFFFFFFFFFFFFFull})
        CHECK(gpu::generate(sp, Seed{seed}) == generate(sp, Seed{seed}));
    GeneratorSpec bad = GeneratorSpec::integer_valued(4, 0.5, 2.5);
    CHECK(expect_throw<std::invalid_argument>([&] { gpu::generate(bad, Seed{1}); }) ==
          expect_throw<std::invalid_argument>([&] { generate(bad, Seed{1}); }));
    bad = GeneratorSpec::real_valued(0, 0.5);
    CHECK(expect_throw<std::invalid_argument>([&] { gpu::generate(bad, Seed{1}); }) ==
          expect_throw<std::invalid_argument>([&] { generate(bad, Seed{1}); }));
    bad = GeneratorSpec::real_valued(3, 1.5);
    CHECK(expect_throw<std::invalid_argument>([&] { gpu::generate(bad, Seed{1}); }) ==
          expect_throw<std::invalid_argument>([&] { generate(bad, Seed{1}); }));
  }
  std::printf("%d checks, %d failures\n", g_checks, g_failures);
  return g_failures == 0 ? 0 : 1;
}
