// afmm_gpu -- the reference CLI's `gen` and `mul` subcommands
// (/root/reference/proj/tools/afmm_cli.cpp:47-60, :137-146) with the B200
// kernels registered next to the reference ones.
//
//   afmm_gpu gen --n N --density D [--role real|int] [--mu M] [--low L] [--high H]
//                [--seed S] [--out FILE]
//   afmm_gpu mul LHS RHS --kernel afmm-a-gpu|afmm-b-gpu|afmm-a|afmm-b|ijk|ikj
//                [--mode order-preserving|fast] [--out FILE]
//
// Matrix text I/O, generation and the CPU kernels are the reference's own
// headers (matrix_io.hpp, random.hpp, kernels.hpp), included at build time;
// the *-gpu kernel ids go through afmm::gpu::run_kernel (libafmm_b200.so).
// Output and exit codes follow the reference CLI: the product in the
// reference text format, then the OpCounts line; 0 ok, 2 error
// (afmm_cli.cpp:173-179). Argument parsing is hand-written (CLI11 is not
// available here).
#include <cstdint>
#include <cstdlib>
#include <iostream>
#include <map>
#include <string>
#include <vector>

#include "afmm/kernels.hpp"
#include "afmm/matrix_io.hpp"
#include "afmm/op_counts.hpp"
#include "afmm/random.hpp"
#include "afmm_b200/kernels.hpp"

namespace {

struct Args {
  std::vector<std::string> positional;
  std::map<std::string, std::string> options;
};

Args parse(int argc, char** argv, int first) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string s = argv[i];
    if (s.rfind("--", 0) == 0) {
      if (i + 1 >= argc) throw std::invalid_argument("option " + s + " needs a value");
      a.options[s.substr(2)] = argv[++i];
    } else {
      a.positional.push_back(s);
    }
  }
  return a;
}

std::string opt(const Args& a, const std::string& key, const std::string& dflt) {
  const auto it = a.options.find(key);
  return it == a.options.end() ? dflt : it->second;
}

afmm::MultiplyResult multiply(const std::string& kernel, const afmm::DenseMatrix& lhs,
                              const afmm::DenseMatrix& rhs, afmm::gpu::Options o) {
  if (const auto g = afmm::gpu::parse_kernel(kernel)) return afmm::gpu::run_kernel(*g, lhs, rhs, o);
  if (const auto c = afmm::parse_kernel(kernel)) {
    switch (*c) {
      case afmm::KernelId::IJK: return afmm::multiply_ijk(lhs, rhs);
      case afmm::KernelId::IKJ: return afmm::multiply_ikj(lhs, rhs);
      case afmm::KernelId::AFMM_A: return afmm::afmm_case_a(lhs, rhs);
      case afmm::KernelId::AFMM_B: return afmm::afmm_case_b(lhs, rhs);
      default: break;
    }
  }
  throw std::invalid_argument("unknown kernel '" + kernel + "'");
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) throw std::invalid_argument("usage: afmm_gpu gen|mul ...");
    const std::string cmd = argv[1];
    const Args a = parse(argc, argv, 2);
    if (cmd == "gen") {
      const std::size_t n = std::stoull(opt(a, "n", "0"));
      const double density = std::stod(opt(a, "density", "-1"));
      const std::string role = opt(a, "role", "real");
      const double mu = std::stod(opt(a, "mu", "1"));
      const std::uint64_t seed = std::stoull(opt(a, "seed", "0"));
      const afmm::GeneratorSpec spec =
          role == "int" ? afmm::GeneratorSpec::integer_valued(n, density, mu)
                        : afmm::GeneratorSpec::real_valued(n, density,
                                                           std::stod(opt(a, "low", "0.5")),
                                                           std::stod(opt(a, "high", "1.5")));
      const auto m = afmm::generate(spec, afmm::Seed{seed});
      const std::string out = opt(a, "out", "");
      if (out.empty()) afmm::write_matrix(std::cout, m);
      else afmm::save_matrix(out, m);
    } else if (cmd == "mul") {
      if (a.positional.size() != 2) throw std::invalid_argument("mul needs LHS and RHS files");
      const auto lhs = afmm::load_matrix(a.positional[0]);
      const auto rhs = afmm::load_matrix(a.positional[1]);
      afmm::gpu::Options o;
      o.mode = opt(a, "mode", "order-preserving") == "fast" ? afmm::gpu::Mode::Fast
                                                             : afmm::gpu::Mode::OrderPreserving;
      const auto result = multiply(opt(a, "kernel", "afmm-a-gpu"), lhs, rhs, o);
      const std::string out = opt(a, "out", "");
      if (out.empty()) afmm::write_matrix(std::cout, result.product);
      else afmm::save_matrix(out, result.product);
      std::cout << result.counts << '\n';
    } else {
      throw std::invalid_argument("unknown subcommand '" + cmd + "'");
    }
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  }
  return 0;
}
