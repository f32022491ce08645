// afmm_gpu -- the reference CLI's `gen`, `mul` and `bench` subcommands
// (/root/reference/proj/tools/afmm_cli.cpp:47-60, :81-101, :137-157) with the
// B200 kernels registered next to the reference ones (SURVEY.md 8(f) ranks 1
// and 3).
//
//   afmm_gpu gen --n N --density D [--role real|int] [--mu M] [--low L] [--high H]
//                [--seed S] [--out FILE]
//   afmm_gpu mul LHS RHS --kernel afmm-a-gpu|afmm-b-gpu|afmm-a|afmm-b|ijk|ikj
//                [--mode order-preserving|fast] [--out FILE]
//   afmm_gpu bench --kernel K --sizes N1,N2,... --d1 D1 --d2 D2 [--mu M] [--reps R]
//                [--warmups W] [--seed S] [--cutoff C] [--mode ...] [--out FILE]
//
// `bench` is the reference's run_plan (bench.hpp:120-154) for any kernel id:
// per (size, replication) the cell seed (bench.hpp:78-81), the factor pair of
// make_factor_pair (bench.hpp:86-99; the *-gpu ids draw the pairs of their CPU
// counterparts, so the CSVs compare cell by cell), W untimed warm-up calls,
// one call timed on steady_clock around the whole C-ABI product (H2D, device
// pipeline, D2H: the drop-in cost a reference caller sees), records under
// 100x the timer resolution discarded with the same warning, and the stable
// CSV schema of report.hpp:24-39 (kCsvHeader, format_double / format_fixed).
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

#include <chrono>
#include <fstream>
#include <sstream>

#include "afmm/bench.hpp"
#include "afmm/kernels.hpp"
#include "afmm/matrix_io.hpp"
#include "afmm/report.hpp"
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

std::vector<std::size_t> parse_sizes(const std::string& text) {
  std::vector<std::size_t> sizes;
  std::stringstream ss(text);
  std::string item;
  while (std::getline(ss, item, ',')) sizes.push_back(std::stoull(item));
  return sizes;
}

int bench(const Args& a) {
  const std::string kernel = opt(a, "kernel", "");
  const auto gpu_id = afmm::gpu::parse_kernel(kernel);
  const auto cpu_id = afmm::parse_kernel(kernel);
  if (!gpu_id && !cpu_id) throw std::invalid_argument("unknown kernel '" + kernel + "'");
  afmm::ExperimentPlan plan;
  plan.kernel = gpu_id ? (*gpu_id == afmm::gpu::KernelId::AFMM_A_GPU ? afmm::KernelId::AFMM_A
                                                                        : afmm::KernelId::AFMM_B)
                       : *cpu_id;
  plan.sizes = parse_sizes(opt(a, "sizes", ""));
  plan.d1 = std::stod(opt(a, "d1", "-1"));
  plan.d2 = std::stod(opt(a, "d2", "-1"));
  plan.mu_prime = std::stod(opt(a, "mu", "1"));
  plan.replications = std::stoull(opt(a, "reps", "20"));
  plan.warmups = std::stoull(opt(a, "warmups", "2"));
  plan.base_seed = afmm::Seed{std::stoull(opt(a, "seed", "0"))};
  plan.strassen_cutoff = std::stoull(opt(a, "cutoff", "64"));
  afmm::validate(plan);
  afmm::gpu::Options o;
  o.mode = opt(a, "mode", "order-preserving") == "fast" ? afmm::gpu::Mode::Fast
                                                         : afmm::gpu::Mode::OrderPreserving;
  auto call = [&](const afmm::DenseMatrix& lhs, const afmm::DenseMatrix& rhs) {
    return gpu_id ? afmm::gpu::run_kernel(*gpu_id, lhs, rhs, o)
                  : afmm::run_kernel(plan.kernel, lhs, rhs, plan.strassen_cutoff);
  };
  using clock = std::chrono::steady_clock;
  const double min_elapsed = 100.0 * afmm::timer_resolution();
  std::ostringstream csv;
  csv << afmm::kCsvHeader << '\n';
  for (const std::size_t n : plan.sizes) {
    for (std::size_t rep = 0; rep < plan.replications; ++rep) {
      const std::uint64_t seed = afmm::cell_seed(plan.base_seed, n, rep);
      const auto [lhs, rhs] =
          afmm::make_factor_pair(plan.kernel, n, plan.d1, plan.d2, plan.mu_prime, seed);
      for (std::size_t w = 0; w < plan.warmups; ++w) (void)call(lhs, rhs);
      const auto start = clock::now();
      const afmm::MultiplyResult result = call(lhs, rhs);
      const double elapsed = std::chrono::duration<double>(clock::now() - start).count();
      if (elapsed < min_elapsed) {
        std::cerr << "warning: n=" << n << " rep=" << rep << " elapsed " << elapsed
                  << "s is under 100x timer resolution; record discarded\n";
        continue;
      }
      csv << kernel << ',' << n << ',' << afmm::detail::format_double(plan.d1) << ','
          << afmm::detail::format_double(plan.d2) << ','
          << afmm::detail::format_double(plan.mu_prime) << ',' << seed << ',' << rep << ','
          << afmm::detail::format_fixed(elapsed, 9) << ',' << result.counts.additions << ','
          << result.counts.multiplications << ',' << result.counts.zero_skips << '\n';
    }
  }
  const std::string out = opt(a, "out", "");
  if (out.empty()) {
    std::cout << csv.str();
  } else {
    std::ofstream f(out);
    if (!f) throw std::runtime_error("cannot open for writing: " + out);
    f << csv.str();
    if (!f.good()) throw std::runtime_error("write failed: " + out);
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) throw std::invalid_argument("usage: afmm_gpu gen|mul|bench ...");
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
    } else if (cmd == "bench") {
      return bench(a);
    } else {
      throw std::invalid_argument("unknown subcommand '" + cmd + "'");
    }
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  }
  return 0;
}
