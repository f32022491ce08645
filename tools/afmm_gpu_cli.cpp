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
//                [--warmups W] [--seed S] [--cutoff C] [--mode ...] [--devices 0,1,..]
//                [--device-time 1] [--out FILE]
//   afmm_gpu report CSV... [--device-time 1] [--out FILE]
//   afmm_gpu plot-data CSV... --out-dir DIR
//
// `report` / `plot-data` are the reference's emit_table / emit_plot_data
// (report.hpp:160-331) over record CSVs that may mix CPU and GPU kernel ids:
// the reference's own parser rejects the *-gpu ids (report.hpp:85-86, it
// resolves names through op_counts.hpp:47-54), so the table is rebuilt here
// with string kernel ids -- same columns, labels, cells and reductions vs
// the ikj column. --device-time 1 in `bench` appends a twelfth CSV column,
// device_seconds (CUDA events around the whole call on the device:
// afmm_options.timing), which `report --device-time 1` tabulates instead of
// the wall-clock elapsed_seconds.
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
#include <filesystem>
#include <fstream>
#include <optional>
#include <sstream>

#include "afmm/bench.hpp"
#include "afmm/analysis.hpp"
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

// --mode order-preserving | fast | fast-ladder
afmm::gpu::Mode parse_mode(const std::string& text) {
  if (text == "order-preserving") return afmm::gpu::Mode::OrderPreserving;
  if (text == "fast") return afmm::gpu::Mode::Fast;
  if (text == "fast-ladder") return afmm::gpu::Mode::FastLadder;
  throw std::invalid_argument("unknown --mode " + text);
}

std::vector<int> parse_ints(const std::string& text) {
  std::vector<int> v;
  std::stringstream ss(text);
  std::string item;
  while (std::getline(ss, item, ',')) v.push_back(std::stoi(item));
  return v;
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
  const bool device_time = opt(a, "device-time", "0") == "1";
  if (device_time && !gpu_id) throw std::invalid_argument("--device-time needs a *-gpu kernel");
  afmm_timing timing{};
  afmm::gpu::Options o;
  o.mode = parse_mode(opt(a, "mode", "order-preserving"));
  o.devices = parse_ints(opt(a, "devices", ""));
  if (device_time) o.timing = &timing;
  auto call = [&](const afmm::DenseMatrix& lhs, const afmm::DenseMatrix& rhs) {
    return gpu_id ? afmm::gpu::run_kernel(*gpu_id, lhs, rhs, o)
                  : afmm::run_kernel(plan.kernel, lhs, rhs, plan.strassen_cutoff);
  };
  using clock = std::chrono::steady_clock;
  const double min_elapsed = 100.0 * afmm::timer_resolution();
  std::ostringstream csv;
  csv << afmm::kCsvHeader << (device_time ? ",device_seconds" : "") << '\n';
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
          << result.counts.multiplications << ',' << result.counts.zero_skips;
      if (device_time) csv << ',' << afmm::detail::format_fixed(timing.total_ms * 1e-3, 9);
      csv << '\n';
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

// ---- report / plot-data over CSVs with CPU and GPU kernel ids ----

struct Record {
  std::string kernel;
  std::size_t n = 0;
  double d1 = 0, d2 = 0, mu = 0;
  double elapsed = 0;
  std::optional<double> device_seconds;
};

bool known_kernel(std::string_view k) {
  return afmm::parse_kernel(k).has_value() || afmm::gpu::parse_kernel(k).has_value();
}
bool afmm_kernel(std::string_view k) { return k.rfind("afmm-", 0) == 0; }

std::vector<Record> load_records(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open for reading: " + path);
  std::string line;
  if (!std::getline(in, line)) throw std::runtime_error(path + ": csv: empty input");
  if (!line.empty() && line.back() == '\r') line.pop_back();
  const std::string h11(afmm::kCsvHeader), h12 = h11 + ",device_seconds";
  if (line != h11 && line != h12)
    throw std::runtime_error(path + ": csv: unexpected header '" + line + "'");
  const std::size_t nf = line == h12 ? 12 : 11;
  std::vector<Record> out;
  std::size_t line_no = 1;
  while (std::getline(in, line)) {
    ++line_no;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    const auto f = afmm::detail::split_fields(line);
    const auto fail = [&](const std::string& what) {
      return std::runtime_error(path + ": csv line " + std::to_string(line_no) + ": " + what);
    };
    if (f.size() != nf) throw fail("expected " + std::to_string(nf) + " fields");
    if (!known_kernel(f[0])) throw fail("unknown kernel '" + std::string(f[0]) + "'");
    Record r;
    r.kernel = std::string(f[0]);
    const auto n = afmm::detail::parse_u64(f[1]);
    const auto d1 = afmm::detail::parse_double(f[2]);
    const auto d2 = afmm::detail::parse_double(f[3]);
    const auto mu = afmm::detail::parse_double(f[4]);
    const auto el = afmm::detail::parse_double(f[7]);
    if (!n || !d1 || !d2 || !mu || !el) throw fail("malformed field");
    r.n = *n;
    r.d1 = *d1;
    r.d2 = *d2;
    r.mu = *mu;
    r.elapsed = *el;
    if (nf == 12) {
      const auto ds = afmm::detail::parse_double(f[11]);
      if (!ds) throw fail("malformed device_seconds");
      r.device_seconds = *ds;
    }
    out.push_back(std::move(r));
  }
  return out;
}

struct Column {
  std::string kernel;
  double d1, d2, mu;
  std::string label;
};

// build_report (report.hpp:160-225) over string kernel ids
struct Table {
  std::vector<std::size_t> sizes;
  std::vector<Column> columns;
  std::vector<std::vector<afmm::SampleStats>> cells;
  std::optional<std::size_t> ikj;
  std::vector<std::vector<std::optional<double>>> reductions;
};

Table build_table(const std::vector<Record>& records, bool device_time) {
  if (records.empty()) throw std::runtime_error("report: no records");
  Table t;
  auto column_of = [&](const Record& r) -> std::size_t {
    for (std::size_t c = 0; c < t.columns.size(); ++c) {
      const auto& col = t.columns[c];
      if (col.kernel == r.kernel && col.d1 == r.d1 && col.d2 == r.d2 && col.mu == r.mu) return c;
    }
    std::string label = r.kernel;
    if (afmm_kernel(r.kernel)) label += " mu'=" + afmm::detail::format_double(r.mu);
    for (const auto& e : t.columns)
      if (e.label == label) {
        label += " d1=" + afmm::detail::format_double(r.d1) +
                 " d2=" + afmm::detail::format_double(r.d2);
        break;
      }
    t.columns.push_back({r.kernel, r.d1, r.d2, r.mu, label});
    return t.columns.size() - 1;
  };
  std::map<std::size_t, std::map<std::size_t, std::vector<double>>> grid;
  for (const auto& r : records) {
    if (device_time && !r.device_seconds)
      throw std::runtime_error("report: --device-time needs device_seconds in every CSV");
    grid[r.n][column_of(r)].push_back(device_time ? *r.device_seconds : r.elapsed);
  }
  std::string missing;
  for (const auto& [n, row] : grid)
    for (std::size_t c = 0; c < t.columns.size(); ++c)
      if (!row.count(c)) missing += " (n=" + std::to_string(n) + ", " + t.columns[c].label + ")";
  if (!missing.empty()) throw std::runtime_error("report: missing cells:" + missing);
  for (std::size_t c = 0; c < t.columns.size(); ++c)
    if (t.columns[c].kernel == "ikj") {
      t.ikj = c;
      break;
    }
  for (const auto& [n, row] : grid) {
    t.sizes.push_back(n);
    std::vector<afmm::SampleStats> cells;
    for (std::size_t c = 0; c < t.columns.size(); ++c) cells.push_back(afmm::summarize(row.at(c)));
    std::vector<std::optional<double>> red(t.columns.size());
    if (t.ikj)
      for (std::size_t c = 0; c < t.columns.size(); ++c)
        if (afmm_kernel(t.columns[c].kernel))
          red[c] = afmm::percent_reduction(cells[*t.ikj].mean, cells[c].mean);
    t.cells.push_back(std::move(cells));
    t.reductions.push_back(std::move(red));
  }
  return t;
}

// format_markdown (report.hpp:229-262)
std::string markdown(const Table& t) {
  std::ostringstream out;
  out << "| n |";
  for (const auto& c : t.columns) out << ' ' << c.label << " |";
  out << "\n|";
  for (std::size_t c = 0; c <= t.columns.size(); ++c) out << " ---: |";
  out << '\n';
  for (std::size_t r = 0; r < t.sizes.size(); ++r) {
    out << "| " << t.sizes[r] << " |";
    for (const auto& st : t.cells[r]) out << ' ' << afmm::detail::format_general(st.mean, 6) << " |";
    out << '\n';
  }
  if (t.ikj)
    for (std::size_t r = 0; r < t.sizes.size(); ++r) {
      bool any = false;
      for (const auto& v : t.reductions[r]) any = any || v.has_value();
      if (!any) continue;
      out << "| reduction vs ikj (%), n=" << t.sizes[r] << " |";
      for (const auto& v : t.reductions[r]) {
        out << ' ';
        if (v) out << afmm::detail::format_fixed(*v, 1);
        out << " |";
      }
      out << '\n';
    }
  return out.str();
}

std::vector<Record> load_all(const Args& a) {
  if (a.positional.empty()) throw std::invalid_argument("needs at least one CSV");
  std::vector<Record> all;
  for (const auto& p : a.positional) {
    auto r = load_records(p);
    all.insert(all.end(), r.begin(), r.end());
  }
  return all;
}

int report(const Args& a) {
  const std::string text = markdown(build_table(load_all(a), opt(a, "device-time", "0") == "1"));
  const std::string out = opt(a, "out", "");
  if (out.empty()) {
    std::cout << text;
  } else {
    std::ofstream f(out);
    if (!f) throw std::runtime_error("cannot open for writing: " + out);
    f << text;
  }
  return 0;
}

// emit_plot_data (report.hpp:288-331)
int plot_data(const Args& a) {
  const std::string dir = opt(a, "out-dir", "");
  if (dir.empty()) throw std::invalid_argument("plot-data needs --out-dir");
  const Table t = build_table(load_all(a), opt(a, "device-time", "0") == "1");
  std::filesystem::create_directories(dir);
  std::ofstream manifest(std::filesystem::path(dir) / "manifest.txt");
  if (!manifest) throw std::runtime_error("cannot open for writing: manifest.txt");
  for (std::size_t c = 0; c < t.columns.size(); ++c) {
    const std::string name =
        "series_" + std::to_string(c) + "_" + afmm::detail::slugify(t.columns[c].label) + ".dat";
    std::ofstream f(std::filesystem::path(dir) / name);
    if (!f) throw std::runtime_error("cannot open for writing: " + name);
    for (std::size_t r = 0; r < t.sizes.size(); ++r)
      f << t.sizes[r] << ' ' << afmm::detail::format_double(t.cells[r][c].mean) << ' '
        << afmm::detail::format_double(t.cells[r][c].std_dev) << '\n';
    manifest << name << ' ' << t.columns[c].label << '\n';
  }
  std::cerr << "wrote " << t.columns.size() + 1 << " files under " << dir << '\n';
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) throw std::invalid_argument("usage: afmm_gpu gen|mul|bench|report|plot-data ...");
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
      o.mode = parse_mode(opt(a, "mode", "order-preserving"));
      const auto result = multiply(opt(a, "kernel", "afmm-a-gpu"), lhs, rhs, o);
      const std::string out = opt(a, "out", "");
      if (out.empty()) afmm::write_matrix(std::cout, result.product);
      else afmm::save_matrix(out, result.product);
      std::cout << result.counts << '\n';
    } else if (cmd == "bench") {
      return bench(a);
    } else if (cmd == "report") {
      return report(a);
    } else if (cmd == "plot-data") {
      return plot_data(a);
    } else {
      throw std::invalid_argument("unknown subcommand '" + cmd + "'");
    }
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  }
  return 0;
}
