// acceptance_gpu -- the reference's acceptance gate (proj/tests/
// acceptance_main.cpp + acceptance.hpp) with every AFMM call on the B200
// (acceptance_gpu_shim.hpp). One shared Context, criteria in the order of
// run_suite(Suite::All) (acceptance.hpp:375-415), except c11 report-fidelity,
// which reads the paper's table CSV from the reference tree and calls no
// AFMM kernel. Prints the reference's [PASS]/[FAIL] lines and the number of
// GPU products; exits 1 if any criterion fails.
#include "acceptance_gpu_shim.hpp"
// (after the shim: its AFMM calls resolve to the B200 wrappers)
#include "afmm/acceptance.hpp"

#include <algorithm>
#include <iostream>

int main() {
  using namespace afmm::acceptance;
  using namespace afmm::acceptance::detail;
  Context ctx;
  std::vector<CriterionResult> results;
  results.push_back(c01_oracle_equivalence(ctx));
  results.push_back(c02_tolerant_equivalence(ctx));
  results.push_back(c03_expected_additions(ctx));
  results.push_back(c05_parameter_independence(ctx));
  results.push_back(c06_cubic_growth(ctx));
  results.push_back(c07_quadratic_regime(ctx));
  results.push_back(c10_timing_monotonicity(ctx));
  results.push_back(c12_fit_recovery(ctx));
  results.push_back(c08_afmm_vs_strassen(ctx));
  results.push_back(c09_strassen_structure(ctx));
  results.push_back(c04_multiplication_freedom(ctx));  // last: covers every run above
  std::sort(results.begin(), results.end(),
            [](const CriterionResult& a, const CriterionResult& b) { return a.id < b.id; });
  const bool ok = print_results(results, std::cout);
  std::cout << "b200 products: " << afmm::g_gpu_calls << '\n';
  return ok ? 0 : 1;
}
