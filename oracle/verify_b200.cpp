// `planc verify` with the B200 executor dropped in (reference
// tools/planc.cpp:63-100): the reference loads the plan and graph, draws its
// seeded integer inputs, runs its sequential oracle (run_reference), and the
// plan is executed by planc_b200::run_plan (include/planc_b200.hpp) instead
// of the CPU planc::run_plan; the reference's own compare_outputs decides.
// Built by oracle/Makefile against the reference objects and the product
// library: the integration INTEGRATION.md describes, compiled and run.
//
//   verify_b200 --plan P --graph G [--seed N] [--tol T] [--lanes-on-one-gpu]
//   exit 0 PASS, 3 mismatch, 4 input error (tools/planc.cpp:18-20)
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

#include "planc/refexec.hpp"
#include "planc/simulate.hpp"
#include "planc_b200.hpp"

namespace {

std::string read_file(const std::string& p) {
  std::ifstream f(p);
  if (!f) throw planc::SchemaError("cannot read " + p);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

}  // namespace

int main(int argc, char** argv) {
  std::string plan_path, graph_path;
  std::uint64_t seed = 1;
  double tol = 0.0;
  bool one_gpu = false;
  int magnitude = 4;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    if (a == "--plan" && i + 1 < argc) plan_path = argv[++i];
    else if (a == "--graph" && i + 1 < argc) graph_path = argv[++i];
    else if (a == "--seed" && i + 1 < argc) seed = std::strtoull(argv[++i], nullptr, 10);
    else if (a == "--tol" && i + 1 < argc) tol = std::strtod(argv[++i], nullptr);
    else if (a == "--lanes-on-one-gpu") one_gpu = true;
    else if (a == "--magnitude" && i + 1 < argc) magnitude = std::atoi(argv[++i]);
  }
  try {
    // The reference front end's objects, exactly as `planc verify` uses them.
    planc::ExecutionPlan plan = planc::load_plan(read_file(plan_path));
    planc::PlanGraph graph = planc::load_graph(read_file(graph_path));
    auto inputs = planc::random_integer_inputs(graph, seed, magnitude);
    auto expected = planc::run_reference(graph, inputs);
    // The drop-in: the plan crosses the ABI in its save_plan wire form.
    std::vector<int> lanes;
    if (one_gpu) lanes.assign(plan.lanes.size(), 0);
    planc::TensorMap actual = planc_b200::run_plan(planc::save_plan(plan), inputs, lanes);
    auto report = planc::compare_outputs(expected, actual, tol);
    if (!report.ok) {
      std::cout << "FAIL: " << report.to_string() << "\n";
      return 3;
    }
    std::cout << "PASS: plan matches reference on seed " << seed << " (" << actual.size()
              << " tensors, executed by planc_b200)\n";
    return 0;
  } catch (const planc::SchemaError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 4;
  } catch (const planc::UsageError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 4;
  } catch (const planc_b200::UsageError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 4;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
