// TEST INFRASTRUCTURE — the exact-signature drop-in INTEGRATION.md describes,
// compiled: `planc::TensorMap run_plan_b200(const ExecutionPlan&, const
// TensorMap&)` (the signature of reference include/planc/refexec.hpp:43)
// serialises the plan with the reference's own save_plan
// (simulate.cpp:492-602) and executes it through the product's C ABI
// (include/planc_b200.h) on the B200; errors come back as the reference's
// exception classes (util.hpp:17-29).
//
// Linked with `-Wl,--wrap=<mangled planc::run_plan>` every reference call
// of planc::run_plan — testutil.cpp:386 oracle_ok, and through it the
// reference's own acceptance suite (acceptance.cpp:36-71 criterion 1: 220
// randomized plans; criteria 7 and 9) — lands here instead of the CPU
// executor (refexec.cpp:361-557), unmodified reference sources otherwise.
// Lanes go round-robin over PLANC_B200_NUM_GPUS devices (default 1: every
// lane on GPU 0, each lane with its own streams).
#include <cstdlib>
#include <string>
#include <vector>

#include "planc/refexec.hpp"
#include "planc/simulate.hpp"
#include "planc/util.hpp"
#include "planc_b200.h"

namespace planc {

TensorMap run_plan_b200(const ExecutionPlan& plan, const TensorMap& inputs) {
  const std::string doc = save_plan(plan);
  planc_b200_exec* h = nullptr;
  auto check = [&](int rc) {
    if (rc == PLANC_B200_OK) return;
    std::string msg = planc_b200_last_error();
    if (h) planc_b200_close(h);
    h = nullptr;
    if (rc == PLANC_B200_EUSAGE) {
      if (msg.rfind("SchemaError", 0) == 0) throw SchemaError(msg);
      throw UsageError(msg);
    }
    throw InternalError(msg);
  };
  const char* env = std::getenv("PLANC_B200_NUM_GPUS");
  const int ngpu = env && std::atoi(env) > 0 ? std::atoi(env) : 1;
  std::vector<int> gpus(static_cast<std::size_t>(ngpu));
  for (int i = 0; i < ngpu; ++i) gpus[static_cast<std::size_t>(i)] = i;
  check(planc_b200_open(doc.c_str(), gpus.data(), ngpu, 0, &h));
  for (const auto& [pt, t] : inputs) {
    check(planc_b200_set_input(h, pt, t.data.data(), t.shape.data(), static_cast<int>(t.shape.size())));
  }
  check(planc_b200_run(h, 0, nullptr));
  TensorMap out;
  const int n = planc_b200_num_outputs(h);
  std::vector<int> ids(n > 0 ? static_cast<std::size_t>(n) : 0);
  if (n > 0 && planc_b200_output_ids(h, ids.data(), n) != n) throw InternalError("planc_b200_output_ids");
  for (int pt : ids) {
    ConcreteTensor t;
    std::int64_t shape[16];
    int rank = 0;
    check(planc_b200_ptensor_shape(h, pt, shape, 16, &rank));
    t.shape.assign(shape, shape + rank);
    t.data.resize(static_cast<std::size_t>(t.volume()));
    check(planc_b200_get_output(h, pt, t.data.data(), t.volume()));
    out[pt] = std::move(t);
  }
  planc_b200_close(h);
  return out;
}

}  // namespace planc

// The linker's --wrap target for planc::run_plan.
planc::TensorMap wrapped_run_plan(const planc::ExecutionPlan& plan, const planc::TensorMap& inputs) asm(
    "__wrap__ZN5planc8run_planERKNS_13ExecutionPlanERKSt3mapIiNS_14ConcreteTensorESt4lessIiESaISt4pairIKiS4_EEE");
planc::TensorMap wrapped_run_plan(const planc::ExecutionPlan& plan, const planc::TensorMap& inputs) {
  return planc::run_plan_b200(plan, inputs);
}
