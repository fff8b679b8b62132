// planc_b200.hpp — header-only C++ face of the C ABI (planc_b200.h) shaped
// like the reference's executor API (proj/include/planc/refexec.hpp:38-60):
//
//   auto outputs = planc_b200::run_plan(plan_json, inputs);
//
// `inputs` / the result are any std::map<int, T> whose T has
// `std::vector<int64_t> shape` and `std::vector<double> data` — the
// reference's own planc::TensorMap / ConcreteTensor work unchanged. Errors
// are thrown as planc_b200::SchemaError / UsageError / InternalError /
// CudaError (the reference's class names, util.hpp:17-29).
#pragma once

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "planc_b200.h"

namespace planc_b200 {

struct Error : std::runtime_error {
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};
struct SchemaError : Error {
  using Error::Error;
};
struct UsageError : Error {
  using Error::Error;
};
struct InternalError : Error {
  using Error::Error;
};
struct CudaError : Error {
  using Error::Error;
};

inline void check(int rc) {
  if (rc == PLANC_B200_OK) return;
  std::string msg = planc_b200_last_error();
  if (rc == PLANC_B200_EUSAGE) {
    if (msg.rfind("SchemaError", 0) == 0) throw SchemaError(msg);
    throw UsageError(msg);
  }
  if (rc == PLANC_B200_ECUDA) throw CudaError(msg);
  throw InternalError(msg);
}

// RAII handle over one compiled plan.
class Executor {
 public:
  explicit Executor(const std::string& plan_json, const std::vector<int>& lane_gpus = {}, uint32_t flags = 0) {
    check(planc_b200_open(plan_json.c_str(), lane_gpus.empty() ? nullptr : lane_gpus.data(),
                          static_cast<int>(lane_gpus.size()), flags, &h_));
  }
  ~Executor() { planc_b200_close(h_); }
  Executor(const Executor&) = delete;
  Executor& operator=(const Executor&) = delete;

  template <class Tensor>
  void set_input(int ptensor, const Tensor& t) {
    check(planc_b200_set_input(h_, ptensor, t.data.data(), t.shape.data(), static_cast<int>(t.shape.size())));
  }
  double run(int iters = 0) {
    double ms = 0;
    check(planc_b200_run(h_, iters, &ms));
    return ms;
  }
  std::vector<int> output_ids() {
    int n = planc_b200_num_outputs(h_);
    std::vector<int> ids(n > 0 ? n : 0);
    if (n > 0) planc_b200_output_ids(h_, ids.data(), n);
    return ids;
  }
  template <class Tensor>
  Tensor output(int ptensor) {
    Tensor t;
    int64_t shape[16];
    int rank = 0;
    check(planc_b200_ptensor_shape(h_, ptensor, shape, 16, &rank));
    t.shape.assign(shape, shape + rank);
    int64_t vol = 1;
    for (auto e : t.shape) vol *= e;
    t.data.resize(static_cast<std::size_t>(vol));
    check(planc_b200_get_output(h_, ptensor, t.data.data(), vol));
    return t;
  }
  planc_b200_exec* handle() { return h_; }

 private:
  planc_b200_exec* h_ = nullptr;
};

// Drop-in for planc::run_plan (refexec.hpp:43): same inputs, same outputs
// (every pTensor produced by a non-inserted op, reassembled).
template <class TensorMap>
TensorMap run_plan(const std::string& plan_json, const TensorMap& inputs, const std::vector<int>& lane_gpus = {},
                   uint32_t flags = 0) {
  using Tensor = typename TensorMap::mapped_type;
  Executor ex(plan_json, lane_gpus, flags);
  for (const auto& [id, t] : inputs) ex.set_input(id, t);
  ex.run(0);
  TensorMap out;
  for (int id : ex.output_ids()) out[id] = ex.template output<Tensor>(id);
  return out;
}

}  // namespace planc_b200
