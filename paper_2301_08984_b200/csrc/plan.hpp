// ExecutionPlan data model and plan.json reader for the B200 executor.
//
// Mirrors the reference's plan types so a plan emitted by the reference front
// end is consumed unchanged:
//   Interval/Region/Mask   reference include/planc/graph.hpp:48-77
//   PTensor / VTensor      graph.hpp:85-109
//   OpNode (+ comm fields) graph.hpp:134-170
//   CollectiveGroup        include/planc/materialize.hpp:26-33
//   Task / DeviceLane      include/planc/simulate.hpp:20-35
//   ExecutionPlan          simulate.hpp:41-48
//   load_plan              proj/src/simulate.cpp:604-739 (same keys, same
//                          SchemaError on malformed documents)
// Error types keep the reference's names and meaning (util.hpp:17-29).
#pragma once

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

namespace planc_b200 {

struct SchemaError : std::runtime_error {
  explicit SchemaError(const std::string& m) : std::runtime_error(m) {}
};
struct UsageError : std::runtime_error {
  explicit UsageError(const std::string& m) : std::runtime_error(m) {}
};
struct InternalError : std::runtime_error {
  explicit InternalError(const std::string& m) : std::runtime_error(m) {}
};

struct Interval {
  std::int64_t lo = 0;
  std::int64_t hi = 0;
  std::int64_t length() const { return hi - lo; }
  bool operator==(const Interval& o) const { return lo == o.lo && hi == o.hi; }
};
using Region = std::vector<Interval>;

std::int64_t region_volume(const Region& r);
bool region_intersect(const Region& a, const Region& b, Region* out);
std::string region_to_string(const Region& r);

struct Mask {
  Region region;
  int value_index = 0;
  int value_count = 1;
  int replica_index = 0;
  int replica_count = 1;
};

enum class TensorKind { weight, activation, gradient, optimizer_state };

struct PTensor {
  int id = 0;
  std::vector<std::int64_t> shape;
  std::int64_t elem_size = 4;
  TensorKind kind = TensorKind::activation;
  int grad_of = -1;
  std::int64_t volume() const {
    std::int64_t v = 1;
    for (auto e : shape) v *= e;
    return v;
  }
};

struct VTensor {
  int id = 0;
  int ptensor = 0;
  Mask mask;
  bool producer_output = false;  // side "out"
  std::string owner_op;
};

enum class OpKind {
  matmul, ew_add, ew_mul, ew_max, reduce_sum, embedding_lookup, embedding_grad, identity,
  split, concat, reduce_assemble, send, recv, collective, free_buffer,
  // Schema extension (not in the reference: document.cpp:43-53 rejects
  // them): row-wise transformer sub-operators over the last axis in
  // segments of `segment` elements (0 = the whole axis), and GELU.
  softmax, softmax_grad, layernorm, layernorm_grad, gelu, gelu_grad,
  // O = softmax(Q·Kᵀ/sqrt(head_dim) [causal])·V per sequence of `seq` rows
  // and head of `head_dim` columns (inputs Q, K, V; output O, all [T, D]).
  attention,
  // its gradient with respect to Q, K or V (`wrt`): inputs Q, K, V, O, dO
  attention_grad,
};
const char* op_kind_name(OpKind k);

struct OpNode {
  std::string id;
  OpKind kind = OpKind::identity;
  std::vector<int> inputs;
  std::vector<int> outputs;
  std::string direction;
  double flops = 0;
  int doc_order = 0;
  bool inserted = false;
  int axis = -1;  // reduce-sum (absent -> 0, refexec.cpp:195)
  bool transpose_a = false;
  bool transpose_b = false;
  int micro_batch = -1;
  int channel = -1;
  int coll_group = -1;
  int free_vtensor = -1;
  std::string primitive;
  std::int64_t segment = 0;  // extension: row-wise segment width (0 = whole last axis)
  double eps = 1e-5;         // extension: layernorm epsilon
  std::int64_t head_dim = 0;  // extension: attention head width
  std::int64_t seq = 0;       // extension: attention rows per sequence
  bool causal = false;        // extension: attention causal mask
  char wrt = 'q';             // extension: attention-grad output ('q', 'k' or 'v')

  bool is_elementwise() const {
    return kind == OpKind::ew_add || kind == OpKind::ew_mul || kind == OpKind::ew_max;
  }
};

struct CollectiveGroup {
  int id = 0;
  std::string primitive;
  int k = 1;
  std::int64_t message_bytes = 0;
  bool inter_group = false;
  std::vector<std::string> ops;
};

enum class TaskKind { compute, send, recv, collective, free_buffer };

struct Task {
  TaskKind kind = TaskKind::compute;
  std::string op;
  double duration = 0;
  std::int64_t bytes = 0;
  int channel = -1;
  int coll_group = -1;
  int peer_device = -1;
};

struct DeviceLane {
  int device = 0;
  std::vector<Task> tasks;
};

struct ExecutionPlan {
  std::map<int, PTensor> ptensors;
  std::map<int, VTensor> vtensors;
  std::vector<OpNode> ops;  // document order
  std::map<std::string, int> assignment;
  std::map<int, int> feeds;  // consumer vt -> producer vt
  std::map<int, CollectiveGroup> coll_groups;
  std::vector<std::pair<std::string, std::string>> sync_edges;
  std::vector<DeviceLane> lanes;
  int num_cluster_devices = 0;

  // Indexes (built by load_plan / index()).
  std::unordered_map<std::string, int> op_index;
  std::vector<bool> pt_is_graph_input_cache;

  void index();
  const OpNode& op(const std::string& id) const;
  int op_idx(const std::string& id) const;
  const VTensor& vt(int id) const;
  const PTensor& pt(int id) const;
  bool is_graph_input(int ptensor) const;

 private:
  std::map<int, bool> graph_input_;
};

ExecutionPlan load_plan(const std::string& document);

}  // namespace planc_b200
