#include "plan.hpp"

#include <algorithm>

#include "json.hpp"

namespace planc_b200 {

std::int64_t region_volume(const Region& r) {
  std::int64_t v = 1;
  for (const auto& iv : r) v *= iv.length();
  return v;
}

// reference proj/src/graph.cpp:63-73
bool region_intersect(const Region& a, const Region& b, Region* out) {
  if (a.size() != b.size()) throw UsageError("region_intersect: rank mismatch");
  Region r(a.size());
  for (std::size_t i = 0; i < a.size(); ++i) {
    r[i].lo = std::max(a[i].lo, b[i].lo);
    r[i].hi = std::min(a[i].hi, b[i].hi);
    if (r[i].lo >= r[i].hi) return false;
  }
  if (out) *out = std::move(r);
  return true;
}

std::string region_to_string(const Region& r) {
  std::string s;
  for (std::size_t i = 0; i < r.size(); ++i) {
    if (i) s += "x";
    s += "[" + std::to_string(r[i].lo) + "," + std::to_string(r[i].hi) + ")";
  }
  return s;
}

const char* op_kind_name(OpKind k) {
  switch (k) {
    case OpKind::matmul: return "matmul";
    case OpKind::ew_add: return "add";
    case OpKind::ew_mul: return "mul";
    case OpKind::ew_max: return "max";
    case OpKind::reduce_sum: return "reduce-sum";
    case OpKind::embedding_lookup: return "embedding-lookup";
    case OpKind::embedding_grad: return "embedding-grad";
    case OpKind::identity: return "identity";
    case OpKind::split: return "split";
    case OpKind::concat: return "concat";
    case OpKind::reduce_assemble: return "reduce-assemble";
    case OpKind::send: return "send";
    case OpKind::recv: return "recv";
    case OpKind::collective: return "collective";
    case OpKind::free_buffer: return "free";
    case OpKind::attention: return "attention";
    case OpKind::attention_grad: return "attention-grad";
    case OpKind::softmax: return "softmax";
    case OpKind::softmax_grad: return "softmax-grad";
    case OpKind::layernorm: return "layernorm";
    case OpKind::layernorm_grad: return "layernorm-grad";
    case OpKind::gelu: return "gelu";
    case OpKind::gelu_grad: return "gelu-grad";
  }
  return "?";
}

namespace {

// simulate.cpp:452-470 (op_kind_from_doc)
OpKind op_kind_from_doc(const std::string& s) {
  static const std::map<std::string, OpKind> m = {
      {"matmul", OpKind::matmul}, {"add", OpKind::ew_add}, {"mul", OpKind::ew_mul},
      {"max", OpKind::ew_max}, {"reduce-sum", OpKind::reduce_sum},
      {"embedding-lookup", OpKind::embedding_lookup}, {"embedding-grad", OpKind::embedding_grad},
      {"identity", OpKind::identity}, {"split", OpKind::split}, {"concat", OpKind::concat},
      {"reduce-assemble", OpKind::reduce_assemble}, {"send", OpKind::send}, {"recv", OpKind::recv},
      {"collective", OpKind::collective}, {"free", OpKind::free_buffer},
      // schema extension (oracle/planc_oracle.py eval_ext)
      {"softmax", OpKind::softmax}, {"softmax-grad", OpKind::softmax_grad}, {"layernorm", OpKind::layernorm},
      {"layernorm-grad", OpKind::layernorm_grad}, {"gelu", OpKind::gelu}, {"gelu-grad", OpKind::gelu_grad},
      {"attention", OpKind::attention}, {"attention-grad", OpKind::attention_grad}};
  auto it = m.find(s);
  if (it == m.end()) throw SchemaError("plan document: unknown op kind " + s);
  return it->second;
}

TensorKind tensor_kind_from(const std::string& s) {
  if (s == "weight") return TensorKind::weight;
  if (s == "activation") return TensorKind::activation;
  if (s == "gradient") return TensorKind::gradient;
  if (s == "optimizer-state") return TensorKind::optimizer_state;
  throw SchemaError("plan document: unknown tensor kind " + s);
}

TaskKind task_kind_from(const std::string& s) {
  if (s == "compute") return TaskKind::compute;
  if (s == "send") return TaskKind::send;
  if (s == "recv") return TaskKind::recv;
  if (s == "collective") return TaskKind::collective;
  if (s == "free") return TaskKind::free_buffer;
  throw SchemaError("plan document: unknown task kind " + s);
}

std::vector<int> int_list(const json::Value& v) {
  std::vector<int> out;
  for (const auto& e : v.arr) out.push_back(static_cast<int>(e.as_int()));
  return out;
}

}  // namespace

void ExecutionPlan::index() {
  op_index.clear();
  for (std::size_t i = 0; i < ops.size(); ++i) {
    if (!op_index.emplace(ops[i].id, static_cast<int>(i)).second) {
      throw SchemaError("plan document: duplicate op id " + ops[i].id);
    }
  }
  graph_input_.clear();
  for (const auto& [id, p] : ptensors) graph_input_[id] = true;
  for (const auto& o : ops) {
    for (int v : o.outputs) graph_input_[vt(v).ptensor] = false;
  }
}

const OpNode& ExecutionPlan::op(const std::string& id) const { return ops[op_idx(id)]; }

int ExecutionPlan::op_idx(const std::string& id) const {
  auto it = op_index.find(id);
  if (it == op_index.end()) throw UsageError("unknown op " + id);
  return it->second;
}

const VTensor& ExecutionPlan::vt(int id) const {
  auto it = vtensors.find(id);
  if (it == vtensors.end()) throw UsageError("unknown vtensor " + std::to_string(id));
  return it->second;
}

const PTensor& ExecutionPlan::pt(int id) const {
  auto it = ptensors.find(id);
  if (it == ptensors.end()) throw UsageError("unknown ptensor " + std::to_string(id));
  return it->second;
}

// graph.cpp:230-237: a pTensor with no producing op.
bool ExecutionPlan::is_graph_input(int ptensor) const {
  auto it = graph_input_.find(ptensor);
  if (it == graph_input_.end()) throw UsageError("unknown ptensor " + std::to_string(ptensor));
  return it->second;
}

ExecutionPlan load_plan(const std::string& document) {
  json::Value j;
  try {
    j = json::parse(document);
  } catch (const json::ParseError& e) {
    throw SchemaError(std::string("plan document is not valid JSON: ") + e.what());
  }
  ExecutionPlan plan;
  try {
    for (const auto& p : j.at("ptensors").arr) {
      PTensor pt;
      pt.id = static_cast<int>(p.at("id").as_int());
      for (const auto& e : p.at("shape").arr) pt.shape.push_back(e.as_int());
      pt.elem_size = p.at("elem_size").as_int();
      pt.kind = tensor_kind_from(p.at("kind").as_string());
      if (p.contains("grad_of")) pt.grad_of = static_cast<int>(p.at("grad_of").as_int());
      plan.ptensors[pt.id] = pt;
    }
    for (const auto& v : j.at("vtensors").arr) {
      VTensor vt;
      vt.id = static_cast<int>(v.at("id").as_int());
      vt.ptensor = static_cast<int>(v.at("ptensor").as_int());
      for (const auto& iv : v.at("region").arr) {
        vt.mask.region.push_back({iv.at(0).as_int(), iv.at(1).as_int()});
      }
      vt.mask.value_index = static_cast<int>(v.at("value").at(0).as_int());
      vt.mask.value_count = static_cast<int>(v.at("value").at(1).as_int());
      vt.mask.replica_index = static_cast<int>(v.at("replica").at(0).as_int());
      vt.mask.replica_count = static_cast<int>(v.at("replica").at(1).as_int());
      vt.producer_output = v.at("side").as_string() == "out";
      vt.owner_op = v.at("owner").as_string();
      plan.vtensors[vt.id] = vt;
    }
    for (const auto& o : j.at("ops").arr) {
      OpNode op;
      op.id = o.at("id").as_string();
      op.kind = op_kind_from_doc(o.at("kind").as_string());
      op.inputs = int_list(o.at("inputs"));
      op.outputs = int_list(o.at("outputs"));
      op.direction = o.at("direction").as_string();
      op.flops = o.at("flops").as_double();
      op.doc_order = static_cast<int>(o.at("doc_order").as_int());
      op.inserted = o.at("inserted").as_bool();
      if (o.contains("axis")) op.axis = static_cast<int>(o.at("axis").as_int());
      if (o.contains("transpose_a")) op.transpose_a = true;
      if (o.contains("transpose_b")) op.transpose_b = true;
      if (o.contains("micro_batch")) op.micro_batch = static_cast<int>(o.at("micro_batch").as_int());
      if (o.contains("channel")) op.channel = static_cast<int>(o.at("channel").as_int());
      if (o.contains("coll_group")) op.coll_group = static_cast<int>(o.at("coll_group").as_int());
      if (o.contains("free_vtensor")) op.free_vtensor = static_cast<int>(o.at("free_vtensor").as_int());
      if (o.contains("primitive")) op.primitive = o.at("primitive").as_string();
      if (o.contains("segment")) op.segment = o.at("segment").as_int();
      if (o.contains("eps")) op.eps = o.at("eps").as_double();
      if (o.contains("head_dim")) op.head_dim = o.at("head_dim").as_int();
      if (o.contains("seq")) op.seq = o.at("seq").as_int();
      if (o.contains("causal")) op.causal = o.at("causal").as_bool();
      if (o.contains("wrt")) {
        const std::string w = o.at("wrt").as_string();
        if (w != "q" && w != "k" && w != "v") throw SchemaError("attention-grad wrt must be q, k or v");
        op.wrt = w[0];
      }
      if (op.segment < 0 || !(op.eps >= 0)) throw SchemaError("plan document: bad segment / eps on op " + op.id);
      plan.ops.push_back(std::move(op));
    }
    for (const auto& kv : j.at("assignment").obj) {
      plan.assignment[kv.first] = static_cast<int>(kv.second.as_int());
    }
    for (const auto& f : j.at("feeds").arr) {
      plan.feeds[static_cast<int>(f.at(0).as_int())] = static_cast<int>(f.at(1).as_int());
    }
    for (const auto& g : j.at("coll_groups").arr) {
      CollectiveGroup grp;
      grp.id = static_cast<int>(g.at("id").as_int());
      grp.primitive = g.at("primitive").as_string();
      grp.k = static_cast<int>(g.at("k").as_int());
      grp.message_bytes = g.at("bytes").as_int();
      grp.inter_group = g.at("inter").as_bool();
      for (const auto& s : g.at("ops").arr) grp.ops.push_back(s.as_string());
      plan.coll_groups[grp.id] = grp;
    }
    if (j.contains("sync_edges")) {
      for (const auto& s : j.at("sync_edges").arr) {
        plan.sync_edges.push_back({s.at(0).as_string(), s.at(1).as_string()});
      }
    }
    for (const auto& lj : j.at("lanes").arr) {
      DeviceLane lane;
      lane.device = static_cast<int>(lj.at("device").as_int());
      for (const auto& tj : lj.at("tasks").arr) {
        Task t;
        t.kind = task_kind_from(tj.at("kind").as_string());
        t.op = tj.at("op").as_string();
        t.duration = tj.at("duration").as_double();
        t.bytes = tj.at("bytes").as_int();
        if (tj.contains("channel")) t.channel = static_cast<int>(tj.at("channel").as_int());
        if (tj.contains("coll_group")) t.coll_group = static_cast<int>(tj.at("coll_group").as_int());
        if (tj.contains("peer")) t.peer_device = static_cast<int>(tj.at("peer").as_int());
        lane.tasks.push_back(std::move(t));
      }
      plan.lanes.push_back(std::move(lane));
    }
    plan.num_cluster_devices = static_cast<int>(j.at("cluster").at("devices").size());
  } catch (const json::ParseError& e) {
    throw SchemaError(std::string("malformed plan document: ") + e.what());
  }
  plan.index();
  return plan;
}

}  // namespace planc_b200
