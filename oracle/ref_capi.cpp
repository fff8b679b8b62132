// TEST INFRASTRUCTURE — the reference-side checker, never the product.
//
// A thin extern "C" shim over the UNMODIFIED reference planc library, built
// from /root/reference/proj sources into oracle/_ref/libplanc_ref.so by
// oracle/Makefile. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs load it. It exposes:
//   * the reference front end (load_graph -> strategy -> compile -> save_plan),
//     reference proj/src/compile.cpp:7-67, strategies.cpp:679-712;
//   * the reference fixtures' graph documents (proj/tests/testutil.cpp:28-368);
//   * the oracle (run_reference, refexec.cpp:264-350), the CPU plan executor
//     the product replaces (run_plan, refexec.cpp:361-557), seeded inputs
//     (random_integer_inputs, refexec.cpp:559-590) and compare_outputs.
// Tensor maps cross the ABI as a flat int64/double blob:
//   int64 count; per tensor: int64 id, int64 rank, int64 shape[rank],
//   double data[volume].
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "planc/compile.hpp"
#include "planc/refexec.hpp"
#include "planc/simulate.hpp"
#include "planc/strategies.hpp"
#include "planc/transform.hpp"
#include "testutil.hpp"

using namespace planc;

namespace {

thread_local std::string g_err;

char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

std::map<std::string, std::string> parse_kv(const char* spec) {
  std::map<std::string, std::string> kv;
  std::stringstream ss(spec ? spec : "");
  std::string item;
  while (std::getline(ss, item, ';')) {
    auto eq = item.find('=');
    if (eq == std::string::npos) continue;
    kv[item.substr(0, eq)] = item.substr(eq + 1);
  }
  return kv;
}

std::vector<std::string> split_csv(const std::string& s) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, ',')) {
    if (!item.empty()) out.push_back(item);
  }
  return out;
}

std::vector<char> encode(const TensorMap& m) {
  std::vector<char> out;
  auto put = [&](const void* p, std::size_t n) {
    out.insert(out.end(), static_cast<const char*>(p),
               static_cast<const char*>(p) + n);
  };
  std::int64_t count = static_cast<std::int64_t>(m.size());
  put(&count, 8);
  for (const auto& [id, t] : m) {
    std::int64_t i = id, r = static_cast<std::int64_t>(t.shape.size());
    put(&i, 8);
    put(&r, 8);
    put(t.shape.data(), 8 * t.shape.size());
    put(t.data.data(), 8 * t.data.size());
  }
  return out;
}

TensorMap decode(const char* blob) {
  TensorMap m;
  const char* p = blob;
  auto get = [&](void* dst, std::size_t n) {
    std::memcpy(dst, p, n);
    p += n;
  };
  std::int64_t count = 0;
  get(&count, 8);
  for (std::int64_t c = 0; c < count; ++c) {
    std::int64_t id = 0, rank = 0;
    get(&id, 8);
    get(&rank, 8);
    ConcreteTensor t;
    t.shape.resize(static_cast<std::size_t>(rank));
    get(t.shape.data(), 8 * rank);
    t.data.resize(static_cast<std::size_t>(t.volume()));
    get(t.data.data(), 8 * t.data.size());
    m[static_cast<int>(id)] = std::move(t);
  }
  return m;
}

char* blob_out(const TensorMap& m, std::int64_t* nbytes) {
  auto v = encode(m);
  char* p = static_cast<char*>(std::malloc(v.size()));
  std::memcpy(p, v.data(), v.size());
  if (nbytes) *nbytes = static_cast<std::int64_t>(v.size());
  return p;
}

// Megatron-style tensor parallelism written as an sProgram over op_trans, the
// way the reference's own TP test does it (proj/tests/test_refexec.cpp:100-140):
// forward ops whose id starts with "col" split output dim 1 (column-parallel
// GEMM), "row" value-split (row-parallel GEMM -> partial sums), "tp" split
// output dim 1 (elementwise ops between the column- and row-parallel GEMMs),
// "sp" split output dim 0 (sequence parallelism: the residual ops between
// the row- and column-parallel GEMMs hold a slice of the tokens, so the
// front end materialises reduce-scatter after row-parallel GEMMs and
// all-gather before column-parallel ones — Megatron-SP), everything else is
// replicated. Backward ops follow their forward op through
// adapt_backward (transform.cpp:503); optimizer ops "optc" / "optr" split like
// their column- / row-parallel weight (dim 1 / dim 0), others are replicated.
StrategyInfo megatron_tp(PlanGraph& g, const ClusterSpec& env,
                         const StrategyConfig& cfg) {
  int n = cfg.devices;
  std::vector<std::string> snapshot;
  for (const auto& op : g.ops) snapshot.push_back(op.id);
  auto has_backward = [&](const std::string& fwd) {
    for (const auto& o : g.ops) {
      if (o.backward_of && *o.backward_of == fwd) return true;
    }
    return false;
  };
  for (const auto& oid : snapshot) {
    if (!g.has_op(oid)) continue;
    const OpNode& op = g.op(oid);
    if (op.direction == OpDirection::backward) continue;
    TransformAlgo algo = replica_algo(n);
    // Role prefix of the op id's last '.'-separated component.
    std::string role = oid.substr(oid.rfind('.') == std::string::npos
                                      ? 0
                                      : oid.rfind('.') + 1);
    auto is = [&](const char* p) { return role.rfind(p, 0) == 0; };
    if (op.direction == OpDirection::forward) {
      if (is("col") || is("tp")) {
        algo = split_algo(1, n);
      } else if (is("sp")) {
        algo = split_algo(0, n);
      } else if (is("row")) {
        algo = value_split_algo(n);
      }
    } else if (op.direction == OpDirection::optimizer) {
      if (is("optc")) algo = split_algo(1, n);
      if (is("optr")) algo = split_algo(0, n);
    }
    std::vector<std::string> bwd;
    if (has_backward(oid)) bwd = adapt_backward(g, oid, algo);
    auto ids = op_trans(g, oid, algo);
    for (std::size_t i = 0; i < ids.size(); ++i) {
      op_assign(g, env, ids[i], static_cast<int>(i % n));
    }
    for (std::size_t i = 0; i < bwd.size(); ++i) {
      op_assign(g, env, bwd[i], static_cast<int>(i % n));
    }
  }
  return {};
}

// Hand-written sProgram in the style of the reference's adapter tests
// (test_refexec.cpp:100-140, test_commplan.cpp:303-366): target_ops lists
// "op@algo[@offset[@count]]" with algo v (value split), sD (split output dim
// D), r (replica) or e (vocabulary-sharded embedding), fanned out `count`
// ways (default: devices); replacement i goes to device offset + i. An algo
// "sD:n/sE:m" splits a forward op on dim D n ways, then each part on dim E m
// ways (a 2-D tiling, e.g. the D(2,2) consumer of SURVEY fact 6).
// Paired backward ops follow through adapt_backward. Unlisted ops stay whole
// on device 0.
StrategyInfo manual(PlanGraph& g, const ClusterSpec& env,
                    const StrategyConfig& cfg) {
  int n = cfg.devices;
  struct Target {
    std::string algo;
    int offset = 0;
    int count = 0;
  };
  std::map<std::string, Target> algo_of;
  for (const auto& t : cfg.target_ops) {
    std::vector<std::string> f;
    std::stringstream ss(t);
    std::string item;
    while (std::getline(ss, item, '@')) f.push_back(item);
    if (f.size() < 2) throw UsageError("manual: bad target " + t);
    Target tg{f[1], f.size() > 2 ? std::stoi(f[2]) : 0,
              f.size() > 3 ? std::stoi(f[3]) : n};
    algo_of[f[0]] = tg;
  }
  std::vector<std::string> snapshot;
  for (const auto& op : g.ops) snapshot.push_back(op.id);
  for (const auto& oid : snapshot) {
    if (!g.has_op(oid)) continue;
    auto it = algo_of.find(oid);
    if (it == algo_of.end()) continue;
    const std::string& a = it->second.algo;
    int cnt = it->second.count, off = it->second.offset;
    if (a.find('/') != std::string::npos) {
      // Nested splits "sD:n/sE:m" (forward ops without a backward pair):
      // op_trans by the first algo, then every replacement by the next;
      // replacement i (row-major over the levels) goes to device off + i.
      std::vector<std::string> ids{oid};
      std::stringstream ls(a);
      std::string lvl;
      while (std::getline(ls, lvl, '/')) {
        auto c = lvl.find(':');
        if (lvl.empty() || lvl[0] != 's' || c == std::string::npos) throw UsageError("manual: bad level " + lvl);
        TransformAlgo la = split_algo(std::stoi(lvl.substr(1, c - 1)), std::stoi(lvl.substr(c + 1)));
        std::vector<std::string> next;
        for (const auto& id : ids) {
          auto r = op_trans(g, id, la);
          next.insert(next.end(), r.begin(), r.end());
        }
        ids = next;
      }
      for (std::size_t i = 0; i < ids.size(); ++i) op_assign(g, env, ids[i], off + static_cast<int>(i));
      continue;
    }
    TransformAlgo algo = replica_algo(cnt);
    if (a == "v") algo = value_split_algo(cnt);
    else if (a == "e") algo = shard_embed_algo(cnt);
    else if (a[0] == 's') algo = split_algo(std::stoi(a.substr(1)), cnt);
    bool paired = false;
    for (const auto& o : g.ops) {
      if (o.backward_of && *o.backward_of == oid) paired = true;
    }
    std::vector<std::string> bwd;
    if (paired) bwd = adapt_backward(g, oid, algo);
    auto ids = op_trans(g, oid, algo);
    for (std::size_t i = 0; i < ids.size(); ++i) {
      op_assign(g, env, ids[i], off + static_cast<int>(i % cnt));
    }
    for (std::size_t i = 0; i < bwd.size(); ++i) {
      op_assign(g, env, bwd[i], off + static_cast<int>(i % cnt));
    }
  }
  for (const auto& op : g.ops) {
    if (!g.assignment.count(op.id)) op_assign(g, env, op.id, 0);
  }
  return {};
}

bool has_backward_pair(const PlanGraph& g, const std::string& fwd) {
  for (const auto& o : g.ops) {
    if (o.backward_of && *o.backward_of == fwd) return true;
  }
  return false;
}

// op_trans preceded by adapt_backward when the op has declared backward
// pairs (the composition the reference's own strategies use,
// strategies.cpp:43-53); backward replacement i of every backward op is
// appended to *bwd in op order.
std::vector<std::string> trans_with_backward(PlanGraph& g, const std::string& oid, const TransformAlgo& algo,
                                             std::vector<std::string>* bwd) {
  if (has_backward_pair(g, oid)) {
    auto b = adapt_backward(g, oid, algo);
    bwd->insert(bwd->end(), b.begin(), b.end());
  }
  return op_trans(g, oid, algo);
}

std::string role_of(const std::string& oid) {
  auto dot = oid.rfind('.');
  return dot == std::string::npos ? oid : oid.substr(dot + 1);
}

// Config C4: co-shard x `shards` composed with `devices`-way
// data parallelism. Forward ops split their batch dim across the DP ranks
// (plan_data_parallel, strategies.cpp:120-146); optimizer adds split dim 0
// across the ranks (a sharded, ZeRO-style optimizer: rank i updates rows
// slice i), "agw*" publication ops stay replicated; then on every rank the
// `target_ops` replacements are co-sharded with the reference's own
// plan_coshard (strategies.cpp:278-396: time-multiplexed sub-operators with
// recompute, chained split choice, shard i before shard i+1).
StrategyInfo coshard_dp(PlanGraph& g, const ClusterSpec& env, const StrategyConfig& cfg) {
  const int n = cfg.devices;
  std::map<std::string, std::vector<std::string>> dp_ids;
  std::vector<std::string> snapshot;
  for (const auto& op : g.ops) snapshot.push_back(op.id);
  for (const auto& oid : snapshot) {
    if (!g.has_op(oid)) continue;
    const OpNode& op = g.op(oid);
    if (op.direction == OpDirection::backward) continue;
    TransformAlgo algo = replica_algo(n);
    if (op.direction == OpDirection::forward) {
      if (!op.attrs.batch_dim) throw UsageError("coshard_dp: forward op " + oid + " has no batch_dim");
      algo = split_algo(*op.attrs.batch_dim, n);
    } else if (role_of(oid).rfind("agw", 0) != 0) {
      algo = split_algo(0, n);
    }
    std::vector<std::string> bwd;
    auto ids = trans_with_backward(g, oid, algo, &bwd);
    for (std::size_t i = 0; i < ids.size(); ++i) op_assign(g, env, ids[i], static_cast<int>(i % n));
    for (std::size_t i = 0; i < bwd.size(); ++i) op_assign(g, env, bwd[i], static_cast<int>(i % n));
    dp_ids[oid] = ids;
  }
  // Each target_ops entry is one co-shard group ("a+b+c": a chain of ops
  // sharded together, shard i of the group before shard i+1); groups are
  // co-sharded independently, so a whole op between two chains (a residual
  // add) never sits inside one group's shard order.
  if (cfg.shards > 1) {
    for (int d = 0; d < n; ++d) {
      for (const auto& entry : cfg.target_ops) {
        std::vector<std::string> targets;
        std::stringstream ss(entry);
        std::string t;
        while (std::getline(ss, t, '+')) {
          auto it = dp_ids.find(t);
          if (it == dp_ids.end()) throw UsageError("coshard_dp: unknown target op " + t);
          targets.push_back(it->second.at(static_cast<std::size_t>(d)));
        }
        plan_coshard(g, env, targets, cfg.shards, d);
      }
    }
  }
  return {};
}

// Config C5: the 3F1B schedule (plan_3f1b, strategies.cpp:
// 524-653) over `stages` pipeline stages of `dap` devices each, with the
// micro-batches declared by the document (op id suffix "#k"), every
// micro-batch sub-operator split DAP-style inside its stage (Dynamic Axial
// Parallelism): "row*" ops on dim 0 (rows), "col*" ops on dim 1 (channels),
// so consecutive row / column ops switch layout D(dap,1) <-> D(1,dap) — the
// all-to-all adapters (rvd.cpp:286-326). Optimizer adds split dim 0 over
// the stage's DAP group. Stage of a layer: contiguous equal count (as
// stage_of_layer, strategies.cpp:72-103). Per stage the task order is the
// 3F1B priority list (backward first, then forward passes 3, 2, 1, lowest
// micro-batch first), enforced with op_order between consecutive groups.
StrategyInfo threef1b_dap(PlanGraph& g, const ClusterSpec& env, const StrategyConfig& cfg) {
  const int S = cfg.stages, K = cfg.micro_batches;
  const int dap = cfg.inner_dp > 0 ? cfg.inner_dp : 1;
  if (S * dap != cfg.devices) throw UsageError("threef1b_dap: devices must equal stages x dap");
  std::set<int> layer_set;
  for (const auto& op : g.ops) {
    if (op.direction == OpDirection::forward && op.attrs.layer) layer_set.insert(*op.attrs.layer);
  }
  std::vector<int> layers(layer_set.begin(), layer_set.end());
  if (static_cast<int>(layers.size()) < S) throw UsageError("threef1b_dap: fewer layers than stages");
  std::map<int, int> stage_of;
  for (std::size_t i = 0; i < layers.size(); ++i)
    stage_of[layers[i]] = static_cast<int>(i * static_cast<std::size_t>(S) / layers.size());
  auto layer = [&](const OpNode& op) {
    if (!op.attrs.layer) throw UsageError("threef1b_dap: op " + op.id + " has no layer");
    return *op.attrs.layer;
  };
  // 1. micro-batches are explicit in the document: op ids end in "#k"
  // (docs.evoformer_doc) — one pTensor family per micro-batch, so the
  // collective pattern matching (rvd.cpp:785-870) sees whole families.
  for (auto& op : g.ops) {
    if (op.direction == OpDirection::optimizer || op.is_reserved_kind()) continue;
    auto h = op.id.rfind('#');
    if (h == std::string::npos) throw UsageError("threef1b_dap: op " + op.id + " lacks a #micro-batch suffix");
    op.micro_batch = std::stoi(op.id.substr(h + 1));
    if (*op.micro_batch >= K) throw UsageError("threef1b_dap: micro-batch of " + op.id + " >= micro_batches");
    if (op.direction == OpDirection::forward && !op.attrs.pass_index) throw UsageError("threef1b_dap: no pass on " + op.id);
  }
  // 2. per-stage 3F1B order over (pass, micro-batch) groups; pass 0 = backward
  using Task = std::pair<int, int>;
  std::vector<std::set<Task>> done(S);
  std::vector<std::vector<Task>> seq(S);
  auto ready = [&](int s, Task t) {
    if (t.first == 0) return (s + 1 == S || done[s + 1].count(t)) && done[s].count({3, t.second}) > 0;
    if (s > 0) return done[s - 1].count(t) > 0;
    return t.first == 1 || done[S - 1].count({t.first - 1, t.second}) > 0;
  };
  for (int total = 0, guard = 0; total < 4 * S * K; ++guard) {
    if (guard > 16 * S * K + 16) throw InternalError("threef1b_dap: schedule stalled");
    std::vector<Task> pick(S, {-1, -1});
    for (int s = 0; s < S; ++s) {
      for (int pass : {0, 3, 2, 1}) {
        for (int mb = 0; mb < K && pick[s].first < 0; ++mb) {
          if (!done[s].count({pass, mb}) && ready(s, {pass, mb})) pick[s] = {pass, mb};
        }
        if (pick[s].first >= 0) break;
      }
    }
    for (int s = 0; s < S; ++s) {
      if (pick[s].first < 0) continue;
      done[s].insert(pick[s]);
      seq[s].push_back(pick[s]);
      ++total;
    }
  }
  auto group = [&](int s, Task t) {
    std::vector<std::string> out;
    for (const auto& op : g.ops) {
      if (op.is_reserved_kind() || !op.micro_batch || *op.micro_batch != t.second) continue;
      if (op.direction == OpDirection::optimizer || stage_of.at(layer(op)) != s) continue;
      const bool b = op.direction == OpDirection::backward;
      if (t.first == 0 ? !b : (b || op.attrs.pass_index.value_or(-1) != t.first)) continue;
      out.push_back(op.id);
    }
    return out;
  };
  StrategyInfo info;
  info.stage_task_sequences.resize(S);
  for (int s = 0; s < S; ++s) {
    std::vector<std::string> prev;
    for (const auto& t : seq[s]) {
      auto ops = group(s, t);
      if (ops.empty()) throw InternalError("threef1b_dap: empty group");
      for (const auto& a : prev)
        for (const auto& b : ops) op_order(g, a, b);
      prev = ops;
      info.stage_task_sequences[s].push_back(ops);
    }
  }
  // 3. DAP inside each stage (happen-before edges follow the replacements)
  std::vector<std::string> snapshot;
  for (const auto& op : g.ops) snapshot.push_back(op.id);
  for (const auto& oid : snapshot) {
    if (!g.has_op(oid)) continue;
    const OpNode& op = g.op(oid);
    if (op.direction == OpDirection::backward || op.is_reserved_kind()) continue;
    const int s = stage_of.at(layer(op));
    const std::string r = role_of(oid.substr(0, oid.find('#')));
    TransformAlgo algo = split_algo(0, dap);
    if (op.direction == OpDirection::forward && r.rfind("col", 0) == 0) algo = split_algo(1, dap);
    std::vector<std::string> bwd;
    std::vector<std::string> ids{oid};
    if (dap > 1) ids = trans_with_backward(g, oid, algo, &bwd);
    for (std::size_t i = 0; i < ids.size(); ++i) op_assign(g, env, ids[i], s * dap + static_cast<int>(i % dap));
    for (std::size_t i = 0; i < bwd.size(); ++i) op_assign(g, env, bwd[i], s * dap + static_cast<int>(i % dap));
  }
  for (const auto& op : g.ops) {
    if (!g.assignment.count(op.id) && !op.is_reserved_kind()) op_assign(g, env, op.id, stage_of.at(layer(op)) * dap);
  }
  // stage sequences are reported at micro-batch granularity (pre-DAP ids)
  info.stage_task_sequences.clear();
  return info;
}

struct Registrar {
  Registrar() {
    register_strategy("megatron_tp", megatron_tp);
    register_strategy("manual", manual);
    register_strategy("coshard_dp", coshard_dp);
    register_strategy("threef1b_dap", threef1b_dap);
  }
} registrar;

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

char* ref_mlp_doc(int layers, std::int64_t batch, std::int64_t hidden,
                  int optimizer, int bias, int weight_grads) {
  testutil::MlpSpec s;
  s.layers = layers;
  s.batch = batch;
  s.hidden = hidden;
  s.optimizer = optimizer != 0;
  s.bias = bias != 0;
  s.weight_grads = weight_grads != 0;
  return dup_string(testutil::mlp_doc(s));
}

char* ref_coshard_doc(std::int64_t b, std::int64_t h, std::int64_t m) {
  return dup_string(testutil::coshard_doc({b, h, m}));
}

char* ref_embed_doc(int stage_layers, std::int64_t b, std::int64_t v,
                    std::int64_t h) {
  return dup_string(testutil::embed_doc({stage_layers, b, v, h}));
}

char* ref_three_pass_doc(int layers, std::int64_t b, std::int64_t h) {
  return dup_string(testutil::three_pass_doc({layers, b, h}));
}

char* ref_chain_doc() { return dup_string(testutil::chain_doc()); }

// spec: "strategy=...;devices=N;micro_batches=K;stages=S;shards=n;
//        target_ops=a,b;inner_dp=d;pattern_match=0|1;cluster_devices=N;
//        group_size=G;intra_bw=..;intra_lat=..;inter_bw=..;inter_lat=..;
//        throughput=..;testutil_cluster=0|1"
char* ref_compile(const char* graph_doc, const char* spec) {
  try {
    auto kv = parse_kv(spec);
    auto geti = [&](const char* k, int d) {
      return kv.count(k) ? std::stoi(kv[k]) : d;
    };
    auto getd = [&](const char* k, double d) {
      return kv.count(k) ? std::stod(kv[k]) : d;
    };
    StrategyConfig c;
    c.strategy = kv.count("strategy") ? kv["strategy"] : "none";
    c.devices = geti("devices", 1);
    c.micro_batches = geti("micro_batches", 1);
    c.stages = geti("stages", 1);
    c.shards = geti("shards", 1);
    c.inner_dp = geti("inner_dp", 1);
    if (kv.count("target_ops")) c.target_ops = split_csv(kv["target_ops"]);
    int ndev = geti("cluster_devices", c.devices);
    ClusterSpec cluster;
    if (geti("testutil_cluster", 0)) {
      cluster = testutil::make_cluster(ndev, geti("group_size", 0));
    } else {
      cluster = ClusterSpec::uniform(
          ndev, geti("group_size", ndev), std::int64_t{180} << 30,
          {getd("intra_bw", 900e9), getd("intra_lat", 3e-6)},
          {getd("inter_bw", 50e9), getd("inter_lat", 10e-6)},
          getd("throughput", 1.39e15));
    }
    auto result = compile(load_graph(graph_doc), cluster, c,
                          geti("pattern_match", 1) != 0);
    return dup_string(save_plan(result.plan));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

char* ref_random_inputs(const char* graph_doc, std::uint64_t seed,
                        int magnitude, std::int64_t* nbytes) {
  try {
    auto g = load_graph(graph_doc);
    return blob_out(random_integer_inputs(g, seed, magnitude), nbytes);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

char* ref_run_reference(const char* graph_doc, const char* inputs,
                        std::int64_t* nbytes) {
  try {
    auto g = load_graph(graph_doc);
    return blob_out(run_reference(g, decode(inputs)), nbytes);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// Runs the reference CPU plan executor `iters` times; reports mean seconds
// per run_plan call (plan parsing excluded) and returns the last outputs.
char* ref_run_plan(const char* plan_json, const char* inputs, int iters,
                   double* seconds_per_iter, std::int64_t* nbytes) {
  try {
    auto plan = load_plan(plan_json);
    auto in = decode(inputs);
    TensorMap out;
    if (iters < 1) iters = 1;
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < iters; ++i) out = run_plan(plan, in);
    auto t1 = std::chrono::steady_clock::now();
    if (seconds_per_iter) {
      *seconds_per_iter =
          std::chrono::duration<double>(t1 - t0).count() / iters;
    }
    return blob_out(out, nbytes);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// The reference's discrete-event simulator (simulate.cpp:102-318): returns
// {"report": to_json(), "timeline": timeline_json()} for a plan document.
char* ref_simulate(const char* plan_json) {
  try {
    auto rep = simulate(load_plan(plan_json));
    return dup_string("{\"report\":" + rep.to_json() + ",\"timeline\":" + rep.timeline_json() + "}");
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// Re-serializes a plan through the reference's own load_plan/save_plan.
char* ref_roundtrip_plan(const char* plan_json) {
  try {
    return dup_string(save_plan(load_plan(plan_json)));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// 0 = equal (within rel_tol), 1 = mismatch (message in ref_last_error()).
int ref_compare(const char* expected, const char* actual, double rel_tol) {
  auto r = compare_outputs(decode(expected), decode(actual), rel_tol);
  g_err = r.to_string();
  return r.ok ? 0 : 1;
}

}  // extern "C"
