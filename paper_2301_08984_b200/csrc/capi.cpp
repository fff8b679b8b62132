// extern "C" boundary (include/planc_b200.h): exceptions become return
// codes, mirroring the reference's error classes (util.hpp:17-29).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>

#include "../../include/planc_b200.h"
#include "nccl_api.hpp"
#include "runtime.hpp"

using namespace planc_b200;

struct planc_b200_exec {
  Executor* ex = nullptr;
};

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return PLANC_B200_OK;
  } catch (const SchemaError& e) {
    g_last_error = std::string("SchemaError: ") + e.what();
    return PLANC_B200_EUSAGE;
  } catch (const UsageError& e) {
    g_last_error = std::string("UsageError: ") + e.what();
    return PLANC_B200_EUSAGE;
  } catch (const InternalError& e) {
    g_last_error = std::string("InternalError: ") + e.what();
    return PLANC_B200_EINTERNAL;
  } catch (const std::exception& e) {
    g_last_error = std::string("CudaError: ") + e.what();
    return PLANC_B200_ECUDA;
  } catch (...) {
    g_last_error = "unknown error";
    return PLANC_B200_EINTERNAL;
  }
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

}  // namespace

// One translation of the open flags, shared by every entry point, so that
// every rank of a multi-process run lowers the same program from the same
// flags (no lowering switch is read from the environment).
ExecOptions exec_options(uint32_t flags) {
  ExecOptions opt;
  opt.use_graph = (flags & PLANC_B200_NO_GRAPH) == 0;
  opt.allow_tensor_cores = (flags & PLANC_B200_NO_TENSOR_CORES) == 0;
  opt.value_split_extension = (flags & PLANC_B200_STRICT_VALUE) == 0;
  if (flags & PLANC_B200_SERIAL_LANES) opt.streams_per_lane = 1;
  opt.fuse_epilogues = (flags & PLANC_B200_NO_FUSION) == 0;
  opt.fuse_act = (flags & PLANC_B200_FUSE_ACT) != 0;
  opt.group_gemms = (flags & PLANC_B200_NO_GROUPING) == 0;
  opt.alias_copies = (flags & PLANC_B200_NO_ALIAS) == 0;
  opt.alias_views = (flags & PLANC_B200_NO_ALIAS_VIEWS) == 0;
  opt.scatter_allreduce = (flags & PLANC_B200_NO_SCATTER) == 0;
  opt.reuse_memory = (flags & PLANC_B200_REUSE_MEMORY) != 0;
  opt.batch_boxes = (flags & PLANC_B200_BATCH) != 0;
  opt.gather_operands = (flags & PLANC_B200_NO_GATHER) == 0;
  opt.fuse_box_ew = (flags & PLANC_B200_NO_BOX_EW) == 0;
  opt.gather_cols = (flags & PLANC_B200_GATHER_COLS) != 0;
  return opt;
}

ProgramOptions describe_options(uint32_t flags) {
  const bool tc = (flags & PLANC_B200_NO_TENSOR_CORES) == 0;
  ProgramOptions po = program_options((flags & PLANC_B200_STRICT_VALUE) == 0,
                                      (flags & PLANC_B200_NO_FUSION) == 0 && tc);
  po.fuse_act = (flags & PLANC_B200_FUSE_ACT) != 0;
  po.group_gemms = (flags & PLANC_B200_NO_GROUPING) == 0 && tc;
  po.scatter_allreduce = (flags & PLANC_B200_NO_SCATTER) == 0 && tc;
  po.gather_operands = (flags & PLANC_B200_NO_GATHER) == 0 && tc;
  po.fuse_box_ew = (flags & PLANC_B200_NO_BOX_EW) == 0;
  po.gather_cols = (flags & PLANC_B200_GATHER_COLS) != 0;
  return po;
}

extern "C" {

const char* planc_b200_last_error(void) { return g_last_error.c_str(); }

const char* planc_b200_version(void) { return "planc_b200 0.1.0 sm_100a"; }

void planc_b200_free(void* p) { std::free(p); }

int planc_b200_open(const char* plan_json, const int* lane_gpu, int num_lane_gpu, uint32_t flags,
                    planc_b200_exec** out) {
  return guarded([&] {
    if (!plan_json || !out) throw UsageError("planc_b200_open: null argument");
    const ExecOptions opt = exec_options(flags);
    std::vector<int> lanes;
    for (int i = 0; lane_gpu && i < num_lane_gpu; ++i) lanes.push_back(lane_gpu[i]);
    auto* h = new planc_b200_exec;
    try {
      h->ex = new Executor(plan_json, lanes, opt);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int planc_b200_nccl_unique_id(unsigned char id_out[128]) {
  return guarded([&] {
    if (!id_out) throw UsageError("null argument");
    ncclUniqueId id;
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(id_out, id.internal, 128);
  });
}

int planc_b200_open_rank(const char* plan_json, int rank, int world, const int* lane_rank, int num_lanes,
                         int local_gpu, const unsigned char nccl_id[128], uint32_t flags, planc_b200_exec** out) {
  return guarded([&] {
    const bool peer = (flags & PLANC_B200_PEER_MEMORY) != 0;
    if (!plan_json || !out || !lane_rank || (!nccl_id && !peer)) throw UsageError("planc_b200_open_rank: null argument");
    if (num_lanes < 1) throw UsageError("planc_b200_open_rank: the plan's lanes need owners");
    const ExecOptions opt = exec_options(flags);
    RankConfig rc;
    rc.rank = rank;
    rc.world = world;
    rc.lane_rank.assign(lane_rank, lane_rank + num_lanes);
    rc.local_gpu = local_gpu;
    if (nccl_id) std::memcpy(rc.nccl_id, nccl_id, 128);
    rc.peer_memory = peer;
    auto* h = new planc_b200_exec;
    try {
      h->ex = new Executor(plan_json, {}, opt, &rc);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int planc_b200_describe_rank(const char* plan_json, const int* lane_rank, int num_lanes, uint32_t flags,
                             char** json_out) {
  return guarded([&] {
    if (!plan_json || !json_out || !lane_rank) throw UsageError("null argument");
    ProgramOptions po = describe_options(flags);
    ExecutionPlan plan = load_plan(plan_json);
    const std::vector<int> lr(lane_rank, lane_rank + num_lanes);
    if ((flags & PLANC_B200_PEER_MEMORY) == 0) {
      po.two_phase_allreduce = false;  // NCCL exchange steps: whole-buffer ncclAllReduce
      po.gather_operands = false;      // pieces on other ranks are not addressable
      po.fuse_box_ew = false;          // as in Executor (NCCL exchange steps)
      *json_out = dup(localize(build_program(plan, po), lr).describe_json());
      return;
    }
    // Peer-memory mode: the global program plus its cross-rank flag schedule.
    Program p = build_program(plan, po);
    PeerSync ps = peer_sync_schedule(p, lr);
    std::string js = p.describe_json();
    std::ostringstream os;
    os << ",\"peer_sync\":{\"slots\":[";
    for (std::size_t r = 0; r < ps.slots.size(); ++r) os << (r ? "," : "") << ps.slots[r];
    os << "],\"waits\":[";
    for (std::size_t i = 0; i < ps.waits.size(); ++i) {
      os << (i ? "," : "") << "[";
      for (std::size_t j = 0; j < ps.waits[i].size(); ++j) os << (j ? "," : "") << ps.waits[i][j];
      os << "]";
    }
    os << "],\"signals\":[";
    for (std::size_t i = 0; i < ps.signals.size(); ++i) {
      os << (i ? "," : "") << "[";
      for (std::size_t j = 0; j < ps.signals[i].size(); ++j)
        os << (j ? "," : "") << "[" << ps.signals[i][j].first << "," << ps.signals[i][j].second << "]";
      os << "]";
    }
    os << "]}}";
    js.pop_back();  // closing brace of the program object
    *json_out = dup(js + os.str());
  });
}

int64_t planc_b200_peer_blob_bytes(planc_b200_exec* h) {
  if (!h) return -1;
  return peer_blob_bytes(h->ex->program().num_lanes);
}

int planc_b200_peer_export(planc_b200_exec* h, unsigned char* blob, int64_t capacity) {
  return guarded([&] {
    if (!h || !blob) throw UsageError("planc_b200_peer_export: null argument");
    std::vector<unsigned char> b = h->ex->peer_export();
    if (capacity < static_cast<int64_t>(b.size())) throw UsageError("planc_b200_peer_export: blob capacity too small");
    std::memcpy(blob, b.data(), b.size());
  });
}

int planc_b200_peer_import(planc_b200_exec* h, const unsigned char* blobs, int64_t blob_bytes) {
  return guarded([&] {
    if (!h || !blobs) throw UsageError("planc_b200_peer_import: null argument");
    h->ex->peer_import(blobs, blob_bytes);
  });
}

void planc_b200_close(planc_b200_exec* h) {
  if (!h) return;
  delete h->ex;
  delete h;
}

int planc_b200_set_input(planc_b200_exec* h, int ptensor, const double* data, const int64_t* shape, int rank) {
  return guarded([&] {
    if (!h || !data || (rank > 0 && !shape)) throw UsageError("planc_b200_set_input: null argument");
    std::vector<std::int64_t> s(shape, shape + rank);
    h->ex->set_input(ptensor, data, s);
  });
}

int planc_b200_run(planc_b200_exec* h, int iters, double* ms_per_step) {
  return guarded([&] {
    if (!h) throw UsageError("planc_b200_run: null handle");
    double ms = h->ex->run(iters);
    if (ms_per_step) *ms_per_step = ms;
  });
}

int planc_b200_run_e2e(planc_b200_exec* h, int iters, double* ms_per_step, int64_t* h2d, int64_t* d2h) {
  return guarded([&] {
    if (!h) throw UsageError("planc_b200_run_e2e: null handle");
    std::int64_t a = 0, b = 0;
    double ms = h->ex->run_e2e(iters, &a, &b);
    if (ms_per_step) *ms_per_step = ms;
    if (h2d) *h2d = a;
    if (d2h) *d2h = b;
  });
}

int planc_b200_num_outputs(planc_b200_exec* h) { return h ? static_cast<int>(h->ex->output_ids().size()) : -1; }

int planc_b200_output_ids(planc_b200_exec* h, int* ids, int cap) {
  if (!h) return -1;
  auto v = h->ex->output_ids();
  for (int i = 0; i < cap && i < static_cast<int>(v.size()); ++i) ids[i] = v[i];
  return static_cast<int>(v.size());
}

int planc_b200_num_inputs(planc_b200_exec* h) {
  return h ? static_cast<int>(h->ex->input_ids().size()) : -1;
}

int planc_b200_input_ids(planc_b200_exec* h, int* ids, int cap) {
  if (!h) return -1;
  const std::vector<int> v = h->ex->input_ids();
  for (int i = 0; i < cap && i < static_cast<int>(v.size()); ++i) ids[i] = v[i];
  return static_cast<int>(v.size());
}

int planc_b200_ptensor_shape(planc_b200_exec* h, int ptensor, int64_t* shape, int cap, int* rank) {
  return guarded([&] {
    if (!h) throw UsageError("null handle");
    const PTensor& pt = h->ex->plan().pt(ptensor);
    if (rank) *rank = static_cast<int>(pt.shape.size());
    for (int i = 0; i < cap && i < static_cast<int>(pt.shape.size()); ++i) shape[i] = pt.shape[i];
  });
}

int planc_b200_get_output(planc_b200_exec* h, int ptensor, double* out, int64_t capacity) {
  return guarded([&] {
    if (!h || !out) throw UsageError("planc_b200_get_output: null argument");
    h->ex->get_output_into(ptensor, out, capacity);
  });
}

int64_t planc_b200_read_buffer(planc_b200_exec* h, int buffer, double* out, int64_t capacity) {
  std::int64_t n = -1;
  int rc = guarded([&] {
    if (!h) throw UsageError("null handle");
    auto v = h->ex->read_buffer(buffer);
    n = static_cast<std::int64_t>(v.size());
    if (out) std::memcpy(out, v.data(), sizeof(double) * std::min<std::int64_t>(n, capacity));
  });
  return rc == PLANC_B200_OK ? n : -1;
}

int planc_b200_get_stats(planc_b200_exec* h, planc_b200_stats* s) {
  return guarded([&] {
    if (!h || !s) throw UsageError("null argument");
    const Program& p = h->ex->program();
    const ExecutionPlan& pl = h->ex->plan();
    std::memset(s, 0, sizeof(*s));
    s->num_lanes = p.num_lanes;
    for (const auto& l : pl.lanes) s->num_tasks += static_cast<int>(l.tasks.size());
    s->num_instructions = static_cast<int>(p.instrs.size());
    s->kernels_per_step = h->ex->kernels_per_step();
    s->gemm_tc_per_step = h->ex->gemm_tc_launches();
    s->graph_captured = h->ex->graph_captured() ? 1 : 0;
    s->flops = p.total_flops;
    s->hbm_bytes = p.total_bytes;
    s->wire_bytes = p.total_wire_bytes;
    std::vector<double> gf(p.num_lanes, 0);
    for (const auto& in : p.instrs)
      if (in.kind == InstrKind::gemm) gf[in.lane] += in.flops;
    for (int l = 0; l < p.num_lanes; ++l) {
      s->max_lane_gemm_flops = std::max(s->max_lane_gemm_flops, gf[l]);
      s->max_lane_hbm_bytes = std::max(s->max_lane_hbm_bytes, p.lane_bytes[l]);
      s->max_lane_wire_bytes = std::max(s->max_lane_wire_bytes, p.lane_wire_bytes[l]);
      s->device_bytes += p.lane_arena_bytes[l];
    }
  });
}

int planc_b200_profile(planc_b200_exec* h, char** json_out) {
  return guarded([&] {
    if (!h || !json_out) throw UsageError("null argument");
    auto st = h->ex->profile();
    std::ostringstream os;
    os.precision(17);
    os << "[";
    for (std::size_t i = 0; i < st.size(); ++i) {
      os << (i ? "," : "") << "{\"kind\":\"" << st[i].kind << "\",\"launches\":" << st[i].launches
         << ",\"ms\":" << st[i].ms << ",\"flops\":" << st[i].flops << ",\"bytes\":" << st[i].bytes
         << ",\"wire_bytes\":" << st[i].wire_bytes << "}";
    }
    os << "]";
    *json_out = dup(os.str());
  });
}

int planc_b200_gemm_config(int64_t m, int64_t n, int64_t k, int ta, int tb, int a_bf16, int b_bf16, int c_bf16,
                           int* tensor_cores, int* tile_n) {
  GemmArgs a{};
  a.m = m;
  a.n = n;
  a.k = k;
  a.ta = ta != 0;
  a.tb = tb != 0;
  a.da = a_bf16 ? DT_BF16 : DT_F32;
  a.db = b_bf16 ? DT_BF16 : DT_F32;
  a.dc = c_bf16 ? DT_BF16 : DT_F32;
  const bool tc = gemm_sm100_eligible(a);
  if (tensor_cores) *tensor_cores = tc ? 1 : 0;
  if (tile_n) *tile_n = tc ? gemm_sm100_tile_n(a) : 0;
  return PLANC_B200_OK;
}

int planc_b200_gemm_schedule(int64_t m, int64_t n, int64_t k, int ta, int tb, int c_bf16, int sms, int group,
                             int* tile_n, int* grid, int* dp_tiles, int* sk_ctas, int* splits, int* half_items,
                             int* variant, int64_t* ws_bytes) {
  return guarded([&] {
    if (sms <= 0) throw UsageError("sms must be positive");
    if (group < 1 || group > kMaxGemmGroup) throw UsageError("group must be in [1, 8]");
    GemmArgs a{};
    a.group = group;
    a.m = m;
    a.n = n;
    a.k = k;
    a.ta = ta != 0;
    a.tb = tb != 0;
    a.da = DT_BF16;
    a.db = DT_BF16;
    a.dc = c_bf16 ? DT_BF16 : DT_F32;
    if (!gemm_sm100_eligible(a)) throw UsageError("shape does not take the tensor-core path");
    GemmSchedule sc = gemm_sm100_schedule(a, sms);
    if (tile_n) *tile_n = sc.bn;
    if (grid) *grid = sc.grid;
    if (dp_tiles) *dp_tiles = sc.dp_tiles;
    if (sk_ctas) *sk_ctas = sc.sk_ctas;
    if (splits) *splits = sc.splits;
    if (half_items) *half_items = sc.half_items;
    if (variant) *variant = sc.occ;
    if (ws_bytes) *ws_bytes = sc.ws_bytes;
  });
}

int planc_b200_timeline(planc_b200_exec* h, char** json_out) {
  return guarded([&] {
    if (!h || !json_out) throw UsageError("null argument");
    *json_out = dup(h->ex->timeline_json());
  });
}

int planc_b200_describe(const char* plan_json, uint32_t flags, char** json_out) {
  return guarded([&] {
    if (!plan_json || !json_out) throw UsageError("null argument");
    ProgramOptions po = describe_options(flags);
    ExecutionPlan plan = load_plan(plan_json);
    Program p = build_program(plan, po);
    std::string js = p.describe_json();
    if (flags & PLANC_B200_REUSE_MEMORY) {
      // The timed-mode memory plan with every lane in this process, 4
      // streams per lane, no same-GPU aliases.
      std::vector<int> lane(p.instrs.size());
      for (const auto& in : p.instrs) lane[in.id] = in.lane;
      const std::vector<int> streams = assign_streams(p, lane, 4);
      MemoryPlan mp = plan_memory(p, plan, lane, streams, 4, {});
      std::ostringstream os;
      os << ",\"memory_plan\":{\"bytes_before\":" << mp.bytes_before << ",\"bytes_after\":" << mp.bytes_after
         << ",\"reused\":" << mp.reused << ",\"streams\":[";
      for (std::size_t i = 0; i < streams.size(); ++i) os << (i ? "," : "") << streams[i];
      os << "],\"offset\":[";
      for (std::size_t i = 0; i < mp.offset.size(); ++i) os << (i ? "," : "") << mp.offset[i];
      os << "],\"lane_bytes\":[";
      for (std::size_t i = 0; i < mp.lane_bytes.size(); ++i) os << (i ? "," : "") << mp.lane_bytes[i];
      os << "],\"overwritten\":[";
      for (std::size_t i = 0; i < mp.overwritten.size(); ++i) os << (i ? "," : "") << (mp.overwritten[i] ? 1 : 0);
      os << "]}}";
      js.pop_back();
      js += os.str();
    }
    *json_out = dup(js);
  });
}

}  // extern "C"
