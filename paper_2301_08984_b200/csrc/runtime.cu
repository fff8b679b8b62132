#include "runtime.hpp"

#include <cuda_bf16.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <set>
#include <sstream>
#include <stdexcept>
#include <thread>

#include "nccl_api.hpp"

namespace planc_b200 {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

int dt_of(DType d) { return d == DType::bf16 ? DT_BF16 : d == DType::i32 ? DT_I32 : DT_F32; }

std::uint16_t f32_to_bf16_rne(float f) {
  std::uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<std::uint16_t>((u >> 16) | 0x40);  // NaN
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<std::uint16_t>(u >> 16);
}

float bf16_to_f32(std::uint16_t h) {
  std::uint32_t u = static_cast<std::uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

// Host-side value of element i of a device-typed buffer.
double host_elem(const std::vector<char>& raw, DType d, std::int64_t i) {
  switch (d) {
    case DType::f32: {
      float f;
      std::memcpy(&f, raw.data() + 4 * i, 4);
      return f;
    }
    case DType::bf16: {
      std::uint16_t h;
      std::memcpy(&h, raw.data() + 2 * i, 2);
      return bf16_to_f32(h);
    }
    case DType::i32: {
      std::int32_t v;
      std::memcpy(&v, raw.data() + 4 * i, 4);
      return v;
    }
  }
  return 0;
}

void put_elem(char* dst, DType d, std::int64_t i, double v) {
  switch (d) {
    case DType::f32: {
      float f = static_cast<float>(v);
      std::memcpy(dst + 4 * i, &f, 4);
      break;
    }
    case DType::bf16: {
      std::uint16_t h = f32_to_bf16_rne(static_cast<float>(v));
      std::memcpy(dst + 2 * i, &h, 2);
      break;
    }
    case DType::i32: {
      std::int32_t x = static_cast<std::int32_t>(v);
      std::memcpy(dst + 4 * i, &x, 4);
      break;
    }
  }
}

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) ck(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

// Host-side parallel loop over [0, n) in contiguous chunks (the float64 <->
// device-type conversions of the drop-in TensorMap path): one chunk per
// hardware thread, inline below `min_work` items.
template <class F>
void parallel_for(std::int64_t n, std::int64_t work_per_item, F&& f) {
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  const std::int64_t T = std::min<std::int64_t>(hw, n);
  if (T <= 1 || n * work_per_item < (std::int64_t(1) << 16)) {
    f(std::int64_t(0), n);
    return;
  }
  std::vector<std::thread> th;
  const std::int64_t chunk = (n + T - 1) / T;
  for (std::int64_t t = 0; t < T; ++t) {
    const std::int64_t lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo < hi) th.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  for (auto& x : th) x.join();
}

inline double load_elem(const char* base, DType d, std::int64_t i) {
  switch (d) {
    case DType::f32: {
      float f;
      std::memcpy(&f, base + 4 * i, 4);
      return f;
    }
    case DType::bf16: {
      std::uint16_t h;
      std::memcpy(&h, base + 2 * i, 2);
      return bf16_to_f32(h);
    }
    case DType::i32: {
      std::int32_t v;
      std::memcpy(&v, base + 4 * i, 4);
      return v;
    }
  }
  return 0;
}

}  // namespace

namespace {
bool tc_fusable(const Instr& g, DType a, DType b, DType c) {
  GemmArgs x{};
  x.m = g.m;
  x.n = g.n;
  x.k = g.k;
  x.ta = g.ta;
  x.tb = g.tb;
  x.da = dt_of(a);
  x.db = dt_of(b);
  x.dc = dt_of(c);
  return c == DType::bf16 && gemm_sm100_eligible(x);
}
bool tc_groupable(const Instr& g, DType a, DType b, DType c) {
  static_assert(kMaxGemmGroupInstr == kMaxGemmGroup, "group size limits differ");
  // Grouped launches and the reduce-scatter epilogue are bf16-operand
  // variants (fp32 GEMMs take the single-launch 3xTF32 kernel).
  if (a != DType::bf16 || b != DType::bf16) return false;
  GemmArgs x{};
  x.m = g.m;
  x.n = g.n;
  x.k = g.k;
  x.ta = g.ta;
  x.tb = g.tb;
  x.da = dt_of(a);
  x.db = dt_of(b);
  x.dc = dt_of(c);
  return gemm_sm100_eligible(x);
}
}  // namespace

ProgramOptions program_options(bool value_split_extension, bool fuse_epilogues) {
  ProgramOptions po;
  po.value_split_extension = value_split_extension;
  po.fuse_epilogues = fuse_epilogues;
  po.gemm_fusable = &tc_fusable;
  po.gemm_groupable = &tc_groupable;
  // A/B knob, read once per process (every rank of a run shares its env):
  // PLANC_B200_FUSE_MIN_TILES=0 fuses single-wave GEMMs too.
  static const int min_tiles = [] {
    const char* e = std::getenv("PLANC_B200_FUSE_MIN_TILES");
    return e ? std::atoi(e) : 148;
  }();
  po.fuse_min_tiles = min_tiles;
  return po;
}

Executor::Executor(const std::string& plan_json, const std::vector<int>& lane_gpu, const ExecOptions& opt,
                   const RankConfig* rank)
    : opt_(opt) {
  plan_ = load_plan(plan_json);
  ProgramOptions po = program_options(opt.value_split_extension, opt.fuse_epilogues && opt.allow_tensor_cores);
  po.group_gemms = opt.group_gemms && opt.allow_tensor_cores;
  po.fuse_act = opt.fuse_act;
  if (const char* e = std::getenv("PLANC_B200_SYNC_EDGES")) po.honor_sync_edges = e[0] != '0';  // A/B only
  // NCCL exchange steps lower whole-buffer all-reduce groups to
  // ncclAllReduce; every other mode runs them as two box phases.
  po.two_phase_allreduce = !(rank && !rank->peer_memory);
  // Gathered operands read pieces in place: not across NCCL ranks.
  po.gather_operands = opt.gather_operands && opt.allow_tensor_cores && !(rank && !rank->peer_memory);
  po.gather_cols = opt.gather_cols;
  // Box -> elementwise fusion: single-process and peer-memory modes
  // (PLANC_B200_BOX_EW=0 for A/B).
  static const bool box_ew_env = [] {
    const char* e = std::getenv("PLANC_B200_BOX_EW");
    return !(e && e[0] == '0');
  }();
  po.fuse_box_ew = opt.fuse_box_ew && box_ew_env && !(rank && !rank->peer_memory);
  // The scatter epilogue pays when the slices cross GPUs (the transfer rides
  // in the GEMM); with every lane on one GPU it only trades TMA stores for
  // plain ones (measured ~2 % slower, profiles/r01/ab_scatter.jsonl).
  bool multi_gpu = rank != nullptr;
  for (std::size_t i = 1; i < lane_gpu.size(); ++i) multi_gpu = multi_gpu || lane_gpu[i] != lane_gpu[0];
  po.scatter_allreduce = opt.allow_tensor_cores && opt.scatter_allreduce && multi_gpu;
  prog_ = build_program(plan_, po);
  if (rank) {
    rank_mode_ = true;
    rc_ = *rank;
    if (rc_.world < 1 || rc_.rank < 0 || rc_.rank >= rc_.world) throw UsageError("bad rank / world");
    for (int r : rc_.lane_rank) {
      if (r < 0 || r >= rc_.world) throw UsageError("lane_rank entry outside [0, world)");
    }
    if (rc_.peer_memory) {
      if (rc_.world > kPeerMaxRanks) throw UsageError("peer-memory mode supports at most 64 ranks");
      peer_ = true;
      psync_ = peer_sync_schedule(prog_, rc_.lane_rank);
    } else {
      prog_ = localize(prog_, rc_.lane_rank);
    }
  }
  int ndev = 0;
  ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  lanes_.resize(prog_.num_lanes);
  owned_.assign(prog_.num_lanes, true);
  std::set<int> gset;
  for (int l = 0; l < prog_.num_lanes; ++l) {
    int g = rank_mode_ ? rc_.local_gpu : lane_gpu.empty() ? 0 : lane_gpu[l % lane_gpu.size()];
    if (g < 0 || g >= ndev) throw UsageError("lane " + std::to_string(l) + " mapped to missing GPU " + std::to_string(g));
    lanes_[l].gpu = g;
    if (rank_mode_) owned_[l] = rc_.lane_rank[l] == rc_.rank;
    if (owned_[l]) gset.insert(g);
  }
  if (gset.empty()) throw UsageError("this rank owns no plan lane");
  gpus_.assign(gset.begin(), gset.end());
  // Which lane's streams run each instruction in this process.
  exec_lane_.assign(prog_.instrs.size(), -1);
  for (const auto& in : prog_.instrs) {
    if (in.kind != InstrKind::xfer) {
      if (owned_[in.lane]) exec_lane_[in.id] = in.lane;
      continue;
    }
    for (const auto& x : in.xfers) {
      if (in.allreduce ? owned_[x.src_lane] : owned_[x.src_lane] != owned_[x.dst_lane]) {
        exec_lane_[in.id] = owned_[x.src_lane] ? x.src_lane : x.dst_lane;
        break;
      }
    }
  }
  // Stream of each instruction within its lane: continue the stream of the
  // most recent dependency that ended a stream's chain, else take the least
  // recently used stream. Only data dependencies (and sync edges) then order
  // a lane's work, via events between streams.
  int nstreams = 1;
  {
    int want = opt_.streams_per_lane;
    if (const char* e = std::getenv("PLANC_B200_STREAMS")) {
      if (want > 1) want = std::atoi(e);  // A/B of the stream count (SERIAL_LANES keeps 1)
    }
    nstreams = std::max(1, std::min(want, kLaneStreams));
    exec_stream_ = assign_streams(prog_, exec_lane_, nstreams);
  }
  if (rank_mode_ && !peer_) {
    DeviceGuard dg(rc_.local_gpu);
    ncclUniqueId id;
    std::memcpy(id.internal, rc_.nccl_id, sizeof(id.internal));
    ncclComm_t c = nullptr;
    nccl_check(nccl().comm_init_rank(&c, rc_.world, id, rc_.rank), "ncclCommInitRank");
    comm_ = c;
  }
  // Lanes on different GPUs read each other's buffers through NVLink peer
  // mappings inside the box kernels.
  for (int a : gpus_) {
    DeviceGuard dg(a);
    for (int b : gpus_) {
      if (a == b) continue;
      int can = 0;
      ck(cudaDeviceCanAccessPeer(&can, a, b), "cudaDeviceCanAccessPeer");
      if (!can) throw UsageError("GPU " + std::to_string(a) + " cannot map GPU " + std::to_string(b));
      cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else ck(e, "cudaDeviceEnablePeerAccess");
    }
  }
  irt_.resize(prog_.instrs.size());
  if (!peer_) plan_aliases();  // (before the memory plan: an alias extends its source's lifetime)
  if (opt_.reuse_memory) {
    // Timed mode honouring the plan's frees: released bytes are reused
    // within the step (single process: every reader's stream is ours).
    if (rank_mode_) throw UsageError("REUSE_MEMORY needs the single-process executor");
    MemoryPlan mp = plan_memory(prog_, plan_, exec_lane_, exec_stream_, nstreams, alias_);
    for (std::size_t b = 0; b < prog_.buffers.size(); ++b) prog_.buffers[b].offset = mp.offset[b];
    prog_.lane_arena_bytes = mp.lane_bytes;
    overwritten_ = mp.overwritten;
  }
  for (int l = 0; l < prog_.num_lanes; ++l) {
    if (!owned_[l]) continue;
    DeviceGuard dg(lanes_[l].gpu);
    std::int64_t bytes = std::max<std::int64_t>(prog_.lane_arena_bytes[l], 256);
    ck(cudaMalloc(&lanes_[l].arena, bytes), "cudaMalloc(arena)");
    for (auto& s : lanes_[l].stream) ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  }
  for (int l = 0; l < prog_.num_lanes; ++l) {
    if (owned_[l]) {
      first_lane_ = l;
      break;
    }
  }
  {
    DeviceGuard dg(lanes_[first_lane_].gpu);
    ck(cudaStreamCreateWithFlags(&origin_, cudaStreamNonBlocking), "origin stream");
    ck(cudaEventCreateWithFlags(&ev_begin_, cudaEventDisableTiming), "event");
    ck(cudaEventCreate(&ev_end_), "event");
  }
  for (int l = 0; l < prog_.num_lanes; ++l) {
    DeviceGuard dg(lanes_[l].gpu);
    for (int s = 0; s < kLaneStreams; ++s) {
      cudaEvent_t e = nullptr;
      if (owned_[l]) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      lane_join_.push_back(e);
    }
  }
  // Element types must agree across an elementwise op's operands; fused
  // attention shapes the kernel supports (bf16, head_dim 64 / 128, seq % 128).
  for (const auto& in : prog_.instrs) {
    if (in.kind == InstrKind::attention) {
      const int dt = dt_of(prog_.buffers[in.out_bufs[0]].dtype);
      for (int b : in.in_bufs)
        if (prog_.buffers[b].dtype != prog_.buffers[in.out_bufs[0]].dtype)
          throw UsageError("attention " + plan_.ops[in.op].id + " mixes element sizes");
      if (const char* why = attention_unsupported(in.att_rows, in.att_cols, in.att_seq, in.att_dh, dt))
        throw UsageError("attention " + plan_.ops[in.op].id + ": " + why);
    }
    if (in.kind == InstrKind::ew || in.kind == InstrKind::rowwise) {
      DType d = prog_.buffers[in.out_bufs[0]].dtype;
      if (in.kind == InstrKind::rowwise && d == DType::i32) {
        throw UsageError("op " + plan_.ops[in.op].id + ": row-wise operators need fp32 or bf16 tensors");
      }
      for (int b : in.in_bufs) {
        if (prog_.buffers[b].dtype != d) {
          throw UsageError("elementwise op " + plan_.ops[in.op].id + " mixes element sizes");
        }
      }
    }
  }
  // Events for producer -> consumer edges that cross streams.
  irt_.resize(prog_.instrs.size());
  for (const auto& in : prog_.instrs) {
    if (exec_lane_[in.id] < 0) continue;
    for (int d : in.deps) {
      const Instr& p = prog_.instrs[d];
      if (exec_lane_[d] < 0) continue;  // ordered by the exchange step instead
      (void)p;
      if ((exec_lane_[d] != exec_lane_[in.id] || exec_stream_[d] != exec_stream_[in.id]) && !irt_[d].done) {
        DeviceGuard dg(lanes_[exec_lane_[d]].gpu);
        ck(cudaEventCreateWithFlags(&irt_[d].done, cudaEventDisableTiming), "event");
      }
    }
    if (in.kind == InstrKind::emb_grad) {
      DeviceGuard dg(lanes_[in.lane].gpu);
      ck(cudaMalloc(&irt_[in.id].scratch, emb_grad_scratch_bytes(in.n_idx, in.h)), "cudaMalloc(scratch)");
    }
    if (in.kind == InstrKind::attention && in.att_grad) {
      DeviceGuard dg(lanes_[in.lane].gpu);
      ck(cudaMalloc(&irt_[in.id].scratch, attention_grad_scratch_bytes(in.att_rows, in.att_cols, in.att_dh)),
         "cudaMalloc(attention statistics)");
    }
    if (in.kind == InstrKind::reduce) {
      const std::int64_t b =
          reduce_scratch_bytes(in.outer, in.axis_len, in.inner, dt_of(prog_.buffers[in.out_bufs[0]].dtype));
      if (b > 0) {
        DeviceGuard dg(lanes_[in.lane].gpu);
        ck(cudaMalloc(&irt_[in.id].scratch, b), "cudaMalloc(reduce scratch)");
      }
    }
  }
  if (peer_) {
    // This rank's flag block: epoch, step barrier slots, ready slots.
    DeviceGuard dg(rc_.local_gpu);
    const std::size_t words = kFlagReady + static_cast<std::size_t>(psync_.slots[rc_.rank]) + 1;
    ck(cudaMalloc(&flags_, words * sizeof(unsigned)), "cudaMalloc(peer flags)");
    ck(cudaMemset(flags_, 0, words * sizeof(unsigned)), "memset(peer flags)");
    ck(cudaHostAlloc(reinterpret_cast<void**>(&peer_err_), 8 * sizeof(unsigned), cudaHostAllocMapped), "cudaHostAlloc");
    std::memset(peer_err_, 0, 8 * sizeof(unsigned));
    double secs = 60.0;
    if (const char* t = std::getenv("PLANC_B200_PEER_TIMEOUT_S")) secs = std::max(0.1, std::atof(t));
    peer_timeout_ns_ = static_cast<unsigned long long>(secs * 1e9);
    lane_mapped_.assign(prog_.num_lanes, false);
    // Box tables need every rank's arena: built by peer_import.
  } else {
    build_box_tables();
    plan_box_batches();
  }
  kernels_per_step_ = 0;
  for (const auto& b : batches_) kernels_per_step_ += static_cast<int>(b.launches.size());
  for (const auto& in : prog_.instrs) {
    if (exec_lane_[in.id] < 0) continue;
    if (peer_) {
      kernels_per_step_ += static_cast<int>((psync_.waits[in.id].size() + kMaxPeerFlags - 1) / kMaxPeerFlags);
      kernels_per_step_ += static_cast<int>((psync_.signals[in.id].size() + kMaxPeerFlags - 1) / kMaxPeerFlags);
    }
    switch (in.kind) {
      case InstrKind::nop: break;
      case InstrKind::box:  // peer: at import; batched: counted with the batch
        if (batch_of_.empty() || batch_of_[in.id] < 0) kernels_per_step_ += static_cast<int>(irt_[in.id].box.size());
        break;
      case InstrKind::emb_grad: kernels_per_step_ += in.n_idx > 0 ? 2 : 1; break;
      case InstrKind::attention:
        kernels_per_step_ += in.att_grad ? 1 + (in.att_out[0] >= 0 ? 1 : 0) + (in.att_out[1] >= 0 || in.att_out[2] >= 0 ? 1 : 0) : 1;
        break;
      case InstrKind::reduce:
        kernels_per_step_ += reduce_launches(in.outer, in.axis_len, in.inner, dt_of(prog_.buffers[in.out_bufs[0]].dtype));
        break;
      case InstrKind::ew:
        if (!irt_[in.id].box.empty()) {
          if (batch_of_.empty() || batch_of_[in.id] < 0) kernels_per_step_ += static_cast<int>(irt_[in.id].box.size());
        } else {
          kernels_per_step_ += 1 + (in.count % 8 != 0 ? 1 : 0);
        }
        break;
      default: kernels_per_step_ += 1;
    }
    if (in.kind == InstrKind::gemm) {
      GemmArgs a{};
      a.m = in.m;
      a.n = in.n;
      a.k = in.k;
      a.ta = in.ta;
      a.tb = in.tb;
      a.da = dt_of(prog_.buffers[in.in_bufs[0]].dtype);
      a.db = dt_of(prog_.buffers[in.in_bufs[1]].dtype);
      a.dc = dt_of(prog_.buffers[in.out_bufs[0]].dtype);
      a.group = in.group;
      a.scatter = in.scatter;
      a.scatter_rows = in.scatter_rows;
      a.allow_streamk = gemm_streamk_ok(exec_lane_[in.id]);
    a.gpu_share = gpu_share(exec_lane_[in.id]);
      a.gpu_share = gpu_share(exec_lane_[in.id]);
      if (opt_.allow_tensor_cores && gemm_sm100_eligible(a)) {
        ++gemm_tc_per_step_;
        kernels_per_step_ += gemm_sm100_launches(a) - 1;  // split-K reduce kernel
        LaneRt& lr = lanes_[exec_lane_[in.id]];
        DeviceGuard dg(lr.gpu);
        std::int64_t& need = lr.gemm_ws_bytes[exec_stream_[in.id]];
        need = std::max(need, gemm_sm100_workspace_bytes(a));
      }
    }
  }
  for (auto& lr : lanes_) {
    for (int k = 0; k < kLaneStreams; ++k) {
      if (lr.gemm_ws_bytes[k] == 0) continue;
      DeviceGuard dg(lr.gpu);
      ck(cudaMalloc(&lr.gemm_ws[k], lr.gemm_ws_bytes[k]), "cudaMalloc(gemm workspace)");
      ck(cudaMemset(lr.gemm_ws[k], 0, lr.gemm_ws_bytes[k]), "memset(gemm workspace)");  // stream-K counters
    }
  }
  if (!peer_) build_gather_maps();  // peer mode: at import (pieces may live on other ranks)
}

Executor::~Executor() {
  for (std::size_t i = 0; i < lanes_.size(); ++i) {
    auto& l = lanes_[i];
    cudaSetDevice(l.gpu);
    for (auto& s : l.stream)
      if (s) cudaStreamDestroy(s);
    for (void* w : l.gemm_ws)
      if (w) cudaFree(w);
    if (l.arena && !(i < lane_mapped_.size() && lane_mapped_[i])) cudaFree(l.arena);
  }
  for (void* p : ipc_mapped_) cudaIpcCloseMemHandle(p);
  if (flags_) cudaFree(flags_);
  if (peer_err_) cudaFreeHost(peer_err_);
  for (auto& r : irt_) {
    if (r.done) cudaEventDestroy(r.done);
    if (r.scratch) cudaFree(r.scratch);
  }
  for (void* p : table_allocs_) cudaFree(p);
  for (auto e : lane_join_)
    if (e) cudaEventDestroy(e);
  if (comm_) nccl().comm_destroy(static_cast<ncclComm_t>(comm_));
  if (host_stage_) cudaFreeHost(host_stage_);
  for (void* p : pinned_in_) cudaFreeHost(p);
  for (void* p : pinned_out_) cudaFreeHost(p);
  for (int k = 0; k < 2; ++k) {
    for (void* p : e2e_stage_in_[k]) cudaFree(p);
    for (void* p : e2e_stage_out_[k]) cudaFree(p);
    for (cudaEvent_t e : {ev_h2d_[k], ev_in_free_[k], ev_out_ready_[k], ev_out_free_[k]})
      if (e) cudaEventDestroy(e);
  }
  if (h2d_stream_) cudaStreamDestroy(h2d_stream_);
  if (d2h_stream_) cudaStreamDestroy(d2h_stream_);
  if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
  if (graph_) cudaGraphDestroy(graph_);
  for (auto& b : batches_)
    if (b.done) cudaEventDestroy(b.done);
  for (auto e : batch_join_) cudaEventDestroy(e);
  for (auto& kv : batch_streams_)
    for (auto st : kv.second) cudaStreamDestroy(st);
  if (ev_begin_) cudaEventDestroy(ev_begin_);
  if (ev_end_) cudaEventDestroy(ev_end_);
  if (origin_) cudaStreamDestroy(origin_);
}

int Executor::gpu_share(int lane) const {
  int sharing = 0;
  for (int l = 0; l < prog_.num_lanes; ++l)
    if (owned_[l] && lanes_[l].gpu == lanes_[lane].gpu) ++sharing;
  return std::max(sharing, 1);
}

bool Executor::gemm_streamk_ok(int lane) const { return gpu_share(lane) == 1; }

bool Executor::released(int b) const {
  while (!alias_.empty() && alias_[b] >= 0) b = alias_[b];
  return !overwritten_.empty() && overwritten_[b];
}

void* Executor::buf_ptr(int b) const {
  std::int64_t off = 0;  // bytes into the aliased source (a view of a sub-range)
  while (!alias_.empty() && alias_[b] >= 0) {
    off += alias_off_[b];
    b = alias_[b];
  }
  const BufferDesc& d = prog_.buffers[b];
  return lanes_[d.lane].arena + d.offset + off;
}

// A box instruction that copies one whole buffer — or one contiguous
// sub-range of it (a split along the outermost dimension) — into another
// buffer of the same dense layout (a recv whose send lane shares the GPU, an
// identity op, C5's DAP splits) moves no data when both lanes' arenas sit in
// the same HBM: the output becomes an alias of the source range (single
// assignment: neither is rewritten within the step; sub-ranges start on a
// 256-byte boundary, as arena buffers do) and the instruction launches
// nothing — its events still order its consumers after its producers.
// Across GPUs or ranks the copy stays.
void Executor::plan_aliases() {
  alias_.assign(prog_.buffers.size(), -1);
  alias_off_.assign(prog_.buffers.size(), 0);
  if (rank_mode_ || !opt_.alias_copies) return;
  static const bool views_env = [] {  // A/B: PLANC_B200_ALIAS_VIEWS=0 keeps sub-range copies
    const char* e = std::getenv("PLANC_B200_ALIAS_VIEWS");
    return !(e && e[0] == '0');
  }();
  const bool views = opt_.alias_views && views_env;
  std::vector<int> writers(prog_.buffers.size(), 0);
  for (const auto& in : prog_.instrs)
    for (int b : in.out_bufs) ++writers[b];
  for (const auto& in : prog_.instrs) {
    if (in.kind != InstrKind::box || exec_lane_[in.id] < 0 || in.out_bufs.size() != 1 || in.cells.size() != 1) continue;
    const Cell& c = in.cells[0];
    if (c.terms.size() != 1 || c.terms[0].add || c.terms[0].fold >= 0 || c.rank != 1 || c.dst_offset != 0 ||
        c.dst_strides[0] != 1 || c.terms[0].strides[0] != 1)
      continue;
    const BufferDesc& ob = prog_.buffers[in.out_bufs[0]];
    const BufferDesc& sb = prog_.buffers[c.terms[0].buffer];
    const std::int64_t off = c.terms[0].offset;
    const std::int64_t off_bytes = off * static_cast<std::int64_t>(dtype_size(sb.dtype));
    if (ob.graph_input || writers[ob.id] != 1 || ob.dtype != sb.dtype || c.elems() != ob.elems || off < 0 ||
        off + ob.elems > sb.elems || off_bytes % 256 != 0 || (off != 0 && !views))
      continue;
    if (!owned_[sb.lane] || lanes_[ob.lane].gpu != lanes_[sb.lane].gpu) continue;
    alias_[ob.id] = sb.id;
    alias_off_[ob.id] = off_bytes;
    irt_[in.id].aliased = true;
  }
}

cudaStream_t Executor::stream_of(const Instr& in) const {
  return lanes_[exec_lane_[in.id]].stream[exec_stream_[in.id]];
}

// One exchange step: this rank's sends and receives of the step, grouped so
// NCCL posts them together (every rank walks the same step sequence).
void Executor::launch_xfer(const Instr& in, cudaStream_t s) {
  const NcclApi& api = nccl();
  ncclComm_t comm = static_cast<ncclComm_t>(comm_);
  if (in.allreduce) {
    // One member per rank; this rank's member sums every rank's partial.
    for (const auto& x : in.xfers) {
      if (!owned_[x.src_lane]) continue;
      const BufferDesc& b = prog_.buffers[x.dst];
      ncclDataType_t dt = b.dtype == DType::bf16 ? ncclBfloat16 : b.dtype == DType::i32 ? ncclInt32 : ncclFloat32;
      nccl_check(api.all_reduce(buf_ptr(x.src), buf_ptr(x.dst), static_cast<std::size_t>(b.elems), dt, ncclSum, comm, s),
                 "ncclAllReduce");
    }
    return;
  }
  nccl_check(api.group_start(), "ncclGroupStart");
  for (const auto& x : in.xfers) {
    bool src_here = owned_[x.src_lane], dst_here = owned_[x.dst_lane];
    if (src_here && !dst_here) {
      nccl_check(api.send(buf_ptr(x.src), static_cast<std::size_t>(x.bytes), ncclUint8, rc_.lane_rank[x.dst_lane], comm,
                          s),
                 "ncclSend");
    } else if (dst_here && !src_here) {
      nccl_check(api.recv(buf_ptr(x.dst), static_cast<std::size_t>(x.bytes), ncclUint8, rc_.lane_rank[x.src_lane], comm,
                          s),
                 "ncclRecv");
    }
  }
  nccl_check(api.group_end(), "ncclGroupEnd");
}

// ---- peer-memory rank mode -----------------------------------------------

std::vector<unsigned char> Executor::peer_export() const {
  if (!peer_) throw UsageError("peer_export: executor was not opened in peer-memory rank mode");
  std::vector<unsigned char> blob(static_cast<std::size_t>(peer_blob_bytes(prog_.num_lanes)), 0);
  const std::uint32_t hdr[5] = {0x50423250u /* "PB2P" */, 1u, static_cast<std::uint32_t>(rc_.rank),
                                static_cast<std::uint32_t>(rc_.world), static_cast<std::uint32_t>(prog_.num_lanes)};
  std::memcpy(blob.data(), hdr, sizeof(hdr));
  const std::size_t hs = sizeof(cudaIpcMemHandle_t);
  DeviceGuard dg(rc_.local_gpu);
  for (int l = 0; l < prog_.num_lanes; ++l) {
    if (!owned_[l]) continue;
    cudaIpcMemHandle_t h;
    ck(cudaIpcGetMemHandle(&h, lanes_[l].arena), "cudaIpcGetMemHandle(arena)");
    std::memcpy(blob.data() + kPeerBlobHeader + hs * l, &h, hs);
  }
  cudaIpcMemHandle_t h;
  ck(cudaIpcGetMemHandle(&h, flags_), "cudaIpcGetMemHandle(flags)");
  std::memcpy(blob.data() + kPeerBlobHeader + hs * prog_.num_lanes, &h, hs);
  return blob;
}

void Executor::peer_import(const unsigned char* blobs, std::int64_t blob_bytes) {
  if (!peer_) throw UsageError("peer_import: executor was not opened in peer-memory rank mode");
  if (peer_ready_) throw UsageError("peer_import: peers already mapped");
  if (blob_bytes != peer_blob_bytes(prog_.num_lanes)) throw UsageError("peer_import: blob size mismatch");
  const std::size_t hs = sizeof(cudaIpcMemHandle_t);
  DeviceGuard dg(rc_.local_gpu);
  peer_flags_.assign(rc_.world, nullptr);
  peer_flags_[rc_.rank] = flags_;
  for (int r = 0; r < rc_.world; ++r) {
    const unsigned char* b = blobs + blob_bytes * r;
    std::uint32_t hdr[5];
    std::memcpy(hdr, b, sizeof(hdr));
    if (hdr[0] != 0x50423250u || hdr[1] != 1u || hdr[2] != static_cast<std::uint32_t>(r) ||
        hdr[3] != static_cast<std::uint32_t>(rc_.world) || hdr[4] != static_cast<std::uint32_t>(prog_.num_lanes)) {
      throw UsageError("peer_import: blob " + std::to_string(r) + " is not rank " + std::to_string(r) +
                       "'s export of this plan");
    }
    if (r == rc_.rank) continue;
    for (int l = 0; l < prog_.num_lanes; ++l) {
      if (rc_.lane_rank[l] != r) continue;
      cudaIpcMemHandle_t h;
      std::memcpy(&h, b + kPeerBlobHeader + hs * l, hs);
      void* p = nullptr;
      ck(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle(arena)");
      ipc_mapped_.push_back(p);
      lanes_[l].arena = static_cast<char*>(p);
      lane_mapped_[l] = true;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, b + kPeerBlobHeader + hs * prog_.num_lanes, hs);
    void* p = nullptr;
    ck(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle(flags)");
    ipc_mapped_.push_back(p);
    peer_flags_[r] = static_cast<unsigned*>(p);
  }
  peer_ready_ = true;
  build_box_tables();
  build_gather_maps();
  for (const auto& in : prog_.instrs)
    if (in.kind == InstrKind::box && exec_lane_[in.id] >= 0) kernels_per_step_ += static_cast<int>(irt_[in.id].box.size());
  kernels_per_step_ += 1 + (rc_.world > 1 ? 1 : 0);  // epoch + step barrier
}

void Executor::peer_check_ready() const {
  if (peer_ && !peer_ready_) {
    throw UsageError("peer-memory rank mode: exchange the ranks' peer_export blobs with peer_import first");
  }
}

void Executor::peer_flags(const std::vector<unsigned*>& sig, const std::vector<const unsigned*>& wait, unsigned code,
                          cudaStream_t s) {
  std::size_t is = 0, iw = 0;
  while (is < sig.size() || iw < wait.size()) {
    PeerFlags f;
    f.code = code;
    while (is < sig.size() && f.n_sig < kMaxPeerFlags) f.sig[f.n_sig++] = sig[is++];
    while (iw < wait.size() && f.n_wait < kMaxPeerFlags) f.wait[f.n_wait++] = wait[iw++];
    launch_peer_flags(flags_, f, peer_timeout_ns_, peer_err_, s);
  }
}

void Executor::peer_wait(int id, cudaStream_t s) {
  if (!peer_ || psync_.waits[id].empty()) return;
  std::vector<const unsigned*> w;
  for (int slot : psync_.waits[id]) w.push_back(flags_ + kFlagReady + slot);
  peer_flags({}, w, static_cast<unsigned>(id) + 1u, s);
}

void Executor::peer_signal(int id, cudaStream_t s) {
  if (!peer_ || psync_.signals[id].empty()) return;
  std::vector<unsigned*> sg;
  for (const auto& [r, slot] : psync_.signals[id]) sg.push_back(peer_flags_[r] + kFlagReady + slot);
  peer_flags(sg, {}, static_cast<unsigned>(id) + 1u, s);
}

void Executor::peer_step_begin(cudaStream_t s) {
  if (peer_) launch_peer_epoch(flags_, s);
}

// Step-end barrier: no rank starts the next step (and rewrites a buffer)
// before every rank has finished reading this step's pieces.
void Executor::peer_step_end(cudaStream_t s) {
  if (!peer_ || rc_.world == 1) return;
  std::vector<unsigned*> sg;
  std::vector<const unsigned*> w;
  for (int r = 0; r < rc_.world; ++r) {
    if (r == rc_.rank) continue;
    sg.push_back(peer_flags_[r] + kFlagBarrier + rc_.rank);
    w.push_back(flags_ + kFlagBarrier + r);
  }
  peer_flags(sg, w, ~0u, s);
}

// Synchronises every device this process drives; a peer wait that timed out
// is reported as such instead of as a bare launch failure.
void Executor::sync_all(const char* what) {
  for (int g : gpus_) {
    DeviceGuard dg(g);
    check_sync(cudaDeviceSynchronize(), what);
  }
}

void Executor::check_sync(cudaError_t e, const char* what) const {
  if (e == cudaSuccess) return;
  if (peer_err_ && *peer_err_) {
    const unsigned c = *peer_err_;
    const unsigned long long addr =
        static_cast<unsigned long long>(peer_err_[3]) | (static_cast<unsigned long long>(peer_err_[4]) << 32);
    const long long word = static_cast<long long>(addr - reinterpret_cast<unsigned long long>(flags_)) / 4;
    std::string where = word >= static_cast<long long>(kFlagReady) ? "ready slot " + std::to_string(word - kFlagReady)
                        : word >= static_cast<long long>(kFlagBarrier)
                            ? "barrier slot of rank " + std::to_string(word - kFlagBarrier)
                            : "flag word " + std::to_string(word);
    where += " saw " + std::to_string(peer_err_[1]) + ", awaited epoch " + std::to_string(peer_err_[2]);
    throw InternalError(std::string("peer-memory rank mode: rank ") + std::to_string(rc_.rank) +
                        (c == ~0u ? " timed out in the step barrier"
                                  : " timed out waiting for the producers of instruction " + std::to_string(c - 1)) +
                        " (" + where + "; " + cudaGetErrorString(e) + ")");
  }
  ck(e, what);
}

void Executor::build_box_tables() {
  if (alias_.empty()) {
    alias_.assign(prog_.buffers.size(), -1);
    alias_off_.assign(prog_.buffers.size(), 0);
  }
  for (const auto& in : prog_.instrs) {
    if (in.kind != InstrKind::box || exec_lane_[in.id] < 0 || irt_[in.id].aliased) continue;
    const BufferDesc& ob = prog_.buffers[in.out_bufs[0]];
    const std::int64_t V = 16 / dtype_size(ob.dtype);
    std::vector<const Cell*> groups[2];
    for (const auto& c : in.cells) {
      bool vec = c.dst_strides[c.rank - 1] == 1 && c.extents[c.rank - 1] % V == 0 && c.dst_offset % V == 0;
      for (int d = 0; d + 1 < c.rank; ++d) vec = vec && c.dst_strides[d] % V == 0;
      for (const auto& t : c.terms) {
        vec = vec && t.strides[c.rank - 1] == 1 && t.offset % V == 0;
        for (int d = 0; d + 1 < c.rank; ++d) vec = vec && t.strides[d] % V == 0;
      }
      groups[vec ? 1 : 0].push_back(&c);
    }
    for (int g = 0; g < 2; ++g) {
      if (groups[g].empty()) continue;
      std::int64_t width = g ? V : 1;
      // A block owns up to kBoxChunkUnits vector units of one cell. Smaller
      // chunks for small boxes (>= 2 waves of blocks) measured slower (C5
      // 2.33 -> 3.10 ms: the lanes' concurrent launches already fill the
      // SMs); PLANC_B200_BOX_CHUNK=<units> sets a fixed size for A/B.
      static const char* fixed = std::getenv("PLANC_B200_BOX_CHUNK");
      const std::int64_t kChunkUnits =
          fixed ? std::max<std::int64_t>(1, std::min<std::int64_t>(kBoxChunkUnits, std::atoll(fixed))) : kBoxChunkUnits;
      std::vector<DevCell> cells;
      std::vector<DevTerm> terms;
      std::vector<DevChunk> chunks;
      // Launch rank: 1, 2 or kBoxRank; lower-rank cells get leading unit
      // dims so the kernel indexes coordinates statically.
      int max_rank = 1;
      for (const Cell* c : groups[g]) max_rank = std::max(max_rank, c->rank);
      const int R = max_rank <= 1 ? 1 : max_rank <= 2 ? 2 : kBoxRank;
      max_rank = R;
      for (const Cell* c : groups[g]) {
        const int pad = R - c->rank;
        DevCell dc{};
        dc.rank = R;
        for (int d = 0; d < R; ++d) {
          dc.ext[d] = d < pad ? 1 : c->extents[d - pad];
          dc.dst_str[d] = d < pad ? 0 : c->dst_strides[d - pad];
        }
        dc.dst = buf_ptr(in.out_bufs[0]);
        dc.dst_off = c->dst_offset;
        dc.elems = c->elems();
        dc.nterms = static_cast<int>(c->terms.size());
        dc.term0 = static_cast<int>(terms.size());
        dc.vec = static_cast<int>(width);
        for (const auto& t : c->terms) {
          DevTerm dt{};
          dt.src = buf_ptr(t.buffer);
          dt.offset = t.offset;
          for (int d = 0; d < R; ++d) dt.str[d] = d < pad ? 0 : t.strides[d - pad];
          dt.op = t.fold >= 0 ? t.fold + 1 : t.add ? 1 : 0;  // EwOp add / mul / max -> box 1 / 2 / 3
          terms.push_back(dt);
        }
        int ci = static_cast<int>(cells.size());
        cells.push_back(dc);
        std::int64_t units = dc.elems / width;
        if (units >= (std::int64_t(1) << 32)) throw UsageError("adapter cell above 2^32 vector units");
        for (std::int64_t b = 0; b < units; b += kChunkUnits) {
          DevChunk ch{};
          ch.cell = ci;
          ch.begin = b;
          ch.count = std::min(kChunkUnits, units - b);
          chunks.push_back(ch);
        }
      }
      if (chunks.empty()) continue;
      BoxLaunch bl;
      bl.nchunks = static_cast<int>(chunks.size());
      bl.vec = g;
      bl.max_rank = max_rank;
      bl.dtype = dt_of(ob.dtype);
      bl.h_cells = std::move(cells);
      bl.h_terms = std::move(terms);
      bl.h_chunks = std::move(chunks);
      upload_box(bl, lanes_[in.lane].gpu);
      irt_[in.id].box.push_back(bl);
    }
  }
}

// Elementwise instructions as box cells (with batching on): one rank-1
// cell per instruction, terms = the operands in fold order (copy, then the
// op) — the same fp32 fold and single rounding as ew_kernel, so the same
// bits; 16-byte vectors for the aligned body, a scalar cell for the tail.
// (More than 8 operands keep ew_kernel: it rounds every 8-operand chunk.)
void Executor::build_ew_tables() {
  for (const auto& in : prog_.instrs) {
    if (in.kind != InstrKind::ew || exec_lane_[in.id] < 0 || in.in_bufs.empty() || in.in_bufs.size() > 8) continue;
    if (in.ew != EwOp::add && in.ew != EwOp::mul && in.ew != EwOp::max) continue;
    const BufferDesc& ob = prog_.buffers[in.out_bufs[0]];
    if (ob.dtype == DType::i32) continue;
    const std::int64_t V = 16 / dtype_size(ob.dtype);
    const int opc = in.ew == EwOp::add ? 1 : in.ew == EwOp::mul ? 2 : 3;
    bool aligned = reinterpret_cast<std::uintptr_t>(buf_ptr(in.out_bufs[0])) % 16 == 0;
    for (int b : in.in_bufs) aligned = aligned && reinterpret_cast<std::uintptr_t>(buf_ptr(b)) % 16 == 0;
    const std::int64_t body = aligned ? in.count / V * V : 0;
    for (int g = 1; g >= 0; --g) {
      const std::int64_t lo = g ? 0 : body, n = g ? body : in.count - body;
      if (n <= 0) continue;
      const std::int64_t width = g ? V : 1;
      BoxLaunch bl;
      bl.vec = g;
      bl.max_rank = 1;
      bl.dtype = dt_of(ob.dtype);
      DevCell dc{};
      dc.dst = buf_ptr(in.out_bufs[0]);
      dc.rank = 1;
      dc.ext[0] = n;
      dc.dst_str[0] = 1;
      dc.dst_off = lo;
      dc.elems = n;
      dc.nterms = static_cast<int>(in.in_bufs.size());
      dc.term0 = 0;
      dc.vec = static_cast<int>(width);
      for (std::size_t t = 0; t < in.in_bufs.size(); ++t) {
        DevTerm dt{};
        dt.src = buf_ptr(in.in_bufs[t]);
        dt.offset = lo;
        dt.str[0] = 1;
        dt.op = t == 0 ? 0 : opc;
        bl.h_terms.push_back(dt);
      }
      bl.h_cells.push_back(dc);
      const std::int64_t units = n / width;
      if (units >= (std::int64_t(1) << 32)) continue;
      for (std::int64_t b = 0; b < units; b += kBoxChunkUnits) {
        DevChunk ch{};
        ch.cell = 0;
        ch.begin = b;
        ch.count = std::min<std::int64_t>(kBoxChunkUnits, units - b);
        bl.h_chunks.push_back(ch);
      }
      upload_box(bl, lanes_[in.lane].gpu);
      irt_[in.id].box.push_back(std::move(bl));
    }
  }
}

void Executor::upload_box(BoxLaunch& bl, int gpu) {
  DeviceGuard dg(gpu);
  const std::size_t cb = bl.h_cells.size() * sizeof(DevCell), tb = bl.h_terms.size() * sizeof(DevTerm),
                    hb = bl.h_chunks.size() * sizeof(DevChunk);
  char* mem = nullptr;
  ck(cudaMalloc(&mem, cb + tb + hb + 64), "cudaMalloc(box table)");
  table_allocs_.push_back(mem);
  ck(cudaMemcpy(mem, bl.h_cells.data(), cb, cudaMemcpyHostToDevice), "box table");
  if (tb) ck(cudaMemcpy(mem + cb, bl.h_terms.data(), tb, cudaMemcpyHostToDevice), "box table");
  ck(cudaMemcpy(mem + cb + tb, bl.h_chunks.data(), hb, cudaMemcpyHostToDevice), "box table");
  bl.cells = reinterpret_cast<DevCell*>(mem);
  bl.terms = reinterpret_cast<DevTerm*>(mem + cb);
  bl.chunks = reinterpret_cast<DevChunk*>(mem + cb + tb);
  bl.nchunks = static_cast<int>(bl.h_chunks.size());
}

// Greedy over the issue order, one open batch per GPU: a box instruction
// joins its GPU's open batch; an instruction that depends on a member first
// closes (launches) that batch. Members are therefore pairwise independent
// and every consumer is issued after its batch.
void Executor::plan_box_batches() {
  const std::size_t n = prog_.instrs.size();
  batch_of_.assign(n, -1);
  flush_before_.assign(prog_.issue_order.size(), {});
  flush_end_.clear();
  batches_.clear();
  // PLANC_B200_BATCH: 1 = one open batch per GPU (lanes sharing it are
  // batched together), 2 = one per lane; unset / 0 = ExecOptions.
  const char* env = std::getenv("PLANC_B200_BATCH");
  const int mode = env ? std::atoi(env) : (opt_.batch_boxes ? 1 : 0);
  if (mode == 0 || rank_mode_ || peer_ || opt_.reuse_memory) return;
  build_ew_tables();
  const bool per_lane = mode == 2;
  std::map<int, std::vector<int>> open;  // gpu (or lane) -> members
  std::vector<char> pending(n, 0);
  auto key_of = [&](int id) { return per_lane ? exec_lane_[id] : lanes_[exec_lane_[id]].gpu; };
  auto close = [&](int key, std::vector<int>* where) {
    auto& mem = open[key];
    if (mem.empty()) return;
    BoxBatch b;
    b.members = mem;
    b.gpu = lanes_[exec_lane_[mem[0]]].gpu;
    for (int m : mem) {
      batch_of_[m] = static_cast<int>(batches_.size());
      pending[m] = 0;
    }
    where->push_back(static_cast<int>(batches_.size()));
    batches_.push_back(std::move(b));
    mem.clear();
  };
  for (std::size_t pos = 0; pos < prog_.issue_order.size(); ++pos) {
    const int id = prog_.issue_order[pos];
    if (exec_lane_[id] < 0) continue;
    const Instr& in = prog_.instrs[id];
    for (int d : in.deps)
      if (d >= 0 && pending[d]) close(key_of(d), &flush_before_[pos]);
    if ((in.kind == InstrKind::box || in.kind == InstrKind::ew) && !irt_[id].aliased && !irt_[id].box.empty()) {
      open[key_of(id)].push_back(id);
      pending[id] = 1;
    }
  }
  for (auto& kv : open) close(kv.first, &flush_end_);
  // Merged tables per (element type, vector width, rank); streams; events.
  constexpr int kBatchStreams = 4;
  std::map<int, int> next_stream;
  for (auto& b : batches_) {
    DeviceGuard dg(b.gpu);
    auto& pool = batch_streams_[b.gpu];
    if (pool.empty()) {
      pool.resize(kBatchStreams);
      for (auto& st : pool) ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "batch stream");
      for (std::size_t k = 0; k < pool.size(); ++k) {
        cudaEvent_t e = nullptr;
        ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        batch_join_.push_back(e);
      }
    }
    // per lane: the first member's own stream (no cross-lane coupling)
    b.stream = per_lane ? stream_of(prog_.instrs[b.members[0]]) : pool[next_stream[b.gpu]++ % kBatchStreams];
    ck(cudaEventCreateWithFlags(&b.done, cudaEventDisableTiming), "event");
    std::map<std::tuple<int, int, int>, BoxLaunch> merged;
    for (int m : b.members) {
      for (const BoxLaunch& bl : irt_[m].box) {
        BoxLaunch& t = merged[{bl.dtype, bl.vec, bl.max_rank}];
        t.dtype = bl.dtype;
        t.vec = bl.vec;
        t.max_rank = bl.max_rank;
        const int cell0 = static_cast<int>(t.h_cells.size()), term0 = static_cast<int>(t.h_terms.size());
        for (DevCell c : bl.h_cells) {
          c.term0 += term0;
          t.h_cells.push_back(c);
        }
        t.h_terms.insert(t.h_terms.end(), bl.h_terms.begin(), bl.h_terms.end());
        for (DevChunk ch : bl.h_chunks) {
          ch.cell += cell0;
          t.h_chunks.push_back(ch);
        }
      }
      // the member's dependencies are awaited by events from the batch stream
      for (int d : prog_.instrs[m].deps) {
        if (d < 0 || exec_lane_[d] < 0 || batch_of_[d] >= 0 || irt_[d].done) continue;
        DeviceGuard dg2(lanes_[exec_lane_[d]].gpu);
        ck(cudaEventCreateWithFlags(&irt_[d].done, cudaEventDisableTiming), "event");
      }
    }
    for (auto& kv : merged) {
      if (b.members.size() == 1) {
        b.launches = irt_[b.members[0]].box;  // the member's own tables
        break;
      }
      upload_box(kv.second, b.gpu);
      b.launches.push_back(std::move(kv.second));
    }
  }
  // Non-members whose consumers moved to a batch keep their events; a
  // member's consumer waits for the batch event.
}

cudaStream_t Executor::issued_stream(int id) const {
  return batch_of_.empty() || batch_of_[id] < 0 ? stream_of(prog_.instrs[id]) : batches_[batch_of_[id]].stream;
}

cudaEvent_t Executor::done_event(int id) const {
  return batch_of_.empty() || batch_of_[id] < 0 ? irt_[id].done : batches_[batch_of_[id]].done;
}

void Executor::launch_batch(int bi) {
  BoxBatch& b = batches_[bi];
  if (gpus_.size() > 1) ck(cudaSetDevice(b.gpu), "cudaSetDevice");
  for (int m : b.members)
    for (int d : prog_.instrs[m].deps)
      if (d >= 0 && exec_lane_[d] >= 0 && issued_stream(d) != b.stream)
        ck(cudaStreamWaitEvent(b.stream, done_event(d), 0), "wait dep (batch)");
  for (const auto& bl : b.launches) launch_box(bl.dtype, bl.cells, bl.terms, bl.chunks, bl.nchunks, bl.vec, bl.max_rank, b.stream);
  ck(cudaEventRecord(b.done, b.stream), "record batch");
}

char* Executor::host_stage(std::int64_t bytes) {
  if (bytes > host_stage_bytes_) {
    if (host_stage_) cudaFreeHost(host_stage_);
    host_stage_ = nullptr;
    host_stage_bytes_ = 0;
    ck(cudaMallocHost(&host_stage_, static_cast<std::size_t>(bytes)), "cudaMallocHost (staging)");
    host_stage_bytes_ = bytes;
  }
  return static_cast<char*>(host_stage_);
}

// Graph-input placement (refexec.cpp:366-376 + ConcreteTensor::extract
// :75-83): each placement buffer of the pTensor receives its view's region,
// converted to the device element type — rows of the region converted in
// parallel into pinned staging, one H2D copy per buffer. Placed at once (the
// caller keeps ownership of `data`); run() checks every input was placed.
void Executor::set_input(int ptensor, const double* data, const std::vector<std::int64_t>& shape) {
  bool synced = false;
  for (const auto& b : prog_.buffers) {
    if (!b.graph_input || !owned_[b.lane] || b.ptensor != ptensor) continue;
    const PTensor& pt = plan_.pt(b.ptensor);
    if (shape != pt.shape) throw UsageError("input tensor " + std::to_string(ptensor) + " has the wrong shape");
    if (!synced) {  // no step in flight may still read the old values
      for (int g : gpus_) {
        DeviceGuard dg(g);
        ck(cudaDeviceSynchronize(), "sync before input placement");
      }
      synced = true;
    }
    const int rank = static_cast<int>(b.shape.size());
    std::vector<std::int64_t> gstr(rank, 1);
    for (int d = rank - 2; d >= 0; --d) gstr[d] = gstr[d + 1] * pt.shape[d + 1];
    const std::int64_t inner = rank ? b.shape[rank - 1] : 1;
    const std::int64_t rows = inner ? b.elems / inner : 0;
    char* host = host_stage(std::max<std::int64_t>(b.bytes, 1));
    parallel_for(rows, inner, [&](std::int64_t lo, std::int64_t hi) {
      for (std::int64_t r = lo; r < hi; ++r) {
        std::int64_t rem = r, g = 0;
        for (int d = rank - 2; d >= 0; --d) {
          g += (b.mask.region[d].lo + rem % b.shape[d]) * gstr[d];
          rem /= b.shape[d];
        }
        if (rank) g += b.mask.region[rank - 1].lo;
        const double* src = data + g;
        const std::int64_t e0 = r * inner;
        for (std::int64_t j = 0; j < inner; ++j) put_elem(host, b.dtype, e0 + j, src[j]);
      }
    });
    DeviceGuard dg(lanes_[b.lane].gpu);
    ck(cudaMemcpy(buf_ptr(b.id), host, b.bytes, cudaMemcpyHostToDevice), "input placement");
  }
  placed_.insert(ptensor);
}

void Executor::place_inputs() {
  for (const auto& b : prog_.buffers) {
    if (b.graph_input && owned_[b.lane] && !placed_.count(b.ptensor))
      throw UsageError("run_plan: missing input tensor " + std::to_string(b.ptensor));
  }
}

GemmArgs Executor::gemm_args(const Instr& in) const {
  GemmArgs a{};
  a.A = buf_ptr(in.in_bufs[0]);
  a.B = buf_ptr(in.in_bufs[1]);
  a.C = buf_ptr(in.out_bufs[0]);
  a.m = in.m;
  a.n = in.n;
  a.k = in.k;
  a.ta = in.ta;
  a.tb = in.tb;
  a.da = dt_of(prog_.buffers[in.in_bufs[0]].dtype);
  a.db = dt_of(prog_.buffers[in.in_bufs[1]].dtype);
  a.dc = dt_of(prog_.buffers[in.out_bufs[0]].dtype);
  a.group = in.group;
  if (in.scatter > 0) {
    if (in.scatter > kMaxGemmGroup || static_cast<int>(in.out_bufs.size()) != in.scatter || !in.fused.empty())
      throw InternalError("malformed reduce-scatter GEMM instruction");
    a.scatter = in.scatter;
    a.scatter_rows = in.scatter_rows;
    for (int i = 0; i < in.scatter; ++i) a.gC[i] = buf_ptr(in.out_bufs[i]);
    a.C = a.gC[0];
  }
  if (in.group > 1) {
    if (in.group > kMaxGemmGroup || static_cast<int>(in.in_bufs.size()) != 2 * in.group ||
        static_cast<int>(in.out_bufs.size()) != in.group || !in.fused.empty()) {
      throw InternalError("malformed grouped GEMM instruction");
    }
    for (int i = 0; i < in.group; ++i) {
      a.gA[i] = buf_ptr(in.in_bufs[2 * i]);
      a.gB[i] = buf_ptr(in.in_bufs[2 * i + 1]);
      a.gC[i] = buf_ptr(in.out_bufs[i]);
    }
  }
  a.epi.n_ops = static_cast<int>(in.fused.size());
  for (std::size_t f = 0; f < in.fused.size(); ++f) {
    const auto& fe = in.fused[f];
    EpiOp& o = a.epi.ops[f];
    o.op = static_cast<int>(fe.op);
    o.n_in = static_cast<int>(fe.in_bufs.size());
    o.gemm_pos = fe.gemm_pos;
    for (std::size_t j = 0; j < fe.in_bufs.size(); ++j) {
      o.in[j] = buf_ptr(fe.in_bufs[j]);
      if (static_cast<int>(j) != fe.gemm_pos) {
        if (a.epi.n_slots >= kMaxEpiSlots) throw InternalError("fused epilogue needs more than 2 operands");
        a.epi.slot_op[a.epi.n_slots] = static_cast<int>(f);
        a.epi.slot_in[a.epi.n_slots] = static_cast<int>(j);
        ++a.epi.n_slots;
      }
    }
    o.out = buf_ptr(fe.out_buf);
  }
  {
    const LaneRt& lr = lanes_[exec_lane_[in.id]];
    a.ws = lr.gemm_ws[exec_stream_[in.id]];
    a.ws_bytes = lr.gemm_ws_bytes[exec_stream_[in.id]];
    a.allow_streamk = gemm_streamk_ok(exec_lane_[in.id]);
    a.gpu_share = gpu_share(exec_lane_[in.id]);
  }
  if (!in.gather[0].empty() || !in.gather[1].empty()) {
    if (in.group != 1 || in.scatter > 0) throw InternalError("malformed gathered-operand GEMM instruction");
    a.gather_a = static_cast<int>(in.gather[0].size());
    a.gather_b = static_cast<int>(in.gather[1].size());
    a.gather_rows_a = in.gather_rows[0];
    a.gather_rows_b = in.gather_rows[1];
    a.gather_cols_a = in.gather_cols[0];
    a.gather_cols_b = in.gather_cols[1];
    for (int i = 0; i < a.gather_a; ++i) a.gather_a_ptr[i] = buf_ptr(in.gather[0][i]);
    for (int i = 0; i < a.gather_b; ++i) a.gather_b_ptr[i] = buf_ptr(in.gather[1][i]);
    a.gather_maps = irt_[in.id].gather_maps;
  }
  return a;
}

// Tensor maps of every gathered-operand GEMM's pieces (buffers are placed
// and workspaces sized by now), copied to device memory once.
void Executor::build_gather_maps() {
  std::vector<unsigned char> host(kGatherMapSlots * kTensorMapBytes);
  for (const auto& in : prog_.instrs) {
    if (in.kind != InstrKind::gemm || exec_lane_[in.id] < 0 || (in.gather[0].empty() && in.gather[1].empty())) continue;
    const GemmArgs a = gemm_args(in);
    if (!opt_.allow_tensor_cores || !gemm_sm100_eligible(a))
      throw InternalError("gathered-operand GEMM " + in.label + " off the tensor-core path");
    gemm_sm100_gather_maps(a, host.data());
    DeviceGuard dg(lanes_[exec_lane_[in.id]].gpu);
    if (!irt_[in.id].gather_maps) {
      ck(cudaMalloc(&irt_[in.id].gather_maps, host.size()), "cudaMalloc(gather maps)");
      table_allocs_.push_back(irt_[in.id].gather_maps);
    }
    ck(cudaMemcpy(irt_[in.id].gather_maps, host.data(), host.size(), cudaMemcpyHostToDevice), "gather maps");
  }
}

void Executor::launch_instr(const Instr& in, cudaStream_t s) {
  switch (in.kind) {
    case InstrKind::nop:
      return;
    case InstrKind::xfer:
      launch_xfer(in, s);
      return;
    case InstrKind::gemm: {
      GemmArgs a = gemm_args(in);
      if (a.epi.n_ops > 0 && !(opt_.allow_tensor_cores && gemm_sm100_eligible(a))) {
        throw InternalError("fused epilogue on a GEMM the tensor-core path does not take");
      }
      launch_gemm(a, s, opt_.allow_tensor_cores, nullptr);
      return;
    }
    case InstrKind::ew: {
      if (!irt_[in.id].box.empty()) {  // as box cells (build_ew_tables)
        for (const auto& bl : irt_[in.id].box)
          launch_box(bl.dtype, bl.cells, bl.terms, bl.chunks, bl.nchunks, bl.vec, bl.max_rank, s);
        return;
      }
      int dt = dt_of(prog_.buffers[in.out_bufs[0]].dtype);
      std::vector<const void*> ptrs;
      for (int b : in.in_bufs) ptrs.push_back(buf_ptr(b));
      void* out = buf_ptr(in.out_bufs[0]);
      // Left fold in chunks of 8 operands: ((x0∘x1)∘…)∘x7, then (out∘x8)∘…
      std::size_t pos = 0;
      while (pos < ptrs.size()) {
        std::vector<const void*> grp;
        if (pos > 0) grp.push_back(out);
        while (grp.size() < 8 && pos < ptrs.size()) grp.push_back(ptrs[pos++]);
        launch_ew(static_cast<int>(in.ew), dt, grp.data(), static_cast<int>(grp.size()), out, in.count, s);
      }
      return;
    }
    case InstrKind::reduce:
      launch_reduce(dt_of(prog_.buffers[in.out_bufs[0]].dtype), buf_ptr(in.in_bufs[0]), buf_ptr(in.out_bufs[0]),
                    irt_[in.id].scratch, in.outer, in.axis_len, in.inner, s);
      return;
    case InstrKind::emb_lookup:
      launch_emb_lookup(dt_of(prog_.buffers[in.out_bufs[0]].dtype), static_cast<const int*>(buf_ptr(in.in_bufs[0])),
                        buf_ptr(in.in_bufs[1]), buf_ptr(in.out_bufs[0]), in.n_idx, in.rows, in.h, in.lo, s);
      return;
    case InstrKind::emb_grad:
      launch_emb_grad(dt_of(prog_.buffers[in.out_bufs[0]].dtype), static_cast<const int*>(buf_ptr(in.in_bufs[0])),
                      buf_ptr(in.in_bufs[1]), buf_ptr(in.out_bufs[0]), irt_[in.id].scratch, in.n_idx, in.rows, in.h,
                      in.lo, s);
      return;
    case InstrKind::attention:
      if (in.att_grad) {
        auto out = [&](int w) { return in.att_out[w] >= 0 ? buf_ptr(in.att_out[w]) : nullptr; };
        launch_attention_grad(buf_ptr(in.in_bufs[0]), buf_ptr(in.in_bufs[1]), buf_ptr(in.in_bufs[2]),
                              buf_ptr(in.in_bufs[3]), buf_ptr(in.in_bufs[4]), out(0), out(1), out(2),
                              irt_[in.id].scratch, in.att_rows, in.att_cols, in.att_seq, in.att_dh, in.causal,
                              dt_of(prog_.buffers[in.out_bufs[0]].dtype), s);
        return;
      }
      launch_attention(buf_ptr(in.in_bufs[0]), buf_ptr(in.in_bufs[1]), buf_ptr(in.in_bufs[2]), buf_ptr(in.out_bufs[0]),
                       in.att_rows, in.att_cols, in.att_seq, in.att_dh, in.causal,
                       dt_of(prog_.buffers[in.out_bufs[0]].dtype), s);
      return;
    case InstrKind::rowwise:
      launch_rowwise(static_cast<int>(in.row_op), dt_of(prog_.buffers[in.out_bufs[0]].dtype), buf_ptr(in.in_bufs[0]),
                     in.in_bufs.size() > 1 ? buf_ptr(in.in_bufs[1]) : nullptr, buf_ptr(in.out_bufs[0]), in.count, in.seg,
                     static_cast<float>(in.eps), s);
      return;
    case InstrKind::box: {
      for (const auto& bl : irt_[in.id].box) {
        launch_box(bl.dtype, bl.cells, bl.terms, bl.chunks, bl.nchunks, bl.vec, bl.max_rank, s);
      }
      return;
    }
  }
}

void Executor::issue_step(bool, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>*) {
  int cur = -1;
  auto set_dev = [&](int g) {
    if (g != cur && gpus_.size() > 1) {
      ck(cudaSetDevice(g), "cudaSetDevice");
    }
    cur = g;
  };
  set_dev(lanes_[first_lane_].gpu);
  peer_step_begin(origin_);
  ck(cudaEventRecord(ev_begin_, origin_), "record begin");
  for (int l = 0; l < prog_.num_lanes; ++l)
    if (owned_[l])
      for (auto s : lanes_[l].stream) ck(cudaStreamWaitEvent(s, ev_begin_, 0), "wait begin");
  for (auto& kv : batch_streams_)
    for (auto s : kv.second) ck(cudaStreamWaitEvent(s, ev_begin_, 0), "wait begin");
  for (std::size_t pos = 0; pos < prog_.issue_order.size(); ++pos) {
    if (!flush_before_.empty())
      for (int b : flush_before_[pos]) {
        launch_batch(b);
        cur = batches_[b].gpu;
      }
    const int id = prog_.issue_order[pos];
    const int el = exec_lane_[id];
    if (el < 0) continue;  // another rank's instruction
    if (!batch_of_.empty() && batch_of_[id] >= 0) continue;  // launched with its batch
    const Instr& in = prog_.instrs[id];
    cudaStream_t s = stream_of(in);
    set_dev(lanes_[el].gpu);
    for (int d : in.deps) {
      if (exec_lane_[d] < 0) continue;
      if (issued_stream(d) != s) ck(cudaStreamWaitEvent(s, done_event(d), 0), "wait dep");
    }
    peer_wait(id, s);
    launch_instr(in, s);
    peer_signal(id, s);
    if (irt_[id].done) ck(cudaEventRecord(irt_[id].done, s), "record done");
  }
  for (int b : flush_end_) launch_batch(b);
  join_lanes();
  peer_step_end(origin_);
}

// The origin stream waits for every lane stream (ends on the origin's device).
void Executor::join_lanes() {
  for (int l = 0; l < prog_.num_lanes; ++l) {
    if (!owned_[l]) continue;
    if (gpus_.size() > 1) ck(cudaSetDevice(lanes_[l].gpu), "cudaSetDevice");
    for (int k = 0; k < kLaneStreams; ++k)
      ck(cudaEventRecord(lane_join_[kLaneStreams * l + k], lanes_[l].stream[k]), "record join");
  }
  std::size_t j = 0;
  for (auto& kv : batch_streams_) {
    if (gpus_.size() > 1) ck(cudaSetDevice(kv.first), "cudaSetDevice");
    for (auto st : kv.second) ck(cudaEventRecord(batch_join_[j++], st), "record join");
  }
  ck(cudaSetDevice(lanes_[first_lane_].gpu), "cudaSetDevice");
  for (auto e : lane_join_)
    if (e) ck(cudaStreamWaitEvent(origin_, e, 0), "wait join");
  for (auto e : batch_join_) ck(cudaStreamWaitEvent(origin_, e, 0), "wait join");
}

void Executor::ensure_graph() {
  if (!opt_.use_graph || graph_exec_) return;
  DeviceGuard dg(lanes_[first_lane_].gpu);
  ck(cudaStreamBeginCapture(origin_, cudaStreamCaptureModeThreadLocal), "begin capture");
  bool ok = true;
  try {
    issue_step(false, nullptr);
  } catch (const std::exception&) {
    ok = false;
  }
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(origin_, &g);
  if (!ok || e != cudaSuccess || !g) {
    cudaGetLastError();
    if (g) cudaGraphDestroy(g);
    opt_.use_graph = false;  // eager issue from here on
    return;
  }
  e = cudaGraphInstantiate(&graph_exec_, g, 0);
  if (e != cudaSuccess) {
    cudaGetLastError();
    cudaGraphDestroy(g);
    graph_exec_ = nullptr;
    opt_.use_graph = false;
    return;
  }
  graph_ = g;
}

double Executor::run(int iters) {
  peer_check_ready();
  place_inputs();
  ensure_graph();
  DeviceGuard dg(lanes_[first_lane_].gpu);
  auto step = [&]() {
    if (graph_exec_) ck(cudaGraphLaunch(graph_exec_, origin_), "graph launch");
    else issue_step(false, nullptr);
  };
  if (iters <= 0) {
    step();
    check_sync(cudaStreamSynchronize(origin_), "step");
    return 0;
  }
  cudaEvent_t t0, t1;
  ck(cudaEventCreate(&t0), "event");
  ck(cudaEventCreate(&t1), "event");
  ck(cudaEventRecord(t0, origin_), "record");
  for (int i = 0; i < iters; ++i) step();
  ck(cudaEventRecord(t1, origin_), "record");
  check_sync(cudaEventSynchronize(t1), "sync");
  float ms = 0;
  ck(cudaEventElapsedTime(&ms, t0, t1), "elapsed");
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  return ms / iters;
}

double Executor::run_e2e(int iters, std::int64_t* h2d_bytes, std::int64_t* d2h_bytes) {
  peer_check_ready();
  place_inputs();
  ensure_graph();
  DeviceGuard dg(lanes_[first_lane_].gpu);
  if (pinned_in_.empty() && pinned_out_.empty()) {
    // Step inputs: non-weight graph-input placements, staged from pinned host
    // memory in device element type (weights stay resident, like a trainer).
    for (const auto& b : prog_.buffers) {
      if (!b.graph_input || b.weight || !owned_[b.lane]) continue;
      void* h = nullptr;
      ck(cudaMallocHost(&h, std::max<std::int64_t>(b.bytes, 1)), "cudaMallocHost");
      ck(cudaMemcpy(h, buf_ptr(b.id), b.bytes, cudaMemcpyDeviceToHost), "stage input");
      pinned_in_.push_back(h);
      e2e_in_bufs_.push_back(b.id);
    }
    // Step results: every piece of a terminal (never consumed), non-weight
    // produced pTensor.
    std::set<int> consumed;
    for (const auto& op : plan_.ops)
      for (int v : op.inputs) consumed.insert(plan_.vt(v).ptensor);
    for (const auto& [pt, bufs] : prog_.outputs) {
      TensorKind k = plan_.pt(pt).kind;
      if (consumed.count(pt) || k == TensorKind::weight || k == TensorKind::optimizer_state) continue;
      for (int b : bufs) {
        if (!local(b)) continue;
        void* h = nullptr;
        ck(cudaMallocHost(&h, std::max<std::int64_t>(prog_.buffers[b].bytes, 1)), "cudaMallocHost");
        pinned_out_.push_back(h);
        e2e_out_bufs_.push_back(b);
      }
    }
  }
  std::int64_t hb = 0, db = 0;
  for (int b : e2e_in_bufs_) hb += prog_.buffers[b].bytes;
  for (int b : e2e_out_bufs_) db += prog_.buffers[b].bytes;
  if (h2d_bytes) *h2d_bytes = hb;
  if (d2h_bytes) *d2h_bytes = db;
  // Pipelined steps: step i+1's inputs cross PCIe (copy stream) while step i
  // computes, and step i's results cross back while step i+1 computes.
  // Every step still moves all of its own bytes: H2D into one of two device
  // staging sets, a device copy into the placement buffers at step start,
  // the step, a device copy of the results into one of two result sets, D2H.
  if (e2e_stage_in_[0].empty()) {
    for (int k = 0; k < 2; ++k) {
      for (int b : e2e_in_bufs_) {
        void* d = nullptr;
        ck(cudaMalloc(&d, std::max<std::int64_t>(prog_.buffers[b].bytes, 1)), "cudaMalloc(stage)");
        e2e_stage_in_[k].push_back(d);
      }
      for (int b : e2e_out_bufs_) {
        void* d = nullptr;
        ck(cudaMalloc(&d, std::max<std::int64_t>(prog_.buffers[b].bytes, 1)), "cudaMalloc(stage)");
        e2e_stage_out_[k].push_back(d);
      }
    }
    ck(cudaStreamCreateWithFlags(&h2d_stream_, cudaStreamNonBlocking), "h2d stream");
    ck(cudaStreamCreateWithFlags(&d2h_stream_, cudaStreamNonBlocking), "d2h stream");
    for (int k = 0; k < 2; ++k) {
      for (cudaEvent_t* e : {&ev_h2d_[k], &ev_in_free_[k], &ev_out_ready_[k], &ev_out_free_[k]}) {
        ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
      }
    }
  }
  auto issue_h2d = [&](int slot) {  // inputs of the step using staging set `slot`
    ck(cudaStreamWaitEvent(h2d_stream_, ev_in_free_[slot], 0), "wait stage free");
    for (std::size_t i = 0; i < e2e_in_bufs_.size(); ++i) {
      ck(cudaMemcpyAsync(e2e_stage_in_[slot][i], pinned_in_[i], prog_.buffers[e2e_in_bufs_[i]].bytes,
                         cudaMemcpyHostToDevice, h2d_stream_),
         "h2d");
    }
    ck(cudaEventRecord(ev_h2d_[slot], h2d_stream_), "record h2d");
  };
  auto compute = [&](int slot) {
    ck(cudaStreamWaitEvent(origin_, ev_h2d_[slot], 0), "wait h2d");
    for (std::size_t i = 0; i < e2e_in_bufs_.size(); ++i) {
      const auto& b = prog_.buffers[e2e_in_bufs_[i]];
      launch_copy_bytes(buf_ptr(b.id), e2e_stage_in_[slot][i], b.bytes, origin_);  // SMs: copy engines carry PCIe
    }
    ck(cudaEventRecord(ev_in_free_[slot], origin_), "record stage free");
    if (graph_exec_) ck(cudaGraphLaunch(graph_exec_, origin_), "graph launch");
    else issue_step(false, nullptr);
    ck(cudaStreamWaitEvent(origin_, ev_out_free_[slot], 0), "wait out free");
    for (std::size_t i = 0; i < e2e_out_bufs_.size(); ++i) {
      const auto& b = prog_.buffers[e2e_out_bufs_[i]];
      launch_copy_bytes(e2e_stage_out_[slot][i], buf_ptr(b.id), b.bytes, origin_);
    }
    ck(cudaEventRecord(ev_out_ready_[slot], origin_), "record out ready");
  };
  auto issue_d2h = [&](int slot) {
    ck(cudaStreamWaitEvent(d2h_stream_, ev_out_ready_[slot], 0), "wait out ready");
    for (std::size_t i = 0; i < e2e_out_bufs_.size(); ++i) {
      ck(cudaMemcpyAsync(pinned_out_[i], e2e_stage_out_[slot][i], prog_.buffers[e2e_out_bufs_[i]].bytes,
                         cudaMemcpyDeviceToHost, d2h_stream_),
         "d2h");
    }
    ck(cudaEventRecord(ev_out_free_[slot], d2h_stream_), "record out free");
  };
  auto run_steps = [&](int n, cudaEvent_t start) {
    if (start) {
      ck(cudaStreamWaitEvent(h2d_stream_, start, 0), "wait start");
      ck(cudaStreamWaitEvent(d2h_stream_, start, 0), "wait start");
    }
    issue_h2d(0);
    for (int i = 0; i < n; ++i) {
      if (i + 1 < n) issue_h2d((i + 1) & 1);
      compute(i & 1);
      issue_d2h(i & 1);
    }
    cudaEvent_t done;
    ck(cudaEventCreateWithFlags(&done, cudaEventDisableTiming), "event");
    ck(cudaEventRecord(done, d2h_stream_), "record done");
    ck(cudaStreamWaitEvent(origin_, done, 0), "join d2h");
    cudaEventDestroy(done);
  };
  run_steps(2, nullptr);
  check_sync(cudaStreamSynchronize(origin_), "warmup");
  cudaEvent_t t0, t1;
  ck(cudaEventCreate(&t0), "event");
  ck(cudaEventCreate(&t1), "event");
  ck(cudaEventRecord(t0, origin_), "record");
  run_steps(std::max(iters, 1), t0);
  ck(cudaEventRecord(t1, origin_), "record");
  check_sync(cudaEventSynchronize(t1), "sync");
  float ms = 0;
  ck(cudaEventElapsedTime(&ms, t0, t1), "elapsed");
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  return ms / std::max(iters, 1);
}

std::string Executor::timeline_json() {
  peer_check_ready();
  place_inputs();
  DeviceGuard dg(lanes_[first_lane_].gpu);
  sync_all("timeline sync");
  cudaSetDevice(lanes_[first_lane_].gpu);
  const std::size_t n = prog_.instrs.size();
  std::vector<cudaEvent_t> ev0(n, nullptr), ev1(n, nullptr);
  cudaEvent_t base;
  ck(cudaEventCreate(&base), "event");
  peer_step_begin(origin_);
  ck(cudaEventRecord(base, origin_), "record base");
  for (int l = 0; l < prog_.num_lanes; ++l)
    if (owned_[l])
      for (auto s : lanes_[l].stream) ck(cudaStreamWaitEvent(s, base, 0), "wait base");
  for (int id : prog_.issue_order) {
    const int el = exec_lane_[id];
    if (el < 0) continue;
    const Instr& in = prog_.instrs[id];
    cudaSetDevice(lanes_[el].gpu);
    cudaStream_t s = stream_of(in);
    for (int d : in.deps) {
      if (exec_lane_[d] < 0) continue;
      if (exec_lane_[d] != el || exec_stream_[d] != exec_stream_[id])
        ck(cudaStreamWaitEvent(s, irt_[d].done ? irt_[d].done : ev1[d], 0), "wait dep");
    }
    ck(cudaEventCreate(&ev0[id]), "event");
    ck(cudaEventCreate(&ev1[id]), "event");
    peer_wait(id, s);
    ck(cudaEventRecord(ev0[id], s), "record");
    launch_instr(in, s);
    ck(cudaEventRecord(ev1[id], s), "record");
    peer_signal(id, s);
    if (irt_[id].done) ck(cudaEventRecord(irt_[id].done, s), "record done");
  }
  if (peer_) {
    join_lanes();
    peer_step_end(origin_);
  }
  sync_all("timeline sync");
  auto task_kind = [&](const Instr& in) -> const char* {
    if (in.kind == InstrKind::xfer) return "collective";
    const OpNode& op = plan_.ops[in.op];
    switch (op.kind) {
      case OpKind::recv: return "recv";
      case OpKind::send: return "send";
      case OpKind::collective: return "collective";
      default: return "compute";
    }
  };
  std::ostringstream os;
  os.precision(9);
  os << "[";
  bool first = true;
  for (int id : prog_.issue_order) {
    if (!ev0[id]) continue;
    const Instr& in = prog_.instrs[id];
    float a = 0, b = 0;
    ck(cudaEventElapsedTime(&a, base, ev0[id]), "elapsed");
    ck(cudaEventElapsedTime(&b, base, ev1[id]), "elapsed");
    os << (first ? "" : ",") << "{\"device\":" << prog_.lane_device[exec_lane_[id]] << ",\"op\":\""
       << (in.op >= 0 ? plan_.ops[in.op].id : in.label) << "\",\"kind\":\"" << task_kind(in) << "\",\"instr\":\""
       << instr_kind_name(in.kind) << "\",\"stream\":" << exec_stream_[id] << ",\"start\":" << a * 1e-3
       << ",\"end\":" << b * 1e-3 << "}";
    first = false;
    cudaEventDestroy(ev0[id]);
    cudaEventDestroy(ev1[id]);
  }
  os << "]";
  cudaEventDestroy(base);
  return os.str();
}

std::vector<KernelStat> Executor::profile() {
  peer_check_ready();
  place_inputs();
  {
    DeviceGuard dg(lanes_[first_lane_].gpu);
    peer_step_begin(origin_);
    sync_all("profile sync");
  }
  std::map<std::string, KernelStat> acc;
  std::vector<std::string> order;
  // Each instruction runs alone, enqueued behind a host gate: start event,
  // launches, end event are all queued before the gate opens, so the
  // interval holds the instruction's kernels back to back — not the host's
  // launch latency (which would dominate a 2-us kernel's measurement).
  unsigned* gate = nullptr;
  ck(cudaHostAlloc(reinterpret_cast<void**>(&gate), sizeof(unsigned), cudaHostAllocMapped | cudaHostAllocPortable),
     "cudaHostAlloc (profile gate)");
  struct GateFree {
    unsigned* p;
    ~GateFree() { cudaFreeHost(p); }
  } gate_free{gate};
  for (int id : prog_.issue_order) {
    const Instr& in = prog_.instrs[id];
    const int el = exec_lane_[id];
    if (in.kind == InstrKind::nop || el < 0) continue;
    DeviceGuard dg(lanes_[el].gpu);
    cudaStream_t s = lanes_[el].stream[0];
    sync_all("profile sync");
    cudaSetDevice(lanes_[el].gpu);
    cudaEvent_t a, b;
    ck(cudaEventCreate(&a), "event");
    ck(cudaEventCreate(&b), "event");
    peer_wait(id, s);
    unsigned* gate_dev = nullptr;
    ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&gate_dev), gate, 0), "gate pointer");
    *reinterpret_cast<volatile unsigned*>(gate) = 0;
    launch_host_gate(gate_dev, s);
    ck(cudaEventRecord(a, s), "record");
    launch_instr(in, s);
    ck(cudaEventRecord(b, s), "record");
    std::atomic_thread_fence(std::memory_order_seq_cst);
    *reinterpret_cast<volatile unsigned*>(gate) = 1;
    peer_signal(id, s);
    check_sync(cudaEventSynchronize(b), "sync");
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, a, b), "elapsed");
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    std::string kind;
    switch (in.kind) {
      case InstrKind::gemm: {
        GemmArgs g{};
        g.m = in.m;
        g.n = in.n;
        g.k = in.k;
        g.ta = in.ta;
        g.tb = in.tb;
        g.da = dt_of(prog_.buffers[in.in_bufs[0]].dtype);
        g.db = dt_of(prog_.buffers[in.in_bufs[1]].dtype);
        g.dc = dt_of(prog_.buffers[in.out_bufs[0]].dtype);
        // One family per GEMM path: a fused elementwise epilogue is part of
        // the GEMM kernel (its flops stay the GEMM's; the fused op's bytes ride along).
        kind = opt_.allow_tensor_cores && gemm_sm100_eligible(g) ? "gemm_tc" : "gemm_simt";
        break;
      }
      case InstrKind::ew: kind = "ew"; break;
      case InstrKind::rowwise: kind = "rowwise"; break;
      case InstrKind::attention: kind = in.att_grad ? "attention_grad" : "attention"; break;
      case InstrKind::reduce: kind = "reduce"; break;
      case InstrKind::emb_lookup:
      case InstrKind::emb_grad: kind = "embedding"; break;
      case InstrKind::xfer: kind = "xfer_nccl"; break;
      case InstrKind::box:
        // Collective member outputs are labelled "<primitive>:<op>".
        kind = irt_[in.id].aliased                      ? "alias"
               : in.label.find(':') != std::string::npos ? "box_collective"
               : in.wire_bytes > 0                     ? "box_p2p"
                                                       : "box_local";
        break;
      default: kind = "other";
    }
    auto& st = acc[kind];
    if (st.kind.empty()) {
      st.kind = kind;
      order.push_back(kind);
    }
    st.launches += 1;
    st.ms += ms;
    st.flops += in.flops;
    if (in.kind == InstrKind::gemm) {
      // GEMM families: only the bytes of fused elementwise epilogues (the
      // operand / result traffic of a compute-bound GEMM is not its bound).
      double base = 0;
      for (std::size_t i = 0; i < static_cast<std::size_t>(2 * in.group) && i < in.in_bufs.size(); ++i)
        base += static_cast<double>(prog_.buffers[in.in_bufs[i]].bytes);
      for (int i = 0; i < in.group && i < static_cast<int>(in.out_bufs.size()); ++i)
        base += static_cast<double>(prog_.buffers[in.out_bufs[i]].bytes);
      st.bytes += in.fused.empty() ? 0.0 : std::max(0.0, in.bytes - base);
    } else {
      st.bytes += in.bytes;
    }
    st.wire_bytes += in.wire_bytes;
  }
  {
    DeviceGuard dg(lanes_[first_lane_].gpu);
    peer_step_end(origin_);
    sync_all("profile sync");
  }
  std::vector<KernelStat> out;
  for (const auto& k : order) out.push_back(acc[k]);
  return out;
}

std::vector<double> Executor::read_buffer(int buffer) {
  if (buffer < 0 || buffer >= static_cast<int>(prog_.buffers.size())) throw UsageError("no such buffer");
  const BufferDesc& bd = prog_.buffers[buffer];
  peer_check_ready();
  if (!readable(bd.lane)) throw UsageError("buffer " + std::to_string(buffer) + " lives on another rank");
  if (released(buffer)) throw UsageError("buffer " + std::to_string(buffer) + " was reused in the step (REUSE_MEMORY)");
  DeviceGuard dg(lanes_[bd.lane].gpu);
  for (int g : gpus_) {
    cudaSetDevice(g);
    ck(cudaDeviceSynchronize(), "sync before readback");
  }
  cudaSetDevice(lanes_[bd.lane].gpu);
  std::vector<char> r(bd.bytes);
  ck(cudaMemcpy(r.data(), buf_ptr(buffer), bd.bytes, cudaMemcpyDeviceToHost), "readback");
  std::vector<double> out(bd.elems);
  for (std::int64_t i = 0; i < bd.elems; ++i) out[i] = host_elem(r, bd.dtype, i);
  return out;
}

std::vector<int> Executor::input_ids() const {
  std::set<int> ids;
  for (const auto& b : prog_.buffers)
    if (b.graph_input && owned_[b.lane]) ids.insert(b.ptensor);
  return std::vector<int>(ids.begin(), ids.end());
}

std::vector<int> Executor::output_ids() const {
  std::vector<int> ids;
  for (const auto& o : prog_.outputs) ids.push_back(o.first);
  return ids;
}

// Reassembly of a produced pTensor (refexec.cpp:532-556): the deduplicated
// producer pieces are read back and reconstructed into the full tensor on
// the host in double, like the reference returns them.
HostTensor Executor::get_output(int ptensor) {
  const PTensor& pt = plan_.pt(ptensor);
  HostTensor out;
  out.shape = pt.shape;
  out.data.assign(pt.volume(), 0.0);
  get_output_into(ptensor, out.data.data(), static_cast<std::int64_t>(out.data.size()));
  return out;
}

// The pieces are read back through pinned staging and reconstructed (same
// cells as every adapter, reconstruct_cells) in parallel over cell rows.
void Executor::get_output_into(int ptensor, double* out, std::int64_t capacity) {
  const std::vector<int>* bufs = nullptr;
  for (const auto& o : prog_.outputs)
    if (o.first == ptensor) bufs = &o.second;
  if (!bufs) throw UsageError("ptensor " + std::to_string(ptensor) + " is not a plan output");
  const PTensor& pt = plan_.pt(ptensor);
  if (pt.volume() > capacity) throw UsageError("output buffer too small");
  for (auto& l : lanes_) {
    DeviceGuard dg(l.gpu);
    ck(cudaDeviceSynchronize(), "sync before readback");
  }
  Mask full;
  for (auto e : pt.shape) full.region.push_back({0, e});
  std::vector<std::pair<const Mask*, int>> pieces;
  std::map<int, std::int64_t> off;
  std::int64_t total = 0;
  for (int b : *bufs) {
    const BufferDesc& bd = prog_.buffers[b];
    if (!readable(bd.lane)) {
      throw UsageError("ptensor " + std::to_string(ptensor) + " has pieces on another rank; read buffers instead");
    }
    if (released(b)) {
      throw UsageError("ptensor " + std::to_string(ptensor) +
                       " was freed by the plan and its bytes reused in the step (REUSE_MEMORY)");
    }
    pieces.push_back({&bd.mask, b});
    off[b] = total;
    total += (bd.bytes + 255) / 256 * 256;
  }
  char* stage = host_stage(std::max<std::int64_t>(total, 1));
  for (int b : *bufs) {
    const BufferDesc& bd = prog_.buffers[b];
    DeviceGuard dg(lanes_[bd.lane].gpu);
    ck(cudaMemcpy(stage + off[b], buf_ptr(b), bd.bytes, cudaMemcpyDeviceToHost), "readback");
  }
  auto cells = reconstruct_cells(full, pt.shape, pieces, prog_.buffers, opt_.value_split_extension,
                                 "output " + std::to_string(ptensor));
  for (const auto& c : cells) {
    const int rank = c.rank;
    const std::int64_t inner_all = rank ? c.extents[rank - 1] : 1;
    const std::int64_t rows = inner_all ? c.elems() / inner_all : 0;
    // work item = (row, 64 Ki-element piece of it): collapsed cells are often
    // one long row
    constexpr std::int64_t kPiece = 1 << 16;
    const std::int64_t pieces_per_row = std::max<std::int64_t>(1, (inner_all + kPiece - 1) / kPiece);
    parallel_for(rows * pieces_per_row, std::min(inner_all, kPiece) * static_cast<std::int64_t>(c.terms.size()),
                 [&](std::int64_t lo, std::int64_t hi) {
      for (std::int64_t item = lo; item < hi; ++item) {
        const std::int64_t r = item / pieces_per_row, j0 = (item % pieces_per_row) * kPiece;
        const std::int64_t inner = std::min(kPiece, inner_all - j0);
        std::int64_t rem = r, doff = c.dst_offset;
        std::int64_t idx[kMaxCellRank] = {};
        for (int d = rank - 2; d >= 0; --d) {
          idx[d] = rem % c.extents[d];
          rem /= c.extents[d];
          doff += idx[d] * c.dst_strides[d];
        }
        const std::int64_t dstep = rank ? c.dst_strides[rank - 1] : 1;
        doff += j0 * dstep;
        for (std::int64_t j = 0; j < inner; ++j) out[doff + j * dstep] = 0.0;
        for (const auto& t : c.terms) {
          std::int64_t so = t.offset;
          for (int d = 0; d + 1 < rank; ++d) so += idx[d] * t.strides[d];
          const std::int64_t sstep = rank ? t.strides[rank - 1] : 1;
          so += j0 * sstep;
          const char* base = stage + off.at(t.buffer);
          const DType dt = prog_.buffers[t.buffer].dtype;
          for (std::int64_t j = 0; j < inner; ++j) {
            const double x = load_elem(base, dt, so + j * sstep);
            double& v = out[doff + j * dstep];
            v = t.fold == 0 ? v + x : t.fold == 1 ? v * x : t.fold == 2 ? std::max(v, x) : t.add ? v + x : x;
          }
        }
      }
    });
  }
}

}  // namespace planc_b200
