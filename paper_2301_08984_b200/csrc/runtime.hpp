// B200 plan executor runtime: device memory, per-lane streams, cross-lane
// events, CUDA-graph capture of one plan step, inputs/outputs.
//
// The drop-in replacement for the reference's
//   TensorMap planc::run_plan(const ExecutionPlan&, const TensorMap&)
// (reference include/planc/refexec.hpp:43, proj/src/refexec.cpp:361-557).
// One Executor owns one plan; every plan lane ("device" of the plan) is
// mapped to a CUDA device ordinal (several lanes may share one B200, each
// with its own streams, which is how multi-device plans are parity-tested on
// one GPU). Lanes on different GPUs of one process read each other's buffers
// through NVLink peer mappings inside the same fused box kernels.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <set>
#include <memory>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "plan.hpp"
#include "program.hpp"

namespace planc_b200 {

struct HostTensor {
  std::vector<std::int64_t> shape;
  std::vector<double> data;
};

struct KernelStat {
  std::string kind;  // gemm_tc, gemm_simt, ew, reduce, emb, box_local, box_coll, box_recv
  int launches = 0;
  double ms = 0;
  double flops = 0;
  double bytes = 0;
  double wire_bytes = 0;
};

// Streams per lane. Instructions of a lane are spread over them so that only
// true data dependencies (and sync edges) order work: independent GEMMs,
// elementwise ops and adapters of one lane overlap on the GPU.
constexpr int kLaneStreams = 8;  // capacity; streams used per lane: ExecOptions / PLANC_B200_STREAMS (default 4)

struct ExecOptions {
  bool use_graph = true;       // capture one step into a CUDA graph
  bool allow_tensor_cores = true;
  bool value_split_extension = true;
  int streams_per_lane = 4;             // 1 = issue a lane strictly in plan order
  bool fuse_epilogues = true;           // elementwise consumers computed in GEMM epilogues
  bool fuse_act = false;                // ...GELU / GELU-grad as well (PLANC_B200_FUSE_ACT)
  bool group_gemms = true;              // same-shape independent GEMMs in one grouped launch
  bool alias_copies = true;             // same-GPU whole-buffer copies (recv, identity) become aliases
  bool alias_views = true;              // ...and contiguous sub-range copies (splits) views of their source
  bool scatter_allreduce = true;        // all-reduce partials leave the GEMM epilogue as reduce-scatter slices
  bool reuse_memory = false;            // timed mode: bytes the plan frees are reused within the step
  // Independent adapter (box) and elementwise instructions of one GPU in
  // shared launches. Off by default: it couples the lanes sharing a GPU
  // (C4 5.55 -> 7.19 ms, C5 2.68 -> 4.48 ms per step measured,
  // profiles/r02/ab_batch.jsonl); PLANC_B200_BATCH=1 / 2 (per lane) for A/B.
  bool batch_boxes = false;
  bool gather_operands = true;          // concat / all-gather feeding only GEMMs: GEMMs read the pieces in place
  bool fuse_box_ew = true;              // elementwise ops on a pure-copy adapter output run inside the box
  bool gather_cols = false;             // column-piece gathers too (opt-in)
};

// ProgramOptions as the executor uses them: epilogue fusion only for GEMMs
// the tcgen05 path takes (it implements the fused epilogue).
ProgramOptions program_options(bool value_split_extension, bool fuse_epilogues);

// One-process-per-GPU mode: this process owns the lanes with
// lane_rank[l] == rank, all on `local_gpu`; pieces owned by other ranks
// arrive through NCCL point-to-point exchange steps (program.hpp localize).
//
// With `peer_memory` there is no NCCL: every rank maps the other ranks' lane
// arenas (CUDA IPC, NVLink) and runs the global program's instructions of its
// own lanes; box terms read other ranks' pieces in place and cross-rank
// dependencies are device flags (program.hpp PeerSync). The arenas are
// exchanged by the caller between construction and the first step
// (peer_export on every rank, all-gather, peer_import).
struct RankConfig {
  int rank = 0;
  int world = 1;
  std::vector<int> lane_rank;
  int local_gpu = 0;
  unsigned char nccl_id[128] = {0};
  bool peer_memory = false;
};

// Flag block layout (32-bit words): [0] step epoch, [kFlagBarrier + r] step
// barrier slot written by rank r, [kFlagReady + i] ready slot i.
constexpr int kPeerMaxRanks = 64;
constexpr std::size_t kFlagBarrier = 64;
constexpr std::size_t kFlagReady = kFlagBarrier + kPeerMaxRanks;

// Peer-memory export blob: header + one cudaIpcMemHandle per plan lane (zero
// for lanes another rank owns) + the rank's flag block handle.
constexpr std::int64_t kPeerBlobHeader = 32;
inline std::int64_t peer_blob_bytes(int num_lanes) {
  return kPeerBlobHeader + static_cast<std::int64_t>(sizeof(cudaIpcMemHandle_t)) * (num_lanes + 1);
}

class Executor {
 public:
  Executor(const std::string& plan_json, const std::vector<int>& lane_gpu, const ExecOptions& opt,
           const RankConfig* rank = nullptr);
  ~Executor();
  Executor(const Executor&) = delete;
  Executor& operator=(const Executor&) = delete;

  const ExecutionPlan& plan() const { return plan_; }
  const Program& program() const { return prog_; }

  void set_input(int ptensor, const double* data, const std::vector<std::int64_t>& shape);
  // Runs `iters` plan steps; returns mean device milliseconds per step
  // (CUDA events on the origin stream, after one untimed warm-up when
  // iters > 0 and the graph is not yet built).
  double run(int iters);
  // End-to-end: per step, H2D of every non-weight graph-input placement from
  // pinned host memory, the step, D2H of every terminal output piece.
  double run_e2e(int iters, std::int64_t* h2d_bytes, std::int64_t* d2h_bytes);
  // Per-kernel-family device time of one eagerly issued, serialised step.
  std::vector<KernelStat> profile();
  // Measured timeline of one eagerly issued step (streams and overlap as in
  // a timed step), in the reference simulator's timeline_json shape
  // (simulate.cpp:373-383): [{device, op, kind, start, end}] in seconds.
  std::string timeline_json();
  HostTensor get_output(int ptensor);
  // Reassembles a produced pTensor straight into `out` (volume elements).
  void get_output_into(int ptensor, double* out, std::int64_t capacity);
  // Raw value of one device buffer (a vTensor piece) as doubles.
  std::vector<double> read_buffer(int buffer);
  std::vector<int> output_ids() const;
  // Graph-input pTensors this process places (rank mode: its own lanes').
  std::vector<int> input_ids() const;
  int kernels_per_step() const { return kernels_per_step_; }
  int gemm_tc_launches() const { return gemm_tc_per_step_; }
  bool graph_captured() const { return graph_exec_ != nullptr; }
  // Peer-memory mode: this rank's blob, and every rank's blobs (rank order,
  // `world` x peer_blob_bytes) to map the other ranks' arenas and flags.
  std::vector<unsigned char> peer_export() const;
  void peer_import(const unsigned char* blobs, std::int64_t blob_bytes);

 private:
  struct LaneRt {
    int gpu = 0;
    char* arena = nullptr;
    cudaStream_t stream[kLaneStreams] = {};
    // Stream-K GEMM workspace per stream (GEMMs on one stream never overlap).
    void* gemm_ws[kLaneStreams] = {};
    std::int64_t gemm_ws_bytes[kLaneStreams] = {};
  };
  struct BoxLaunch {
    DevCell* cells = nullptr;
    DevTerm* terms = nullptr;
    DevChunk* chunks = nullptr;
    int nchunks = 0;
    int vec = 0;
    int max_rank = 1;
    int dtype = 0;
    // host copies (merged into batched launches)
    std::vector<DevCell> h_cells;
    std::vector<DevTerm> h_terms;
    std::vector<DevChunk> h_chunks;
  };
  // Adapter batching (ExecOptions::batch_boxes): box instructions of one GPU
  // that are pending together in issue order — none depends on another,
  // nothing issued so far consumes them — run as one launch per (element
  // type, vector width, cell rank): their cell tables concatenated, each
  // cell writing its own destination. The batch runs on one of the GPU's
  // batch streams after every member's dependencies; its event orders every
  // member's consumers. Many small adapter launches (split / concat /
  // all-to-all pieces of co-sharded and pipelined plans) become a few.
  struct BoxBatch {
    std::vector<int> members;
    int gpu = 0;
    cudaStream_t stream = nullptr;
    std::vector<BoxLaunch> launches;
    cudaEvent_t done = nullptr;
  };
  struct InstrRt {
    std::vector<BoxLaunch> box;
    bool aliased = false;        // whole-buffer copy on one GPU: output shares the source's memory
    cudaEvent_t done = nullptr;  // recorded when a later instruction on another stream depends on it
    float* scratch = nullptr;
    void* gather_maps = nullptr;  // device tensor maps of a gathered-operand GEMM's pieces
  };

  void* buf_ptr(int b) const;
  bool released(int b) const;  // REUSE_MEMORY: bytes taken over by a later buffer
  void plan_aliases();
  bool gemm_streamk_ok(int lane) const;
  int gpu_share(int lane) const;  // the lane has its GPU to itself
  cudaStream_t stream_of(const Instr& in) const;
  void build_box_tables();
  void plan_box_batches();
  void build_ew_tables();
  void upload_box(BoxLaunch& bl, int gpu);
  void launch_batch(int b);
  cudaStream_t issued_stream(int id) const;
  cudaEvent_t done_event(int id) const;
  void place_inputs();
  void issue_step(bool timing_events, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* ev);
  void launch_instr(const Instr& in, cudaStream_t s);
  GemmArgs gemm_args(const Instr& in) const;
  void build_gather_maps();
  void ensure_graph();

  bool local(int buffer) const { return owned_[prog_.buffers[buffer].lane]; }
  // Readable here: owned, or mapped from its rank in peer-memory mode.
  bool readable(int lane) const { return owned_[lane] || (peer_ && peer_ready_); }
  void launch_xfer(const Instr& in, cudaStream_t s);
  // Peer-memory mode: flag launches around one instruction / a step.
  void peer_check_ready() const;
  void peer_wait(int id, cudaStream_t s);
  void peer_signal(int id, cudaStream_t s);
  void peer_step_begin(cudaStream_t s);
  void peer_step_end(cudaStream_t s);
  void peer_flags(const std::vector<unsigned*>& sig, const std::vector<const unsigned*>& wait, unsigned code,
                  cudaStream_t s);
  void sync_all(const char* what);
  void join_lanes();
  void check_sync(cudaError_t e, const char* what) const;

  ExecutionPlan plan_;
  Program prog_;
  ExecOptions opt_;
  bool rank_mode_ = false;
  RankConfig rc_;
  std::vector<bool> owned_;     // per lane: runs in this process
  std::vector<int> exec_lane_;  // per instruction: lane whose streams run it here (-1: elsewhere)
  std::vector<int> exec_stream_;  // per instruction: stream index within its lane
  void* comm_ = nullptr;        // ncclComm_t in rank mode (NCCL exchange steps)
  // Peer-memory rank mode.
  bool peer_ = false;
  bool peer_ready_ = false;               // other ranks' arenas / flags mapped
  PeerSync psync_;
  unsigned* flags_ = nullptr;             // this rank's flag block (epoch, barrier, ready slots)
  std::vector<unsigned*> peer_flags_;     // per rank: its flag block as mapped here
  std::vector<void*> ipc_mapped_;         // cudaIpcOpenMemHandle results (closed, not freed)
  std::vector<bool> lane_mapped_;         // lane arena is an IPC mapping
  unsigned* peer_err_ = nullptr;          // host-mapped timeout report
  unsigned long long peer_timeout_ns_ = 0;
  int first_lane_ = 0;          // first lane this process runs (origin stream's device)
  std::vector<LaneRt> lanes_;
  std::vector<InstrRt> irt_;
  std::vector<int> alias_;  // per buffer: -1, or the buffer whose memory it shares
  std::vector<std::int64_t> alias_off_;  // per aliased buffer: byte offset into its source
  std::vector<int> gpus_;  // distinct devices
  std::vector<void*> table_allocs_;
  std::vector<BoxBatch> batches_;
  std::vector<int> batch_of_;                    // per instruction: its batch, or -1
  std::vector<std::vector<int>> flush_before_;   // per issue position: batches launched before it
  std::vector<int> flush_end_;                   // batches launched after the last instruction
  std::map<int, std::vector<cudaStream_t>> batch_streams_;  // per GPU
  std::vector<cudaEvent_t> batch_join_;
  std::vector<bool> overwritten_;       // REUSE_MEMORY: buffers whose bytes a later buffer takes
  std::set<int> placed_;                // graph inputs placed by set_input
  void* host_stage_ = nullptr;          // pinned staging for set_input / get_output conversions
  std::int64_t host_stage_bytes_ = 0;
  char* host_stage(std::int64_t bytes);
  cudaStream_t origin_ = nullptr;
  cudaEvent_t ev_begin_ = nullptr, ev_end_ = nullptr;
  std::vector<cudaEvent_t> lane_join_;
  cudaGraph_t graph_ = nullptr;
  cudaGraphExec_t graph_exec_ = nullptr;
  int kernels_per_step_ = 0;
  int gemm_tc_per_step_ = 0;
  // e2e staging
  std::vector<void*> pinned_in_, pinned_out_;
  std::vector<int> e2e_in_bufs_, e2e_out_bufs_;
  std::vector<void*> e2e_stage_in_[2], e2e_stage_out_[2];  // device staging, double-buffered
  cudaStream_t h2d_stream_ = nullptr, d2h_stream_ = nullptr;
  cudaEvent_t ev_h2d_[2] = {}, ev_in_free_[2] = {}, ev_out_ready_[2] = {}, ev_out_free_[2] = {};
};

}  // namespace planc_b200
