// Host-side plan compiler: ExecutionPlan -> per-lane device programs.
//
// Replaces the interpretation loop of the reference's run_plan
// (proj/src/refexec.cpp:361-557) with a one-time lowering:
//   * every producer-output vTensor gets its own device buffer on its lane;
//     consumer views alias their feed (plan.feeds, exact mask match) and
//     graph-input views get a placement buffer (refexec.cpp:366-376);
//   * every task becomes zero or more device instructions: sub-operator
//     kernels for compute ops (eval_compute, refexec.cpp:142-257) and
//     box-copy/accumulate "cell" programs for every adapter — split, concat,
//     reduce-assemble, recv and each collective member's output — restating
//     reconstruct (refexec.cpp:102-140) as a static schedule of
//     (destination box, ordered source terms, copy|add) cells;
//   * the host issue order is the reference's round-robin lane-cursor loop
//     (refexec.cpp:483-522) with "issued" as readiness, so pairing deadlocks
//     are reported exactly where run_plan reports them (refexec.cpp:523-530);
//   * cross-lane dependencies (send->recv, collective rendezvous, sync_edges)
//     become explicit producer->consumer instruction edges, realised on the
//     GPU as CUDA events between per-lane streams.
// Nothing in this file touches CUDA; the lowering is unit-tested on CPU.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "plan.hpp"

namespace planc_b200 {

enum class DType : std::uint8_t { f32 = 0, bf16 = 1, i32 = 2 };
inline std::int64_t dtype_size(DType d) { return d == DType::bf16 ? 2 : 4; }
const char* dtype_name(DType d);

constexpr int kMaxCellRank = 6;

struct BufferDesc {
  int id = 0;
  int lane = 0;
  int ptensor = 0;
  Mask mask;
  DType dtype = DType::f32;
  std::vector<std::int64_t> shape;  // region extents, row-major dense
  std::int64_t elems = 0;
  std::int64_t bytes = 0;
  std::int64_t offset = 0;     // byte offset inside the lane arena
  bool graph_input = false;    // filled by placement from host inputs
  bool weight = false;         // graph input of kind weight / optimizer state
  int producer = -1;           // instruction writing it (-1: placement)
  int vt = -1;                 // producing vTensor (or first placed view)
  bool dead = false;           // replaced (reduce-scatter GEMM epilogue): never written nor read
};

// One source of a cell: a box of another buffer, copied or accumulated.
struct Term {
  int buffer = 0;
  std::int64_t offset = 0;  // element offset of the cell origin in the source
  std::int64_t strides[kMaxCellRank] = {0};
  bool add = false;
  // >= 0: an elementwise op folded into the box (fuse_box_elementwise):
  // value = value (EwOp add | mul | max) term, in the ew kernel's fp32 fold.
  int fold = -1;
};

// Destination box of an adapter output with its ordered source terms.
// value = 0; for term in terms: value = term (copy) | value += term (add)
// | value = value fold term.
struct Cell {
  int rank = 0;
  std::int64_t extents[kMaxCellRank] = {0};
  std::int64_t dst_offset = 0;
  std::int64_t dst_strides[kMaxCellRank] = {0};
  std::vector<Term> terms;
  std::int64_t elems() const {
    std::int64_t v = 1;
    for (int i = 0; i < rank; ++i) v *= extents[i];
    return v;
  }
};

constexpr int kMaxGemmGroupInstr = 8;  // members of one grouped GEMM launch (kernels.cuh kMaxGemmGroup)

enum class InstrKind { gemm, ew, reduce, emb_lookup, emb_grad, box, xfer, nop, rowwise, attention };

// Row-wise / activation sub-operators of the schema extension.
enum class RowOp { softmax = 0, softmax_grad = 1, layernorm = 2, layernorm_grad = 3, gelu = 4, gelu_grad = 5 };

// One cross-rank piece movement of an exchange step (one-process-per-GPU
// mode): the whole `src` buffer of lane src_lane lands in `dst` (a shadow
// buffer on dst_lane) before the box program that reads it.
struct Xfer {
  int src = 0;
  int dst = 0;
  int src_lane = 0;
  int dst_lane = 0;
  std::int64_t bytes = 0;
};
const char* instr_kind_name(InstrKind k);

// gelu / gelu_grad occur only as fused GEMM epilogue ops (Instr::FusedEw),
// taken over from RowOp::gelu / gelu_grad instructions.
enum class EwOp { add = 0, mul = 1, max = 2, gelu = 3, gelu_grad = 4 };

struct Instr {
  int id = 0;
  InstrKind kind = InstrKind::nop;
  int lane = 0;
  int stream = 0;  // 0 = lane compute stream, 1 = lane adapter stream
  int op = -1;     // index into plan.ops
  std::vector<int> in_bufs;
  std::vector<int> out_bufs;
  std::vector<int> deps;  // producer instructions (all, incl. same stream)
  // gemm: C[m,n] = op(A)·op(B); a grouped GEMM (group > 1) computes
  // out_bufs[i] = op(in_bufs[2i])·op(in_bufs[2i+1]) for i < group.
  std::int64_t m = 0, n = 0, k = 0;
  int group = 1;
  // gemm with a reduce-scatter epilogue: rows [i*scatter_rows, (i+1)*scatter_rows)
  // of the product go to out_bufs[i] (receive buffers on the slice owners' lanes).
  int scatter = 0;
  std::int64_t scatter_rows = 0;
  bool ta = false, tb = false;
  // ew
  EwOp ew = EwOp::add;
  std::int64_t count = 0;
  // reduce: in [outer, axis_len, inner] -> out [outer, inner]
  std::int64_t outer = 0, axis_len = 0, inner = 0;
  // embedding: idx[n_idx], table/grad rows, width h, vocab offset lo
  std::int64_t n_idx = 0, rows = 0, h = 0, lo = 0;
  // rowwise: `count` elements = count / seg segments of `seg` contiguous
  // elements (gelu / gelu_grad: seg unused); in_bufs = x (or y) [, dy]
  RowOp row_op = RowOp::softmax;
  std::int64_t seg = 0;
  double eps = 0;
  // attention: in_bufs = Q, K, V, out_bufs = O, each a [rows, cols] piece of
  // whole sequences (att_seq rows) and whole heads (att_dh columns).
  // attention gradient (att_grad != 0): in_bufs = Q, K, V, O, dO; att_out[0..2]
  // = the dQ / dK / dV buffers it writes (-1: not requested) — the
  // attention-grad ops of one lane with the same operands share one
  // instruction (one statistics pass); out_bufs lists the written ones.
  std::int64_t att_rows = 0, att_cols = 0, att_seq = 0, att_dh = 0;
  bool causal = false;
  int att_grad = 0;
  int att_out[3] = {-1, -1, -1};
  // box
  std::vector<Cell> cells;
  int coll_group = -1;  // collective group a box instruction belongs to
  // xfer (exchange step, identical on every rank): the piece movements; or,
  // when `allreduce`, one whole-buffer sum across all ranks where each
  // entry is a member lane's (src = its partial input, dst = its output)
  // and every dst receives the sum of all srcs (ncclAllReduce).
  std::vector<Xfer> xfers;
  bool allreduce = false;
  // gemm: elementwise consumers computed in this GEMM's epilogue (the fused
  // ew instruction becomes a nop). Operand `gemm_pos` of each is the GEMM's
  // own (output-rounded) value; the others are read in place.
  struct FusedEw {
    int ew_instr = -1;
    EwOp op = EwOp::add;
    std::vector<int> in_bufs;  // in fold order; in_bufs[gemm_pos] == this GEMM's output
    int gemm_pos = 0;
    int out_buf = -1;
  };
  std::vector<FusedEw> fused;
  // gemm operand gathered in place (all-gather / concat -> GEMM prologue,
  // SURVEY §8f rank 1): operand j (0 = A, 1 = B) is the row-wise
  // concatenation, in its stored layout, of gather[j] (pieces of
  // gather_rows[j] rows each, in order) — the concatenating box instruction
  // is gone (a nop), its output buffer is dead and in_bufs[j] names the
  // first piece; the GEMM's TMA loads read each piece where its producer
  // left it.
  // ...or, with gather_cols[j] > 0, the column-wise concatenation of pieces
  // of gather_cols[j] stored columns each (DAP's column halves -> GEMM: a
  // K- or N-split of the operand); gather_rows[j] is then 0.
  std::vector<int> gather[2];
  std::int64_t gather_rows[2] = {0, 0};
  std::int64_t gather_cols[2] = {0, 0};
  // accounting (algorithmic, from masks)
  double flops = 0;
  double bytes = 0;       // HBM bytes read + written
  double wire_bytes = 0;  // NCCL bus-bandwidth convention bytes (adapters)
  std::string label;
};

struct ProgramOptions {
  bool value_split_extension = true;  // V(m*v) -> V(v) sums
  bool honor_sync_edges = true;
  // Fuse elementwise ops that consume a fresh GEMM output on the same lane
  // into that GEMM's epilogue (local form), for GEMMs the
  // predicate accepts (the tensor-core path implements the fused epilogue).
  bool fuse_epilogues = false;
  // ...GELU / GELU-grad too (opt-in: bit-identical, but measured slower than
  // the separate pass on C2x, profiles/r01/ab_fuse_gelu.jsonl).
  bool fuse_act = false;
  // ...not into long GEMMs (m·n·k >= 2^34) of at most this many 128x256
  // output tiles (one wave: every CTA has a single tile, so the fused
  // epilogue cannot overlap a next tile's MMAs and is exposed; the separate
  // elementwise pass runs beside other work instead, and the GEMM may take
  // split-K / stream-K). 0 = fuse regardless.
  int fuse_min_tiles = 148;
  // All-reduce groups (every member output = the sum of the same k whole
  // member inputs) as two box phases: member j sums slice j of all inputs
  // (reduce-scatter), then copies the other members' reduced slices
  // (all-gather). Same terms in the same order, so the same bits; each
  // member reads ~2n instead of k*n (over NVLink when members sit on other
  // GPUs or ranks).
  bool two_phase_allreduce = true;
  // ...and when every member's partial comes straight from a GEMM (a
  // row-parallel / value-split matmul consumed only by the all-reduce), that
  // GEMM's epilogue stores each row slice into a receive buffer on the lane
  // owning that slice (tile by tile, over NVLink when the owner is another
  // GPU): the reduce-scatter transfer rides in the GEMM, the phase-1 box sums
  // local pieces in the reference's order. Needs the tensor-core predicate.
  bool scatter_allreduce = true;
  // Independent GEMMs of one shape on one lane that become ready together
  // (each one's dependencies are ancestors of the other's) run as one
  // grouped tensor-core launch (one tile space: no per-GEMM wave tail, one
  // launch instead of several) — for GEMMs the predicate accepts.
  bool group_gemms = true;
  // A box instruction that only concatenates whole row blocks of its pieces
  // into a buffer read by nothing but tensor-core GEMMs (as an operand) is
  // dropped: those GEMMs read the pieces in place (Instr::gather) — the
  // all-gather / concat -> GEMM prologue. Single-process and peer-memory
  // modes (the pieces must be addressable by the GEMM's lane).
  bool gather_operands = true;
  // ...column pieces too (opt-in, flag GATHER_COLS): along K only; measured
  // ~3 % slower on C5 than the materialised concat (profiles/r02/ab_col_gather.jsonl).
  bool gather_cols = false;
  // An elementwise op (add / mul / max) whose operand is the output of a
  // pure-copy box instruction (an all-to-all / all-gather / layout adapter)
  // read by nothing else runs inside that box: the other operands become
  // fold terms of every cell and the box writes the op's output — one launch
  // and one HBM round trip of the adapter output fewer, the same bits (the
  // copy is exact, the fold is the ew kernel's fp32 fold in operand order).
  bool fuse_box_ew = true;
  bool (*gemm_groupable)(const Instr& gemm, DType a, DType b, DType c) = nullptr;
  bool (*gemm_fusable)(const Instr& gemm, DType a, DType b, DType c) = nullptr;
};

struct Program {
  int num_lanes = 0;
  std::vector<int> lane_device;          // plan device id per lane
  std::vector<BufferDesc> buffers;
  std::vector<Instr> instrs;
  std::vector<int> issue_order;          // instruction ids, global host order
  std::vector<std::int64_t> lane_arena_bytes;
  std::vector<int> vt_buffer;            // vt id -> buffer (-1 if none)
  // Output reassembly (refexec.cpp:532-556): per produced pTensor, the
  // deduplicated (region, value part) producer buffers, in op order.
  struct OutputPiece {
    int buffer;
  };
  std::vector<std::pair<int, std::vector<int>>> outputs;  // pt -> buffers
  std::vector<int> graph_inputs;         // pTensor ids needing host data
  double total_flops = 0, total_bytes = 0, total_wire_bytes = 0;
  std::vector<double> lane_flops, lane_bytes, lane_wire_bytes;

  std::string describe_json() const;
};

Program build_program(const ExecutionPlan& plan, const ProgramOptions& opt = {});

// Epilogue fusion pass (run by build_program when opt.fuse_epilogues): an
// elementwise op whose operand is a bf16 GEMM output on the same lane, whose
// other operands are ready before that GEMM, is computed in the GEMM's
// epilogue; the op's instruction becomes a nop.
void fuse_gemm_epilogues(Program& p, const ProgramOptions& opt);

// GEMM grouping pass (run by build_program after fusion when
// opt.group_gemms): members become nops, the first member of each group
// carries every member's operands and results.
void group_gemms(Program& p, const ProgramOptions& opt);

// Gather-prologue pass (opt.gather_operands; run after epilogue fusion,
// before grouping): see ProgramOptions::gather_operands.
void gather_gemm_operands(Program& p, const ProgramOptions& opt);
// Box -> elementwise fusion pass (opt.fuse_box_ew; after epilogue fusion).
void fuse_box_elementwise(Program& p, const ProgramOptions& opt);

// The two-phase all-reduce pass (ProgramOptions::two_phase_allreduce), run
// by build_program before epilogue fusion. Rebuilds the program in issue
// order (instruction ids stay dense and ascending along the issue order).
void two_phase_allreduce(Program& p, const ProgramOptions& opt = {});

// Peer-memory one-process-per-GPU mode: every rank runs the global program's
// instructions of its own lanes and reads other ranks' buffers in place
// (CUDA IPC mappings of their arenas over NVLink). A dependency edge between
// instructions of different ranks becomes a device flag: after the producer,
// its rank writes the step epoch into a ready slot owned by the consumer's
// rank; before the consumer, its rank waits until that slot reaches the
// epoch. Slots are numbered per consumer rank in instruction order, so every
// rank derives the same numbering. (Cross-step reuse of a buffer is ordered by
// a step-end barrier across ranks.)
struct PeerSync {
  std::vector<std::vector<int>> waits;                    // per instr: ready slots on its own rank
  std::vector<std::vector<std::pair<int, int>>> signals;  // per instr: (consumer rank, slot)
  std::vector<int> slots;                                 // per rank: number of ready slots
};
PeerSync peer_sync_schedule(const Program& p, const std::vector<int>& lane_rank);

// One-process-per-GPU lowering: the same global program on every rank, with
// every box term that lives on another rank's lane redirected to a shadow
// buffer on the consuming lane and filled by an `xfer` exchange step placed
// just before its consumers in the global issue order (all box outputs of a
// collective group share one step). Every rank derives the identical step
// sequence, so the per-rank point-to-point groups are matched in order and
// cannot deadlock. `lane_rank[l]` is the rank owning lane l; instructions of
// lanes other ranks own stay in the program (the caller skips them).
Program localize(const Program& global, const std::vector<int>& lane_rank);

// Stream of each instruction within its lane (exec_lane[i] < 0: not run in
// this process): continue the stream of the most recent dependency that
// ended a stream's chain, else take the least recently used of `ns` streams.
std::vector<int> assign_streams(const Program& p, const std::vector<int>& exec_lane, int ns);

// Static memory plan of one step for timed mode (the plan's `free` tasks,
// refexec.cpp:416-417 / insert_frees materialize.cpp:340-465, made real):
// a buffer the plan frees (or an executor-internal buffer) may hand its
// arena bytes to a later buffer once every use of it — reads and writes,
// through aliases, on any lane's stream — is ordered before every write of
// the newcomer by the step's dependency edges and stream order (vector
// clocks over the (lane, stream) queues). Graph inputs, terminal outputs
// and buffers the plan never frees keep their own bytes.
struct MemoryPlan {
  std::vector<std::int64_t> offset;      // per buffer: byte offset in its lane arena
  std::vector<std::int64_t> lane_bytes;  // per lane: arena size
  std::vector<bool> overwritten;         // per buffer: its bytes are reused later in the step
  std::int64_t bytes_before = 0, bytes_after = 0;
  int reused = 0;                        // buffers placed in released bytes
};
MemoryPlan plan_memory(const Program& p, const ExecutionPlan& plan, const std::vector<int>& exec_lane,
                       const std::vector<int>& exec_stream, int ns, const std::vector<int>& alias);

// Reconstruct-as-cells (refexec.cpp:102-140): target buffer box from ordered
// pieces. Exposed for tests.
std::vector<Cell> reconstruct_cells(const Mask& target, const std::vector<std::int64_t>& target_shape,
                                    const std::vector<std::pair<const Mask*, int>>& pieces,
                                    const std::vector<BufferDesc>& buffers, bool vv_extension,
                                    const std::string& ctx);

}  // namespace planc_b200
