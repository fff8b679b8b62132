// Device kernels of the B200 plan executor (sm_100a).
//
// Sub-operators (reference eval_compute, proj/src/refexec.cpp:142-257):
//   gemm   matmul with transpose_a / transpose_b       (refexec.cpp:142-168)
//   ew     N-ary add / mul / max, same shape           (refexec.cpp:178-193)
//   reduce reduce-sum over one axis                    (refexec.cpp:194-215)
//   emb    embedding lookup / grad with vocab offset   (refexec.cpp:216-250)
// Adapters (reference reconstruct, refexec.cpp:102-140): one "box" kernel
// executes a static cell program — every destination cell is written once as
// 0 ∘ term_0 ∘ term_1 … (∘ = copy | add, in piece order). Sources may be
// local buffers, other lanes' buffers on the same GPU, or NVLink peer
// pointers, so split / concat / reduce-assemble / recv / every collective
// member output is one fused gather(-reduce) launch with no pack/unpack pass.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>

namespace planc_b200 {

enum DT : int { DT_F32 = 0, DT_BF16 = 1, DT_I32 = 2 };

constexpr int kBoxRank = 6;

struct DevTerm {
  const void* src;
  std::int64_t offset;
  std::int64_t str[kBoxRank];
  int op;  // 0 copy, 1 add, 2 mul, 3 max (elementwise instructions run as box cells)
  int pad;
};

struct DevCell {
  void* dst;  // destination buffer (cells of a batched launch write different buffers)
  std::int64_t ext[kBoxRank];
  std::int64_t dst_str[kBoxRank];
  std::int64_t dst_off;
  std::int64_t elems;
  int rank;
  int nterms;
  int term0;
  int vec;  // elements per vector access (1, 4 or 8), innermost contiguous
};

struct DevChunk {
  int cell;
  int pad;
  std::int64_t begin;  // in vector units
  std::int64_t count;  // in vector units
};

// Elementwise ops fused into a GEMM's epilogue (bf16): out = fold(op, in[0..n_in))
// where in[gemm_pos] is the GEMM's own bf16-rounded output value and the
// other operands are [m, n] row-major bf16 tensors read in place — the same
// bits the separate elementwise kernel would produce.
constexpr int kMaxEpiOps = 1;
constexpr int kMaxEpiIn = 4;
struct EpiOp {
  int op = 0;  // 0 add, 1 mul, 2 max, 3 gelu (unary), 4 gelu-grad (x, dy)
  int n_in = 0;
  int gemm_pos = 0;
  const void* in[kMaxEpiIn] = {};
  void* out = nullptr;
};
struct EpiParams {
  int n_ops = 0;
  EpiOp ops[kMaxEpiOps];
  // Non-GEMM operands, one prefetch slot each (at most kMaxEpiSlots): slot
  // s holds operand slot_in[s] of op slot_op[s].
  int n_slots = 0;
  int slot_op[2] = {0, 0};
  int slot_in[2] = {0, 0};
};
constexpr int kMaxEpiSlots = 2;

// Grouped launch: up to kMaxGemmGroup independent GEMMs of one shape share
// one persistent launch (one tile space, no per-GEMM wave tail).
constexpr int kMaxGemmGroup = 8;

struct GemmArgs {
  const void* A;
  const void* B;
  void* C;
  // group > 1: members 0..group-1 are (gA[i], gB[i], gC[i]); A/B/C unused.
  int group = 1;
  // Reduce-scatter epilogue (scatter > 0, group == 1): output rows
  // [i * scatter_rows, (i + 1) * scatter_rows) are stored to gC[i] — each a
  // [scatter_rows][n] buffer, typically on the rank that owns reduce-scatter
  // slice i (NVLink peer memory, plain 16-byte stores) — instead of C, tile
  // by tile as the GEMM runs: the transfer of the partial sums overlaps the
  // math. C is unused.
  int scatter = 0;
  std::int64_t scatter_rows = 0;
  const void* gA[kMaxGemmGroup] = {};
  const void* gB[kMaxGemmGroup] = {};
  void* gC[kMaxGemmGroup] = {};
  std::int64_t m, n, k;
  bool ta, tb;
  int da, db, dc;
  EpiParams epi;
  // Stream-K workspace (counters + fp32 partials), owned by the caller and
  // used by one launch at a time; null / too small -> data-parallel only.
  void* ws = nullptr;
  std::int64_t ws_bytes = 0;
  // Stream-K spends more SM-time than whole tiles for a shorter critical
  // path: worth it when the GPU has nothing else to run (one lane per GPU),
  // not when co-resident lanes fill the idle SMs with their own work.
  bool allow_streamk = true;
  int gpu_share = 1;  // lanes co-resident on this GPU (their launches run concurrently)
  // No workspace at all: the schedule is chosen among data-parallel
  // variants only (no stream-K, no split-K).
  bool no_workspace = false;
  // Gathered operands (all-gather / concat -> GEMM prologue, group == 1):
  // A (B) is the row-wise concatenation, in stored layout, of gather_a
  // (gather_b) pieces of gather_rows_a (_b) rows each; gather_maps = device
  // copy of their tensor maps (gemm_sm100_gather_maps; 16 slots).
  // With gather_cols_a (_b) > 0 the pieces are column blocks of that many
  // stored columns instead (gather_rows_* = 0).
  int gather_a = 0, gather_b = 0;
  std::int64_t gather_rows_a = 0, gather_rows_b = 0;
  std::int64_t gather_cols_a = 0, gather_cols_b = 0;
  const void* gather_a_ptr[kMaxGemmGroup] = {};
  const void* gather_b_ptr[kMaxGemmGroup] = {};
  const void* gather_maps = nullptr;
};

// Launch schedule of the tcgen05 GEMM: tile width, persistent grid, and the
// stream-K tail (tiles [dp_tiles, tiles) shared by sk_ctas CTAs in equal
// k-iteration ranges).
struct GemmSchedule {
  int bn = 256;
  int grid = 0;
  std::int64_t tiles = 0;
  std::int64_t num_k = 0;
  int dp_tiles = 0;
  int sk_ctas = 0;
  long long sk_iters = 0;
  std::int64_t counter_bytes = 0;
  // Split-K (small output, long k): every tile's k-blocks split into
  // `splits` equal ranges, one work item each; fp32 partials land in the
  // workspace (splits stacked copies of the padded output) and a separate
  // reduce kernel sums them in split order — every SM pulls a slice, no CTA
  // waits on another. 0 = off.
  int splits = 0;
  // Half-width tail (data-parallel only): tiles [dp_tiles, tiles) run as
  // half_items = 2 x (tiles - dp_tiles) tiles of 128 x bn/2.
  int half_items = 0;
  int occ = 1;  // CTAs per SM (2: small-k variant with a ~100 KB ring)
  std::int64_t ws_bytes = 0;  // 0 without stream-K / split-K
  double model_us = 0;
};

// Launchers (all asynchronous on `s`).
// `vec` != 0: every chunk's cell is innermost-contiguous with 16-byte
// aligned offsets (the executor splits a box program into vector / scalar
// launches).
// `max_rank` is the highest cell rank in the launch; every chunk covers at
// most kBoxChunkUnits vector units of one cell.
constexpr int kBoxChunkUnits = 1024;
void launch_box(int dtype, const DevCell* cells, const DevTerm* terms, const DevChunk* chunks,
                int nchunks, int vec, int max_rank, cudaStream_t s);
// Profiling: blocks stream s until the host writes a nonzero *flag
// (mapped pinned memory), at most 2 s.
void launch_host_gate(const unsigned* flag, cudaStream_t s);
void launch_ew(int op, int dtype, const void* const* ins, int nin, void* out, std::int64_t count, cudaStream_t s);
// reduce-sum over the middle axis of [outer][axis_len][inner]; column
// reductions (inner > 1) split the axis over blocks with fp32 partials in
// `scratch` (reduce_scratch_bytes; null = no split), summed in split order.
std::int64_t reduce_scratch_bytes(std::int64_t outer, std::int64_t axis_len, std::int64_t inner, int dtype);
int reduce_launches(std::int64_t outer, std::int64_t axis_len, std::int64_t inner, int dtype);
void launch_reduce(int dtype, const void* in, void* out, void* scratch, std::int64_t outer, std::int64_t axis_len,
                   std::int64_t inner, cudaStream_t s);
void launch_emb_lookup(int dtype, const int* idx, const void* table, void* out, std::int64_t n, std::int64_t rows,
                       std::int64_t h, std::int64_t lo, cudaStream_t s);
// Deterministic embedding-grad: per-block sorted segment sums, then one warp
// per output row adds the blocks' partials in block order (no atomics).
std::int64_t emb_grad_scratch_bytes(std::int64_t n, std::int64_t h);
void launch_emb_grad(int dtype, const int* idx, const void* gout, void* out, void* scratch, std::int64_t n,
                     std::int64_t rows, std::int64_t h, std::int64_t lo, cudaStream_t s);
void launch_gemm_simt(const GemmArgs& a, cudaStream_t s);
// Schema extension (program.hpp RowOp): softmax / softmax_grad / layernorm /
// layernorm_grad over `count / seg` contiguous segments of `seg` elements
// (one warp per segment, fp32 statistics, 16-byte vectors), gelu / gelu_grad
// elementwise. `b` is the second operand (dy) of the *_grad ops.
void launch_rowwise(int op, int dtype, const void* a, const void* b, void* out, std::int64_t count, std::int64_t seg,
                    float eps, cudaStream_t s);
void launch_convert(int dtype_out, void* out, const float* in, std::int64_t count, cudaStream_t s);
// Fused attention (attention.cu; schema extension): O = softmax(Q·Kᵀ/sqrt(dh)
// [+ causal mask])·V per (sequence of `seq` rows, head of `head_dim` cols)
// of a [rows, cols] bf16 piece. attention_unsupported: why a shape cannot
// run (nullptr when it can).
const char* attention_unsupported(std::int64_t rows, std::int64_t cols, std::int64_t seq, std::int64_t head_dim,
                                  int dtype);
void launch_attention(const void* q, const void* k, const void* v, void* o, std::int64_t rows, std::int64_t cols,
                      std::int64_t seq, std::int64_t head_dim, bool causal, int dtype, cudaStream_t s);
// Its gradient: a statistics pass (per-row log-sum-exp of the scores and
// D = rowsum(dO ∘ O) into `scratch`), then dQ (query-block CTAs) and dK / dV
// (key-block CTAs) — any of dq / dk / dv may be null.
std::int64_t attention_grad_scratch_bytes(std::int64_t rows, std::int64_t cols, std::int64_t head_dim);
void launch_attention_grad(const void* q, const void* k, const void* v, const void* o, const void* dout, void* dq,
                           void* dk, void* dv, void* scratch, std::int64_t rows, std::int64_t cols, std::int64_t seq,
                           std::int64_t head_dim, bool causal, int dtype, cudaStream_t s);
void launch_fill_zero_f32(float* p, std::int64_t count, cudaStream_t s);
// Device-to-device copy on the SMs (16-byte vectors): keeps the copy engines
// free for the host-link transfers running beside it (end-to-end mode).
void launch_copy_bytes(void* dst, const void* src, std::int64_t bytes, cudaStream_t s);

// Cross-rank ordering in peer-memory mode (program.hpp PeerSync). One
// launch first publishes the step epoch (*epoch) to every `sig` flag
// (release at system scope: the stream's earlier writes are visible to a
// peer that acquires the flag), then waits until every `wait` flag has
// reached the epoch (acquire, system scope). A wait that does not complete
// within timeout_ns records `code` in err[0] (host-mapped; err[1] the value
// seen, err[2] the epoch awaited, err[3..4] the flag address) and traps, so a
// broken schedule fails the context instead of hanging the GPU.
constexpr int kMaxPeerFlags = 16;
struct PeerFlags {
  int n_sig = 0;
  int n_wait = 0;
  unsigned* sig[kMaxPeerFlags] = {};
  const unsigned* wait[kMaxPeerFlags] = {};
  unsigned code = 0;  // reported on timeout (instruction id + 1, or ~0u for the step barrier)
};
void launch_peer_epoch(unsigned* epoch, cudaStream_t s);
void launch_peer_flags(const unsigned* epoch, const PeerFlags& f, unsigned long long timeout_ns, unsigned* err,
                       cudaStream_t s);

// tcgen05 / TMEM / TMA GEMM (gemm_sm100.cu).
bool gemm_sm100_eligible(const GemmArgs& a);
int gemm_sm100_tile_n(const GemmArgs& a);  // 256, 128 or 64
GemmSchedule gemm_sm100_schedule(const GemmArgs& a, int sms);
std::int64_t gemm_sm100_workspace_bytes(const GemmArgs& a);  // on the current device
int gemm_sm100_launches(const GemmArgs& a);                   // kernels per GEMM (2 with split-K)
void launch_gemm_sm100(const GemmArgs& a, cudaStream_t s);
// Host: the 16 tensor maps (A pieces, then B pieces at slot 8) of a GEMM
// with gathered operands, boxed for the launch the schedule will choose;
// the caller copies them to device memory and passes it as gather_maps.
constexpr int kGatherMapSlots = 2 * kMaxGemmGroup;
constexpr std::size_t kTensorMapBytes = 128;
void gemm_sm100_gather_maps(const GemmArgs& a, void* host_out /* kGatherMapSlots * 128 bytes */);
// 3xTF32 tcgen05 GEMM for fp32 operands and output (gemm_x3.cu); reached
// through the gemm_sm100_* entry points above.
bool gemm_x3_eligible(const GemmArgs& a);
GemmSchedule gemm_x3_schedule(const GemmArgs& a, int sms);
void launch_gemm_x3(const GemmArgs& a, cudaStream_t s);

// Dispatch: tcgen05 path when eligible, SIMT tile kernel otherwise (a
// group then runs member by member).
inline void launch_gemm(const GemmArgs& a, cudaStream_t s, bool allow_tc, bool* used_tc) {
  bool tc = allow_tc && gemm_sm100_eligible(a);
  if (used_tc) *used_tc = tc;
  if (a.scatter > 0 && !tc) throw std::runtime_error("reduce-scatter GEMM epilogue needs the tensor-core path");
  if (tc) {
    launch_gemm_sm100(a, s);
  } else if (a.group > 1) {
    for (int i = 0; i < a.group; ++i) {
      GemmArgs one = a;
      one.group = 1;
      one.A = a.gA[i];
      one.B = a.gB[i];
      one.C = a.gC[i];
      launch_gemm_simt(one, s);
    }
  } else {
    launch_gemm_simt(a, s);
  }
}

}  // namespace planc_b200
