/*
 * planc_b200 — C ABI of the B200-native SuperScaler plan executor.
 *
 * Drop-in boundary for the reference's plan-execution path:
 *
 *   TensorMap planc::run_plan(const ExecutionPlan& plan, const TensorMap& inputs)
 *     reference /root/reference/proj/include/planc/refexec.hpp:43,
 *     implementation proj/src/refexec.cpp:361-557
 *
 * The plan crosses the ABI in its wire form, the plan.json text produced by
 * planc::save_plan (proj/src/simulate.cpp:492-602) and read with the same keys
 * as planc::load_plan (simulate.cpp:604-739). TensorMap values cross as
 * dense row-major double arrays keyed by pTensor id, exactly the
 * ConcreteTensor{shape, data} layout (refexec.hpp:19-32).
 *
 * Error behaviour mirrors the reference's exception classes
 * (proj/include/planc/util.hpp:17-29) as return codes; the message is
 * available from planc_b200_last_error():
 *   PLANC_B200_OK        0
 *   PLANC_B200_EINTERNAL 1  InternalError (no feed, pairing deadlock,
 *                            uncovered reconstruct region, ...)
 *   PLANC_B200_ECUDA     2  CUDA runtime / device failure
 *   PLANC_B200_EUSAGE    4  SchemaError / UsageError (malformed plan, missing
 *                            input, partial-value graph input, unsupported op
 *                            kind) — the CLI's exit code 4 (tools/planc.cpp:18-20)
 * No exception crosses the ABI. One handle is used from one host thread.
 */
#ifndef PLANC_B200_H_
#define PLANC_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PLANC_B200_OK 0
#define PLANC_B200_EINTERNAL 1
#define PLANC_B200_ECUDA 2
#define PLANC_B200_EUSAGE 4

/* Open flags. */
#define PLANC_B200_NO_GRAPH 0x1u        /* issue eagerly instead of replaying a CUDA graph */
#define PLANC_B200_NO_TENSOR_CORES 0x2u /* force the SIMT GEMM (debug / A-B checks) */
#define PLANC_B200_STRICT_VALUE 0x4u    /* reference value-part rule only: V(m*v)->V(v) pieces are
                                           skipped like refexec.cpp:110-117 instead of summed */
#define PLANC_B200_FUSE_EPILOGUES 0x10u /* (default, kept for compatibility) an elementwise op consuming a
                                           fresh bf16 GEMM output on the same lane runs in that GEMM's
                                           epilogue — same bits as the separate kernel */
#define PLANC_B200_FUSE_ACT 0x400u      /* also run GELU / GELU-grad in the producing GEMM's epilogue
                                           (opt-in: same bits, measured slower on C2x) */
#define PLANC_B200_REUSE_MEMORY 0x800u  /* timed mode: the bytes of every buffer the plan frees (free tasks,
                                           refexec.cpp:416-417) are reused within the step once all its uses
                                           are ordered before the new writer; outputs whose bytes were reused
                                           are unavailable (UsageError). Single-process executor only */
#define PLANC_B200_NO_FUSION 0x80u      /* every elementwise op its own kernel (no epilogue fusion) */
#define PLANC_B200_NO_SCATTER 0x200u    /* all-reduce partials stored whole by their GEMM and pulled by the
                                           reduce-scatter phase (default: a GEMM whose output only feeds an
                                           all-reduce stores each row slice straight into the receive buffer
                                           of the lane owning it — the transfer rides in the GEMM epilogue) */
#define PLANC_B200_NO_ALIAS 0x100u      /* copy even when a whole-buffer copy (recv, identity) stays on one
                                           GPU (default: the output aliases the source, no kernel) */
#define PLANC_B200_PEER_MEMORY 0x20u     /* planc_b200_open_rank / describe_rank: peer-memory transport
                                           (CUDA IPC over NVLink, device flags) instead of NCCL */
#define PLANC_B200_NO_GROUPING 0x40u    /* every GEMM its own launch (default: independent same-shape
                                           GEMMs of a lane that become ready together share one grouped
                                           tensor-core launch) */
#define PLANC_B200_BATCH 0x1000u        /* box and elementwise instructions of one GPU pending together in issue
                                           order (pairwise independent) share one launch per element type
                                           (default off: measured slower — it couples the lanes of a GPU) */
#define PLANC_B200_NO_GATHER 0x2000u    /* materialise every concat / all-gather (default: one whose output only
                                           feeds tensor-core GEMMs as an operand is dropped and the GEMMs' TMA
                                           loads read the row pieces in place — the all-gather -> GEMM prologue) */
#define PLANC_B200_NO_BOX_EW 0x4000u    /* keep an add / mul / max on a pure-copy adapter output (all-to-all,
                                           all-gather, layout change) as its own kernel (default: it runs inside
                                           the adapter's box launch as fold terms — same bits) */
#define PLANC_B200_GATHER_COLS 0x10000u  /* the gather prologue also takes concats of column blocks along K
                                           (opt-in: measured ~3 % slower on C5 than the materialised concat) */
#define PLANC_B200_NO_ALIAS_VIEWS 0x8000u /* copy contiguous sub-ranges (splits) instead of aliasing them as views
                                           of their source on the same GPU (NO_ALIAS turns off every alias) */
#define PLANC_B200_SERIAL_LANES 0x8u    /* one stream per lane: a lane's tasks run strictly in plan
                                           order (default: only data dependencies and sync edges order
                                           a lane's work, spread over several streams) */

typedef struct planc_b200_exec planc_b200_exec;

/* Last error of the calling thread (handle-less calls) or of any handle. */
const char* planc_b200_last_error(void);

/* Compiles a plan for the GPU: buffers, kernels, cross-lane events, box
 * programs. lane_gpu[i] is the CUDA device ordinal that runs plan lane i
 * (lanes are the plan's DeviceLanes in document order, simulate.hpp:32-35);
 * NULL or num_lane_gpu == 0 maps every lane to device 0, fewer entries than
 * lanes wrap around. Replaces load_plan + the set-up half of run_plan. */
int planc_b200_open(const char* plan_json, const int* lane_gpu, int num_lane_gpu, uint32_t flags,
                    planc_b200_exec** out);
void planc_b200_close(planc_b200_exec* h);

/* One process per GPU (torchrun): this process runs the plan lanes l with
 * lane_rank[l] == rank on CUDA device local_gpu. Pieces produced on another
 * rank's lane reach their consumers through NCCL point-to-point exchange
 * steps placed in the global issue order (identical on every rank, so the
 * grouped sends/receives match without deadlock). nccl_id is the 128-byte
 * ncclUniqueId from planc_b200_nccl_unique_id on rank 0, broadcast by the
 * caller. NCCL is loaded at run time (libnccl.so.2). */
int planc_b200_nccl_unique_id(unsigned char id_out[128]);
int planc_b200_open_rank(const char* plan_json, int rank, int world, const int* lane_rank, int num_lanes,
                         int local_gpu, const unsigned char nccl_id[128], uint32_t flags,
                         planc_b200_exec** out);
/* Host-only: the rank-localised program (same on every rank), as JSON.
 * With PLANC_B200_PEER_MEMORY: the global program and its cross-rank flag
 * schedule ("peer_sync": per-instruction wait slots and (rank, slot) signals). */
int planc_b200_describe_rank(const char* plan_json, const int* lane_rank, int num_lanes, uint32_t flags,
                             char** json_out);

/* Peer-memory transport (open_rank with PLANC_B200_PEER_MEMORY; nccl_id may
 * be NULL). No NCCL: each rank maps every other rank's lane arenas through
 * CUDA IPC (NVLink peer memory); adapter box kernels — split / concat /
 * reduce-assemble / recv / every collective member output, all-reduces as a
 * reduce-scatter phase plus an all-gather phase — read the pieces in place on
 * the peer GPU, and cross-rank dependencies are device flags (release /
 * acquire at system scope, a step-end barrier across ranks). Before the first
 * step every rank exports a blob of planc_b200_peer_blob_bytes bytes, the
 * caller all-gathers them (rank order, concatenated) and every rank imports
 * the lot. After import, get_output / read_buffer read any rank's pieces. */
int64_t planc_b200_peer_blob_bytes(planc_b200_exec* h);
int planc_b200_peer_export(planc_b200_exec* h, unsigned char* blob, int64_t capacity);
int planc_b200_peer_import(planc_b200_exec* h, const unsigned char* blobs, int64_t blob_bytes);

/* Binds one graph-input pTensor (refexec.cpp:366-376); `data` is dense
 * row-major with `rank` extents `shape`. Copied; placed on the GPU at the
 * next run. */
int planc_b200_set_input(planc_b200_exec* h, int ptensor, const double* data, const int64_t* shape, int rank);

/* Executes the plan `iters` times (>= 1) back to back; *ms_per_step receives
 * the mean device time per step (CUDA events, origin stream). iters == 0
 * runs one untimed step (verification). */
int planc_b200_run(planc_b200_exec* h, int iters, double* ms_per_step);

/* End-to-end steps: per step H2D of every non-weight graph input from
 * pinned host memory, the plan step, D2H of every terminal non-weight
 * output piece. */
int planc_b200_run_e2e(planc_b200_exec* h, int iters, double* ms_per_step, int64_t* h2d_bytes_per_step,
                       int64_t* d2h_bytes_per_step);

/* Produced pTensors (refexec.cpp:532-556), ascending id. Returns the count;
 * writes up to `cap` ids. */
int planc_b200_num_outputs(planc_b200_exec* h);
int planc_b200_output_ids(planc_b200_exec* h, int* ids, int cap);
/* Rank / shape of a pTensor. */
int planc_b200_ptensor_shape(planc_b200_exec* h, int ptensor, int64_t* shape, int cap, int* rank);
/* Reassembled value of a produced pTensor as doubles (volume elements). */
int planc_b200_get_output(planc_b200_exec* h, int ptensor, double* out, int64_t capacity);

/* Debug / verification: the value of one device buffer (a vTensor piece,
 * ids as in planc_b200_describe) as doubles. Returns its element count. */
int64_t planc_b200_read_buffer(planc_b200_exec* h, int buffer, double* out, int64_t capacity);

/* Graph-input pTensors the plan places (ascending id); in one-process-per-GPU
 * mode, those placed on this rank's lanes (the only inputs it needs). */
int planc_b200_num_inputs(planc_b200_exec* h);
int planc_b200_input_ids(planc_b200_exec* h, int* ids, int cap);

/* Step accounting (algorithmic, from task masks). */
typedef struct planc_b200_stats {
  int num_lanes;
  int num_tasks;
  int num_instructions;
  int kernels_per_step;   /* kernel launches of one step */
  int gemm_tc_per_step;   /* of which tcgen05 GEMMs */
  int graph_captured;     /* 1 when steps replay one CUDA graph */
  double flops;           /* total GEMM + elementwise FLOPs of one step */
  double hbm_bytes;       /* memory-bound kernels' bytes (reads + writes) */
  double wire_bytes;      /* adapter bytes by NCCL bus-bandwidth convention */
  double max_lane_gemm_flops;
  double max_lane_hbm_bytes;
  double max_lane_wire_bytes;
  int64_t device_bytes;   /* arena bytes over all lanes */
} planc_b200_stats;
int planc_b200_get_stats(planc_b200_exec* h, planc_b200_stats* out);

/* Per-kernel-family timing of one eagerly issued, serialised step.
 * Returns a JSON array [{"kind","launches","ms","flops","bytes","wire_bytes"}]
 * (caller frees with planc_b200_free). */
int planc_b200_profile(planc_b200_exec* h, char** json_out);

/* Measured timeline of one step (per-task CUDA events, streams and overlap as
 * in a timed step) in the shape of the reference simulator's
 * SimReport::timeline_json (simulate.cpp:373-383): a JSON array of
 * {"device","op","kind","start","end"} (seconds) plus "instr" / "stream".
 * Caller frees with planc_b200_free. */
int planc_b200_timeline(planc_b200_exec* h, char** json_out);

/* Host-only: which GEMM path a matmul of this shape takes — tcgen05 tensor
 * cores (1: kind::f16 for bf16 operands, 3xTF32 kind::tf32 when operands and
 * output are all fp32) or the SIMT kernel (0) — and the tensor-core tile
 * width. */
int planc_b200_gemm_config(int64_t m, int64_t n, int64_t k, int ta, int tb, int a_bf16, int b_bf16, int c_bf16,
                           int* tensor_cores, int* tile_n);

/* Host-only: the tcgen05 GEMM's launch schedule on a GPU with `sms` SMs for
 * `group` independent GEMMs of this shape in one launch (1 = a single GEMM)
 * — tile width, persistent grid, and either tiles done whole (data-parallel
 * waves) followed by half_items half-width tiles (the last partial wave,
 * 128 x tile_n/2 each) or by the CTAs sharing the remaining tiles by k-range
 * (stream-K), or the number of k-splits per tile (split-K: fp32 partials + a
 * reduce kernel); with the workspace either needs (0 without). `variant` is
 * the kernel variant: 1 one CTA per SM, 2 two CTAs per SM (short k, grid up
 * to 2 x sms), 3 eight epilogue warps (short k), 4 cluster pairs sharing B by
 * multicast, 5 2-SM pairs (one 256-row tcgen05 MMA per pair). bf16 operands. */
int planc_b200_gemm_schedule(int64_t m, int64_t n, int64_t k, int ta, int tb, int c_bf16, int sms, int group,
                             int* tile_n, int* grid, int* dp_tiles, int* sk_ctas, int* splits, int* half_items,
                             int* variant, int64_t* ws_bytes);

/* Host-only lowering (no GPU needed): the executor's device program for a
 * plan as JSON — buffers, instructions, box cells, issue order. */
int planc_b200_describe(const char* plan_json, uint32_t flags, char** json_out);
void planc_b200_free(void* p);

/* Library identity: "planc_b200 <version> sm_100a". */
const char* planc_b200_version(void);

#ifdef __cplusplus
}
#endif

#endif /* PLANC_B200_H_ */
