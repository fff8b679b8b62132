// tcgen05 / TMEM / TMA GEMM for the plan's matmul sub-operators (sm_100a) —
// kernel templates and launch helpers, included by gemm_sm100.cu (schedule,
// dispatch) and the gemm_sm100_ab*.cu instantiation units.
//
// C[m,n] = op(A)[m,k] · op(B)[k,n] with bf16 operands, fp32 accumulation in
// tensor memory, bf16 or fp32 output — the reference's matmul_eval
// (proj/src/refexec.cpp:142-168) including transpose_a / transpose_b, which
// are not materialised: a transposed operand is simply loaded MN-major and the
// UMMA instruction descriptor's major bits say so.
//
// Structure: persistent, one CTA per SM, 128xBN output tiles (BN 256 / 128 /
// 64 chosen per shape) in grouped raster order (8 M-blocks per group for L2
// reuse of B), 6 warps:
//   warp 0      TMA producer: smem ring filling ~192 KB (A 16 KB + B BN*128 B
//               per stage, 128B-swizzled), mbarrier full/empty pipeline
//               running across tiles
//   warp 1      TMEM allocator (two BN-column fp32 accumulators) + single-
//               thread tcgen05.mma issuer (kind::f16, M=128, N=BN, K=16 per
//               instruction); commits free smem stages and, per tile, the
//               accumulator it just finished
//   warps 2..5  epilogue: tcgen05.ld 32x32b.x32 TMEM -> registers, convert,
//               64B/128B-swizzled smem staging, TMA bulk tensor store
//               (double-buffered per warp); releases the accumulator so the
//               MMA warp fills it with the tile after next while this one
//               drains. An optional fused elementwise consumer (FUSE)
//               reads its operands one chunk ahead and leaves by TMA store.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <type_traits>

#pragma once

#include "gelu.cuh"
#include "kernels.cuh"
#include "launch.cuh"

namespace planc_b200 {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 128 bytes of bf16: one 128B swizzle row
constexpr int A_STAGE_BYTES = BM * BK * 2;  // 16 KB
constexpr int NUM_THREADS = 192;
// Launch variants (template OCC): 1 = one CTA per SM, 4 epilogue warps;
// 2 = two CTAs per SM (short-k GEMMs that cannot fill the GPU); 3 = one CTA
// per SM with 8 epilogue warps, two per TMEM lane quarter splitting a tile's
// columns (short-k GEMMs whose tile epilogue outlasts its MMAs).
// 4 = one CTA per SM in clusters of two along M: the pair shares each B
// tile — every CTA loads half of it and multicasts to both (TMA
// .multicast::cluster), halving B's L2 -> SM traffic.
// Eight epilogue warps (two per TMEM lane quarter, each taking half of a
// tile's columns) for short-k launches (OCC 3) and for the 2-SM variant
// (OCC 5), whose fused elementwise epilogues otherwise outlast the pair's
// MMAs (C2's FFN GEMM with its fused ReLU: 250 us vs 169 us plain, r01).
__host__ __device__ constexpr int epi_warps(int occ) { return occ == 3 || occ == 5 ? 8 : 4; }
__host__ __device__ constexpr int cta_threads(int occ) { return 64 + 32 * epi_warps(occ); }
constexpr int GROUP_M = 8;
constexpr int kSkDepth = 2;  // stream-K partials loaded per round trip

// Tile width BN in {256, 128, 64}: smem ring depth fills ~200 KB, TMEM holds
// two BN-column fp32 accumulators (power of two >= 32 columns).
// OCC = 2 ("small" GEMMs: k <= 1024, BN <= 128, no fusion / stream-K): a
// ~100 KB ring and <= 256 TMEM columns so two CTAs share an SM — two tiles'
// prologue / epilogue latencies overlap, or two concurrent small GEMMs from
// different streams run side by side instead of one after the other.
template <int BN_, bool FUSE = false, int OCC = 1>
struct Cfg {
  static constexpr int BN = BN_;
  // 2-SM pairs (OCC 5): each CTA holds only its BN/2 columns of the B tile.
  static constexpr int B_STAGE_BYTES = (OCC == 5 ? BN / 2 : BN) * BK * 2;
  // + epilogue staging: 4 (8) warps x 2 buffers x (32 rows x 32 cols, <= 4 B);
  // FUSE (bf16): warps x 2 x {C, fused result} 2 KB chunks — same size.
  static constexpr int STAGING_BYTES = epi_warps(OCC) * 2 * 4096;
  static constexpr int RING_BYTES =
      OCC == 5 ? 227 * 1024 - STAGING_BYTES - 3 * 1024 : (OCC == 1 || OCC >= 4 ? 200 : OCC == 2 ? 76 : 159) * 1024;
  static constexpr int STAGES_RAW = RING_BYTES / (A_STAGE_BYTES + B_STAGE_BYTES);
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int SMEM_BYTES =
      STAGES * (A_STAGE_BYTES + B_STAGE_BYTES) + STAGING_BYTES + 1024 /*align*/ + 1024 /*barriers + align*/;
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory per CTA above the sm_100 limit");
};

// Tensor map of a fused epilogue's result: [m][n] bf16 in the C layout
// (32x32 boxes, 64B swizzle).
struct EpiMaps {
  CUtensorMap out[1];
  // Split-K partials: fp32 [group][splits][m_pad] x [n_pad] (32x32 boxes,
  // 128B swizzle), row of (member p, split s, output row r) =
  // (p * splits + s) * m_pad + r.
  CUtensorMap ws;
};

// Operand / result maps of the launch's GEMMs (one, or a group of
// independent same-shape GEMMs sharing the tile space: tile t belongs to
// member t / tiles_per_gemm).
// NG = capacity (1 for single launches: kernel parameters stay small, which
// keeps graph launch latency down; kMaxGemmGroup for grouped launches).
template <int NG>
struct GroupMaps {
  CUtensorMap a[NG];
  CUtensorMap b[NG];
  CUtensorMap c[NG];
};

// Stream-K tail (data-parallel waves, then the remaining tiles' k-iterations
// split evenly over the CTAs): tiles [0, dp_tiles) go whole to CTA
// t % gridDim.x; CTA b < sk_ctas then takes k-iterations [lo(b), lo(b+1)) of
// the linearised (tile, k-block) space of tiles [dp_tiles, tiles). A tile
// covered by several CTAs is reduced by whichever of them arrives last (per
// 32-row quarter: a counter per quarter, no CTA ever waits on another), in
// fixed CTA (= k) order from fp32 partials — the same bits whatever the
// arrival order.
struct SkParams {
  int dp_tiles = 0;
  int sk_ctas = 0;
  int splits = 0;  // split-K: every work item is (tile, split), stored to ws_map
  // Half-width tail: after dp_tiles whole tiles, the remaining tiles run as
  // half_items tiles of 128 x BN/2 (item h: half h & 1 of tile dp_tiles + h / 2),
  // so a last wave of r < grid/2 tiles takes half a tile-time.
  int half_items = 0;
  // Reduce-scatter epilogue: row y of C goes to row y % scatter_rows of the
  // [scatter_rows][n] buffer scatter_dst[y / scatter_rows] (0 = off) — by
  // plain 16-byte stores from registers, valid for NVLink peer memory.
  int scatter_rows = 0;
  void* scatter_dst[kMaxGemmGroup] = {};
  // Raster: M-blocks (pair rows for 2-SM launches) per group (tiles_coords).
  int group_m = GROUP_M;
  // L2 eviction priority of the A / B operand loads (0: default, 1:
  // evict_first — streamed once, 2: evict_last — re-read across raster
  // groups while the other operand streams past it).
  int hint_a = 0, hint_b = 0;
  // Gathered operands (all-gather / concat -> GEMM prologue): operand A (B)
  // is the row-wise concatenation of pieces of gather_rows_a (_b) rows each,
  // stored row-major wherever their producers left them (this lane, another
  // lane, NVLink peer memory). Their tensor maps live in global memory
  // (gather_maps: A pieces [0, 8), B pieces [8, 16)); a TMA box at stored
  // row r reads piece r / gather_rows at row r % gather_rows (pieces are
  // whole multiples of every box height).
  int gather_rows_a = 0, gather_rows_b = 0;
  int gather_cols_a = 0, gather_cols_b = 0;  // column pieces: a box at stored column x reads piece x / cols
  int gather_na = 0, gather_nb = 0;          // piece counts (boxes past the last piece stay in it, out of bounds)
  const CUtensorMap* gather_maps = nullptr;
  long long sk_iters = 0;
  float* partials = nullptr;  // [sk_ctas][2 slots][4 quarters][BN/32 chunks][8][32] float4
  int* counters = nullptr;    // [(tiles - dp_tiles) * 4], zero between launches
};

__device__ __forceinline__ long long sk_lo(const SkParams& sk, int b) {
  return static_cast<long long>(b) * sk.sk_iters / sk.sk_ctas;
}

// CTA whose stream-K range holds iteration x: max b with lo(b) <= x.
__device__ __forceinline__ int sk_owner(const SkParams& sk, long long x) {
  return static_cast<int>(((x + 1) * sk.sk_ctas - 1) / sk.sk_iters);
}

// Calls f(tile, kb0, kb1, half) for this CTA's work items in order; half is
// -1 for a whole tile, else which 128 x BN/2 half of the tile.
template <typename F>
__device__ __forceinline__ void for_each_work(int num_k, const SkParams& sk, F&& f) {
  if (sk.splits > 1) {
    // Split-K: item (tile t, split s) covers k-blocks [s*K/S, (s+1)*K/S).
    const int items = sk.dp_tiles * sk.splits;
    for (int x = blockIdx.x; x < items; x += gridDim.x) {
      const int t = x / sk.splits, sp = x - t * sk.splits;
      f(t, sp * num_k / sk.splits, (sp + 1) * num_k / sk.splits, -1);
    }
    return;
  }
  if (sk.half_items > 0) {
    for (int x = blockIdx.x; x < sk.dp_tiles + sk.half_items; x += gridDim.x) {
      if (x < sk.dp_tiles) f(x, 0, num_k, -1);
      else f(sk.dp_tiles + (x - sk.dp_tiles) / 2, 0, num_k, (x - sk.dp_tiles) & 1);
    }
    return;
  }
  for (int t = blockIdx.x; t < sk.dp_tiles; t += gridDim.x) f(t, 0, num_k, -1);
  if (static_cast<int>(blockIdx.x) < sk.sk_ctas) {
    long long it = sk_lo(sk, blockIdx.x);
    const long long hi = sk_lo(sk, blockIdx.x + 1);
    while (it < hi) {
      const int j = static_cast<int>(it / num_k);
      const int kb0 = static_cast<int>(it - static_cast<long long>(j) * num_k);
      const int kb1 = static_cast<int>(min(static_cast<long long>(num_k), kb0 + (hi - it)));
      f(sk.dp_tiles + j, kb0, kb1, -1);
      it += kb1 - kb0;
    }
  }
}

// ---- PTX wrappers ------------------------------------------------------------

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(std::uint64_t* bar, std::uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(std::uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, std::uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, std::uint32_t parity) {
  std::uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra.uni DONE;\n"
      "bra.uni LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, std::uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<std::uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// Same, with an L2 eviction-priority policy (createpolicy).
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int c0, int c1, std::uint64_t* bar,
                                                 std::uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<std::uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// L2 policy for operand loads: 1 = evict_first, 2 = evict_last, else normal.
__device__ __forceinline__ std::uint64_t l2_policy(int hint) {
  std::uint64_t p;
  if (hint == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else if (hint == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Bulk tensor store smem -> global (clips rows / cols outside the tensor).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<std::uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// Same, with an L2 eviction-priority policy (createpolicy), no group close.
__device__ __forceinline__ void tma_store_2d_nc_hint(const CUtensorMap* map, const void* src, int c0, int c1,
                                                     std::uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(
          reinterpret_cast<std::uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(smem_u32(src)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ std::uint64_t l2_evict_first_policy() {
  std::uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Multicast load: the box lands at the same smem offset in every CTA of
// ctaMask and completes bytes on each one's mbarrier at the same offset.
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, int c0, int c1, std::uint64_t* bar,
                                               std::uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<std::uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}

__device__ __forceinline__ void tc_commit_mc(std::uint64_t* bar, std::uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"(mask)
               : "memory");
}

// 2-SM variant: TMA load whose completion is counted on the pair leader's
// mbarrier (shared::cluster address), and the leader's MMA commit.
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, int c0, int c1,
                                                std::uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<std::uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_cluster)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d_2sm_hint(void* dst, const CUtensorMap* map, int c0, int c1,
                                                     std::uint32_t bar_cluster, std::uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
      "[%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<std::uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_cluster), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void tc_commit_2sm_mc(std::uint64_t* bar, std::uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"(mask)
               : "memory");
}

__device__ __forceinline__ void tc_mma_2sm(std::uint32_t tmem_d, std::uint64_t adesc, std::uint64_t bdesc,
                                           std::uint32_t idesc, std::uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// shared::cluster address of `p` in CTA `rank` of the cluster.
__device__ __forceinline__ std::uint32_t cluster_addr(const void* p, std::uint32_t rank) {
  std::uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}

// Remote arrive on a pair CTA's mbarrier releasing an accumulator: relaxed.
// It only has to follow this thread's TMEM reads, which have completed
// (tcgen05.wait::ld returned them; tcgen05.fence::before_thread_sync orders
// them) before the peer's MMA warp reuses the columns. A release arrive
// compiles to MEMBAR.ALL.CTA / .GPU, which also wait for the epilogue's
// in-flight operand prefetch loads — the top stall of the fused 2-SM launch
// (~1/5 of its samples; profiles/r02/ncu_fused_gemm_*).
__device__ __forceinline__ void mbar_arrive_cluster(std::uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ std::uint32_t cluster_rank() {
  std::uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// Same, without closing the bulk group (several stores per group).
__device__ __forceinline__ void tma_store_2d_nc(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<std::uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(std::uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_mma(std::uint32_t tmem_d, std::uint64_t adesc, std::uint64_t bdesc,
                                       std::uint32_t idesc, std::uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// Shared-memory matrix descriptor (tcgen05 "version 1"), SWIZZLE_128B.
__device__ __forceinline__ std::uint64_t smem_desc(std::uint32_t addr, std::uint32_t lbo, std::uint32_t sbo) {
  std::uint64_t d = 0;
  d |= static_cast<std::uint64_t>((addr >> 4) & 0x3FFFu);
  d |= static_cast<std::uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<std::uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;  // version
  d |= 2ull << 61;  // SWIZZLE_128B
  return d;
}

// Instruction descriptor: kind::f16, A/B bf16, D f32, M=128, N=BN.
template <int BN, int M = BM>
__host__ __device__ constexpr std::uint32_t make_idesc(bool a_mn, bool b_mn) {
  return (1u << 4)                              // D format f32
         | (1u << 7)                            // A bf16
         | (1u << 10)                           // B bf16
         | ((a_mn ? 1u : 0u) << 15)             // A major
         | ((b_mn ? 1u : 0u) << 16)             // B major
         | (static_cast<std::uint32_t>(BN >> 3) << 17)  // N
         | (static_cast<std::uint32_t>(M >> 4) << 24);  // M
}

// tcgen05.ld without the wait: the registers are valid after tmem_wait_ld()
// (which waits for every outstanding load of the thread).
__device__ __forceinline__ void tmem_ld32_issue(std::uint32_t taddr, std::uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(std::uint32_t taddr, std::uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---- kernel --------------------------------------------------------------------

__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int& mb, int& nb, int group_m = GROUP_M) {
  const int per_group = group_m * tiles_n;
  const int group = t / per_group;
  const int first_m = group * group_m;
  const int gm = min(tiles_m - first_m, group_m);
  const int r = t % per_group;
  mb = first_m + r % gm;
  nb = r / gm;
}

// Fold step of a fused epilogue op (program.hpp EwOp): add / mul / max; ACT
// (compile-time, so the plain ops carry no activation code) 4 = GELU's
// gradient gelu'(a) * b (a = x, b = incoming gradient), 3 = GELU, unary,
// applied after the fold (epi_finish).
template <int ACT>
__device__ __forceinline__ float epi_apply(int op, float a, float b) {
  if constexpr (ACT == 4) return gelu_grad_f(a, b);
  return op == 0 ? a + b : op == 1 ? a * b : fmaxf(a, b);
}
template <int ACT>
__device__ __forceinline__ float epi_finish(float a) {
  if constexpr (ACT == 3) return gelu_f(a);
  return a;
}

// Two floats -> packed bf16x2 (round to nearest even): one F2FP pack on the
// FMA / ALU pipes instead of two F2F conversions on the XU pipe.
__device__ __forceinline__ std::uint32_t bf16_pair(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const std::uint32_t*>(&v);
}

__device__ __forceinline__ void bf16_unpair(std::uint32_t w, float& lo, float& hi) {
  lo = __uint_as_float(w << 16);
  hi = __uint_as_float(w & 0xffff0000u);
}

template <bool A_MN, bool B_MN, bool C_BF16, int BN, bool FUSE, int NG, int OCC>
__global__ void __launch_bounds__(cta_threads(OCC), OCC == 2 ? 2 : 1)
    gemm_tc_kernel(const __grid_constant__ GroupMaps<NG> gm, int ng, int m, int n, int k,
                   const __grid_constant__ EpiParams epi, const __grid_constant__ EpiMaps maps,
                   const __grid_constant__ SkParams sk) {
  static_assert(OCC == 1 || OCC == 3 || OCC == 5 || (!FUSE && (OCC >= 3 || BN <= 128)),
                "two CTAs per SM: no fusion, <= 256 TMEM columns");
  static_assert(OCC < 4 || BN >= 128, "cluster pairs split B tiles in 64-wide halves");
  constexpr bool CL = OCC == 4;   // pair sharing B by multicast, one MMA per CTA
  constexpr bool SM2 = OCC == 5;  // pair running one 256-row MMA (tcgen05 cta_group::2)
  constexpr bool PAIR = CL || SM2;
  constexpr int EPI_WARPS = epi_warps(OCC);
  extern __shared__ std::uint8_t smem_raw[];
  using CF = Cfg<BN, FUSE, OCC>;
  constexpr int STAGES = CF::STAGES;
  constexpr int B_STAGE_BYTES = CF::B_STAGE_BYTES;
  constexpr int TMEM_COLS = CF::TMEM_COLS;
  std::uint8_t* smem =
      smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays a shared-space pointer (STS / LDS)
  std::uint8_t* sA = smem;
  std::uint8_t* sB = smem + STAGES * A_STAGE_BYTES;
  // Epilogue staging (1024-aligned: the 64B / 128B swizzle atoms of the C map).
  std::uint8_t* staging = sB + STAGES * B_STAGE_BYTES;
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(staging + CF::STAGING_BYTES);
  std::uint64_t* empty = full + STAGES;
  std::uint64_t* tfull = empty + STAGES;  // [2] accumulator ready
  std::uint64_t* tempty = tfull + 2;      // [2] accumulator drained
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int tiles_m = (m + BM - 1) / BM;
  const int tiles_n = (n + BN - 1) / BN;
  const int per_gemm = tiles_m * tiles_n;
  const int num_tiles = per_gemm * ng;
  const int num_k = (k + BK - 1) / BK;
  // Tile t of the launch: member t / per_gemm, its tile t % per_gemm.
  auto coords = [&](int t, int& p, int& mb, int& nb) {
    if constexpr (PAIR) {
      // t = 2 * pair + rank: pairs of vertically adjacent tiles sharing nb
      const int tiles_m2 = (tiles_m + 1) / 2;
      const int per_pair = tiles_m2 * tiles_n;
      const int pr = t >> 1;
      p = pr / per_pair;
      int mb2;
      tile_coords(pr - p * per_pair, tiles_m2, tiles_n, mb2, nb, sk.group_m);
      mb = 2 * mb2 + (t & 1);  // may pass tiles_m: a zero tile whose stores are clipped
    } else {
      p = t / per_gemm;
      tile_coords(t - p * per_gemm, tiles_m, tiles_n, mb, nb, sk.group_m);
    }
  };
  const int work_items = PAIR ? 2 * ((tiles_m + 1) / 2) * tiles_n * ng : num_tiles;  // fused epilogue loop bound
  // Work items: for_each_work, or — cluster pairs — pair tiles in lockstep.
  auto work = [&](auto&& f) {
    if constexpr (PAIR) {
      const int pairs = ((tiles_m + 1) / 2) * tiles_n * ng;
      const int rank = static_cast<int>(cluster_rank());
      for (int pr = blockIdx.x / 2; pr < pairs; pr += gridDim.x / 2) f(2 * pr + rank, 0, num_k, -1);
    } else {
      for_each_work(num_k, sk, f);
    }
  };

  if (warp == 0 && lane == 0) {
    for (int p = 0; p < ng; ++p) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&gm.a[p])) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&gm.b[p])) : "memory");
    }
    // Gathered operands' piece maps (global memory, written at open).
    for (int i = 0; i < sk.gather_na; ++i)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(sk.gather_maps + i)) : "memory");
    for (int i = 0; i < sk.gather_nb; ++i)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(sk.gather_maps + kMaxGemmGroup + i))
                   : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL ? 2 : 1);  // cluster pairs: both CTAs' MMAs free a stage
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], SM2 ? 2 * EPI_WARPS : EPI_WARPS);  // one arrive per epilogue warp (2-SM: both CTAs')
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (SM2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync();  // peer barriers initialised before any multicast / remote arrive
  tc_fence_after();
  const std::uint32_t tmem = *tmem_slot;
  // Prologue done (barriers, TMEM, descriptor prefetch): from here on the
  // previous kernel's results are read and the workspace is written.
  pdl_wait();

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;  // global k-block counter across work items (ring position)
      const std::uint64_t pol_a = l2_policy(sk.hint_a), pol_b = l2_policy(sk.hint_b);
      // Gathered operand: the piece holding stored row `row` (row pieces)
      // or stored column `x` (column pieces), coordinates made piece-local.
      // A box past the operand's end (the zero tile of a 2-SM pair, a
      // partial tile) stays in the last piece, out of bounds there: TMA
      // zero-fills it as it would past the concatenated operand.
      auto pick_a = [&](const CUtensorMap* dflt, int& x, int& row) -> const CUtensorMap* {
        if (sk.gather_rows_a != 0) {
          const int q = min(row / sk.gather_rows_a, sk.gather_na - 1);
          row -= q * sk.gather_rows_a;
          return sk.gather_maps + q;
        }
        if (sk.gather_cols_a != 0) {
          const int q = min(x / sk.gather_cols_a, sk.gather_na - 1);
          x -= q * sk.gather_cols_a;
          return sk.gather_maps + q;
        }
        return dflt;
      };
      auto pick_b = [&](const CUtensorMap* dflt, int& x, int& row) -> const CUtensorMap* {
        if (sk.gather_rows_b != 0) {
          const int q = min(row / sk.gather_rows_b, sk.gather_nb - 1);
          row -= q * sk.gather_rows_b;
          return sk.gather_maps + kMaxGemmGroup + q;
        }
        if (sk.gather_cols_b != 0) {
          const int q = min(x / sk.gather_cols_b, sk.gather_nb - 1);
          x -= q * sk.gather_cols_b;
          return sk.gather_maps + kMaxGemmGroup + q;
        }
        return dflt;
      };
      work([&](int t, int kb0, int kb1, int half) {
        int p, mb, nb;
        coords(t, p, mb, nb);
        const CUtensorMap* tmA = &gm.a[p];
        const CUtensorMap* tmB = &gm.b[p];
        // A half tile loads the B rows from its own first column (the box's
        // upper half is unused, and zero-filled past the tensor edge).
        const int m0 = mb * BM, n0 = nb * BN + (half > 0 ? BN / 2 : 0);
        if constexpr (SM2) {
          // 2-SM: this CTA's 128 rows of A and its half of B's columns land
          // in its own smem; both CTAs' bytes are counted on the leader's
          // full barrier, which only the leader arms (with both CTAs' bytes).
          const int r = t & 1;
          for (int kb = kb0; kb < kb1; ++kb, ++it) {
            const int s = it % STAGES;
            const std::uint32_t phase = (it / STAGES) & 1;
            mbar_wait(&empty[s], phase ^ 1);
            if (r == 0) mbar_expect_tx(&full[s], 2 * (A_STAGE_BYTES + B_STAGE_BYTES));  // (B_STAGE: BN/2 columns)
            const std::uint32_t lb = cluster_addr(&full[s], 0);
            std::uint8_t* a = sA + s * A_STAGE_BYTES;
            std::uint8_t* b = sB + s * B_STAGE_BYTES;
            if (A_MN) {
#pragma unroll
              for (int j = 0; j < BM / 64; ++j) {
                int x = m0 + 64 * j, ra = kb * BK;
                const CUtensorMap* mA = pick_a(tmA, x, ra);
                tma_load_2d_2sm_hint(a + j * (64 * BK * 2), mA, x, ra, lb, pol_a);
              }
            } else {
              int x = kb * BK, ra = m0;
              const CUtensorMap* mA = pick_a(tmA, x, ra);
              tma_load_2d_2sm_hint(a, mA, x, ra, lb, pol_a);
            }
            if (B_MN) {
#pragma unroll
              for (int j = 0; j < BN / 128; ++j) {
                int x = n0 + r * (BN / 2) + 64 * j, rb = kb * BK;
                const CUtensorMap* mB = pick_b(tmB, x, rb);
                tma_load_2d_2sm_hint(b + j * (64 * BK * 2), mB, x, rb, lb, pol_b);
              }
            } else {
              int x = kb * BK, rb = n0 + r * (BN / 2);
              const CUtensorMap* mB = pick_b(tmB, x, rb);
              tma_load_2d_2sm_hint(b, mB, x, rb, lb, pol_b);
            }
          }
          return;
        }
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          const std::uint32_t phase = (it / STAGES) & 1;
          mbar_wait(&empty[s], phase ^ 1);
          mbar_expect_tx(&full[s], A_STAGE_BYTES + B_STAGE_BYTES);
          std::uint8_t* a = sA + s * A_STAGE_BYTES;
          std::uint8_t* b = sB + s * B_STAGE_BYTES;
          if (A_MN) {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) {
              int x = m0 + 64 * j, ra = kb * BK;
              const CUtensorMap* mA = pick_a(tmA, x, ra);
              tma_load_2d_hint(a + j * (64 * BK * 2), mA, x, ra, &full[s], pol_a);
            }
          } else {
            int x = kb * BK, ra = m0;
            const CUtensorMap* mA = pick_a(tmA, x, ra);
            tma_load_2d_hint(a, mA, x, ra, &full[s], pol_a);
          }
          if constexpr (CL) {
            // this CTA's half of the B tile, multicast to both CTAs of the pair
            const int r = t & 1;
            if (B_MN) {
#pragma unroll
              for (int j = r * (BN / 128); j < (r + 1) * (BN / 128); ++j) {
                int x = n0 + 64 * j, rb = kb * BK;
                const CUtensorMap* mB = pick_b(tmB, x, rb);
                tma_load_2d_mc(b + j * (64 * BK * 2), mB, x, rb, &full[s], 0x3);
              }
            } else {
              int x = kb * BK, rb = n0 + r * (BN / 2);
              const CUtensorMap* mB = pick_b(tmB, x, rb);
              tma_load_2d_mc(b + r * (BN / 2) * 128, mB, x, rb, &full[s], 0x3);
            }
          } else {
            if (B_MN) {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j) {
                int x = n0 + 64 * j, rb = kb * BK;
                const CUtensorMap* mB = pick_b(tmB, x, rb);
                tma_load_2d_hint(b + j * (64 * BK * 2), mB, x, rb, &full[s], pol_b);
              }
            } else {
              int x = kb * BK, rb = n0;
              const CUtensorMap* mB = pick_b(tmB, x, rb);
              tma_load_2d_hint(b, mB, x, rb, &full[s], pol_b);
            }
          }
        }
      });
    }
  } else if (warp == 1) {
    if (SM2 && cluster_rank() != 0) {
      // 2-SM: the pair leader issues every MMA for both CTAs.
    } else if (lane == 0) {
      constexpr std::uint32_t idesc_full = make_idesc<BN, SM2 ? 2 * BM : BM>(A_MN, B_MN);
      constexpr std::uint32_t idesc_half = make_idesc<(BN >= 128 ? BN / 2 : BN)>(A_MN, B_MN);
      int it = 0, local = 0;
      work([&](int, int kb0, int kb1, int half) {
        const std::uint32_t idesc = half >= 0 ? idesc_half : idesc_full;
        const int acc = local & 1;
        const std::uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);  // epilogue drained this accumulator
        tc_fence_after();
        const std::uint32_t d = tmem + static_cast<std::uint32_t>(acc * BN);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          const std::uint32_t phase = (it / STAGES) & 1;
          mbar_wait(&full[s], phase);
          tc_fence_after();
          const std::uint32_t a_base = smem_u32(sA + s * A_STAGE_BYTES);
          const std::uint32_t b_base = smem_u32(sB + s * B_STAGE_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            // K-major: 16 elements = 32 bytes along the swizzled row; rows of
            // 128 B, 8-row groups 1024 B apart (SBO). MN-major: 16 K-rows =
            // 2048 B; 64-element MN blocks 8 KB apart (LBO), 8-row K groups
            // 1024 B apart (SBO).
            std::uint64_t ad = A_MN ? smem_desc(a_base + kk * 2048, 64 * BK * 2, 1024)
                                    : smem_desc(a_base + kk * 32, 16, 1024);
            std::uint64_t bd = B_MN ? smem_desc(b_base + kk * 2048, 64 * BK * 2, 1024)
                                    : smem_desc(b_base + kk * 32, 16, 1024);
            if constexpr (SM2) tc_mma_2sm(d, ad, bd, idesc, (kb != kb0 || kk != 0) ? 1u : 0u);
            else tc_mma(d, ad, bd, idesc, (kb != kb0 || kk != 0) ? 1u : 0u);
          }
          if constexpr (SM2) tc_commit_2sm_mc(&empty[s], 0x3);   // both CTAs' stages free
          else if constexpr (CL) tc_commit_mc(&empty[s], 0x3);  // both CTAs' producers refill the stage
          else tc_commit(&empty[s]);  // smem stage free once these MMAs retire
        }
        if constexpr (SM2) tc_commit_2sm_mc(&tfull[acc], 0x3);  // both CTAs' accumulator halves complete
        else tc_commit(&tfull[acc]);  // accumulator complete
        ++local;
      });
      pdl_trigger();  // every MMA issued: the next kernel may start its prologue
    }
  } else if constexpr (!FUSE) {
    // Epilogue warps 2..5: warp w may only touch TMEM lanes 32*(w%4)..+31.
    // Each 32x32 output chunk goes TMEM -> registers -> swizzled smem
    // staging (conflict-free 16-byte stores) -> one TMA bulk tensor store
    // (coalesced, clipped at the tensor edge); two staging buffers per warp
    // keep a store in flight while the next chunk is converted.
    const int q = warp % 4;
    const int ew = warp - 2;          // epilogue warp index
    const int col_half = ew / 4;      // 8 epilogue warps: which half of a tile's columns
    std::uint8_t* stg = staging + ew * 2 * 4096;
    int sb = 0;
    int local = 0;
    auto store_chunk = [&](const std::uint32_t(&r)[32], const CUtensorMap* map, bool bf16, int x, int y) {
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // buffer sb is free
      __syncwarp();
      std::uint8_t* buf = stg + sb * 4096;
      if (bf16) {
        // 64 B rows, SWIZZLE_64B: 16-byte chunk v lands at v ^ ((row >> 1) & 3).
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const uint4 w = make_uint4(bf16_pair(__uint_as_float(r[8 * v + 0]), __uint_as_float(r[8 * v + 1])),
                                     bf16_pair(__uint_as_float(r[8 * v + 2]), __uint_as_float(r[8 * v + 3])),
                                     bf16_pair(__uint_as_float(r[8 * v + 4]), __uint_as_float(r[8 * v + 5])),
                                     bf16_pair(__uint_as_float(r[8 * v + 6]), __uint_as_float(r[8 * v + 7])));
          *reinterpret_cast<uint4*>(buf + lane * 64 + ((v ^ ((lane >> 1) & 3)) << 4)) = w;
        }
      } else {
        // 128 B rows, SWIZZLE_128B: 16-byte chunk v lands at v ^ (row & 7).
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          *reinterpret_cast<uint4*>(buf + lane * 128 + ((v ^ (lane & 7)) << 4)) =
              make_uint4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> async proxy
      __syncwarp();
      if (lane == 0) tma_store_2d(map, buf, x, y);
      sb ^= 1;
    };
    const int m_pad = tiles_m * BM;
    // fp32 partial of (CTA b, slot, this quarter, chunk c): 8 float4 per
    // lane, lane-interleaved so every access is one coalesced 512 B row.
    auto partial_ptr = [&](int b, int slot, int c) {
      return reinterpret_cast<float4*>(sk.partials) +
             ((static_cast<std::int64_t>((b * 2 + slot) * 4 + q) * (BN / 32) + c) * 8) * 32 + lane;
    };
    work([&](int t, int kb0, int kb1, int half) {
      int p, mb, nb;
      coords(t, p, mb, nb);
      const int acc = local & 1;
      mbar_wait(&tfull[acc], (local >> 1) & 1);
      ++local;
      tc_fence_after();
      const std::uint32_t base = tmem + (static_cast<std::uint32_t>(q * 32) << 16) + static_cast<std::uint32_t>(acc * BN);
      if ((kb0 == 0 && kb1 == num_k) || sk.splits > 1) {  // whole tile, or one split's fp32 partial
        const bool part = sk.splits > 1;
        // split index of k-range start kb0 = floor(s*K/S): s = ceil(kb0*S/K) (K/S >= 1)
        const int sp = (kb0 * sk.splits + num_k - 1) / num_k;
        const int y = part ? (p * sk.splits + sp) * m_pad + mb * BM + q * 32 : mb * BM + q * 32;
        const int chunks = half >= 0 ? BN / 64 : BN / 32;
        const int x0 = nb * BN + (half > 0 ? BN / 2 : 0);
        const int c_lo = EPI_WARPS == 8 ? col_half * (chunks / 2) : 0;
        const int c_hi = EPI_WARPS == 8 ? c_lo + chunks / 2 : chunks;
        // The TMEM load of chunk c+1 is in flight while chunk c is emitted
        // (ping-pong registers; tcgen05.wait::ld waits for every earlier load).
        auto emit = [&](const std::uint32_t(&r)[32], int c) {
          if (part) {
            store_chunk(r, &maps.ws, false, x0 + c * 32, y);
          } else if (sk.scatter_rows > 0) {
            // lane = row of the 32-row chunk: 32 columns straight to the
            // owner's receive buffer (64 B bf16 / 128 B fp32 per lane).
            const int row = y + lane, col = x0 + c * 32;
            const int dst_i = row / sk.scatter_rows;
            char* dst = static_cast<char*>(sk.scatter_dst[dst_i]) +
                        (static_cast<std::int64_t>(row - dst_i * sk.scatter_rows) * n + col) * (C_BF16 ? 2 : 4);
            if constexpr (C_BF16) {
#pragma unroll
              for (int v = 0; v < 4; ++v)
                if (col + 8 * v < n)
                  reinterpret_cast<uint4*>(dst)[v] =
                      make_uint4(bf16_pair(__uint_as_float(r[8 * v + 0]), __uint_as_float(r[8 * v + 1])),
                                 bf16_pair(__uint_as_float(r[8 * v + 2]), __uint_as_float(r[8 * v + 3])),
                                 bf16_pair(__uint_as_float(r[8 * v + 4]), __uint_as_float(r[8 * v + 5])),
                                 bf16_pair(__uint_as_float(r[8 * v + 6]), __uint_as_float(r[8 * v + 7])));
            } else {
#pragma unroll
              for (int v = 0; v < 8; ++v)
                if (col + 4 * v < n)
                  reinterpret_cast<uint4*>(dst)[v] = make_uint4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
            }
          } else {
            store_chunk(r, &gm.c[p], C_BF16, x0 + c * 32, y);
          }
        };
        auto release = [&] {  // every TMEM read of this accumulator has completed
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (SM2) mbar_arrive_cluster(cluster_addr(&tempty[acc], 0));  // the leader's MMA waits
            else mbar_arrive(&tempty[acc]);
          }
        };
        std::uint32_t ra[32], rb[32];
        tmem_ld32_issue(base + c_lo * 32, ra);
        tmem_wait_ld();
#pragma unroll 1
        for (int c = c_lo; c < c_hi; c += 2) {
          const bool has1 = c + 1 < c_hi;
          if (has1) tmem_ld32_issue(base + (c + 1) * 32, rb);
          else release();
          emit(ra, c);
          if (has1) {
            tmem_wait_ld();
            const bool has2 = c + 2 < c_hi;
            if (has2) tmem_ld32_issue(base + (c + 2) * 32, ra);
            else release();
            emit(rb, c + 1);
            if (has2) tmem_wait_ld();
          }
        }
        return;
      }
      if constexpr (OCC == 1) {
      // Stream-K segment: publish the fp32 partial, count the arrival.
      const int j = t - sk.dp_tiles;
      const long long x0 = static_cast<long long>(j) * num_k;
      const int me = blockIdx.x;
      const int myslot = sk_lo(sk, me) >= x0 ? 0 : 1;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        std::uint32_t r[32];
        tmem_ld32(base + c * 32, r);
        float4* dst = partial_ptr(me, myslot, c);
#pragma unroll
        for (int v = 0; v < 8; ++v)
          __stcg(dst + v * 32, make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                                           __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3])));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      __threadfence();
      __syncwarp();
      int old = 0;
      if (lane == 0) old = atomicAdd(&sk.counters[j * 4 + q], 1);
      old = __shfl_sync(0xffffffffu, old, 0);
      const int b_first = sk_owner(sk, x0), b_last = sk_owner(sk, x0 + num_k - 1);
      if (old != b_last - b_first) return;  // another CTA finishes this quarter
      // Last arrival: sum every segment's partial in k order, store.
      __threadfence();
      if (lane == 0) sk.counters[j * 4 + q] = 0;  // ready for the next launch
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        // Loads of kSkDepth partials in flight, folded in CTA order.
        float4 sum[8];
#pragma unroll 1
        for (int b0 = b_first; b0 <= b_last; b0 += kSkDepth) {
          float4 p[kSkDepth][8];
#pragma unroll
          for (int d = 0; d < kSkDepth; ++d) {
            const int b = b0 + d;
            if (b <= b_last) {
              const float4* src = partial_ptr(b, sk_lo(sk, b) >= x0 ? 0 : 1, c);
#pragma unroll
              for (int v = 0; v < 8; ++v) p[d][v] = __ldcg(src + v * 32);
            }
          }
#pragma unroll
          for (int d = 0; d < kSkDepth; ++d) {
            const int b = b0 + d;
            if (b > b_last) break;
#pragma unroll
            for (int v = 0; v < 8; ++v) {
              if (b == b_first) {
                sum[v] = p[d][v];
              } else {
                sum[v].x += p[d][v].x;
                sum[v].y += p[d][v].y;
                sum[v].z += p[d][v].z;
                sum[v].w += p[d][v].w;
              }
            }
          }
        }
        std::uint32_t r[32];
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          r[4 * v] = __float_as_uint(sum[v].x);
          r[4 * v + 1] = __float_as_uint(sum[v].y);
          r[4 * v + 2] = __float_as_uint(sum[v].z);
          r[4 * v + 3] = __float_as_uint(sum[v].w);
        }
        store_chunk(r, &gm.c[p], C_BF16, nb * BN + c * 32, mb * BM + q * 32);
      }
      }  // OCC == 1
    });
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete
  } else {
    // Fused epilogue (bf16, one elementwise consumer): lane = output row of
    // the 32x32 chunk. The op's other operands (<= 2) are read straight into
    // registers one chunk ahead — the first chunk of a tile while its
    // accumulator is still being built — alternating between two register
    // sets so no load is waited on before its chunk. C and the op result
    // are staged swizzled side by side and leave as two TMA stores in one
    // bulk group. Bits equal the separate kernels': the op folds its inputs
    // in order, reading the GEMM's bf16-rounded C.
    const int q = warp % 4;
    std::uint8_t* stg = staging + (warp - 2) * 2 * 4096;  // [2][C 2 KB | result 2 KB]
    // 8 epilogue warps: warps q and q + 4 share TMEM lane quarter q, each
    // taking half of the tile's 32-column chunks.
    constexpr int NCH = BN / 32;
    const int c_lo = EPI_WARPS == 8 ? ((warp - 2) / 4) * (NCH / 2) : 0;
    const int c_hi = EPI_WARPS == 8 ? c_lo + NCH / 2 : NCH;
    const int swz = (lane >> 1) & 3;
    const int nst = epi.n_slots;
    const __nv_bfloat16* src0 =
        static_cast<const __nv_bfloat16*>(epi.ops[0].in[epi.slot_in[0]]);
    const __nv_bfloat16* src1 =
        static_cast<const __nv_bfloat16*>(epi.ops[0].in[epi.slot_in[1]]);
    auto load = [&](int t_, int c_, uint4(&d)[kMaxEpiSlots][4]) {
      int mb_, nb_;
      int p_;
      coords(t_, p_, mb_, nb_);
      const int grow = mb_ * BM + q * 32 + lane;
      const int gcol = nb_ * BN + c_ * 32;
      const std::int64_t off = static_cast<std::int64_t>(grow) * n + gcol;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const bool ok = grow < m && gcol + 8 * v < n;  // n % 8 == 0: whole vectors
        // Streaming loads (evict-first): the fused operand is read once and
        // must not push the GEMM's A / B panels out of L2.
        d[0][v] = ok && nst > 0 ? __ldcs(reinterpret_cast<const uint4*>(src0 + off) + v) : make_uint4(0, 0, 0, 0);
        d[1][v] = ok && nst > 1 ? __ldcs(reinterpret_cast<const uint4*>(src1 + off) + v) : make_uint4(0, 0, 0, 0);
      }
    };
    int g = 0;  // chunk counter of this warp (staging ring position)
    auto chunk = [&](int t, int mb, int nb, int c, std::uint32_t base, int acc, uint4(&cur)[kMaxEpiSlots][4],
                     uint4(&nxt)[kMaxEpiSlots][4]) {
      if (c + 1 < c_hi) load(t, c + 1, nxt);
      else if (t + static_cast<int>(gridDim.x) < work_items) load(t + gridDim.x, c_lo, nxt);
      std::uint32_t r[32];
      tmem_ld32(base + c * 32, r);
      if (c == c_hi - 1) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (SM2) mbar_arrive_cluster(cluster_addr(&tempty[acc], 0));  // the leader's MMA waits
          else mbar_arrive(&tempty[acc]);
        }
      }
      std::uint32_t cw[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) cw[i] = bf16_pair(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // ring entry g&1 is free
      __syncwarp();
      std::uint8_t* buf = stg + (g & 1) * 4096;
      // Fold + store, specialised on the activation so the plain ops'
      // loop carries no GELU code (a runtime select would evaluate both).
      auto fold_store = [&](auto act) {
        constexpr int ACT = decltype(act)::value;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          *reinterpret_cast<uint4*>(buf + lane * 64 + ((v ^ swz) << 4)) =
              make_uint4(cw[4 * v], cw[4 * v + 1], cw[4 * v + 2], cw[4 * v + 3]);
          float accv[8];
#pragma unroll
          for (int i = 0; i < kMaxEpiIn; ++i) {
            if (i >= epi.ops[0].n_in) break;
            const uint4 w = i == epi.ops[0].gemm_pos ? make_uint4(cw[4 * v], cw[4 * v + 1], cw[4 * v + 2], cw[4 * v + 3])
                            : (nst > 1 && epi.slot_in[1] == i) ? cur[1][v]
                                                               : cur[0][v];
            float x[8];
            bf16_unpair(w.x, x[0], x[1]);
            bf16_unpair(w.y, x[2], x[3]);
            bf16_unpair(w.z, x[4], x[5]);
            bf16_unpair(w.w, x[6], x[7]);
#pragma unroll
            for (int e = 0; e < 8; ++e) accv[e] = i == 0 ? x[e] : epi_apply<ACT>(epi.ops[0].op, accv[e], x[e]);
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) accv[e] = epi_finish<ACT>(accv[e]);
          *reinterpret_cast<uint4*>(buf + 2048 + lane * 64 + ((v ^ swz) << 4)) =
              make_uint4(bf16_pair(accv[0], accv[1]), bf16_pair(accv[2], accv[3]), bf16_pair(accv[4], accv[5]),
                         bf16_pair(accv[6], accv[7]));
        }
      };
      const int eop = epi.ops[0].op;
      if (eop == 3) fold_store(std::integral_constant<int, 3>{});
      else if (eop == 4) fold_store(std::integral_constant<int, 4>{});
      else fold_store(std::integral_constant<int, 0>{});
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        const int c0 = nb * BN + c * 32, c1 = mb * BM + q * 32;
        // The fused op streams a tensor as large as C through L2: its
        // results leave evict-first so the GEMM's A / B panels stay resident.
        const std::uint64_t pol = l2_evict_first_policy();
        tma_store_2d_nc_hint(&gm.c[0], buf, c0, c1, pol);
        tma_store_2d_nc_hint(&maps.out[0], buf + 2048, c0, c1, pol);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      ++g;
    };
    uint4 pa[kMaxEpiSlots][4], pb[kMaxEpiSlots][4];
    if (static_cast<int>(blockIdx.x) < work_items) load(blockIdx.x, c_lo, pa);
    int local = 0;
    // Work items t = blockIdx.x + i * gridDim.x: plain tiles, or (pairs)
    // 2 * pair + rank — the same stride, cluster rank = blockIdx.x % 2.
    for (int t = blockIdx.x; t < work_items; t += gridDim.x, ++local) {
      int mb, nb;
      int p;
      coords(t, p, mb, nb);
      const int acc = local & 1;
      mbar_wait(&tfull[acc], (local >> 1) & 1);
      tc_fence_after();
      const std::uint32_t base = tmem + (static_cast<std::uint32_t>(q * 32) << 16) + static_cast<std::uint32_t>(acc * BN);
#pragma unroll 1
      for (int c = c_lo; c < c_hi; c += 2) {
        chunk(t, mb, nb, c, base, acc, pa, pb);
        chunk(t, mb, nb, c + 1, base, acc, pb, pa);
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync();  // no CTA leaves while its peer may still multicast / arrive into it
  if (warp == 1) {
    tc_fence_after();
    if constexpr (SM2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
  }
}

// Split-K reduction: C_p[row][col..col+3] = sum over splits s (in order) of
// ws[(p*S + s)*m_pad + row][col..col+3] — coalesced on both sides.
struct SplitOut {
  void* c[kMaxGemmGroup];
};

template <bool C_BF16>
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float4* __restrict__ ws, const __grid_constant__ SplitOut out, int S,
                                                            int m, int n, int m_pad, int n_pad, int ng) {
  pdl_wait();
  pdl_trigger();
  const int n4 = n / 4;
  const long long per = static_cast<long long>(m) * n4;
  const long long total = per * ng;
  const int np4 = n_pad / 4;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int p = static_cast<int>(i / per);
    const long long rem = i - p * per;
    const int row = static_cast<int>(rem / n4), c4 = static_cast<int>(rem - static_cast<long long>(row) * n4);
    const float4* src = ws + (static_cast<long long>(p) * S * m_pad + row) * np4 + c4;
    const long long step = static_cast<long long>(m_pad) * np4;
    // kSplitBatch partial loads in flight per thread, summed in split order.
    constexpr int kSplitBatch = 8;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s0 = 0; s0 < S; s0 += kSplitBatch) {
      float4 v[kSplitBatch];
#pragma unroll
      for (int j = 0; j < kSplitBatch; ++j)
        if (s0 + j < S) v[j] = __ldcg(src + (s0 + j) * step);
#pragma unroll
      for (int j = 0; j < kSplitBatch; ++j) {
        if (s0 + j >= S) break;
        if (s0 + j == 0) {
          acc = v[j];
        } else {
          acc.x += v[j].x;
          acc.y += v[j].y;
          acc.z += v[j].z;
          acc.w += v[j].w;
        }
      }
    }
    if constexpr (C_BF16) {
      uint2 w = make_uint2(bf16_pair(acc.x, acc.y), bf16_pair(acc.z, acc.w));
      reinterpret_cast<uint2*>(out.c[p])[rem] = w;
    } else {
      reinterpret_cast<float4*>(out.c[p])[rem] = acc;
    }
  }
}

// ---- host ---------------------------------------------------------------------

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
  });
  if (!fn) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
  return fn;
}

// bf16 row-major [rows][cols] matrix, box {64 cols, box_rows}, 128B swizzle.
CUtensorMap make_map(const void* base, std::int64_t rows, std::int64_t cols, int box_rows) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}

// Output map for the staged epilogue: [m][n] row-major, 32x32 boxes,
// 64B swizzle for bf16 rows (64 B), 128B swizzle for fp32 rows (128 B).
CUtensorMap make_store_map(void* base, std::int64_t m, std::int64_t n, bool bf16) {
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  const std::int64_t es = bf16 ? 2 : 4;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(m)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(n * es)};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base,
                           dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           bf16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled (C) failed: " + std::to_string(r));
  return map;
}

int device_sms() {
  static int num_sms[32] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (num_sms[dev & 31] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    num_sms[dev & 31] = v > 0 ? v : 148;
  }
  return num_sms[dev & 31];
}

// L2 residency of the operands. The grouped raster (GROUP_M rows of tiles,
// N slow) streams each A row-panel through L2 once, shared by the group's
// concurrently running N-tiles, while every group re-reads all of B (and,
// for tall-k shapes, a wide B re-reads A across N-tiles). When the operands
// together outgrow L2 (126 MB), the smaller one (<= 48 MB) is loaded
// evict_last so it survives the other's stream between raster groups — the
// re-reads of it otherwise come from HBM (C2's k = 8192 launches read
// ~2x their algorithmic bytes, profiles/r01/ncu_gemm_dram_c2_tp1_v10.csv).
// The large operand streams evict_first (C2's k = 8192 launches 336 -> 264 MB
// of DRAM reads and 190 -> 184 us, gpurun_out/l2hint r02). PLANC_B200_L2HINT
// =0 disables, =1 marks only the small operand;
// PLANC_B200_GROUP_M sets the raster group height.
inline void l2_plan(const GemmArgs& a, SkParams& sk) {
  static const int mode = [] {
    const char* e = std::getenv("PLANC_B200_L2HINT");
    return e ? std::atoi(e) : 2;
  }();
  static const int group_m = [] {
    const char* e = std::getenv("PLANC_B200_GROUP_M");
    return e && std::atoi(e) > 0 ? std::atoi(e) : GROUP_M;
  }();
  sk.group_m = group_m;
  sk.hint_a = sk.hint_b = 0;
  if (mode == 0) return;
  const double g = std::max(a.group, 1);
  const double bytes_a = g * a.m * a.k * 2.0, bytes_b = g * a.k * a.n * 2.0;
  const double small = std::min(bytes_a, bytes_b), big = std::max(bytes_a, bytes_b);
  // Launches that stream a large output (and, fused, as large an operand
  // and result) through L2 evict the operand every raster group re-reads —
  // all of B, once per group of M-blocks — even when A and B fit together:
  // C2's fused 8192x8192x2048 launches read 356 MB for 201 MB of operands
  // (profiles/r02/l2hint). Keeping B (evict_last) with A streaming was
  // measured worse (C2's fused 8192x8192x2048 launch 228 -> 237 us, 353 ->
  // 473 MB read; profiles/r02/ab_l2_stream.jsonl): opt-in only,
  // PLANC_B200_L2HINT_STREAM=1.
  static const bool stream_rule = [] {
    const char* e = std::getenv("PLANC_B200_L2HINT_STREAM");
    return e && e[0] == '1';
  }();
  const double out_bytes = g * a.m * a.n * (a.dc == DT_BF16 ? 2.0 : 4.0) * (a.epi.n_ops > 0 ? 3.0 : 1.0);
  if (stream_rule && small + big <= 96e6 && out_bytes >= 64e6 && bytes_b <= 48e6) {
    sk.hint_b = 2;
    if (mode == 2) sk.hint_a = 1;
    return;
  }
  if (small + big <= 96e6 || small > 48e6) return;
  const bool a_small = bytes_a <= bytes_b;
  (a_small ? sk.hint_a : sk.hint_b) = 2;
  if (mode == 2) (a_small ? sk.hint_b : sk.hint_a) = 1;
}

template <bool A_MN, bool B_MN, bool C_BF16, int BN, bool FUSE, int NG, int OCC = 1>
void launch_typed_ng(const GemmArgs& a, const GemmSchedule& sc, cudaStream_t s) {
  static unsigned attr_set_mask = 0;  // per device ordinal
  constexpr int SMEM_BYTES = Cfg<BN, FUSE, OCC>::SMEM_BYTES;
  auto kern = gemm_tc_kernel<A_MN, B_MN, C_BF16, BN, FUSE, NG, OCC>;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_set_mask & (1u << dev))) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) throw std::runtime_error(std::string("gemm_tc smem attribute: ") + cudaGetErrorString(e));
    attr_set_mask |= 1u << dev;
  }
  // A: [m][k] (K-major) or, transposed, [k][m] (MN-major); B: [k][n]
  // (MN-major) or, transposed, [n][k] (K-major).
  const int ng = a.group > 1 ? a.group : 1;
  if (ng > NG) throw std::runtime_error("gemm_tc: group above the launch's capacity");
  if (FUSE && ng > 1) throw std::runtime_error("gemm_tc: fused epilogue on a grouped launch");
  GroupMaps<NG> gm;
  std::memset(&gm, 0, sizeof(gm));
  for (int i = 0; i < ng; ++i) {
    const void* A = ng > 1 ? a.gA[i] : a.A;
    const void* B = ng > 1 ? a.gB[i] : a.B;
    void* C = ng > 1 ? a.gC[i] : a.C;
    gm.a[i] = A_MN ? make_map(A, a.k, a.m, BK) : make_map(A, a.m, a.k, BM);
    gm.b[i] = B_MN ? make_map(B, a.k, a.n, BK) : make_map(B, a.n, a.k, OCC >= 4 ? BN / 2 : BN);
    gm.c[i] = make_store_map(a.scatter > 0 ? a.gC[0] : C, a.scatter > 0 ? a.scatter_rows : a.m, a.n, C_BF16);
  }
  if (a.scatter > 0) {
    if (a.scatter > kMaxGemmGroup || ng != 1 || FUSE || sc.splits > 1 || sc.sk_ctas > 0 || sc.half_items > 0 ||
        a.scatter_rows % BM != 0 || a.scatter_rows * a.scatter != a.m)
      throw std::runtime_error("gemm_tc: reduce-scatter epilogue needs a plain data-parallel launch");
  }
  EpiMaps maps;
  std::memset(&maps, 0, sizeof(maps));
  if constexpr (FUSE) maps.out[0] = make_store_map(a.epi.ops[0].out, a.m, a.n, true);
  SkParams sk;
  sk.dp_tiles = sc.dp_tiles;
  sk.sk_ctas = sc.sk_ctas;
  sk.sk_iters = sc.sk_iters;
  sk.splits = sc.splits;
  sk.half_items = sc.half_items;
  sk.scatter_rows = a.scatter > 0 ? static_cast<int>(a.scatter_rows) : 0;
  l2_plan(a, sk);
  for (int i = 0; i < a.scatter; ++i) sk.scatter_dst[i] = a.gC[i];
  if (a.gather_maps) {
    sk.gather_rows_a = static_cast<int>(a.gather_rows_a);
    sk.gather_rows_b = static_cast<int>(a.gather_rows_b);
    sk.gather_cols_a = static_cast<int>(a.gather_cols_a);
    sk.gather_cols_b = static_cast<int>(a.gather_cols_b);
    sk.gather_na = a.gather_a;
    sk.gather_nb = a.gather_b;
    sk.gather_maps = static_cast<const CUtensorMap*>(a.gather_maps);
  }
  const std::int64_t m_pad = (a.m + BM - 1) / BM * BM, n_pad = (a.n + BN - 1) / BN * BN;
  if (sc.splits > 1) {
    // Partials: fp32 [ng * splits * m_pad][n_pad], stored like an fp32 C.
    maps.ws = make_store_map(a.ws, static_cast<std::int64_t>(ng) * sc.splits * m_pad, n_pad, false);
  } else if (sc.sk_ctas > 0) {
    char* ws = static_cast<char*>(a.ws);
    sk.counters = reinterpret_cast<int*>(ws);
    sk.partials = reinterpret_cast<float*>(ws + sc.counter_bytes);
  }
  pdl_launch_cluster("gemm_tc_kernel", kern, dim3(sc.grid), dim3(cta_threads(OCC)), SMEM_BYTES, s, OCC >= 4 ? 2 : 1,
             gm, ng, static_cast<int>(a.m),
             static_cast<int>(a.n), static_cast<int>(a.k), a.epi, maps, sk);
  if (sc.splits > 1) {
    SplitOut out;
    for (int i = 0; i < ng; ++i) out.c[i] = ng > 1 ? a.gC[i] : a.C;
    const long long work = static_cast<long long>(ng) * a.m * (a.n / 4);
    const int blocks = static_cast<int>(std::min<long long>((work + 255) / 256, 4LL * device_sms()));
    pdl_launch("splitk_reduce_kernel", splitk_reduce_kernel<C_BF16>, dim3(blocks), dim3(256), 0, s,
               static_cast<const float4*>(a.ws), out, sc.splits, static_cast<int>(a.m), static_cast<int>(a.n),
               static_cast<int>(m_pad), static_cast<int>(n_pad), ng);
  }
}

// Tensor maps of a gathered operand's pieces with the box the launch of
// schedule `sc` loads (gemm_sm100_gather_maps).
inline void encode_gather_maps(const GemmArgs& a, const GemmSchedule& sc, CUtensorMap* out) {
  const bool a_mn = a.ta, b_mn = !a.tb;
  // Row pieces: (piece rows) x (full stored width); column pieces: (full
  // stored rows) x (piece columns).
  for (int i = 0; i < a.gather_a; ++i) {
    // A: K-major [m][k] boxes of BM rows; MN-major [k][m] boxes of BK rows
    const std::int64_t rows = a.gather_cols_a ? (a_mn ? a.k : a.m) : a.gather_rows_a;
    const std::int64_t cols = a.gather_cols_a ? a.gather_cols_a : (a_mn ? a.m : a.k);
    out[i] = make_map(a.gather_a_ptr[i], rows, cols, a_mn ? BK : BM);
  }
  for (int i = 0; i < a.gather_b; ++i) {
    // B: MN-major [k][n] boxes of BK rows; K-major [n][k] boxes of BN (pairs: BN/2) rows
    const std::int64_t rows = a.gather_cols_b ? (b_mn ? a.k : a.n) : a.gather_rows_b;
    const std::int64_t cols = a.gather_cols_b ? a.gather_cols_b : (b_mn ? a.n : a.k);
    out[kMaxGemmGroup + i] = make_map(a.gather_b_ptr[i], rows, cols, b_mn ? BK : (sc.occ >= 4 ? sc.bn / 2 : sc.bn));
  }
}

template <bool A_MN, bool B_MN, bool C_BF16, int BN, bool FUSE>
void launch_typed(const GemmArgs& a, const GemmSchedule& sc, cudaStream_t s) {
  if constexpr (FUSE) {
    if constexpr (BN >= 128) {
      if (sc.occ == 5) return launch_typed_ng<A_MN, B_MN, C_BF16, BN, FUSE, 1, 5>(a, sc, s);
    }
    if (sc.occ == 3) return launch_typed_ng<A_MN, B_MN, C_BF16, BN, FUSE, 1, 3>(a, sc, s);
    launch_typed_ng<A_MN, B_MN, C_BF16, BN, FUSE, 1>(a, sc, s);
  } else if (sc.occ == 4 || sc.occ == 5) {
    if constexpr (BN >= 128) {
      if (sc.occ == 5) {
        if (a.group > 1) launch_typed_ng<A_MN, B_MN, C_BF16, BN, FUSE, kMaxGemmGroup, 5>(a, sc, s);
        else launch_typed_ng<A_MN, B_MN, C_BF16, BN, FUSE, 1, 5>(a, sc, s);
      } else if (a.group > 1) launch_typed_ng<A_MN, B_MN, C_BF16, BN, FUSE, kMaxGemmGroup, 4>(a, sc, s);
      else launch_typed_ng<A_MN, B_MN, C_BF16, BN, FUSE, 1, 4>(a, sc, s);
    } else {
      throw std::runtime_error("gemm_tc: cluster pairs need BN >= 128");
    }
  } else if (sc.occ == 3) {
    if (a.group > 1) launch_typed_ng<A_MN, B_MN, C_BF16, BN, FUSE, kMaxGemmGroup, 3>(a, sc, s);
    else launch_typed_ng<A_MN, B_MN, C_BF16, BN, FUSE, 1, 3>(a, sc, s);
  } else if constexpr (BN <= 128) {
    const bool wide = a.group > 1;  // member maps
    if (sc.occ == 2) {
      if (wide) launch_typed_ng<A_MN, B_MN, C_BF16, BN, FUSE, kMaxGemmGroup, 2>(a, sc, s);
      else launch_typed_ng<A_MN, B_MN, C_BF16, BN, FUSE, 1, 2>(a, sc, s);
    } else {
      if (wide) launch_typed_ng<A_MN, B_MN, C_BF16, BN, FUSE, kMaxGemmGroup>(a, sc, s);
      else launch_typed_ng<A_MN, B_MN, C_BF16, BN, FUSE, 1>(a, sc, s);
    }
  } else {
    if (a.group > 1) launch_typed_ng<A_MN, B_MN, C_BF16, BN, FUSE, kMaxGemmGroup>(a, sc, s);
    else launch_typed_ng<A_MN, B_MN, C_BF16, BN, FUSE, 1>(a, sc, s);
  }
}

}  // namespace

// One translation unit per operand-major combination instantiates the
// kernels (gemm_sm100_ab*.cu): the variants compile in parallel.
template <bool A_MN, bool B_MN>
void launch_gemm_tc_ab(const GemmArgs& a, const GemmSchedule& sc, cudaStream_t s);

}  // namespace planc_b200
