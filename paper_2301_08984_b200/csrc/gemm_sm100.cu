// tcgen05 / TMEM / TMA GEMM for the plan's matmul sub-operators (sm_100a).
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
//               drains. Optional fused elementwise consumers (FUSE) re-read
//               the staged chunk row-contiguously.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "kernels.cuh"

namespace planc_b200 {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 128 bytes of bf16: one 128B swizzle row
constexpr int A_STAGE_BYTES = BM * BK * 2;  // 16 KB
constexpr int NUM_THREADS = 192;
constexpr int GROUP_M = 8;

// Tile width BN in {256, 128, 64}: smem ring depth fills ~200 KB, TMEM holds
// two BN-column fp32 accumulators (power of two >= 32 columns).
template <int BN_>
struct Cfg {
  static constexpr int BN = BN_;
  static constexpr int B_STAGE_BYTES = BN * BK * 2;
  static constexpr int STAGES_RAW = (200 * 1024) / (A_STAGE_BYTES + B_STAGE_BYTES);
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  // + epilogue staging: 4 warps x 2 buffers x (32 rows x 32 cols, <= 4 B)
  static constexpr int STAGING_BYTES = 4 * 2 * 4096;
  static constexpr int SMEM_BYTES =
      STAGES * (A_STAGE_BYTES + B_STAGE_BYTES) + STAGING_BYTES + 1024 /*align*/ + 1024 /*barriers + align*/;
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
};

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

// Bulk tensor store smem -> global (clips rows / cols outside the tensor).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<std::uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
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
template <int BN>
__host__ __device__ constexpr std::uint32_t make_idesc(bool a_mn, bool b_mn) {
  return (1u << 4)                              // D format f32
         | (1u << 7)                            // A bf16
         | (1u << 10)                           // B bf16
         | ((a_mn ? 1u : 0u) << 15)             // A major
         | ((b_mn ? 1u : 0u) << 16)             // B major
         | (static_cast<std::uint32_t>(BN >> 3) << 17)  // N
         | (static_cast<std::uint32_t>(BM >> 4) << 24); // M
}

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

__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int& mb, int& nb) {
  const int per_group = GROUP_M * tiles_n;
  const int group = t / per_group;
  const int first_m = group * GROUP_M;
  const int gm = min(tiles_m - first_m, GROUP_M);
  const int r = t % per_group;
  mb = first_m + r % gm;
  nb = r / gm;
}

__device__ __forceinline__ float epi_apply(int op, float a, float b) {
  return op == 0 ? a + b : op == 1 ? a * b : fmaxf(a, b);
}

__device__ __forceinline__ std::uint32_t bf16_pair(float lo, float hi) {
  return static_cast<std::uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(lo))) |
         (static_cast<std::uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(hi))) << 16);
}

__device__ __forceinline__ void bf16_unpair(std::uint32_t w, float& lo, float& hi) {
  lo = __uint_as_float(w << 16);
  hi = __uint_as_float(w & 0xffff0000u);
}

template <bool A_MN, bool B_MN, bool C_BF16, int BN, bool FUSE>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, void* __restrict__ C, int m, int n, int k,
                   const __grid_constant__ EpiParams epi) {
  extern __shared__ std::uint8_t smem_raw[];
  constexpr int STAGES = Cfg<BN>::STAGES;
  constexpr int B_STAGE_BYTES = Cfg<BN>::B_STAGE_BYTES;
  constexpr int TMEM_COLS = Cfg<BN>::TMEM_COLS;
  std::uint8_t* smem =
      reinterpret_cast<std::uint8_t*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  std::uint8_t* sA = smem;
  std::uint8_t* sB = smem + STAGES * A_STAGE_BYTES;
  // Epilogue staging (1024-aligned: the 64B / 128B swizzle atoms of the C map).
  std::uint8_t* staging = sB + STAGES * B_STAGE_BYTES;
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(staging + Cfg<BN>::STAGING_BYTES);
  std::uint64_t* empty = full + STAGES;
  std::uint64_t* tfull = empty + STAGES;  // [2] accumulator ready
  std::uint64_t* tempty = tfull + 2;      // [2] accumulator drained
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int tiles_m = (m + BM - 1) / BM;
  const int tiles_n = (n + BN - 1) / BN;
  const int num_tiles = tiles_m * tiles_n;
  const int num_k = (k + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tmB)) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;  // global k-block counter across tiles (ring position)
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(t, tiles_m, tiles_n, mb, nb);
        const int m0 = mb * BM, n0 = nb * BN;
        for (int kb = 0; kb < num_k; ++kb, ++it) {
          const int s = it % STAGES;
          const std::uint32_t phase = (it / STAGES) & 1;
          mbar_wait(&empty[s], phase ^ 1);
          mbar_expect_tx(&full[s], A_STAGE_BYTES + B_STAGE_BYTES);
          std::uint8_t* a = sA + s * A_STAGE_BYTES;
          std::uint8_t* b = sB + s * B_STAGE_BYTES;
          if (A_MN) {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) tma_load_2d(a + j * (64 * BK * 2), &tmA, m0 + 64 * j, kb * BK, &full[s]);
          } else {
            tma_load_2d(a, &tmA, kb * BK, m0, &full[s]);
          }
          if (B_MN) {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) tma_load_2d(b + j * (64 * BK * 2), &tmB, n0 + 64 * j, kb * BK, &full[s]);
          } else {
            tma_load_2d(b, &tmB, kb * BK, n0, &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr std::uint32_t idesc = make_idesc<BN>(A_MN, B_MN);
      int it = 0, local = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++local) {
        const int acc = local & 1;
        const std::uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);  // epilogue drained this accumulator
        tc_fence_after();
        const std::uint32_t d = tmem + static_cast<std::uint32_t>(acc * BN);
        for (int kb = 0; kb < num_k; ++kb, ++it) {
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
            tc_mma(d, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
          }
          tc_commit(&empty[s]);  // smem stage free once these MMAs retire
        }
        tc_commit(&tfull[acc]);  // accumulator complete
      }
    }
  } else {
    // Epilogue warps 2..5: warp w may only touch TMEM lanes 32*(w%4)..+31.
    // Each 32x32 output chunk goes TMEM -> registers -> swizzled smem
    // staging (conflict-free 16-byte stores) -> one TMA bulk tensor store
    // (coalesced, clipped at the tensor edge); two staging buffers per warp
    // keep a store in flight while the next chunk is converted.
    const int q = warp % 4;
    std::uint8_t* stg = staging + (warp - 2) * 2 * 4096;
    int sb = 0;
    int local = 0;
    // Fused-operand prefetch (FUSE): the 4 row segments this lane handles in
    // a 32x32 chunk, per operand slot; chunk c+1 is in flight while chunk c
    // is processed, and a tile's first chunk while its accumulator is built.
    uint4 pf_cur[kMaxEpiSlots][4], pf_nxt[kMaxEpiSlots][4];
    auto prefetch = [&](int mb_, int nb_, int c_, uint4(&dst)[kMaxEpiSlots][4]) {
#pragma unroll
      for (int s = 0; s < kMaxEpiSlots; ++s) {
        const int o = epi.slot_op[s], i = epi.slot_in[s];
        const __nv_bfloat16* srcb = static_cast<const __nv_bfloat16*>(epi.ops[o].in[i]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint4 val = make_uint4(0u, 0u, 0u, 0u);
          const int rr = (lane >> 2) + 8 * j;
          const int grow = mb_ * BM + q * 32 + rr;
          const int gcol = nb_ * BN + c_ * 32 + 8 * (lane & 3);
          if (s < epi.n_slots && grow < m && gcol < n) {
            const __nv_bfloat16* p = srcb + static_cast<std::int64_t>(grow) * n + gcol;
            if (gcol + 8 <= n) {
              val = __ldg(reinterpret_cast<const uint4*>(p));
            } else {
              std::uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
              for (int e = 0; e < 8; ++e)
                if (gcol + e < n)
                  w[e >> 1] |= static_cast<std::uint32_t>(__bfloat16_as_ushort(p[e])) << (16 * (e & 1));
              val = make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
          dst[s][j] = val;
        }
      }
    };
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++local) {
      int mb, nb;
      tile_coords(t, tiles_m, tiles_n, mb, nb);
      const int acc = local & 1;
      if constexpr (FUSE) prefetch(mb, nb, 0, pf_cur);
      mbar_wait(&tfull[acc], (local >> 1) & 1);
      tc_fence_after();
      const int row = mb * BM + q * 32 + lane;
      (void)row;
      const std::uint32_t base = tmem + (static_cast<std::uint32_t>(q * 32) << 16) + static_cast<std::uint32_t>(acc * BN);
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        if constexpr (FUSE) {
          if (c + 1 < BN / 32) prefetch(mb, nb, c + 1, pf_nxt);
        }
        std::uint32_t r[32];
        tmem_ld32(base + c * 32, r);
        if (c == BN / 32 - 1) {
          // All TMEM reads of this accumulator are complete: hand it back.
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        {
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // buffer sb is free
          __syncwarp();
          std::uint8_t* buf = stg + sb * 4096;
          if constexpr (C_BF16) {
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
          if (lane == 0) tma_store_2d(&tmC, buf, nb * BN + c * 32, mb * BM + q * 32);
          if constexpr (FUSE) {
            // Fused elementwise consumers, in the row-contiguous domain: the
            // staged (bf16-rounded) chunk is re-read so that 4 lanes cover
            // one 64-byte row segment — operand loads and result stores are
            // coalesced. Bits equal the separate elementwise kernel's.
#pragma unroll
            for (int o = 0; o < kMaxEpiOps; ++o) {
              if (o >= epi.n_ops) break;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int rr = (lane >> 2) + 8 * j;
                const int v = lane & 3;
                const int grow = mb * BM + q * 32 + rr;
                const int gcol = nb * BN + c * 32 + 8 * v;
                if (grow >= m || gcol >= n) continue;
                const uint4 cw = *reinterpret_cast<const uint4*>(buf + rr * 64 + ((v ^ ((rr >> 1) & 3)) << 4));
                float cv[8];
                bf16_unpair(cw.x, cv[0], cv[1]);
                bf16_unpair(cw.y, cv[2], cv[3]);
                bf16_unpair(cw.z, cv[4], cv[5]);
                bf16_unpair(cw.w, cv[6], cv[7]);
                const std::int64_t off = static_cast<std::int64_t>(grow) * n + gcol;
                const bool whole = gcol + 8 <= n;
                float acc[8];
#pragma unroll
                for (int i = 0; i < kMaxEpiIn; ++i) {
                  if (i >= epi.ops[o].n_in) break;
                  float x[8];
                  if (i == epi.ops[o].gemm_pos) {
#pragma unroll
                    for (int e = 0; e < 8; ++e) x[e] = cv[e];
                  } else {
                    // prefetched one chunk ahead (static slot selection)
                    const bool s1 = epi.n_slots > 1 && epi.slot_op[1] == o && epi.slot_in[1] == i;
                    const uint4 qv = s1 ? pf_cur[1][j] : pf_cur[0][j];
                    bf16_unpair(qv.x, x[0], x[1]);
                    bf16_unpair(qv.y, x[2], x[3]);
                    bf16_unpair(qv.z, x[4], x[5]);
                    bf16_unpair(qv.w, x[6], x[7]);
                  }
#pragma unroll
                  for (int e = 0; e < 8; ++e) acc[e] = i == 0 ? x[e] : epi_apply(epi.ops[o].op, acc[e], x[e]);
                }
                __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(epi.ops[o].out) + off;
                if (whole) {
                  *reinterpret_cast<uint4*>(dst) = make_uint4(bf16_pair(acc[0], acc[1]), bf16_pair(acc[2], acc[3]),
                                                              bf16_pair(acc[4], acc[5]), bf16_pair(acc[6], acc[7]));
                } else {
#pragma unroll
                  for (int e = 0; e < 8; ++e)
                    if (gcol + e < n) dst[e] = __float2bfloat16_rn(acc[e]);
                }
              }
            }
#pragma unroll
            for (int s = 0; s < kMaxEpiSlots; ++s)
#pragma unroll
              for (int j = 0; j < 4; ++j) pf_cur[s][j] = pf_nxt[s][j];
          }
          sb ^= 1;
        }
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
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

template <bool A_MN, bool B_MN, bool C_BF16, int BN, bool FUSE>
void launch_typed(const GemmArgs& a, cudaStream_t s) {
  static unsigned attr_set_mask = 0;  // per device ordinal
  static int num_sms[32] = {0};
  constexpr int SMEM_BYTES = Cfg<BN>::SMEM_BYTES;
  auto kern = gemm_tc_kernel<A_MN, B_MN, C_BF16, BN, FUSE>;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_set_mask & (1u << dev))) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) throw std::runtime_error(std::string("gemm_tc smem attribute: ") + cudaGetErrorString(e));
    cudaDeviceGetAttribute(&num_sms[dev & 31], cudaDevAttrMultiProcessorCount, dev);
    attr_set_mask |= 1u << dev;
  }
  // A: [m][k] (K-major) or, transposed, [k][m] (MN-major); B: [k][n]
  // (MN-major) or, transposed, [n][k] (K-major).
  CUtensorMap ma = A_MN ? make_map(a.A, a.k, a.m, BK) : make_map(a.A, a.m, a.k, BM);
  CUtensorMap mb = B_MN ? make_map(a.B, a.k, a.n, BK) : make_map(a.B, a.n, a.k, BN);
  CUtensorMap mc = make_store_map(a.C, a.m, a.n, C_BF16);
  const std::int64_t tiles = ((a.m + BM - 1) / BM) * ((a.n + BN - 1) / BN);
  const int grid = static_cast<int>(std::min<std::int64_t>(tiles, num_sms[dev & 31] > 0 ? num_sms[dev & 31] : 148));
  kern<<<grid, NUM_THREADS, SMEM_BYTES, s>>>(ma, mb, mc, a.C, static_cast<int>(a.m), static_cast<int>(a.n),
                                              static_cast<int>(a.k), a.epi);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("gemm_tc_kernel: ") + cudaGetErrorString(e));
}

}  // namespace

// Tile width: the candidate minimising (waves over the SMs) x (per-tile MMA
// time ~ BN, plus a fixed per-tile cost), so narrow / small GEMMs get more,
// narrower tiles. PLANC_B200_GEMM_BN=256|128|64 forces one (experiments).
int gemm_sm100_tile_n(const GemmArgs& a) {
  const char* env = std::getenv("PLANC_B200_GEMM_BN");
  const int forced = env ? std::atoi(env) : 0;
  if (forced == 256 || forced == 128 || forced == 64) return forced;
  const std::int64_t sms = 148;
  int best = 256;
  double best_cost = 1e300;
  for (int bn : {256, 128, 64}) {
    const std::int64_t tiles = ((a.m + BM - 1) / BM) * ((a.n + bn - 1) / bn);
    const std::int64_t waves = (tiles + sms - 1) / sms;
    const double cost = static_cast<double>(waves) * (bn + 64.0);
    if (cost < best_cost * 0.97) {  // prefer wider tiles unless clearly better
      best_cost = cost;
      best = bn;
    }
  }
  return best;
}

bool gemm_sm100_eligible(const GemmArgs& a) {
  if (a.da != DT_BF16 || a.db != DT_BF16 || (a.dc != DT_BF16 && a.dc != DT_F32)) return false;
  if (a.m <= 0 || a.n <= 0 || a.k <= 0) return false;
  if (a.m > (1 << 30) || a.n > (1 << 30) || a.k > (1 << 30)) return false;
  // TMA: 16-byte global row pitch for both operands; 16-byte C vectors.
  if ((a.ta ? a.m : a.k) % 8 != 0) return false;
  if ((a.tb ? a.k : a.n) % 8 != 0) return false;
  if (a.n % 8 != 0) return false;
  // Tiny GEMMs stay on the SIMT path (a 128x256 tile would be mostly idle).
  if (a.m * a.n * a.k < (std::int64_t(1) << 20)) return false;
  return true;
}

void launch_gemm_sm100(const GemmArgs& a, cudaStream_t s) {
  const bool a_mn = a.ta, b_mn = !a.tb, cb = a.dc == DT_BF16;
  const int bn = gemm_sm100_tile_n(a);
  if (a.epi.n_ops > 0) {
    if (!cb) throw std::runtime_error("fused GEMM epilogue needs a bf16 output");
#define PLANC_TCF(AM, BMN)                                                      \
  if (a_mn == AM && b_mn == BMN) {                                             \
    if (bn == 256) return launch_typed<AM, BMN, true, 256, true>(a, s);        \
    if (bn == 128) return launch_typed<AM, BMN, true, 128, true>(a, s);        \
    return launch_typed<AM, BMN, true, 64, true>(a, s);                        \
  }
    PLANC_TCF(false, false)
    PLANC_TCF(false, true)
    PLANC_TCF(true, false)
    PLANC_TCF(true, true)
#undef PLANC_TCF
  }
#define PLANC_TC(AM, BMN, CB)                                                   \
  if (a_mn == AM && b_mn == BMN && cb == CB) {                                 \
    if (bn == 256) return launch_typed<AM, BMN, CB, 256, false>(a, s);         \
    if (bn == 128) return launch_typed<AM, BMN, CB, 128, false>(a, s);         \
    return launch_typed<AM, BMN, CB, 64, false>(a, s);                         \
  }
  PLANC_TC(false, false, false)
  PLANC_TC(false, false, true)
  PLANC_TC(false, true, false)
  PLANC_TC(false, true, true)
  PLANC_TC(true, false, false)
  PLANC_TC(true, false, true)
  PLANC_TC(true, true, false)
  PLANC_TC(true, true, true)
#undef PLANC_TC
}

}  // namespace planc_b200
