// fp32 GEMM on the tensor cores: 3xTF32 (tcgen05.mma kind::tf32) for the
// plan's fp32 matmul sub-operators — the reference's matmul_eval
// (proj/src/refexec.cpp:142-168) at fp32 accuracy instead of the SIMT FFMA
// tile (kernels.cu gemm_simt_kernel).
//
// Every operand element x is split once per launch into x_hi = x rounded to
// TF32 (10 explicit mantissa bits, low 13 bits zero) and x_lo = x - x_hi
// (exact in fp32); the tensor core then accumulates, per k-step and in fp32
// TMEM,
//     A_hi·B_lo + A_lo·B_hi + A_hi·B_hi
// — the product with the A_lo·B_lo term (~2^-22 relative) dropped and x_lo
// itself truncated to TF32 by the MMA (another ~2^-22): ~fp32 accuracy
// (|error| <~ 2^-20 · Σ|a||b|, inside north_star's 1e-5 fp32 bar), at a third
// of the TF32 tensor rate. Integer-valued operands below 2^11 have x_lo = 0,
// so fp32 plans on the reference's integer inputs stay exact while partial
// sums stay below 2^24.
//
// Kernels:
//   x3_split_kernel  one pass over A and B (16-byte vectors): hi / lo planes
//                    into the GEMM's workspace (HBM-bound, 12 B per element).
//   gemm_x3_kernel   persistent, one CTA per SM, 128 x 128 output tiles in
//                    grouped raster order, 6 warps: TMA producer (four planes
//                    per k-block: A_hi, A_lo, B_hi, B_lo, a 3-stage 64 KB
//                    ring; K-major operands 128B-swizzled, MN-major ones in
//                    the 128B / 32-byte-atom swizzle UMMA requires for 32-bit
//                    MN-major operands), single-thread MMA issuer (3 MMAs of
//                    128x128x8 per 32-byte k-step), 4 epilogue warps.
//
// Promotion: the tensor core adds each MMA's products into the fp32 TMEM
// accumulator without round-to-nearest (the error grows ~linearly with the
// number of MMAs: 7e-6 normwise at k = 1000, 3e-5 at k = 4096 measured with
// one accumulator per tile), so every X3_CHUNK_KB k-blocks the MMA warp
// switches to a fresh TMEM accumulator (a ring of four 128-column slots)
// and the epilogue warps add the finished chunk into fp32 registers with
// ordinary (round-to-nearest) adds, storing the tile after its last chunk.
#include "gemm_sm100_impl.cuh"

namespace planc_b200 {

namespace {

constexpr int X3_BN = 128;
constexpr int X3_BK = 32;                        // fp32 elements per 128-byte swizzle row
constexpr int X3_A_BYTES = BM * 128;             // one plane of the A tile, 16 KB
constexpr int X3_B_BYTES = X3_BN * 128;          // one plane of the B tile, 16 KB
constexpr int X3_STAGE_BYTES = 2 * (X3_A_BYTES + X3_B_BYTES);
constexpr int X3_STAGES = 3;
constexpr int X3_EPI_WARPS = 8;                  // two per TMEM lane quarter, 64 columns each
constexpr int X3_THREADS = 64 + 32 * X3_EPI_WARPS;
constexpr int X3_STAGING = X3_EPI_WARPS * 4096;  // one 32x32 fp32 staging buffer per warp
constexpr int X3_SMEM = X3_STAGES * X3_STAGE_BYTES + X3_STAGING + 1024 + 1024;
constexpr int X3_SLOTS = 4;       // TMEM accumulator ring (chunk partials)
constexpr int X3_TMEM_COLS = X3_SLOTS * X3_BN;
constexpr int X3_CHUNK_KB = 8;    // k-blocks (256 k) accumulated in TMEM before promotion
static_assert(X3_SMEM <= 227 * 1024, "3xTF32 ring above the shared memory limit");

// 32-bit MN-major operands: SWIZZLE_128B_BASE32B (32-byte atoms, 4-row
// groups; descriptor layout type 1), the only UMMA layout for MN-major tf32.
__device__ __forceinline__ std::uint64_t smem_desc_b32(std::uint32_t addr, std::uint32_t lbo, std::uint32_t sbo) {
  std::uint64_t d = 0;
  d |= static_cast<std::uint64_t>((addr >> 4) & 0x3FFFu);
  d |= static_cast<std::uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<std::uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;  // version
  d |= 1ull << 61;  // SWIZZLE_128B_BASE32B
  return d;
}

struct X3Maps {
  CUtensorMap ah, al, bh, bl, c;
};

// Instruction descriptor: kind::tf32, A/B tf32, D f32, M=128, N=128.
__host__ __device__ constexpr std::uint32_t x3_idesc(bool a_mn, bool b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         (static_cast<std::uint32_t>(X3_BN >> 3) << 17) | (static_cast<std::uint32_t>(BM >> 4) << 24);
}

__device__ __forceinline__ void tc_mma_tf32(std::uint32_t tmem_d, std::uint64_t adesc, std::uint64_t bdesc,
                                            std::uint32_t idesc, std::uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void x3_split1(float x, float& hi, float& lo) {
  const std::uint32_t u = __float_as_uint(x);
  if ((u & 0x7f800000u) == 0x7f800000u) {  // inf / nan: carried by the hi plane
    hi = x;
    lo = 0.f;
    return;
  }
  hi = __uint_as_float((u + 0x1000u) & 0xffffe000u);  // round half away from zero to 10 mantissa bits
  lo = x - hi;                                         // exact
}

struct X3Split {
  const float* src[2];
  float* hi[2];
  float* lo[2];
  long long count[2];
  long long blocks0;  // blocks of operand 0; the rest split operand 1
};

constexpr int kX3SplitThreads = 256;
constexpr int kX3SplitVec = 4;  // float4 per thread per operand block

__global__ void __launch_bounds__(kX3SplitThreads) x3_split_kernel(const __grid_constant__ X3Split p) {
  pdl_wait();
  pdl_trigger();
  const int op = blockIdx.x < p.blocks0 ? 0 : 1;
  const long long blk = op == 0 ? blockIdx.x : blockIdx.x - p.blocks0;
  const long long nvec = p.count[op] / 4;
  const float4* src = reinterpret_cast<const float4*>(p.src[op]);
  float4* hi = reinterpret_cast<float4*>(p.hi[op]);
  float4* lo = reinterpret_cast<float4*>(p.lo[op]);
  const long long base = blk * kX3SplitThreads * kX3SplitVec + threadIdx.x;
  float4 v[kX3SplitVec];
#pragma unroll
  for (int u = 0; u < kX3SplitVec; ++u) {
    const long long i = base + u * kX3SplitThreads;
    if (i < nvec) v[u] = __ldcs(src + i);
  }
#pragma unroll
  for (int u = 0; u < kX3SplitVec; ++u) {
    const long long i = base + u * kX3SplitThreads;
    if (i >= nvec) continue;
    float4 h, l;
    x3_split1(v[u].x, h.x, l.x);
    x3_split1(v[u].y, h.y, l.y);
    x3_split1(v[u].z, h.z, l.z);
    x3_split1(v[u].w, h.w, l.w);
    hi[i] = h;
    lo[i] = l;
  }
  // Scalar tail (count % 4), by the operand's first block.
  if (blk == 0 && threadIdx.x < (p.count[op] & 3)) {
    const long long i = nvec * 4 + threadIdx.x;
    float h, l;
    x3_split1(p.src[op][i], h, l);
    p.hi[op][i] = h;
    p.lo[op][i] = l;
  }
}

template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(X3_THREADS, 1)
    gemm_x3_kernel(const __grid_constant__ X3Maps mp, int m, int n, int k, int group_m) {
  extern __shared__ std::uint8_t smem_raw[];
  std::uint8_t* smem =
      smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays a shared-space pointer (STS / LDS)
  // Stage s: [A_hi | A_lo | B_hi | B_lo]
  std::uint8_t* ring = smem;
  std::uint8_t* staging = ring + X3_STAGES * X3_STAGE_BYTES;
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(staging + X3_STAGING);
  std::uint64_t* empty = full + X3_STAGES;
  std::uint64_t* tfull = empty + X3_STAGES;
  std::uint64_t* tempty = tfull + X3_SLOTS;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tempty + X3_SLOTS);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int tiles_m = (m + BM - 1) / BM;
  const int tiles_n = (n + X3_BN - 1) / X3_BN;
  const int tiles = tiles_m * tiles_n;
  const int num_k = (k + X3_BK - 1) / X3_BK;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&mp.ah)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&mp.al)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&mp.bh)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&mp.bl)) : "memory");
    for (int s = 0; s < X3_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < X3_SLOTS; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], X3_EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(X3_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = *tmem_slot;
  pdl_wait();  // the split planes (previous kernel on the stream) are visible

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(t, tiles_m, tiles_n, mb, nb, group_m);
        const int m0 = mb * BM, n0 = nb * X3_BN;
        for (int kb = 0; kb < num_k; ++kb, ++it) {
          const int s = it % X3_STAGES;
          mbar_wait(&empty[s], ((it / X3_STAGES) & 1) ^ 1);
          mbar_expect_tx(&full[s], X3_STAGE_BYTES);
          std::uint8_t* st = ring + s * X3_STAGE_BYTES;
          const int k0 = kb * X3_BK;
#pragma unroll
          for (int pl = 0; pl < 2; ++pl) {
            const CUtensorMap* ma = pl == 0 ? &mp.ah : &mp.al;
            const CUtensorMap* mbm = pl == 0 ? &mp.bh : &mp.bl;
            std::uint8_t* a = st + pl * X3_A_BYTES;
            std::uint8_t* b = st + 2 * X3_A_BYTES + pl * X3_B_BYTES;
            // K-major: one box of 128 rows x 32 k (128 B); MN-major: four
            // boxes of 32 k-rows x 32 MN elements (4 KB each).
            if (A_MN) {
#pragma unroll
              for (int j = 0; j < BM / 32; ++j) tma_load_2d(a + j * 4096, ma, m0 + 32 * j, k0, &full[s]);
            } else {
              tma_load_2d(a, ma, k0, m0, &full[s]);
            }
            if (B_MN) {
#pragma unroll
              for (int j = 0; j < X3_BN / 32; ++j) tma_load_2d(b + j * 4096, mbm, n0 + 32 * j, k0, &full[s]);
            } else {
              tma_load_2d(b, mbm, k0, n0, &full[s]);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr std::uint32_t idesc = x3_idesc(A_MN, B_MN);
      int it = 0, q = 0;  // ring position, chunk counter
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        std::uint32_t d = 0;
        for (int kb = 0; kb < num_k; ++kb, ++it) {
          const int slot = q % X3_SLOTS;
          if (kb % X3_CHUNK_KB == 0) {  // a fresh accumulator for this chunk
            mbar_wait(&tempty[slot], ((q / X3_SLOTS) & 1) ^ 1);
            tc_fence_after();
            d = tmem + static_cast<std::uint32_t>(slot * X3_BN);
          }
          const int s = it % X3_STAGES;
          mbar_wait(&full[s], (it / X3_STAGES) & 1);
          tc_fence_after();
          const std::uint32_t base = smem_u32(ring + s * X3_STAGE_BYTES);
          const std::uint32_t ah = base, al = base + X3_A_BYTES;
          const std::uint32_t bh = base + 2 * X3_A_BYTES, bl = bh + X3_B_BYTES;
#pragma unroll
          for (int kk = 0; kk < X3_BK / 8; ++kk) {
            // k-step of 8 fp32: K-major advances 32 B along the 128B-swizzled
            // row (8-row groups 1024 B apart); MN-major advances 8 k-rows =
            // 1024 B in the 32B-atom layout (4-row groups 512 B apart,
            // 32-element MN blocks 4 KB apart).
            auto desc = [&](std::uint32_t b, bool mn) {
              return mn ? smem_desc_b32(b + kk * 1024, 4096, 512) : smem_desc(b + kk * 32, 16, 1024);
            };
            const std::uint64_t dah = desc(ah, A_MN), dal = desc(al, A_MN);
            const std::uint64_t dbh = desc(bh, B_MN), dbl = desc(bl, B_MN);
            const std::uint32_t first = (kb % X3_CHUNK_KB != 0 || kk != 0) ? 1u : 0u;
            // small terms first
            tc_mma_tf32(d, dah, dbl, idesc, first);
            tc_mma_tf32(d, dal, dbh, idesc, 1u);
            tc_mma_tf32(d, dah, dbh, idesc, 1u);
          }
          tc_commit(&empty[s]);
          if (kb % X3_CHUNK_KB == X3_CHUNK_KB - 1 || kb == num_k - 1) {
            tc_commit(&tfull[slot]);  // chunk partial complete
            ++q;
          }
        }
      }
      pdl_trigger();
    }
  } else {
    // Epilogue warps 2..9: TMEM lane quarter qr = warp % 4, column half
    // (warp - 2) / 4, one output row per lane: every chunk partial of the
    // tile is added into 64 fp32 registers (round-to-nearest), then the row
    // half leaves in 32-column pieces through 128B-swizzled staging and TMA
    // stores.
    constexpr int HC = X3_BN / 2;
    const int qr = warp % 4;
    const int c0 = ((warp - 2) / 4) * HC;
    std::uint8_t* stg = staging + (warp - 2) * 4096;
    int q = 0;
    const int nch = (num_k + X3_CHUNK_KB - 1) / X3_CHUNK_KB;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      int mb, nb;
      tile_coords(t, tiles_m, tiles_n, mb, nb, group_m);
      float acc[HC];
#pragma unroll 1
      for (int c = 0; c < nch; ++c, ++q) {
        const int slot = q % X3_SLOTS;
        mbar_wait(&tfull[slot], (q / X3_SLOTS) & 1);
        tc_fence_after();
        const std::uint32_t base = tmem + (static_cast<std::uint32_t>(qr * 32) << 16) +
                                   static_cast<std::uint32_t>(slot * X3_BN + c0);
        if (c == 0) {
#pragma unroll
          for (int j = 0; j < HC / 32; ++j) {
            std::uint32_t r[32];
            tmem_ld32(base + j * 32, r);
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[j * 32 + i] = __uint_as_float(r[i]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < HC / 32; ++j) {
            std::uint32_t r[32];
            tmem_ld32(base + j * 32, r);
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[j * 32 + i] += __uint_as_float(r[i]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[slot]);  // the MMA warp may refill this slot
      }
#pragma unroll
      for (int j = 0; j < HC / 32; ++j) {
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // staging free
        __syncwarp();
#pragma unroll
        for (int v = 0; v < 8; ++v)
          *reinterpret_cast<float4*>(stg + lane * 128 + ((v ^ (lane & 7)) << 4)) =
              make_float4(acc[j * 32 + 4 * v], acc[j * 32 + 4 * v + 1], acc[j * 32 + 4 * v + 2], acc[j * 32 + 4 * v + 3]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) tma_store_2d(&mp.c, stg, nb * X3_BN + c0 + j * 32, mb * BM + qr * 32);
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(X3_TMEM_COLS));
  }
}

// fp32 row-major [rows][cols], box {32 cols (128 B), box_rows}: 128B swizzle
// (K-major operand) or 128B with 32-byte atoms (MN-major operand, `mn`).
CUtensorMap make_map_f32(const void* base, std::int64_t rows, std::int64_t cols, int box_rows, bool mn = false) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 4};
  cuuint32_t box[2] = {32, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           mn ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled (fp32) failed: " + std::to_string(r));
  return m;
}

std::int64_t round256(std::int64_t b) { return (b + 255) / 256 * 256; }

template <bool A_MN, bool B_MN>
void launch_x3_typed(const GemmArgs& a, const GemmSchedule& sc, float* ah, float* al, float* bh, float* bl,
                     cudaStream_t s) {
  static unsigned attr_set_mask = 0;
  auto kern = gemm_x3_kernel<A_MN, B_MN>;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_set_mask & (1u << dev))) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, X3_SMEM);
    if (e != cudaSuccess) throw std::runtime_error(std::string("gemm_x3 smem attribute: ") + cudaGetErrorString(e));
    attr_set_mask |= 1u << dev;
  }
  X3Maps mp;
  std::memset(&mp, 0, sizeof(mp));
  // A: [m][k] (K-major) or [k][m] (MN-major); B: [k][n] (MN-major) or [n][k].
  mp.ah = A_MN ? make_map_f32(ah, a.k, a.m, X3_BK, true) : make_map_f32(ah, a.m, a.k, BM);
  mp.al = A_MN ? make_map_f32(al, a.k, a.m, X3_BK, true) : make_map_f32(al, a.m, a.k, BM);
  mp.bh = B_MN ? make_map_f32(bh, a.k, a.n, X3_BK, true) : make_map_f32(bh, a.n, a.k, X3_BN);
  mp.bl = B_MN ? make_map_f32(bl, a.k, a.n, X3_BK, true) : make_map_f32(bl, a.n, a.k, X3_BN);
  mp.c = make_store_map(a.C, a.m, a.n, false);
  pdl_launch("gemm_x3_kernel", kern, dim3(sc.grid), dim3(X3_THREADS), X3_SMEM, s, mp, static_cast<int>(a.m),
             static_cast<int>(a.n), static_cast<int>(a.k), GROUP_M);
}

}  // namespace

bool gemm_x3_eligible(const GemmArgs& a) {
  const char* off = std::getenv("PLANC_B200_TF32X3");  // =0: fp32 GEMMs on the SIMT kernel
  if (off && off[0] == '0') return false;
  if (a.da != DT_F32 || a.db != DT_F32 || a.dc != DT_F32) return false;
  if (a.group > 1 || a.scatter > 0 || a.epi.n_ops > 0) return false;
  if (a.m <= 0 || a.n <= 0 || a.k <= 0 || a.m > (1 << 30) || a.n > (1 << 30) || a.k > (1 << 30)) return false;
  // TMA: 16-byte row pitch of both operands and of C.
  if ((a.ta ? a.m : a.k) % 4 != 0 || (a.tb ? a.k : a.n) % 4 != 0 || a.n % 4 != 0) return false;
  if (a.m * a.n * a.k < (std::int64_t(1) << 20)) return false;
  return true;
}

GemmSchedule gemm_x3_schedule(const GemmArgs& a, int sms) {
  GemmSchedule sc;
  sc.bn = X3_BN;
  sc.tiles = ((a.m + BM - 1) / BM) * ((a.n + X3_BN - 1) / X3_BN);
  sc.num_k = (a.k + X3_BK - 1) / X3_BK;
  sc.grid = static_cast<int>(std::min<std::int64_t>(sc.tiles, sms));
  sc.dp_tiles = static_cast<int>(sc.tiles);
  sc.occ = 6;  // 3xTF32
  sc.ws_bytes = 2 * round256(a.m * a.k * 4) + 2 * round256(a.k * a.n * 4);
  return sc;
}

void launch_gemm_x3(const GemmArgs& a, cudaStream_t s) {
  const GemmSchedule sc = gemm_x3_schedule(a, device_sms());
  if (a.ws == nullptr || a.ws_bytes < sc.ws_bytes)
    throw std::runtime_error("gemm_x3: workspace missing or too small for the hi / lo planes");
  if ((reinterpret_cast<std::uintptr_t>(a.A) | reinterpret_cast<std::uintptr_t>(a.B) |
       reinterpret_cast<std::uintptr_t>(a.C)) % 16 != 0)
    throw std::runtime_error("gemm_x3: operands must be 16-byte aligned");
  char* ws = static_cast<char*>(a.ws);
  const std::int64_t pa = round256(a.m * a.k * 4), pb = round256(a.k * a.n * 4);
  float* ah = reinterpret_cast<float*>(ws);
  float* al = reinterpret_cast<float*>(ws + pa);
  float* bh = reinterpret_cast<float*>(ws + 2 * pa);
  float* bl = reinterpret_cast<float*>(ws + 2 * pa + pb);
  X3Split sp;
  sp.src[0] = static_cast<const float*>(a.A);
  sp.src[1] = static_cast<const float*>(a.B);
  sp.hi[0] = ah;
  sp.lo[0] = al;
  sp.hi[1] = bh;
  sp.lo[1] = bl;
  sp.count[0] = a.m * a.k;
  sp.count[1] = a.k * a.n;
  constexpr long long per_block = static_cast<long long>(kX3SplitThreads) * kX3SplitVec * 4;
  sp.blocks0 = std::max(1LL, (sp.count[0] + per_block - 1) / per_block);
  const long long blocks1 = std::max(1LL, (sp.count[1] + per_block - 1) / per_block);
  pdl_launch("x3_split_kernel", x3_split_kernel, dim3(static_cast<unsigned>(sp.blocks0 + blocks1)),
             dim3(kX3SplitThreads), 0, s, sp);
  const bool a_mn = a.ta, b_mn = !a.tb;
  if (!a_mn && !b_mn) return launch_x3_typed<false, false>(a, sc, ah, al, bh, bl, s);
  if (!a_mn && b_mn) return launch_x3_typed<false, true>(a, sc, ah, al, bh, bl, s);
  if (a_mn && !b_mn) return launch_x3_typed<true, false>(a, sc, ah, al, bh, bl, s);
  return launch_x3_typed<true, true>(a, sc, ah, al, bh, bl, s);
}

}  // namespace planc_b200
