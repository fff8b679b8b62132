// Fused attention (schema extension): O = softmax(Q·Kᵀ·s)·V
// per (sequence, head) on tcgen05 tensor cores — one kernel, S and P never
// leave the SM (flash-attention structure: online softmax, rescaled
// accumulation).
//
// Layout: Q, K, V, O are a piece's [rows, cols] bf16 tensors (row-major):
// rows = whole sequences of `seq` tokens, cols = whole heads of `dh`
// features. CTA (h, b, qb) computes the 128 query rows qb of head h of
// sequence b.
//
// Warps: 0 TMA producer (Q once; K_j / V_j 128-row tiles through a 2-stage
//          ring), 1 single-thread MMA issuer, 2..5 softmax / accumulation
//          (thread = query row = TMEM lane).
// Per key block j:
//   MMA      S_j = Q·K_jᵀ  -> TMEM S[j%2]   (M=128, N=128, K=dh; both K-major)
//   softmax  row max over S_j (scaled, base 2; causal mask on the diagonal
//            block) -> m_j; P_j = exp2(S_j - m_j) -> bf16 smem P[j%2] in the
//            128B-swizzled K-major layout of an MMA A operand; row sum
//   MMA      O_j = P_j·V_j  -> TMEM O[j%2]   (N=dh; V MN-major)
//   softmax  acc = acc·exp2(m_{j-1} - m_j) + O_j in fp32 registers
// so the tensor core runs S_{j+1} and P_j·V_j while the softmax warps work
// on block j (TMEM: S0 S1 O0 O1 = 512 columns at dh = 128). End: O = acc / l.
#include "gemm_sm100_impl.cuh"

namespace planc_b200 {

namespace {

constexpr int kAttnThreads = 64 + 8 * 32;  // producer, MMA, 8 softmax warps
constexpr int kAttnBlock = 128;  // query / key rows per tile

template <int DH>
struct AttnCfg {
  static constexpr int Q_BYTES = kAttnBlock * DH * 2;   // DH/64 K-major chunks of 16 KB
  static constexpr int K_BYTES = kAttnBlock * DH * 2;
  static constexpr int V_BYTES = kAttnBlock * DH * 2;   // 2 kv chunks x DH/64 n-blocks of 8 KB
  static constexpr int P_BYTES = kAttnBlock * kAttnBlock * 2;  // 2 kv chunks of 16 KB
  // + 1024-byte alignment slack, barriers / TMEM slot (256 B), pair-exchange rows (2 x 128 floats)
  static constexpr int SMEM = Q_BYTES + 2 * (K_BYTES + V_BYTES) + 2 * P_BYTES + 1024 + 256 + 1024;
  static_assert(SMEM <= 227 * 1024, "attention tiles above the shared memory limit");
};

struct AttnMaps {
  CUtensorMap q, k, v;
};

// tcgen05.ld 32x32b.x64: 64 consecutive TMEM columns of this thread's lane,
// one wait (tcgen05.wait::ld) for all of them.
__device__ __forceinline__ void tmem_ld64(std::uint32_t taddr, std::uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
      "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
      "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]),
        "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]),
        "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]),
        "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]),
        "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// (Splitting the exponentials between MUFU ex2 and an FMA-pipe polynomial —
// FA4's balance — measured slower here: forward 794 -> 712 TFLOP/s, causal
// 436 -> 308; the softmax warps are issue / latency bound, not XU bound.)

// STATS (the backward's statistics pass): no V, no P·V — every query row's
// base-2 log-sum-exp lse2 = m + log2(l) of its scaled scores, and
// D = rowsum(dO ∘ O) from the forward output and its incoming gradient,
// into lse_out / d_out [head][row of the piece].
template <int DH, bool CAUSAL, bool STATS = false>
__global__ void __launch_bounds__(kAttnThreads, 1)
    attn_fwd_kernel(const __grid_constant__ AttnMaps mp, __nv_bfloat16* __restrict__ out, int seq, int ld,
                    float scale_log2, float* __restrict__ lse_out = nullptr, float* __restrict__ d_out = nullptr,
                    const __nv_bfloat16* __restrict__ o_in = nullptr, const __nv_bfloat16* __restrict__ do_in = nullptr,
                    int rows = 0) {
  using CF = AttnCfg<DH>;
  extern __shared__ std::uint8_t smem_raw[];
  std::uint8_t* smem =
      smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays a shared-space pointer (STS / LDS)
  std::uint8_t* sQ = smem;
  std::uint8_t* sK = sQ + CF::Q_BYTES;                 // [2][K_BYTES]
  std::uint8_t* sV = sK + 2 * CF::K_BYTES;             // [2][V_BYTES]
  std::uint8_t* sP = sV + 2 * CF::V_BYTES;             // [2][P_BYTES]
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(sP + 2 * CF::P_BYTES);
  std::uint64_t* q_full = bars;
  std::uint64_t* k_full = bars + 1;    // [2]
  std::uint64_t* k_empty = bars + 3;   // [2]
  std::uint64_t* s_full = bars + 5;    // [2]
  std::uint64_t* s_empty = bars + 7;   // [2]
  std::uint64_t* p_full = bars + 9;    // [2]
  std::uint64_t* p_empty = bars + 11;  // [2]
  std::uint64_t* o_full = bars + 13;   // [2]
  std::uint64_t* o_empty = bars + 15;  // [2]
  std::uint64_t* v_full = bars + 17;   // [2]
  std::uint64_t* v_empty = bars + 19;  // [2]
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 21);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // grid (head, sequence, query block), query blocks slowest: with a causal
  // mask the longest blocks (most keys) are dispatched first (LPT order)
  const int qb = CAUSAL ? static_cast<int>(gridDim.z) - 1 - static_cast<int>(blockIdx.z) : static_cast<int>(blockIdx.z);
  const int h = blockIdx.x, b = blockIdx.y;
  const int row0 = b * seq + qb * kAttnBlock;  // first query row of the tile
  const int col0 = h * DH;
  const int nkv = CAUSAL ? qb + 1 : seq / kAttnBlock;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&mp.q)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&mp.k)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&mp.v)) : "memory");
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 8);
      mbar_init(&p_full[i], 8);
      mbar_init(&p_empty[i], 1);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_empty[i], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = *tmem_slot;
  pdl_wait();

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_full, CF::Q_BYTES);
#pragma unroll
      for (int c = 0; c < DH / 64; ++c) tma_load_2d(sQ + c * 16384, &mp.q, col0 + 64 * c, row0, q_full);
      // K_j is freed by S_j, V_j only by P_j·V_j: K runs one block ahead of V
      // so the next score tile never waits for a value tile's release.
      auto load_k = [&](int j) {
        const int st = j & 1;
        mbar_wait(&k_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&k_full[st], CF::K_BYTES);
        std::uint8_t* k = sK + st * CF::K_BYTES;
#pragma unroll
        for (int c = 0; c < DH / 64; ++c)
          tma_load_2d(k + c * 16384, &mp.k, col0 + 64 * c, b * seq + j * kAttnBlock, &k_full[st]);
      };
      auto load_v = [&](int j) {  // V as an MN-major B operand: per 64-key chunk, DH/64 blocks of 64 features
        const int st = j & 1;
        mbar_wait(&v_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&v_full[st], CF::V_BYTES);
        std::uint8_t* v = sV + st * CF::V_BYTES;
#pragma unroll
        for (int kc = 0; kc < 2; ++kc)
#pragma unroll
          for (int nb = 0; nb < DH / 64; ++nb)
            tma_load_2d(v + kc * (DH / 64) * 8192 + nb * 8192, &mp.v, col0 + 64 * nb,
                        b * seq + j * kAttnBlock + 64 * kc, &v_full[st]);
      };
      load_k(0);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) load_k(j + 1);
        if constexpr (!STATS) load_v(j);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr std::uint32_t idesc_s = make_idesc<kAttnBlock>(false, false);
      constexpr std::uint32_t idesc_o = make_idesc<DH>(false, true);
      mbar_wait(q_full, 0);
      auto pv = [&](int i) {  // O[i%2] = P[i%2] · V[i%2]
        const int st = i & 1;
        mbar_wait(&v_full[st], (i >> 1) & 1);
        mbar_wait(&p_full[st], (i >> 1) & 1);
        mbar_wait(&o_empty[st], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const std::uint32_t p = smem_u32(sP + st * CF::P_BYTES), v = smem_u32(sV + st * CF::V_BYTES);
        const std::uint32_t d = tmem + 256 + st * DH;
#pragma unroll
        for (int s = 0; s < kAttnBlock / 16; ++s) {
          const int kc = s / 4, kk = s % 4;
          tc_mma(d, smem_desc(p + kc * 16384 + kk * 32, 16, 1024),
                 smem_desc(v + kc * (DH / 64) * 8192 + kk * 2048, 8192, 1024), idesc_o, s > 0 ? 1u : 0u);
        }
        tc_commit(&o_full[st]);
        tc_commit(&v_empty[st]);  // V_i consumed
        tc_commit(&p_empty[st]);
      };
      const std::uint32_t q = smem_u32(sQ);
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        mbar_wait(&k_full[st], (j >> 1) & 1);
        mbar_wait(&s_empty[st], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const std::uint32_t k = smem_u32(sK + st * CF::K_BYTES);
        const std::uint32_t d = tmem + st * kAttnBlock;
#pragma unroll
        for (int s = 0; s < DH / 16; ++s) {
          const int c = s / 4, kk = s % 4;
          tc_mma(d, smem_desc(q + c * 16384 + kk * 32, 16, 1024), smem_desc(k + c * 16384 + kk * 32, 16, 1024),
                 idesc_s, s > 0 ? 1u : 0u);
        }
        tc_commit(&s_full[st]);
        tc_commit(&k_empty[st]);  // K_j consumed
        if constexpr (!STATS) {
          if (j > 0) pv(j - 1);
        }
      }
      if constexpr (!STATS) pv(nkv - 1);
      pdl_trigger();
    }
  } else {
    // Softmax warps 2..9: row r of the tile = TMEM lane r; the two warps of a
    // lane quarter split its columns (scores: 64 keys each; output: DH/2
    // features each) and exchange row maxima / sums through shared memory
    // under a 64-thread named barrier (one per quarter).
    const int qr = warp % 4, half = (warp - 2) / 4;
    const int r = qr * 32 + lane;
    const std::uint32_t lane_base = tmem + (static_cast<std::uint32_t>(qr * 32) << 16);
    float* xch = reinterpret_cast<float*>(bars + 32);  // [2 halves][128 rows] (bars: 22 words used)
    auto pair_sync = [&] { asm volatile("bar.sync %0, 64;" ::"r"(1 + qr) : "memory"); };
    constexpr int HD = DH / 2;
    float acc[HD];
#pragma unroll
    for (int i = 0; i < HD; ++i) acc[i] = 0.f;
    float m = -INFINITY, l = 0.f, alpha_prev = 1.f;
    auto accumulate = [&](int i, float alpha) {  // acc = acc * alpha + O[i%2] (this warp's features)
      const int st = i & 1;
      mbar_wait(&o_full[st], (i >> 1) & 1);
      tc_fence_after();
      if constexpr (HD == 64) {
        std::uint32_t v[64];
        tmem_ld64(lane_base + 256 + st * DH + half * HD, v);
#pragma unroll
        for (int e = 0; e < 64; ++e) acc[e] = fmaf(acc[e], alpha, __uint_as_float(v[e]));
      } else {
        std::uint32_t v[32];
        tmem_ld32(lane_base + 256 + st * DH + half * HD, v);
#pragma unroll
        for (int e = 0; e < 32; ++e) acc[e] = fmaf(acc[e], alpha, __uint_as_float(v[e]));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[st]);
    };
    for (int j = 0; j < nkv; ++j) {
      const int st = j & 1;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      const std::uint32_t sb = lane_base + st * kAttnBlock + half * 64;
      const bool diag = CAUSAL && j == qb;  // keys above the query row are masked
      const int key0 = half * 64;
      // this warp's 64 scores of the row stay in registers for both passes
      std::uint32_t v[64];
      tmem_ld64(sb, v);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[st]);  // S[st] may be overwritten (S_{j+2})
      // pass 1: row max of the raw scores (the scale is positive), pair-combined
      float mx = -INFINITY;
#pragma unroll
      for (int e = 0; e < 64; ++e)
        if (!diag || key0 + e <= r) mx = fmaxf(mx, __uint_as_float(v[e]));
      xch[half * 128 + r] = mx;
      pair_sync();
      mx = fmaxf(xch[r], xch[128 + r]);
      pair_sync();  // both halves read before the next block's maxima land
      const float m_new = fmaxf(m, mx * scale_log2);
      if constexpr (STATS) {  // only the row sum
        float sum = 0.f;
#pragma unroll
        for (int e = 0; e < 64; ++e)
          if (!diag || key0 + e <= r) sum += ex2(fmaf(__uint_as_float(v[e]), scale_log2, -m_new));
        l = l * ex2(m - m_new) + sum;
        m = m_new;
        continue;
      }
      // pass 2: P = exp2(s * scale - m_new) as bf16 into this warp's 64-key
      // atom of the swizzled A-operand tile
      mbar_wait(&p_empty[st], ((j >> 1) & 1) ^ 1);
      std::uint8_t* prow = sP + st * CF::P_BYTES + half * 16384 + r * 128;
      float sum = 0.f;
#pragma unroll
      for (int cw = 0; cw < 8; ++cw) {  // 16-byte chunk of the 128-byte row; 128B swizzle: chunk ^ (row & 7)
        std::uint32_t w[4];
#pragma unroll
        for (int h2 = 0; h2 < 4; ++h2) {
          const int e = 8 * cw + 2 * h2;
          const float p0 = (!diag || key0 + e <= r) ? ex2(fmaf(__uint_as_float(v[e]), scale_log2, -m_new)) : 0.f;
          const float p1 = (!diag || key0 + e + 1 <= r) ? ex2(fmaf(__uint_as_float(v[e + 1]), scale_log2, -m_new)) : 0.f;
          sum += p0 + p1;
          const __nv_bfloat162 pk = __floats2bfloat162_rn(p0, p1);  // one packed convert (FMA pipe, not XU)
          w[h2] = *reinterpret_cast<const std::uint32_t*>(&pk);
        }
        *reinterpret_cast<uint4*>(prow + ((cw ^ (r & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P visible to the tensor core
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[st]);
      const float alpha = ex2(m - m_new);  // (m = -inf on the first block: alpha = 0, acc is 0)
      l = l * alpha + sum;                  // this warp's keys only; halves added at the end
      m = m_new;
      if (j > 0) accumulate(j - 1, alpha_prev);
      alpha_prev = alpha;
    }
    if constexpr (STATS) {
      // lse2 of the row (pair-combined sums) and D = rowsum(dO ∘ O) over
      // this warp's half of the head's features
      const std::int64_t go = static_cast<std::int64_t>(row0 + r) * ld + col0 + half * HD;
      float dd = 0.f;
#pragma unroll
      for (int g = 0; g < HD / 8; ++g) {
        const uint4 ow = reinterpret_cast<const uint4*>(o_in + go)[g];
        const uint4 gw = reinterpret_cast<const uint4*>(do_in + go)[g];
        const std::uint32_t a4[4] = {ow.x, ow.y, ow.z, ow.w}, b4[4] = {gw.x, gw.y, gw.z, gw.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float a0, a1, b0, b1;
          bf16_unpair(a4[e], a0, a1);
          bf16_unpair(b4[e], b0, b1);
          dd = fmaf(a0, b0, fmaf(a1, b1, dd));
        }
      }
      xch[half * 128 + r] = l;
      pair_sync();
      const float lt = xch[r] + xch[128 + r];
      pair_sync();
      xch[half * 128 + r] = dd;
      pair_sync();
      if (half == 0) {
        lse_out[static_cast<std::int64_t>(h) * rows + row0 + r] = m + __log2f(lt);
        d_out[static_cast<std::int64_t>(h) * rows + row0 + r] = xch[r] + xch[128 + r];
      }
    } else {
    accumulate(nkv - 1, alpha_prev);
    // acc: sum over blocks of P_j·V_j, each rescaled to the running max;
    // l: this warp's share of the row sum (same maxima) — add the pair's.
    xch[half * 128 + r] = l;
    pair_sync();
    const float inv = 1.f / (xch[r] + xch[128 + r]);
    __nv_bfloat16* orow = out + static_cast<std::int64_t>(row0 + r) * ld + col0 + half * HD;
#pragma unroll
    for (int g = 0; g < HD / 8; ++g)
      reinterpret_cast<uint4*>(orow)[g] =
          make_uint4(bf16_pair(acc[8 * g] * inv, acc[8 * g + 1] * inv), bf16_pair(acc[8 * g + 2] * inv, acc[8 * g + 3] * inv),
                     bf16_pair(acc[8 * g + 4] * inv, acc[8 * g + 5] * inv), bf16_pair(acc[8 * g + 6] * inv, acc[8 * g + 7] * inv));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---- backward -----------------------------------------------------------------
// With the statistics (lse2, D) of attn_fwd_kernel<..., STATS>:
//   P = exp2(S·s·log2e - lse2)      (exact softmax, no rescaling)
//   dS = P ∘ (dO·Vᵀ - D)
//   dQ = s · dS·K        (attn_bwd_dq_kernel: CTA = 128 query rows, loop over keys)
//   dK = s · dSᵀ·Q, dV = Pᵀ·dO   (attn_bwd_dkdv_kernel: CTA = 128 keys, loop over queries)
// Tiles are loaded K-major (128 rows x 64-feature chunks, 128B swizzle); a
// tile that an MMA needs as an MN-major B operand (K in dQ, Q and dO in dK /
// dV) is read in place through an MN-major descriptor (LBO = the 16 KB
// feature-chunk stride, SBO = 1 KB per 8 rows).
struct AttnBwdMaps {
  CUtensorMap q, k, v, dout;
};

template <int DH>
struct AttnBwdCfg {
  static constexpr int T_BYTES = kAttnBlock * DH * 2;            // one 128 x DH tile
  static constexpr int P_BYTES = kAttnBlock * kAttnBlock * 2;    // 128 x 128 bf16 A operand
  // dq: Q, dO resident; K, V rings of 2; dS.  dkdv: K, V resident; Q, dO rings of 2; P/dS.
  // Layout: barriers (256 B) and the statistics rows (2 KB) at the (16-byte
  // aligned) start, tiles from the next 1 KB boundary: 3 KB covers both for
  // any start alignment.
  static constexpr int HEAD = 3072;
  static constexpr int SMEM = HEAD + 6 * T_BYTES + P_BYTES;
  static_assert(SMEM <= 227 * 1024, "attention backward tiles above the shared memory limit");
};

__device__ __forceinline__ std::uint64_t kdesc(std::uint32_t base, int s) {  // K-major operand, k-step s (16)
  return smem_desc(base + (s / 4) * 16384 + (s % 4) * 32, 16, 1024);
}
__device__ __forceinline__ std::uint64_t mndesc(std::uint32_t base, int s) {  // K-major tile as MN-major B, k-step s
  return smem_desc(base + s * 2048, 16384, 1024);
}

template <int DH, bool CAUSAL>
__global__ void __launch_bounds__(kAttnThreads, 1)
    attn_bwd_dq_kernel(const __grid_constant__ AttnBwdMaps mp, __nv_bfloat16* __restrict__ dq, int seq, int ld,
                       float scale_log2, float scale, const float* __restrict__ lse, const float* __restrict__ dsum,
                       int rows) {
  using CF = AttnBwdCfg<DH>;
  extern __shared__ std::uint8_t smem_raw[];
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem_raw);
  std::uint8_t* smem = smem_raw + 2304 + ((1024u - ((smem_u32(smem_raw) + 2304u) & 1023u)) & 1023u);
  std::uint8_t* sQ = smem;
  std::uint8_t* sO = sQ + CF::T_BYTES;       // dO
  std::uint8_t* sK = sO + CF::T_BYTES;       // [2]
  std::uint8_t* sV = sK + 2 * CF::T_BYTES;   // [2]
  std::uint8_t* sS = sV + 2 * CF::T_BYTES;   // dS (A operand)
  std::uint64_t* q_full = bars;
  std::uint64_t* k_full = bars + 1;    // [2]
  std::uint64_t* k_empty = bars + 3;   // [2]
  std::uint64_t* v_full = bars + 5;    // [2]
  std::uint64_t* v_empty = bars + 7;   // [2]
  std::uint64_t* s_full = bars + 9;
  std::uint64_t* s_empty = bars + 10;
  std::uint64_t* ds_full = bars + 11;
  std::uint64_t* ds_empty = bars + 12;
  std::uint64_t* acc_full = bars + 13;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 14);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int qb = CAUSAL ? static_cast<int>(gridDim.z) - 1 - static_cast<int>(blockIdx.z) : static_cast<int>(blockIdx.z);
  const int h = blockIdx.x, b = blockIdx.y;
  const int row0 = b * seq + qb * kAttnBlock;
  const int col0 = h * DH;
  const int nkv = CAUSAL ? qb + 1 : seq / kAttnBlock;

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_empty, 8);
    mbar_init(ds_full, 8);
    mbar_init(ds_empty, 1);
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = *tmem_slot;
  pdl_wait();

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_full, 2 * CF::T_BYTES);
#pragma unroll
      for (int c = 0; c < DH / 64; ++c) {
        tma_load_2d(sQ + c * 16384, &mp.q, col0 + 64 * c, row0, q_full);
        tma_load_2d(sO + c * 16384, &mp.dout, col0 + 64 * c, row0, q_full);
      }
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        const int kr = b * seq + j * kAttnBlock;
        mbar_wait(&k_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&k_full[st], CF::T_BYTES);
#pragma unroll
        for (int c = 0; c < DH / 64; ++c)
          tma_load_2d(sK + st * CF::T_BYTES + c * 16384, &mp.k, col0 + 64 * c, kr, &k_full[st]);
        mbar_wait(&v_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&v_full[st], CF::T_BYTES);
#pragma unroll
        for (int c = 0; c < DH / 64; ++c)
          tma_load_2d(sV + st * CF::T_BYTES + c * 16384, &mp.v, col0 + 64 * c, kr, &v_full[st]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr std::uint32_t idesc_s = make_idesc<kAttnBlock>(false, false);
      constexpr std::uint32_t idesc_q = make_idesc<DH>(false, true);
      const std::uint32_t q = smem_u32(sQ), o = smem_u32(sO), ds = smem_u32(sS);
      mbar_wait(q_full, 0);
      // S_j / dP_j are issued as soon as the softmax warps have read the
      // previous block's scores (registers), i.e. before dQ += dS_{j-1}·K_{j-1}:
      // the tensor core computes block j while the softmax warps work on j-1.
      auto scores = [&](int j) {
        const int st = j & 1;
        const std::uint32_t k = smem_u32(sK + st * CF::T_BYTES), v = smem_u32(sV + st * CF::T_BYTES);
        mbar_wait(&k_full[st], (j >> 1) & 1);
        mbar_wait(&v_full[st], (j >> 1) & 1);
        mbar_wait(s_empty, (j & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int s = 0; s < DH / 16; ++s) tc_mma(tmem, kdesc(q, s), kdesc(k, s), idesc_s, s > 0 ? 1u : 0u);
#pragma unroll
        for (int s = 0; s < DH / 16; ++s) tc_mma(tmem + 128, kdesc(o, s), kdesc(v, s), idesc_s, s > 0 ? 1u : 0u);
        tc_commit(s_full);
        tc_commit(&v_empty[st]);  // V_j consumed (dP only)
      };
      auto grad = [&](int j) {  // dQ += dS_j · K_j
        const int st = j & 1;
        const std::uint32_t k = smem_u32(sK + st * CF::T_BYTES);
        mbar_wait(ds_full, j & 1);
        tc_fence_after();
#pragma unroll
        for (int s = 0; s < kAttnBlock / 16; ++s)
          tc_mma(tmem + 256, kdesc(ds, s), mndesc(k, s), idesc_q, (j > 0 || s > 0) ? 1u : 0u);
        tc_commit(ds_empty);
        tc_commit(&k_empty[st]);
      };
      scores(0);
      for (int j = 1; j < nkv; ++j) {
        scores(j);
        grad(j - 1);
      }
      grad(nkv - 1);
      tc_commit(acc_full);
      pdl_trigger();
    }
  } else {
    const int qr = warp % 4, half = (warp - 2) / 4;
    const int r = qr * 32 + lane;
    const std::uint32_t lane_base = tmem + (static_cast<std::uint32_t>(qr * 32) << 16);
    const int key0 = half * 64;
    const float l2 = lse[static_cast<std::int64_t>(h) * rows + row0 + r];
    const float dd = dsum[static_cast<std::int64_t>(h) * rows + row0 + r];
    for (int j = 0; j < nkv; ++j) {
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      std::uint32_t sv[64], pv[64];
      tmem_ld64(lane_base + key0, sv);
      tmem_ld64(lane_base + 128 + key0, pv);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_empty);
      const bool diag = CAUSAL && j == qb;
      mbar_wait(ds_empty, (j & 1) ^ 1);
      std::uint8_t* drow = sS + half * 16384 + r * 128;
#pragma unroll
      for (int cw = 0; cw < 8; ++cw) {
        std::uint32_t w[4];
#pragma unroll
        for (int h2 = 0; h2 < 4; ++h2) {
          const int e = 8 * cw + 2 * h2;
          const float p0 = (!diag || key0 + e <= r) ? ex2(fmaf(__uint_as_float(sv[e]), scale_log2, -l2)) : 0.f;
          const float p1 = (!diag || key0 + e + 1 <= r) ? ex2(fmaf(__uint_as_float(sv[e + 1]), scale_log2, -l2)) : 0.f;
          w[h2] = bf16_pair(p0 * (__uint_as_float(pv[e]) - dd), p1 * (__uint_as_float(pv[e + 1]) - dd));
        }
        *reinterpret_cast<uint4*>(drow + ((cw ^ (r & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
    }
    mbar_wait(acc_full, 0);
    tc_fence_after();
    constexpr int HD = DH / 2;
    __nv_bfloat16* orow = dq + static_cast<std::int64_t>(row0 + r) * ld + col0 + half * HD;
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      std::uint32_t v[32];
      tmem_ld32(lane_base + 256 + half * HD + c * 32, v);
#pragma unroll
      for (int g = 0; g < 4; ++g)
        reinterpret_cast<uint4*>(orow + c * 32)[g] = make_uint4(
            bf16_pair(__uint_as_float(v[8 * g]) * scale, __uint_as_float(v[8 * g + 1]) * scale),
            bf16_pair(__uint_as_float(v[8 * g + 2]) * scale, __uint_as_float(v[8 * g + 3]) * scale),
            bf16_pair(__uint_as_float(v[8 * g + 4]) * scale, __uint_as_float(v[8 * g + 5]) * scale),
            bf16_pair(__uint_as_float(v[8 * g + 6]) * scale, __uint_as_float(v[8 * g + 7]) * scale));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int DH, bool CAUSAL>
__global__ void __launch_bounds__(kAttnThreads, 1)
    attn_bwd_dkdv_kernel(const __grid_constant__ AttnBwdMaps mp, __nv_bfloat16* __restrict__ dk,
                         __nv_bfloat16* __restrict__ dv, int seq, int ld, float scale_log2, float scale,
                         const float* __restrict__ lse, const float* __restrict__ dsum, int rows) {
  using CF = AttnBwdCfg<DH>;
  extern __shared__ std::uint8_t smem_raw[];
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem_raw);
  std::uint8_t* smem = smem_raw + 2304 + ((1024u - ((smem_u32(smem_raw) + 2304u) & 1023u)) & 1023u);
  std::uint8_t* sK = smem;
  std::uint8_t* sV = sK + CF::T_BYTES;
  std::uint8_t* sQ = sV + CF::T_BYTES;       // [2]
  std::uint8_t* sO = sQ + 2 * CF::T_BYTES;   // dO [2]
  std::uint8_t* sP = sO + 2 * CF::T_BYTES;   // Pᵀ, then dSᵀ (A operand)
  std::uint64_t* kv_full = bars;
  std::uint64_t* q_full = bars + 1;    // [2] (Q_i and dO_i)
  std::uint64_t* q_empty = bars + 3;   // [2]
  std::uint64_t* s_full = bars + 5;
  std::uint64_t* s_empty = bars + 6;
  std::uint64_t* p_full = bars + 7;
  std::uint64_t* p_empty = bars + 8;
  std::uint64_t* ds_full = bars + 9;
  std::uint64_t* ds_empty = bars + 10;
  std::uint64_t* acc_full = bars + 11;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 12);
  float* stat = reinterpret_cast<float*>(bars + 32);  // [2 parity][lse2 128 | D 128]

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int kb = blockIdx.z;  // causal: the longest key blocks are the first ones
  const int h = blockIdx.x, b = blockIdx.y;
  const int krow0 = b * seq + kb * kAttnBlock;
  const int col0 = h * DH;
  const int nq = seq / kAttnBlock;
  const int i0 = CAUSAL ? kb : 0;

  if (warp == 0 && lane == 0) {
    mbar_init(kv_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_empty, 8);
    mbar_init(p_full, 8);
    mbar_init(p_empty, 1);
    mbar_init(ds_full, 8);
    mbar_init(ds_empty, 1);
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = *tmem_slot;
  pdl_wait();

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(kv_full, 2 * CF::T_BYTES);
#pragma unroll
      for (int c = 0; c < DH / 64; ++c) {
        tma_load_2d(sK + c * 16384, &mp.k, col0 + 64 * c, krow0, kv_full);
        tma_load_2d(sV + c * 16384, &mp.v, col0 + 64 * c, krow0, kv_full);
      }
      for (int i = i0; i < nq; ++i) {
        const int n = i - i0, st = n & 1;
        const int qrow = b * seq + i * kAttnBlock;
        mbar_wait(&q_empty[st], ((n >> 1) & 1) ^ 1);
        mbar_expect_tx(&q_full[st], 2 * CF::T_BYTES);
#pragma unroll
        for (int c = 0; c < DH / 64; ++c) {
          tma_load_2d(sQ + st * CF::T_BYTES + c * 16384, &mp.q, col0 + 64 * c, qrow, &q_full[st]);
          tma_load_2d(sO + st * CF::T_BYTES + c * 16384, &mp.dout, col0 + 64 * c, qrow, &q_full[st]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr std::uint32_t idesc_s = make_idesc<kAttnBlock>(false, false);
      constexpr std::uint32_t idesc_g = make_idesc<DH>(false, true);
      const std::uint32_t k = smem_u32(sK), v = smem_u32(sV), p = smem_u32(sP);
      mbar_wait(kv_full, 0);
      // Sᵀ / dPᵀ of block i+1 are issued once the softmax warps have read
      // block i's (registers) — before dV / dK of block i.
      auto scores = [&](int i) {  // Sᵀ = K·Q_iᵀ, dPᵀ = V·dO_iᵀ  (keys x queries)
        const int n = i - i0, st = n & 1;
        const std::uint32_t q = smem_u32(sQ + st * CF::T_BYTES), o = smem_u32(sO + st * CF::T_BYTES);
        mbar_wait(&q_full[st], (n >> 1) & 1);
        mbar_wait(s_empty, (n & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int s = 0; s < DH / 16; ++s) tc_mma(tmem, kdesc(k, s), kdesc(q, s), idesc_s, s > 0 ? 1u : 0u);
#pragma unroll
        for (int s = 0; s < DH / 16; ++s) tc_mma(tmem + 128, kdesc(v, s), kdesc(o, s), idesc_s, s > 0 ? 1u : 0u);
        tc_commit(s_full);
      };
      scores(i0);
      for (int i = i0; i < nq; ++i) {
        const int n = i - i0, st = n & 1;
        const std::uint32_t q = smem_u32(sQ + st * CF::T_BYTES), o = smem_u32(sO + st * CF::T_BYTES);
        if (i + 1 < nq) scores(i + 1);
        // dV += Pᵀ · dO_i
        mbar_wait(p_full, n & 1);
        tc_fence_after();
#pragma unroll
        for (int s = 0; s < kAttnBlock / 16; ++s)
          tc_mma(tmem + 256, kdesc(p, s), mndesc(o, s), idesc_g, (n > 0 || s > 0) ? 1u : 0u);
        tc_commit(p_empty);
        // dK += dSᵀ · Q_i   (dSᵀ written into the same tile once P·dO has read it)
        mbar_wait(ds_full, n & 1);
        tc_fence_after();
#pragma unroll
        for (int s = 0; s < kAttnBlock / 16; ++s)
          tc_mma(tmem + 256 + DH, kdesc(p, s), mndesc(q, s), idesc_g, (n > 0 || s > 0) ? 1u : 0u);
        tc_commit(ds_empty);
        tc_commit(&q_empty[st]);
      }
      tc_commit(acc_full);
      pdl_trigger();
    }
  } else {
    // thread = key row r of the block; the two warps of a lane quarter split
    // the 128 query columns of each block (64 each) and the DH features of dK / dV
    const int qr = warp % 4, half = (warp - 2) / 4;
    const int r = qr * 32 + lane;
    const int t = (warp - 2) * 32 + lane;  // 0..255 among the softmax warps
    const std::uint32_t lane_base = tmem + (static_cast<std::uint32_t>(qr * 32) << 16);
    const int q0 = half * 64;
    for (int i = i0; i < nq; ++i) {
      const int n = i - i0;
      float* st = stat + (n & 1) * 256;
      // the block's lse2 / D, staged in shared memory for every key row
      if (t < 128) st[t] = lse[static_cast<std::int64_t>(h) * rows + b * seq + i * kAttnBlock + t];
      else st[t] = dsum[static_cast<std::int64_t>(h) * rows + b * seq + i * kAttnBlock + t - 128];
      asm volatile("bar.sync 5, 256;" ::: "memory");
      mbar_wait(s_full, n & 1);
      tc_fence_after();
      std::uint32_t sv[64], pv[64];
      tmem_ld64(lane_base + q0, sv);
      tmem_ld64(lane_base + 128 + q0, pv);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_empty);
      const bool diag = CAUSAL && i == kb;  // query < key masked
      float pf[64];
#pragma unroll
      for (int e = 0; e < 64; ++e)
        pf[e] = (!diag || r <= q0 + e) ? ex2(fmaf(__uint_as_float(sv[e]), scale_log2, -st[q0 + e])) : 0.f;
      std::uint8_t* prow = sP + half * 16384 + r * 128;
      mbar_wait(ds_empty, (n & 1) ^ 1);  // the previous block's dSᵀ consumed
#pragma unroll
      for (int cw = 0; cw < 8; ++cw)
        *reinterpret_cast<uint4*>(prow + ((cw ^ (r & 7)) << 4)) =
            make_uint4(bf16_pair(pf[8 * cw], pf[8 * cw + 1]), bf16_pair(pf[8 * cw + 2], pf[8 * cw + 3]),
                       bf16_pair(pf[8 * cw + 4], pf[8 * cw + 5]), bf16_pair(pf[8 * cw + 6], pf[8 * cw + 7]));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      mbar_wait(p_empty, n & 1);  // Pᵀ·dO has read the tile
#pragma unroll
      for (int cw = 0; cw < 8; ++cw) {
        std::uint32_t w[4];
#pragma unroll
        for (int h2 = 0; h2 < 4; ++h2) {
          const int e = 8 * cw + 2 * h2;
          w[h2] = bf16_pair(pf[e] * (__uint_as_float(pv[e]) - st[128 + q0 + e]),
                            pf[e + 1] * (__uint_as_float(pv[e + 1]) - st[128 + q0 + e + 1]));
        }
        *reinterpret_cast<uint4*>(prow + ((cw ^ (r & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
    }
    mbar_wait(acc_full, 0);
    tc_fence_after();
    constexpr int HD = DH / 2;
    const std::int64_t go = static_cast<std::int64_t>(krow0 + r) * ld + col0 + half * HD;
#pragma unroll
    for (int which = 0; which < 2; ++which) {  // 0: dV (unscaled), 1: dK (x scale)
      __nv_bfloat16* dst = which == 0 ? dv : dk;
      if (dst == nullptr) continue;
      const float f = which == 0 ? 1.f : scale;
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        std::uint32_t v[32];
        tmem_ld32(lane_base + 256 + which * DH + half * HD + c * 32, v);
#pragma unroll
        for (int g = 0; g < 4; ++g)
          reinterpret_cast<uint4*>(dst + go + c * 32)[g] = make_uint4(
              bf16_pair(__uint_as_float(v[8 * g]) * f, __uint_as_float(v[8 * g + 1]) * f),
              bf16_pair(__uint_as_float(v[8 * g + 2]) * f, __uint_as_float(v[8 * g + 3]) * f),
              bf16_pair(__uint_as_float(v[8 * g + 4]) * f, __uint_as_float(v[8 * g + 5]) * f),
              bf16_pair(__uint_as_float(v[8 * g + 6]) * f, __uint_as_float(v[8 * g + 7]) * f));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// bf16 row-major [rows][cols], box {64 cols, box_rows}, 128B swizzle (make_map).
template <int DH, bool CAUSAL>
void attn_launch(const void* q, const void* k, const void* v, void* o, std::int64_t rows, std::int64_t cols,
                 std::int64_t seq, cudaStream_t s) {
  static unsigned attr_set_mask = 0;
  auto kern = attn_fwd_kernel<DH, CAUSAL>;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_set_mask & (1u << dev))) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, AttnCfg<DH>::SMEM);
    if (e != cudaSuccess) throw std::runtime_error(std::string("attention smem attribute: ") + cudaGetErrorString(e));
    attr_set_mask |= 1u << dev;
  }
  AttnMaps mp;
  mp.q = make_map(q, rows, cols, kAttnBlock);
  mp.k = make_map(k, rows, cols, kAttnBlock);
  mp.v = make_map(v, rows, cols, 64);
  const float scale_log2 = 1.4426950408889634f / std::sqrt(static_cast<float>(DH));
  dim3 grid(static_cast<unsigned>(cols / DH), static_cast<unsigned>(rows / seq), static_cast<unsigned>(seq / kAttnBlock));
  pdl_launch("attn_fwd_kernel", kern, grid, dim3(kAttnThreads), AttnCfg<DH>::SMEM, s, mp,
             static_cast<__nv_bfloat16*>(o), static_cast<int>(seq), static_cast<int>(cols), scale_log2,
             static_cast<float*>(nullptr), static_cast<float*>(nullptr), static_cast<const __nv_bfloat16*>(nullptr),
             static_cast<const __nv_bfloat16*>(nullptr), 0);
}

template <int DH, bool CAUSAL>
void attn_bwd_launch(const void* q, const void* k, const void* v, const void* o, const void* dout, void* dq, void* dk,
                     void* dv, float* ws, std::int64_t rows, std::int64_t cols, std::int64_t seq, cudaStream_t s) {
  static unsigned attr_set_mask = 0;
  auto kst = attn_fwd_kernel<DH, CAUSAL, true>;
  auto kdq = attn_bwd_dq_kernel<DH, CAUSAL>;
  auto kkv = attn_bwd_dkdv_kernel<DH, CAUSAL>;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_set_mask & (1u << dev))) {
    for (auto e : {cudaFuncSetAttribute(kst, cudaFuncAttributeMaxDynamicSharedMemorySize, AttnCfg<DH>::SMEM),
                   cudaFuncSetAttribute(kdq, cudaFuncAttributeMaxDynamicSharedMemorySize, AttnBwdCfg<DH>::SMEM),
                   cudaFuncSetAttribute(kkv, cudaFuncAttributeMaxDynamicSharedMemorySize, AttnBwdCfg<DH>::SMEM)})
      if (e != cudaSuccess) throw std::runtime_error(std::string("attention-grad smem attribute: ") + cudaGetErrorString(e));
    attr_set_mask |= 1u << dev;
  }
  const float scale = 1.f / std::sqrt(static_cast<float>(DH));
  const float scale_log2 = 1.4426950408889634f * scale;
  const std::int64_t heads = cols / DH;
  float* lse = ws;
  float* dsum = ws + heads * rows;
  dim3 grid(static_cast<unsigned>(heads), static_cast<unsigned>(rows / seq), static_cast<unsigned>(seq / kAttnBlock));
  AttnMaps fm;
  fm.q = make_map(q, rows, cols, kAttnBlock);
  fm.k = make_map(k, rows, cols, kAttnBlock);
  fm.v = make_map(v, rows, cols, 64);
  pdl_launch("attn_stats_kernel", kst, grid, dim3(kAttnThreads), AttnCfg<DH>::SMEM, s, fm,
             static_cast<__nv_bfloat16*>(nullptr), static_cast<int>(seq), static_cast<int>(cols), scale_log2, lse, dsum,
             static_cast<const __nv_bfloat16*>(o), static_cast<const __nv_bfloat16*>(dout), static_cast<int>(rows));
  AttnBwdMaps bm;
  bm.q = make_map(q, rows, cols, kAttnBlock);
  bm.k = make_map(k, rows, cols, kAttnBlock);
  bm.v = make_map(v, rows, cols, kAttnBlock);
  bm.dout = make_map(dout, rows, cols, kAttnBlock);
  if (dq)
    pdl_launch("attn_bwd_dq_kernel", kdq, grid, dim3(kAttnThreads), AttnBwdCfg<DH>::SMEM, s, bm,
               static_cast<__nv_bfloat16*>(dq), static_cast<int>(seq), static_cast<int>(cols), scale_log2, scale,
               static_cast<const float*>(lse), static_cast<const float*>(dsum), static_cast<int>(rows));
  if (dk || dv)
    pdl_launch("attn_bwd_dkdv_kernel", kkv, grid, dim3(kAttnThreads), AttnBwdCfg<DH>::SMEM, s, bm,
               static_cast<__nv_bfloat16*>(dk), static_cast<__nv_bfloat16*>(dv), static_cast<int>(seq),
               static_cast<int>(cols), scale_log2, scale, static_cast<const float*>(lse),
               static_cast<const float*>(dsum), static_cast<int>(rows));
}

}  // namespace

std::int64_t attention_grad_scratch_bytes(std::int64_t rows, std::int64_t cols, std::int64_t head_dim) {
  return 2 * rows * (cols / head_dim) * static_cast<std::int64_t>(sizeof(float));
}

void launch_attention_grad(const void* q, const void* k, const void* v, const void* o, const void* dout, void* dq,
                           void* dk, void* dv, void* scratch, std::int64_t rows, std::int64_t cols, std::int64_t seq,
                           std::int64_t head_dim, bool causal, int dtype, cudaStream_t s) {
  if (const char* why = attention_unsupported(rows, cols, seq, head_dim, dtype)) throw std::runtime_error(why);
  float* ws = static_cast<float*>(scratch);
  if (head_dim == 128) {
    if (causal) attn_bwd_launch<128, true>(q, k, v, o, dout, dq, dk, dv, ws, rows, cols, seq, s);
    else attn_bwd_launch<128, false>(q, k, v, o, dout, dq, dk, dv, ws, rows, cols, seq, s);
  } else {
    if (causal) attn_bwd_launch<64, true>(q, k, v, o, dout, dq, dk, dv, ws, rows, cols, seq, s);
    else attn_bwd_launch<64, false>(q, k, v, o, dout, dq, dk, dv, ws, rows, cols, seq, s);
  }
}

const char* attention_unsupported(std::int64_t rows, std::int64_t cols, std::int64_t seq, std::int64_t head_dim,
                                  int dtype) {
  if (dtype != DT_BF16) return "fused attention needs bf16 tensors";
  if (head_dim != 64 && head_dim != 128) return "fused attention supports head_dim 64 or 128";
  if (seq <= 0 || seq % kAttnBlock != 0) return "fused attention needs seq a multiple of 128";
  if (rows % seq != 0 || cols % head_dim != 0) return "attention piece does not hold whole sequences and heads";
  if (rows / seq > 65535 || seq / kAttnBlock > 65535) return "attention piece above the grid limits";
  return nullptr;
}

void launch_attention(const void* q, const void* k, const void* v, void* o, std::int64_t rows, std::int64_t cols,
                      std::int64_t seq, std::int64_t head_dim, bool causal, int dtype, cudaStream_t s) {
  if (const char* why = attention_unsupported(rows, cols, seq, head_dim, dtype)) throw std::runtime_error(why);
  if (head_dim == 128) {
    if (causal) attn_launch<128, true>(q, k, v, o, rows, cols, seq, s);
    else attn_launch<128, false>(q, k, v, o, rows, cols, seq, s);
  } else {
    if (causal) attn_launch<64, true>(q, k, v, o, rows, cols, seq, s);
    else attn_launch<64, false>(q, k, v, o, rows, cols, seq, s);
  }
}

}  // namespace planc_b200
