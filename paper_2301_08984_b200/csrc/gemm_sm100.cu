// tcgen05 GEMM: launch schedules (data-parallel / stream-K / split-K /
// grouped / two-CTAs-per-SM / 8-epilogue-warp variants) and dispatch. Kernel
// templates: gemm_sm100_impl.cuh; instantiations: gemm_sm100_ab*.cu.
#include "gemm_sm100_impl.cuh"

namespace planc_b200 {

namespace {

// Modelled time (us) of one launch, calibrated on B200 single-GEMM graphs
// (profiles/r01/gemm_streamk*.jsonl): per k-block MMA time by tile width
// (128x256 blocks ~0.35 us with every SM busy; 128x128 / 128x64 blocks are
// shared-memory-bandwidth bound at ~0.28 us), a per-tile epilogue cost, and
// for stream-K the fp32 partial writes plus the last arrival's reduction,
// which is L2-latency bound: one ~1 us round trip per kSkDepth partials per
// 32-column chunk.
double kb_us(int bn) { return bn == 256 ? 0.35 : 0.28; }
constexpr double kTileUs = 0.3;
constexpr double kSkRoundTripUs = 1.0;
constexpr double kSkWriteChunkUs = 0.15;
constexpr int kMinSkIters = 4;  // k-blocks per stream-K range, at least

GemmSchedule schedule_for(std::int64_t m, std::int64_t n, std::int64_t k, int bn, bool allow_sk, int sms,
                          bool force_sk = false, int group = 1, bool allow_half = true) {
  GemmSchedule sc;
  sc.bn = bn;
  sc.tiles = ((m + BM - 1) / BM) * ((n + bn - 1) / bn) * std::max(group, 1);
  sc.num_k = (k + BK - 1) / BK;
  const std::int64_t waves = (sc.tiles + sms - 1) / sms;
  sc.grid = static_cast<int>(std::min<std::int64_t>(sc.tiles, sms));
  sc.dp_tiles = sc.tiles;
  sc.model_us = static_cast<double>(waves) * (sc.num_k * kb_us(bn) + kTileUs);
  // Half-width tail: a last wave of r <= sms/2 tiles runs as 2r half tiles.
  const std::int64_t rem = sc.tiles % sms;
  if (allow_half && bn >= 128 && rem > 0 && 2 * rem <= sms && sc.tiles > sms) {
    sc.dp_tiles = static_cast<int>(sc.tiles - rem);
    sc.half_items = static_cast<int>(2 * rem);
    sc.model_us = static_cast<double>(waves - 1) * (sc.num_k * kb_us(bn) + kTileUs) +
                  0.5 * sc.num_k * kb_us(bn) + kTileUs;
  }
  if (!allow_sk || sc.tiles % sms == 0) return sc;
  // Whole waves minus one stay data-parallel; the rest (< 2 waves of tiles)
  // is shared by `ctas` CTAs — every count from ~one segment per tile up to
  // the whole GPU is tried (fewer CTAs = shallower reductions).
  const std::int64_t dp_waves = sc.tiles >= sms ? sc.tiles / sms - 1 : 0;
  const std::int64_t sk_tiles = sc.tiles - dp_waves * sms;
  const long long iters = sk_tiles * sc.num_k;
  const int max_ctas = static_cast<int>(std::min<long long>(sms, iters / kMinSkIters));
  GemmSchedule best = sc;
  if (force_sk) best.model_us = 1e300;
  for (int ctas = static_cast<int>(std::min<std::int64_t>(sk_tiles, sms)); ctas <= max_ctas; ++ctas) {
    const long long per = (iters + ctas - 1) / ctas;
    if (ctas <= sk_tiles && per >= sc.num_k) continue;  // no tile would be shared
    const long long covers = std::min<long long>((sc.num_k + per - 1) / per + 1, ctas);
    const double chunks = bn / 32.0;
    const double fix = chunks * (2 * kSkWriteChunkUs + kSkRoundTripUs * ((covers + kSkDepth - 1) / kSkDepth));
    const double t = static_cast<double>(dp_waves) * (sc.num_k * kb_us(bn) + kTileUs) + per * kb_us(bn) + kTileUs + fix;
    if (t >= best.model_us) continue;
    best.half_items = 0;
    best.dp_tiles = static_cast<int>(dp_waves * sms);
    best.sk_ctas = ctas;
    best.sk_iters = iters;
    best.grid = dp_waves > 0 ? sms : ctas;
    best.counter_bytes = (sk_tiles * 4 * 4 + 255) / 256 * 256;
    best.ws_bytes = best.counter_bytes + static_cast<std::int64_t>(ctas) * 2 * BM * bn * 4;
    best.model_us = t;
  }
  return best;
}

}  // namespace

// Split-K candidate: T tiles (group included) x S splits work items on at
// most `sms` CTAs, S as large as keeps >= kMinSplitIters k-blocks per split;
// the reduce kernel reads S fp32 copies of the padded output and writes C.
constexpr int kMinSplitIters = 4;
constexpr double kReduceLaunchUs = 2.0;
constexpr double kReduceBytesPerUs = 4.0e6;  // ~4 TB/s from L2 / HBM
GemmSchedule splitk_for(std::int64_t m, std::int64_t n, std::int64_t k, int bn, int sms, int group, int es_out) {
  GemmSchedule sc;
  sc.bn = bn;
  const std::int64_t tm = (m + BM - 1) / BM, tn = (n + bn - 1) / bn;
  sc.tiles = tm * tn * std::max(group, 1);
  sc.num_k = (k + BK - 1) / BK;
  const std::int64_t S = std::min<std::int64_t>(sms / std::max<std::int64_t>(sc.tiles, 1), sc.num_k / kMinSplitIters);
  if (S < 2 || n % 4 != 0) {
    sc.model_us = 1e300;
    return sc;
  }
  sc.splits = static_cast<int>(S);
  sc.dp_tiles = static_cast<int>(sc.tiles);
  sc.grid = static_cast<int>(sc.tiles * S);
  const double part_bytes = static_cast<double>(std::max(group, 1)) * S * (tm * BM) * (tn * bn) * 4.0;
  sc.ws_bytes = static_cast<std::int64_t>(part_bytes);
  sc.model_us = static_cast<double>((sc.num_k + S - 1) / S) * kb_us(bn) + kTileUs + kReduceLaunchUs +
                (part_bytes + static_cast<double>(std::max(group, 1)) * m * n * es_out) / kReduceBytesPerUs;
  return sc;
}

// Tile width and stream-K split: the candidate with the least modelled time
// (data-parallel preferred unless stream-K is clearly faster, wider tiles
// unless narrower ones are). PLANC_B200_GEMM_BN=256|128|64 forces a width,
// PLANC_B200_STREAMK=0 disables stream-K, =2 takes it whenever it applies.
GemmSchedule gemm_sm100_schedule(const GemmArgs& a, int sms) {
  if (gemm_x3_eligible(a)) return gemm_x3_schedule(a, sms);
  const char* env = std::getenv("PLANC_B200_GEMM_BN");
  const int forced = env ? std::atoi(env) : 0;
  const char* skenv = std::getenv("PLANC_B200_STREAMK");
  const int skmode = skenv ? std::atoi(skenv) : 1;
  const bool allow_sk =
      skmode != 0 && !a.no_workspace && a.epi.n_ops == 0 && a.scatter == 0 && (a.allow_streamk || skmode == 2);
  // PLANC_B200_SPLITK=0 disables split-K, =2 takes it whenever it applies.
  const char* spenv = std::getenv("PLANC_B200_SPLITK");
  const int splitmode = spenv ? std::atoi(spenv) : 1;
  // Like stream-K, split-K trades SM-time (and a reduce launch) for
  // latency: only when the lane has the GPU to itself. With co-resident
  // lanes (C4 / C5 at N=1: 8 lanes) the reduce launch lengthens every
  // lane's dependency chain and their concurrent work fills the SMs anyway
  // (C5 2.57 -> 2.35 ms, C4 5.34 -> 5.26 ms without it;
  // profiles/r02/ab_knobs_c4_c5.jsonl). =2 forces it.
  // Exception: a long-k GEMM with a tiny output (C5's dW GEMMs: 128 x 128 x
  // 8192 and 256 x 256 x 4096, one or two tiles — 2-4 SMs for 40-60 us, a
  // link of its lane's chain) is split within the lane's share of the SMs
  // (sms / lanes on the GPU) when that gives >= 4 splits: C5 2.42 -> 2.30
  // ms. With 2 splits (C4's 512 x 512 x 16384 dW) the reduce launch costs
  // more than it saves (C4 5.38 -> 5.52 ms; profiles/r02/ab_shared_split.json).
  // PLANC_B200_SPLITK_SHARED=0 disables, =2 allows 2 splits as well.
  const char* shenv = std::getenv("PLANC_B200_SPLITK_SHARED");
  const int shmode = shenv ? std::atoi(shenv) : 1;
  const bool shared_split = shmode != 0 && a.gpu_share > 1;
  const int min_splits = a.allow_streamk || splitmode == 2 || shmode == 2 ? 2 : 4;
  const bool allow_split = splitmode != 0 && !a.no_workspace && a.epi.n_ops == 0 && a.scatter == 0 &&
                           (a.allow_streamk || splitmode == 2 || shared_split);
  const int split_sms = a.allow_streamk ? sms : std::max(2, sms / std::max(a.gpu_share, 1));
  GemmSchedule best;
  bool have = false;
  for (int bn : {256, 128, 64}) {
    if (forced && bn != forced) continue;
    // PLANC_B200_HALF_TAIL=1 enables the half-width tail (off by default:
    // inside a plan step the idle SMs of a partial last wave already run
    // other streams' work, and the A/B on C2 / C2x / C1-L measured the tail
    // 2-3 % slower — profiles/r01/ab_plans_half_tail.jsonl); the fused
    // epilogue walks whole tiles only.
    const char* hv = std::getenv("PLANC_B200_HALF_TAIL");
    const bool allow_half = a.epi.n_ops == 0 && a.scatter == 0 && hv && hv[0] == '1';
    GemmSchedule dp = schedule_for(a.m, a.n, a.k, bn, false, sms, false, a.group, allow_half);
    GemmSchedule sk = schedule_for(a.m, a.n, a.k, bn, allow_sk, sms, skmode == 2, a.group, allow_half);
    GemmSchedule c = (sk.sk_ctas > 0 && (skmode == 2 || sk.model_us < 0.9 * dp.model_us)) ? sk : dp;
    if (allow_split) {
      GemmSchedule sp = splitk_for(a.m, a.n, a.k, bn, split_sms, a.group, a.dc == DT_BF16 ? 2 : 4);
      if (sp.splits >= min_splits && (splitmode == 2 || sp.model_us < 0.9 * c.model_us)) c = sp;
    }
    if (!have || c.model_us < best.model_us * 0.97) {
      best = c;
      have = true;
    }
  }
  // Fused short-k launches: a tile's epilogue (fold + two stores per chunk)
  // outlasts its few k-blocks, and with ~1.7 tiles per CTA (C4's 16384 x 512
  // x 512: 256 tiles of 128 x 256) it barely overlaps the next mainloop
  // (profiles/r02/ncu_fused_shortk_c4.json): 128-wide tiles instead (twice
  // the tiles per CTA, half-length epilogues) — C4 5.27 -> 5.15 ms, 64-wide
  // 5.83 (profiles/r02/ab_fused_short_k_bn.json). PLANC_B200_FUSED_SHORTK_BN=0
  // leaves the width to the model.
  const std::int64_t nk_fs = (a.k + BK - 1) / BK;
  static const int fused_bn = [] {
    const char* e = std::getenv("PLANC_B200_FUSED_SHORTK_BN");
    return e ? std::atoi(e) : 128;
  }();
  if (a.epi.n_ops > 0 && nk_fs <= 16 && !forced && fused_bn == 128 && fused_bn < best.bn)
    best = schedule_for(a.m, a.n, a.k, fused_bn, false, sms, false, a.group, false);
  // Short-k GEMMs (<= 16 k-blocks: latency-bound tiles) that cannot fill
  // the GPU on their own (<= sms tiles of 128 x 128) take the two-CTAs-per-SM
  // variant (BN <= 128, a ~76 KB ring): a concurrent small GEMM of another
  // stream / lane then runs on the same SMs instead of after it (C5 pipeline
  // 0.416 -> 0.344 ms; the grouped 1000+-tile launches of C4 are slower with
  // it, hence the tile bound). PLANC_B200_OCC2=0 disables it, =2 forces it.
  const char* oenv = std::getenv("PLANC_B200_OCC2");
  const int omode = oenv ? std::atoi(oenv) : 1;
  const std::int64_t num_k = (a.k + BK - 1) / BK;
  const std::int64_t tiles128 = ((a.m + BM - 1) / BM) * ((a.n + 127) / 128) * std::max(a.group, 1);
  if (omode != 0 && a.epi.n_ops == 0 && !forced && best.splits <= 1 && best.sk_ctas == 0 &&
      (omode == 2 || (num_k <= 16 && tiles128 <= sms))) {
    const int bn = a.n <= 64 ? 64 : 128;
    GemmSchedule o = schedule_for(a.m, a.n, a.k, bn, false, 2 * sms, false, a.group, false);
    o.occ = 2;
    best = o;
  }
  // Short-k launches that fill the GPU on their own: the tile epilogue
  // (BN/32 TMEM chunks per warp) outlasts the tile's few k-blocks of MMAs,
  // so 8 epilogue warps split each tile's columns. PLANC_B200_EPI8=0
  // disables it, =2 forces it on plain data-parallel launches.
  // Fused elementwise epilogues too (C4's 16384 x 512 x 512 GEMMs with their
  // add / mul: the fold and the second store double the epilogue's work);
  // PLANC_B200_EPI8_FUSED=0 keeps those on four epilogue warps.
  const char* e8 = std::getenv("PLANC_B200_EPI8");
  const int e8mode = e8 ? std::atoi(e8) : 1;
  const char* e8f = std::getenv("PLANC_B200_EPI8_FUSED");
  const bool e8fused = !(e8f && e8f[0] == '0');
  // (fused: >= 128-wide tiles — the fused chunk loop walks column chunks in
  // pairs, and a 64-wide tile gives each of the eight warps a single chunk)
  if (e8mode != 0 && best.occ == 1 && (a.epi.n_ops == 0 || (e8fused && best.bn >= 128)) && a.scatter == 0 &&
      best.splits <= 1 &&
      best.sk_ctas == 0 &&
      best.half_items == 0 && (e8mode == 2 || num_k <= 16)) {
    best.occ = 3;
  }
  // Cluster pairs sharing B tiles by TMA multicast (halves B's L2 -> SM
  // traffic). PLANC_B200_CLUSTER=2 forces it on plain data-parallel
  // launches with tiles >= 128 wide; 0 (default) leaves it off.
  const char* cenv = std::getenv("PLANC_B200_CLUSTER");
  const int cmode = cenv ? std::atoi(cenv) : 0;
  // 2-SM pairs (one 256-row tcgen05 MMA per pair, cta_group::2) for
  // data-parallel launches with more than 16 k-blocks (k > 1024), fused
  // epilogues included: C2 1.733 -> 1.688 ms, C2x 1.906 -> 1.858 ms, C1-L
  // 2.020 -> 1.960 ms, C4 / C5 neutral (profiles/r01/ab_2sm_fused.jsonl;
  // short k keeps the eight-epilogue-warp / two-CTA variants).
  // PLANC_B200_2SM=0 disables, =2 forces.
  const char* senv = std::getenv("PLANC_B200_2SM");
  const int smode = senv ? std::atoi(senv) : 1;
  const bool sm2 = smode == 2 || (smode == 1 && num_k > 16);
  // (the 2-SM variant also carries fused elementwise epilogues)
  if ((cmode == 2 || sm2) && best.occ == 1 && (a.epi.n_ops == 0 || (sm2 && cmode != 2)) && a.scatter == 0 &&
      best.splits <= 1 && best.sk_ctas == 0 && best.half_items == 0 && best.bn >= 128) {
    const std::int64_t pairs =
        ((a.m + 2 * BM - 1) / (2 * BM)) * ((a.n + best.bn - 1) / best.bn) * std::max(a.group, 1);
    best.occ = sm2 ? 5 : 4;
    best.grid = static_cast<int>(2 * std::min<std::int64_t>(pairs, sms / 2));
  }
  return best;
}

int gemm_sm100_launches(const GemmArgs& a) {
  if (gemm_x3_eligible(a)) return 2;  // hi / lo split + GEMM
  return gemm_sm100_schedule(a, device_sms()).splits > 1 ? 2 : 1;
}

void gemm_sm100_gather_maps(const GemmArgs& a, void* host_out) {
  static_assert(sizeof(CUtensorMap) == kTensorMapBytes, "tensor map size");
  GemmSchedule sc = gemm_sm100_schedule(a, device_sms());
  if ((sc.sk_ctas > 0 || sc.splits > 1) && (a.ws == nullptr || a.ws_bytes < sc.ws_bytes)) {
    GemmArgs b = a;
    b.no_workspace = true;
    sc = gemm_sm100_schedule(b, device_sms());
  }
  CUtensorMap* out = static_cast<CUtensorMap*>(host_out);
  std::memset(out, 0, kGatherMapSlots * sizeof(CUtensorMap));
  encode_gather_maps(a, sc, out);
}

int gemm_sm100_tile_n(const GemmArgs& a) { return gemm_sm100_schedule(a, 148).bn; }

std::int64_t gemm_sm100_workspace_bytes(const GemmArgs& a) {
  if (!gemm_sm100_eligible(a)) return 0;
  return gemm_sm100_schedule(a, device_sms()).ws_bytes;
}

bool gemm_sm100_eligible(const GemmArgs& a) {
  if (gemm_x3_eligible(a)) return true;  // fp32: 3xTF32 (gemm_x3.cu)
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
  if (gemm_x3_eligible(a)) return launch_gemm_x3(a, s);
  const bool a_mn = a.ta, b_mn = !a.tb, cb = a.dc == DT_BF16;
  GemmSchedule sc = gemm_sm100_schedule(a, device_sms());
  if ((sc.sk_ctas > 0 || sc.splits > 1) && (a.ws == nullptr || a.ws_bytes < sc.ws_bytes)) {
    // No (or too small a) workspace: the same selection among the
    // data-parallel variants (2-SM, eight epilogue warps, two CTAs per SM).
    GemmArgs b = a;
    b.no_workspace = true;
    sc = gemm_sm100_schedule(b, device_sms());
  }
  if (a.epi.n_ops > 0) {
    if (!cb) throw std::runtime_error("fused GEMM epilogue needs a bf16 output");
    if (a.epi.n_ops != 1 || a.epi.n_slots > kMaxEpiSlots || a.epi.ops[0].n_in > kMaxEpiIn)
      throw std::runtime_error("fused GEMM epilogue: one elementwise op with <= 2 other operands");
  }
  if (!a_mn && !b_mn) return launch_gemm_tc_ab<false, false>(a, sc, s);
  if (!a_mn && b_mn) return launch_gemm_tc_ab<false, true>(a, sc, s);
  if (a_mn && !b_mn) return launch_gemm_tc_ab<true, false>(a, sc, s);
  return launch_gemm_tc_ab<true, true>(a, sc, s);
}

}  // namespace planc_b200
