// Instantiation unit of the tcgen05 GEMM for A_MN = false, B_MN = true
// (gemm_sm100_impl.cuh): every output type, tile width, fusion and launch variant.
#include "gemm_sm100_impl.cuh"

namespace planc_b200 {

template <>
void launch_gemm_tc_ab<false, true>(const GemmArgs& a, const GemmSchedule& sc, cudaStream_t s) {
  const bool cb = a.dc == DT_BF16;
  const int bn = sc.bn;
  if (a.epi.n_ops > 0) {
    if (bn == 256) return launch_typed<false, true, true, 256, true>(a, sc, s);
    if (bn == 128) return launch_typed<false, true, true, 128, true>(a, sc, s);
    return launch_typed<false, true, true, 64, true>(a, sc, s);
  }
  if (cb) {
    if (bn == 256) return launch_typed<false, true, true, 256, false>(a, sc, s);
    if (bn == 128) return launch_typed<false, true, true, 128, false>(a, sc, s);
    return launch_typed<false, true, true, 64, false>(a, sc, s);
  }
  if (bn == 256) return launch_typed<false, true, false, 256, false>(a, sc, s);
  if (bn == 128) return launch_typed<false, true, false, 128, false>(a, sc, s);
  return launch_typed<false, true, false, 64, false>(a, sc, s);
}

}  // namespace planc_b200
