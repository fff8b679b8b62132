// tcgen05 GEMM — placeholder until the tensor-core path lands.
#include "kernels.cuh"

namespace planc_b200 {
bool gemm_sm100_eligible(const GemmArgs&) { return false; }
void launch_gemm_sm100(const GemmArgs& a, cudaStream_t s) { launch_gemm_simt(a, s); }
}  // namespace planc_b200
