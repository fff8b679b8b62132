// GELU and its gradient (erf form), shared by the stand-alone activation
// kernel (kernels.cu act_kernel) and the tcgen05 GEMM's fused epilogue
// (gemm_sm100_impl.cuh): one definition, so both produce the same bits.
#pragma once
#include <cuda_runtime.h>

// Phi(x) = 0.5 (1 + erf(x / sqrt 2)) with erf from Abramowitz & Stegun 7.1.26
// (|error| <= 1.5e-7) on e = exp(-x^2 / 2) — the same exponential GELU's
// gradient needs for the normal pdf. A third of erff's instructions: the
// GELU kernels stay memory-bound.
__device__ __forceinline__ float ex2_ftz(float x) {  // 2^x, denormals flushed (one MUFU.EX2, no range fix-up)
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcp_ftz(float x) {  // 1 / x for x >= 1 (one MUFU.RCP)
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float normal_cdf_e(float x, float e) {
  const float z = fabsf(x) * 0.70710678118654752f;
  const float t = rcp_ftz(fmaf(0.3275911f, z, 1.f));
  const float poly =
      t * fmaf(t, fmaf(t, fmaf(t, fmaf(t, 1.061405429f, -1.453152027f), 1.421413741f), -0.284496736f), 0.254829592f);
  const float erf_abs = fmaf(-poly, e, 1.f);
  return fmaf(0.5f, copysignf(erf_abs, x), 0.5f);
}
// exp(-x^2 / 2) = 2^(x * (x * -log2(e) / 2))
__device__ __forceinline__ float gelu_e(float x) { return ex2_ftz(x * (x * -0.72134752044448170f)); }
__device__ __forceinline__ float gelu_f(float x) { return x * normal_cdf_e(x, gelu_e(x)); }
__device__ __forceinline__ float gelu_grad_f(float x, float g) {
  const float e = gelu_e(x);
  return g * fmaf(x * 0.39894228040143268f, e, normal_cdf_e(x, e));
}
