// Kernel launches with programmatic dependent launch (PDL, sm_90+).
//
// Every executor kernel is launched with programmatic stream serialization:
// it may be scheduled while the previous kernel of its stream is still
// draining, runs its prologue (barrier init, TMEM allocation, descriptor
// prefetch, table loads), and blocks in griddepcontrol.wait until that
// kernel has completed and its memory is visible — so a chain of dependent
// small kernels pays one launch latency instead of one per kernel. Each
// kernel calls pdl_wait() before touching any buffer (reads or writes: the
// split-K workspace is reused by the next GEMM on the stream) and
// pdl_trigger() once its dependents may start their prologues (never before
// a wait on other ranks: see peer_flags_kernel). Inside CUDA
// graph capture the attribute becomes a programmatic edge; PLANC_B200_PDL=0
// launches without it (the instructions are then no-ops).
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>

namespace planc_b200 {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PLANC_B200_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline void pdl_launch(const char* what, void (*kern)(KArgs...), dim3 grid, dim3 block, std::size_t smem,
                       cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Same with a thread-block cluster of `cluster_x` CTAs (1 = none).
template <typename... KArgs, typename... Args>
inline void pdl_launch_cluster(const char* what, void (*kern)(KArgs...), dim3 grid, dim3 block, std::size_t smem,
                               cudaStream_t s, int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = static_cast<unsigned>(cluster_x);
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace planc_b200
