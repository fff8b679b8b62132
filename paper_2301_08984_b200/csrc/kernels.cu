// Memory-bound sub-operator kernels, the fused adapter (box) kernel and the
// SIMT GEMM used for shapes the tcgen05 path does not take. sm_100a only.
#include <cuda_bf16.h>

#include <algorithm>
#include <stdexcept>
#include <string>

#include "gelu.cuh"
#include "kernels.cuh"
#include "launch.cuh"

namespace planc_b200 {

namespace {

inline void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

inline int grid_for(std::int64_t work, int per_block, int cap = 148 * 32) {
  std::int64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<int>(g);
}

// ---- element access --------------------------------------------------------

template <typename T>
struct Acc {
  using type = float;
};
template <>
struct Acc<int> {
  using type = int;
};

template <typename T>
__device__ __forceinline__ typename Acc<T>::type to_acc(T v) {
  return static_cast<typename Acc<T>::type>(v);
}
template <>
__device__ __forceinline__ float to_acc<__nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}
template <typename T>
__device__ __forceinline__ T from_acc(typename Acc<T>::type v) {
  return static_cast<T>(v);
}
template <>
__device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

// V consecutive elements (V*sizeof(T) = 16 bytes when V > 1).
// Unpacking is done with shifts / bit casts on the loaded words (no
// address-taken locals, so nothing is demoted to local memory).
__device__ __forceinline__ void unpack_word(std::uint32_t w, float& lo, float& hi) {
  lo = __uint_as_float(w << 16);
  hi = __uint_as_float(w & 0xffff0000u);
}
__device__ __forceinline__ std::uint32_t pack_word(float lo, float hi) {  // one F2FP pack (RNE)
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const std::uint32_t*>(&v);
}

template <typename T, int V>
__device__ __forceinline__ void load_vec(const T* p, typename Acc<T>::type (&o)[V]) {
  if constexpr (V == 1) {
    o[0] = to_acc<T>(*p);
  } else if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    uint4 r = __ldg(reinterpret_cast<const uint4*>(p));
    unpack_word(r.x, o[0], o[1]);
    unpack_word(r.y, o[2], o[3]);
    unpack_word(r.z, o[4], o[5]);
    unpack_word(r.w, o[6], o[7]);
  } else if constexpr (std::is_same<T, float>::value) {
    float4 r = __ldg(reinterpret_cast<const float4*>(p));
    o[0] = r.x;
    o[1] = r.y;
    o[2] = r.z;
    o[3] = r.w;
  } else {
    int4 r = __ldg(reinterpret_cast<const int4*>(p));
    o[0] = r.x;
    o[1] = r.y;
    o[2] = r.z;
    o[3] = r.w;
  }
}

template <typename T, int V>
__device__ __forceinline__ void store_vec(T* p, const typename Acc<T>::type (&v)[V]) {
  if constexpr (V == 1) {
    *p = from_acc<T>(v[0]);
  } else if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    *reinterpret_cast<uint4*>(p) =
        make_uint4(pack_word(v[0], v[1]), pack_word(v[2], v[3]), pack_word(v[4], v[5]), pack_word(v[6], v[7]));
  } else if constexpr (std::is_same<T, float>::value) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  } else {
    *reinterpret_cast<int4*>(p) = make_int4(v[0], v[1], v[2], v[3]);
  }
}

// Raw 16-byte vector loads, unpacked only after every load of a thread is in
// flight (unpacking at each load lets the compiler recycle one destination
// register set and serialise the loads).
template <typename T>
__device__ __forceinline__ uint4 ld16(const T* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}
template <typename T, int V>
__device__ __forceinline__ void unpack16(const uint4& r, float (&o)[V]) {
  static_assert(V == 16 / sizeof(T), "one 16-byte vector");
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    unpack_word(r.x, o[0], o[1]);
    unpack_word(r.y, o[2], o[3]);
    unpack_word(r.z, o[4], o[5]);
    unpack_word(r.w, o[6], o[7]);
  } else {
    o[0] = __uint_as_float(r.x);
    o[1] = __uint_as_float(r.y);
    o[2] = __uint_as_float(r.z);
    o[3] = __uint_as_float(r.w);
  }
}

__device__ __forceinline__ float load_any(const void* p, int dt, std::int64_t i) {
  if (dt == DT_BF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
  if (dt == DT_I32) return static_cast<float>(reinterpret_cast<const int*>(p)[i]);
  return reinterpret_cast<const float*>(p)[i];
}

__device__ __forceinline__ void store_any(void* p, int dt, std::int64_t i, float v) {
  if (dt == DT_BF16) reinterpret_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
  else if (dt == DT_I32) reinterpret_cast<int*>(p)[i] = static_cast<int>(v);
  else reinterpret_cast<float*>(p)[i] = v;
}

// ---- box: fused reconstruct -------------------------------------------------
// One block per chunk of kBoxThreads*kBoxUnroll vector units of one cell;
// every thread owns kBoxUnroll independent 16-byte vectors (all terms' loads
// in flight before any store). R = highest cell rank of the launch, so the
// common rank-1/2 cells carry no unused coordinates. Cell and term records
// are read through the read-only path (warp-uniform broadcasts); no smem,
// no barriers.

__device__ __forceinline__ float box_max(float a, float b) { return fmaxf(a, b); }  // = ew_kernel's max
__device__ __forceinline__ int box_max(int a, int b) { return a > b ? a : b; }

constexpr int kBoxThreads = 256;
constexpr int kBoxUnroll = 4;

template <typename T, int V, int R>
__global__ void __launch_bounds__(kBoxThreads) box_kernel(const DevCell* __restrict__ cells,
                                                           const DevTerm* __restrict__ terms,
                                                           const DevChunk* __restrict__ chunks) {
  pdl_wait();  // launch.cuh: inputs of the previous kernel visible
  pdl_trigger();
  // Every cell of the launch has exactly rank R (the host pads lower-rank
  // cells with leading unit dims), so all coordinate indexing is static and
  // stays in registers.
  using A = typename Acc<T>::type;
  constexpr int U = kBoxUnroll;
  const DevChunk ch = chunks[blockIdx.x];
  const DevCell* c = cells + ch.cell;
  const int nt = __ldg(&c->nterms);
  const int term0 = __ldg(&c->term0);
  std::int64_t dstr[R];
  std::uint32_t ext[R];
#pragma unroll
  for (int d = 0; d < R; ++d) {
    ext[d] = static_cast<std::uint32_t>(__ldg(&c->ext[d]));
    dstr[d] = __ldg(&c->dst_str[d]);
  }
  const std::int64_t dst_off = __ldg(&c->dst_off);
  T* dst = reinterpret_cast<T*>(__ldg(reinterpret_cast<const unsigned long long*>(&c->dst)));
  const std::uint32_t inner_vecs = ext[R - 1] / V;
  std::int64_t coord[U][R];
  bool live[U];
#pragma unroll
  for (int x = 0; x < U; ++x) {
    const std::int64_t u = threadIdx.x + static_cast<std::int64_t>(x) * kBoxThreads;
    live[x] = u < ch.count;
    const std::int64_t lin = ch.begin + (live[x] ? u : 0);
    if constexpr (R == 1) {
      coord[x][0] = lin * V;
    } else {
      // 32-bit division: chunk tables are built only for cells < 2^32 units.
      std::uint32_t l32 = static_cast<std::uint32_t>(lin);
      coord[x][R - 1] = static_cast<std::int64_t>(l32 % inner_vecs) * V;
      l32 /= inner_vecs;
#pragma unroll
      for (int d = R - 2; d >= 0; --d) {
        coord[x][d] = l32 % ext[d];
        l32 /= ext[d];
      }
    }
  }
  A acc[U][V];
#pragma unroll
  for (int x = 0; x < U; ++x)
#pragma unroll
    for (int i = 0; i < V; ++i) acc[x][i] = A(0);
  for (int t = 0; t < nt; ++t) {
    const DevTerm* tm = terms + term0 + t;
    const T* src = reinterpret_cast<const T*>(__ldg(reinterpret_cast<const unsigned long long*>(&tm->src)));
    const std::int64_t toff = __ldg(&tm->offset);
    const int op = __ldg(&tm->op);
    std::int64_t tstr[R];
#pragma unroll
    for (int d = 0; d < R; ++d) tstr[d] = __ldg(&tm->str[d]);
    A v[U][V];
#pragma unroll
    for (int x = 0; x < U; ++x) {
      std::int64_t soff = toff;
#pragma unroll
      for (int d = 0; d < R; ++d) soff += coord[x][d] * tstr[d];
      if (live[x]) load_vec<T, V>(src + soff, v[x]);
    }
#pragma unroll
    for (int x = 0; x < U; ++x) {
      if (op == 1) {
#pragma unroll
        for (int i = 0; i < V; ++i) acc[x][i] += v[x][i];
      } else if (op == 0) {
#pragma unroll
        for (int i = 0; i < V; ++i) acc[x][i] = v[x][i];
      } else if (op == 2) {
#pragma unroll
        for (int i = 0; i < V; ++i) acc[x][i] *= v[x][i];
      } else {
#pragma unroll
        for (int i = 0; i < V; ++i) acc[x][i] = box_max(acc[x][i], v[x][i]);
      }
    }
  }
#pragma unroll
  for (int x = 0; x < U; ++x) {
    if (!live[x]) continue;
    std::int64_t doff = dst_off;
#pragma unroll
    for (int d = 0; d < R; ++d) doff += coord[x][d] * dstr[d];
    store_vec<T, V>(dst + doff, acc[x]);
  }
}

template <typename T, int V>
void box_rank_dispatch(const DevCell* cells, const DevTerm* terms, const DevChunk* chunks, int nchunks, int max_rank,
                       cudaStream_t s) {
  if (max_rank <= 1) pdl_launch("box_kernel", box_kernel<T, V, 1>, dim3(nchunks), dim3(kBoxThreads), 0, s, cells, terms, chunks);
  else if (max_rank == 2) pdl_launch("box_kernel", box_kernel<T, V, 2>, dim3(nchunks), dim3(kBoxThreads), 0, s, cells, terms, chunks);
  else pdl_launch("box_kernel", box_kernel<T, V, kBoxRank>, dim3(nchunks), dim3(kBoxThreads), 0, s, cells, terms, chunks);
}

template <typename T>
void box_dispatch(const DevCell* cells, const DevTerm* terms, const DevChunk* chunks, int nchunks, int vec,
                  int max_rank, cudaStream_t s) {
  constexpr int VV = 16 / sizeof(T);
  if (vec) box_rank_dispatch<T, VV>(cells, terms, chunks, nchunks, max_rank, s);
  else box_rank_dispatch<T, 1>(cells, terms, chunks, nchunks, max_rank, s);
}

// ---- elementwise -----------------------------------------------------------

constexpr int kMaxEwIn = 8;
struct EwPtrs {
  const void* p[kMaxEwIn];
};

template <int OP>
__device__ __forceinline__ float ew_apply(float a, float b) {
  if constexpr (OP == 0) return a + b;
  if constexpr (OP == 1) return a * b;
  return fmaxf(a, b);
}

// Each thread keeps kEwUnroll independent 16-byte vectors in flight per
// operand; a block covers one contiguous 16 KB span per operand (DRAM page
// locality) with every warp access coalesced.
constexpr int kEwUnroll = 4;

template <typename T, int OP, int NIN>
__global__ void __launch_bounds__(256) ew_kernel(EwPtrs in, T* __restrict__ out, std::int64_t nvec) {
  pdl_wait();  // launch.cuh: inputs of the previous kernel visible
  pdl_trigger();
  constexpr int V = 16 / sizeof(T);
  const std::int64_t stride = blockDim.x;
  for (std::int64_t base = blockIdx.x * static_cast<std::int64_t>(blockDim.x) * kEwUnroll + threadIdx.x; base < nvec;
       base += static_cast<std::int64_t>(gridDim.x) * blockDim.x * kEwUnroll) {
    float acc[kEwUnroll][V], v[kEwUnroll][V];
#pragma unroll
    for (int u = 0; u < kEwUnroll; ++u) {
      const std::int64_t i = base + u * stride;
      if (i < nvec) load_vec<T, V>(static_cast<const T*>(in.p[0]) + i * V, acc[u]);
    }
#pragma unroll
    for (int k = 1; k < NIN; ++k) {  // NIN is static: operand pointers stay in the param bank
#pragma unroll
      for (int u = 0; u < kEwUnroll; ++u) {
        const std::int64_t i = base + u * stride;
        if (i < nvec) load_vec<T, V>(static_cast<const T*>(in.p[k]) + i * V, v[u]);
      }
#pragma unroll
      for (int u = 0; u < kEwUnroll; ++u)
#pragma unroll
        for (int j = 0; j < V; ++j) acc[u][j] = ew_apply<OP>(acc[u][j], v[u][j]);
    }
#pragma unroll
    for (int u = 0; u < kEwUnroll; ++u) {
      const std::int64_t i = base + u * stride;
      if (i < nvec) store_vec<T, V>(out + i * V, acc[u]);
    }
  }
}

template <typename T, int OP, int NIN>
__global__ void ew_tail_kernel(EwPtrs in, T* __restrict__ out, std::int64_t begin, std::int64_t count) {
  pdl_wait();  // launch.cuh: inputs of the previous kernel visible
  pdl_trigger();
  std::int64_t i = begin + blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (i >= begin + count) return;
  float acc = to_acc<T>(static_cast<const T*>(in.p[0])[i]);
#pragma unroll
  for (int k = 1; k < NIN; ++k) acc = ew_apply<OP>(acc, to_acc<T>(static_cast<const T*>(in.p[k])[i]));
  out[i] = from_acc<T>(acc);
}

template <typename T, int OP, int NIN>
void ew_launch(const EwPtrs& p, void* out, std::int64_t nvec, std::int64_t count, cudaStream_t s) {
  constexpr int V = 16 / sizeof(T);
  if (nvec > 0) {
    // One pass: every thread owns kEwUnroll vectors (no grid-stride tail).
    pdl_launch("ew_kernel", ew_kernel<T, OP, NIN>, dim3(grid_for(nvec, 256 * kEwUnroll, 1 << 30)), dim3(256), 0, s, p, static_cast<T*>(out), nvec);
  }
  std::int64_t rest = count - nvec * V;
  if (rest > 0) {
    pdl_launch("ew_tail_kernel", ew_tail_kernel<T, OP, NIN>, dim3(static_cast<int>((rest + 255) / 256)), dim3(256), 0, s, p, static_cast<T*>(out),
                                                                                    nvec * V, rest);
  }
}

template <typename T, int OP>
void ew_typed(const void* const* ins, int nin, void* out, std::int64_t count, cudaStream_t s) {
  constexpr int V = 16 / sizeof(T);
  EwPtrs p{};
  bool aligned = (reinterpret_cast<std::uintptr_t>(out) % 16) == 0;
  for (int i = 0; i < nin; ++i) {
    p.p[i] = ins[i];
    aligned = aligned && (reinterpret_cast<std::uintptr_t>(ins[i]) % 16) == 0;
  }
  std::int64_t nvec = aligned ? count / V : 0;
  switch (nin) {
    case 1: ew_launch<T, OP, 1>(p, out, nvec, count, s); break;
    case 2: ew_launch<T, OP, 2>(p, out, nvec, count, s); break;
    case 3: ew_launch<T, OP, 3>(p, out, nvec, count, s); break;
    case 4: ew_launch<T, OP, 4>(p, out, nvec, count, s); break;
    case 5: ew_launch<T, OP, 5>(p, out, nvec, count, s); break;
    case 6: ew_launch<T, OP, 6>(p, out, nvec, count, s); break;
    case 7: ew_launch<T, OP, 7>(p, out, nvec, count, s); break;
    default: ew_launch<T, OP, 8>(p, out, nvec, count, s); break;
  }
}

// ---- reduce-sum --------------------------------------------------------------

// inner == 1: one warp per output row, lanes stride the reduced axis.
// V > 1: 16-byte vectors (axis_len % V == 0, 16-byte aligned rows), four
// loads in flight per lane.
template <typename T, int V>
__global__ void __launch_bounds__(256) reduce_rows_kernel(const T* __restrict__ in, T* __restrict__ out,
                                                          std::int64_t outer, std::int64_t axis_len) {
  pdl_wait();  // launch.cuh: inputs of the previous kernel visible
  pdl_trigger();
  std::int64_t warp = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) / 32;
  int lane = threadIdx.x & 31;
  std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * blockDim.x / 32;
  const std::int64_t nv = axis_len / V;
  constexpr int U = V > 1 ? 4 : 1;
  for (std::int64_t r = warp; r < outer; r += nwarps) {
    const T* row = in + r * axis_len;
    float acc = 0.f;
    for (std::int64_t a0 = lane; a0 < nv; a0 += 32 * U) {
      float v[U][V];
      if constexpr (V > 1) {  // raw loads first: all U in flight
        uint4 raw[U];
#pragma unroll
        for (int u = 0; u < U; ++u) raw[u] = a0 + 32 * u < nv ? ld16(row + (a0 + 32 * u) * V) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) unpack16<T, V>(raw[u], v[u]);
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (a0 + 32 * u < nv) load_vec<T, V>(row + (a0 + 32 * u) * V, v[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (V > 1 || a0 + 32 * u < nv) {  // V > 1: dead vectors loaded as zeros
#pragma unroll
          for (int j = 0; j < V; ++j) acc += v[u][j];
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[r] = from_acc<T>(acc);
  }
}

// inner > 1: a block owns 32 * V * CV consecutive inner columns of one outer
// index (lane l holds vectors l, l + 32, ... of V elements: a warp reads
// CV * 512 contiguous bytes of every row it visits, DRAM-page friendly) and a
// range of the reduced axis, split over its 8 warps (interleaved rows, two
// rows of loads in flight); the warps' sums are combined in shared memory in
// warp order. When the axis is split over S > 1 blocks (grid.z), each writes
// an fp32 partial [outer][S][inner] to scratch and reduce_cols_finish adds
// the S partials in order — no atomics, the same bits every run.
constexpr int kRedWarps = 8;
constexpr int kRedCV = 4;  // vectors per lane along the kept axis
template <typename T, int V>
__global__ void __launch_bounds__(kRedWarps * 32) reduce_cols_kernel(const T* __restrict__ in, T* __restrict__ out,
                                                                    float* __restrict__ partial, std::int64_t outer,
                                                                    std::int64_t axis_len, std::int64_t inner) {
  pdl_wait();  // launch.cuh: inputs of the previous kernel visible
  pdl_trigger();
  constexpr int TW = 32 * V * kRedCV;  // columns per block
  __shared__ float red[kRedWarps][TW];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const std::int64_t o = blockIdx.y;
  const std::int64_t col0 = static_cast<std::int64_t>(blockIdx.x) * TW;
  const int S = gridDim.z;
  const std::int64_t a_lo = axis_len * blockIdx.z / S, a_hi = axis_len * (blockIdx.z + 1) / S;
  const T* base = in + o * axis_len * inner + col0;
  float acc[kRedCV][V];
#pragma unroll
  for (int c = 0; c < kRedCV; ++c)
#pragma unroll
    for (int j = 0; j < V; ++j) acc[c][j] = 0.f;
  bool live[kRedCV];
#pragma unroll
  for (int c = 0; c < kRedCV; ++c) live[c] = col0 + (c * 32 + lane) * V < inner;  // inner % V == 0 when V > 1
  constexpr int U = 2;
  for (std::int64_t a = a_lo + warp; a < a_hi; a += kRedWarps * U) {
    float v[U][kRedCV][V];
    if constexpr (V > 1) {  // raw loads first: all U x CV in flight
      uint4 raw[U][kRedCV];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int c = 0; c < kRedCV; ++c)
          raw[u][c] = live[c] && a + kRedWarps * u < a_hi
                          ? ld16(base + (a + kRedWarps * u) * inner + (c * 32 + lane) * V)
                          : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int c = 0; c < kRedCV; ++c) unpack16<T, V>(raw[u][c], v[u][c]);
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int c = 0; c < kRedCV; ++c)
          if (live[c] && a + kRedWarps * u < a_hi)
            load_vec<T, V>(base + (a + kRedWarps * u) * inner + (c * 32 + lane) * V, v[u][c]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int c = 0; c < kRedCV; ++c)
        if (V > 1 || (live[c] && a + kRedWarps * u < a_hi)) {  // V > 1: dead vectors loaded as zeros
#pragma unroll
          for (int j = 0; j < V; ++j) acc[c][j] += v[u][c][j];
        }
  }
#pragma unroll
  for (int c = 0; c < kRedCV; ++c)
#pragma unroll
    for (int j = 0; j < V; ++j) red[warp][(c * 32 + lane) * V + j] = acc[c][j];
  __syncthreads();
  for (int i = threadIdx.x; i < TW; i += blockDim.x) {
    const std::int64_t col = col0 + i;
    if (col >= inner) continue;
    float sum = red[0][i];
#pragma unroll
    for (int w = 1; w < kRedWarps; ++w) sum += red[w][i];
    if (S == 1) out[o * inner + col] = from_acc<T>(sum);
    else partial[(o * S + blockIdx.z) * inner + col] = sum;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) reduce_cols_finish(const float* __restrict__ partial, T* __restrict__ out,
                                                          std::int64_t outer, int S, std::int64_t inner) {
  pdl_wait();
  pdl_trigger();
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < outer * inner;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t o = i / inner, c = i - o * inner;
    const float* p = partial + o * S * inner + c;
    // Partials folded in split order; loaded 8 at a time so the chain of S
    // loads costs S / 8 memory round trips, not S.
    float sum = 0.f;
    for (int s0 = 0; s0 < S; s0 += 8) {
      float v[8];
#pragma unroll
      for (int d = 0; d < 8; ++d) v[d] = s0 + d < S ? __ldcg(p + static_cast<std::int64_t>(s0 + d) * inner) : 0.f;
#pragma unroll
      for (int d = 0; d < 8; ++d)
        if (s0 + d < S) sum = s0 + d == 0 ? v[d] : sum + v[d];
    }
    out[i] = from_acc<T>(sum);
  }
}

// ---- embedding ---------------------------------------------------------------

// One warp per index; V > 1 copies 16-byte vectors (h % V == 0, aligned).
template <typename T, int V>
__global__ void __launch_bounds__(256) emb_lookup_kernel(const int* __restrict__ idx, const T* __restrict__ table,
                                                         T* __restrict__ out, std::int64_t n, std::int64_t rows,
                                                         std::int64_t h, std::int64_t lo) {
  pdl_wait();  // launch.cuh: inputs of the previous kernel visible
  pdl_trigger();
  std::int64_t warp = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) / 32;
  int lane = threadIdx.x & 31;
  std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * blockDim.x / 32;
  for (std::int64_t j = warp; j < n; j += nwarps) {
    std::int64_t id = idx[j];
    bool in_shard = id >= lo && id < lo + rows;
    if constexpr (V > 1) {
      const uint4* src = reinterpret_cast<const uint4*>(table + (id - lo) * h);
      uint4* dst = reinterpret_cast<uint4*>(out + j * h);
      for (std::int64_t c = lane; c < h / V; c += 32) dst[c] = in_shard ? __ldg(src + c) : make_uint4(0, 0, 0, 0);
    } else {
      for (std::int64_t c = lane; c < h; c += 32) out[j * h + c] = in_shard ? table[(id - lo) * h + c] : from_acc<T>(0.f);
    }
  }
}

// embedding-grad (refexec.cpp:233-250: out[idx[j] - lo] += gout[j] in
// ascending j), deterministic: no float atomics. Kernel 1 takes 1024
// consecutive indices per block, sorts (row, j) keys in shared memory
// (bitonic, unique keys) and sums each row's gout rows in ascending j into a
// per-block partial; kernel 2 gives each output row one warp that adds the
// blocks' partials in block order (binary search of the block's sorted
// segment rows). Same bits on every run, the reference's j order inside a
// block.
constexpr int kEmbBlock = 1024;

template <typename T>
__global__ void __launch_bounds__(512) emb_grad_block_kernel(const int* __restrict__ idx, const T* __restrict__ gout,
                                                             float* __restrict__ partial, int* __restrict__ seg_row,
                                                             int* __restrict__ nseg, std::int64_t n, std::int64_t rows,
                                                             std::int64_t h, std::int64_t lo) {
  pdl_wait();  // launch.cuh: inputs of the previous kernel visible
  pdl_trigger();
  __shared__ unsigned long long key[kEmbBlock];
  __shared__ int start[kEmbBlock + 1];
  __shared__ int head_scan[kEmbBlock];
  const std::int64_t base = static_cast<std::int64_t>(blockIdx.x) * kEmbBlock;
  for (int i = threadIdx.x; i < kEmbBlock; i += blockDim.x) {
    const std::int64_t j = base + i;
    unsigned long long r = static_cast<unsigned long long>(rows);  // sentinel: not in this shard / padding
    if (j < n) {
      const std::int64_t id = idx[j];
      if (id >= lo && id < lo + rows) r = static_cast<unsigned long long>(id - lo);
    }
    key[i] = (r << 10) | static_cast<unsigned long long>(i);
  }
  __syncthreads();
  for (int k = 2; k <= kEmbBlock; k <<= 1) {
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int i = threadIdx.x; i < kEmbBlock; i += blockDim.x) {
        const int p = i ^ jj;
        if (p > i) {
          const bool up = (i & k) == 0;
          const unsigned long long a = key[i], b = key[p];
          if ((a > b) == up) {
            key[i] = b;
            key[p] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  // segment heads (valid rows only) -> inclusive scan -> segment ids
  for (int i = threadIdx.x; i < kEmbBlock; i += blockDim.x) {
    const unsigned long long r = key[i] >> 10;
    head_scan[i] = (r < static_cast<unsigned long long>(rows) && (i == 0 || (key[i - 1] >> 10) != r)) ? 1 : 0;
  }
  __syncthreads();
  for (int off = 1; off < kEmbBlock; off <<= 1) {
    int v[2];
    for (int q = 0; q < 2; ++q) {
      const int i = threadIdx.x + q * blockDim.x;
      v[q] = (i < kEmbBlock && i >= off) ? head_scan[i - off] : 0;
    }
    __syncthreads();
    for (int q = 0; q < 2; ++q) {
      const int i = threadIdx.x + q * blockDim.x;
      if (i < kEmbBlock) head_scan[i] += v[q];
    }
    __syncthreads();
  }
  const int segs = head_scan[kEmbBlock - 1];
  for (int i = threadIdx.x; i < kEmbBlock; i += blockDim.x) {
    const unsigned long long r = key[i] >> 10;
    const bool head = r < static_cast<unsigned long long>(rows) && (i == 0 || (key[i - 1] >> 10) != r);
    if (head) {
      start[head_scan[i] - 1] = i;
      seg_row[base + head_scan[i] - 1] = static_cast<int>(r);
    }
    // end of the last valid segment: the first sentinel (or the block end)
    if (r >= static_cast<unsigned long long>(rows) && (i == 0 || (key[i - 1] >> 10) < static_cast<unsigned long long>(rows)))
      start[segs] = i;
  }
  if (threadIdx.x == 0) {
    nseg[blockIdx.x] = segs;
    if ((key[kEmbBlock - 1] >> 10) < static_cast<unsigned long long>(rows)) start[segs] = kEmbBlock;
  }
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  for (int sg = warp; sg < segs; sg += nw) {
    const int s0 = start[sg], s1 = start[sg + 1];
    float* dst = partial + (base + sg) * h;
    for (std::int64_t c = lane; c < h; c += 32) {
      float acc = 0.f;
      for (int i = s0; i < s1; ++i) acc += to_acc<T>(gout[(base + static_cast<int>(key[i] & 1023)) * h + c]);
      dst[c] = acc;
    }
  }
}

template <typename T>
__global__ void emb_grad_combine_kernel(const float* __restrict__ partial, const int* __restrict__ seg_row,
                                        const int* __restrict__ nseg, T* __restrict__ out, int nblocks,
                                        std::int64_t rows, std::int64_t h) {
  pdl_wait();  // launch.cuh: inputs of the previous kernel visible
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const std::int64_t warp = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) / 32;
  const std::int64_t nwarps = static_cast<std::int64_t>(gridDim.x) * blockDim.x / 32;
  for (std::int64_t r = warp; r < rows; r += nwarps) {
    for (std::int64_t c0 = 0; c0 < h; c0 += 128) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      for (int b0 = 0; b0 < nblocks; b0 += 32) {
        // lane l looks row r up among block (b0 + l)'s sorted segment rows
        int seg = -1;
        const int b = b0 + lane;
        if (b < nblocks) {
          int lo_i = 0, hi_i = nseg[b];
          const int* rowsb = seg_row + static_cast<std::int64_t>(b) * kEmbBlock;
          while (lo_i < hi_i) {
            const int mid = (lo_i + hi_i) / 2;
            if (rowsb[mid] < r) lo_i = mid + 1;
            else hi_i = mid;
          }
          if (lo_i < nseg[b] && rowsb[lo_i] == r) seg = lo_i;
        }
        unsigned found = __ballot_sync(0xffffffffu, seg >= 0);
        while (found) {  // blocks in ascending order
          const int l = __ffs(found) - 1;
          found &= found - 1;
          const int sg = __shfl_sync(0xffffffffu, seg, l);
          const float* src = partial + (static_cast<std::int64_t>(b0 + l) * kEmbBlock + sg) * h;
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const std::int64_t c = c0 + lane + 32 * v;
            if (c < h) acc[v] += src[c];
          }
        }
      }
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const std::int64_t c = c0 + lane + 32 * v;
        if (c < h) out[r * h + c] = from_acc<T>(acc[v]);
      }
    }
  }
}

__global__ void convert_kernel(int dt, void* out, const float* __restrict__ in, std::int64_t count) {
  pdl_wait();  // launch.cuh: inputs of the previous kernel visible
  pdl_trigger();
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    store_any(out, dt, i, in[i]);
}

__global__ void zero_kernel(float* p, std::int64_t count) {
  pdl_wait();  // launch.cuh: inputs of the previous kernel visible
  pdl_trigger();
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    p[i] = 0.f;
}

// ---- SIMT GEMM (small / unaligned shapes, fp32 plans) ------------------------
// C[m,n] = op(A)[m,k] · op(B)[k,n], fp32 FFMA accumulation in k order.

constexpr int kTM = 64, kTN = 64, kTK = 16;

__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmArgs a) {
  pdl_wait();  // launch.cuh: inputs of the previous kernel visible
  pdl_trigger();
  __shared__ float As[kTK][kTM + 4];
  __shared__ float Bs[kTK][kTN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const std::int64_t m0 = static_cast<std::int64_t>(blockIdx.y) * kTM;
  const std::int64_t n0 = static_cast<std::int64_t>(blockIdx.x) * kTN;
  float acc[4][4] = {};
  // A element (i, kk): ta ? A[kk, i] (A stored [k, m]) : A[i, kk] (stored [m, k])
  for (std::int64_t k0 = 0; k0 < a.k; k0 += kTK) {
    for (int e = threadIdx.x; e < kTK * kTM; e += 256) {
      int kk, ii;
      if (a.ta) {
        ii = e % kTM;
        kk = e / kTM;
      } else {
        kk = e % kTK;
        ii = e / kTK;
      }
      std::int64_t gi = m0 + ii, gk = k0 + kk;
      float v = 0.f;
      if (gi < a.m && gk < a.k) v = load_any(a.A, a.da, a.ta ? gk * a.m + gi : gi * a.k + gk);
      As[kk][ii] = v;
    }
    // B element (kk, j): tb ? B[j, kk] (stored [n, k]) : B[kk, j] (stored [k, n])
    for (int e = threadIdx.x; e < kTK * kTN; e += 256) {
      int kk, jj;
      if (a.tb) {
        kk = e % kTK;
        jj = e / kTK;
      } else {
        jj = e % kTN;
        kk = e / kTN;
      }
      std::int64_t gj = n0 + jj, gk = k0 + kk;
      float v = 0.f;
      if (gj < a.n && gk < a.k) v = load_any(a.B, a.db, a.tb ? gj * a.k + gk : gk * a.n + gj);
      Bs[kk][jj] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kTK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    std::int64_t gi = m0 + ty * 4 + i;
    if (gi >= a.m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      std::int64_t gj = n0 + tx * 4 + j;
      if (gj < a.n) store_any(a.C, a.dc, gi * a.n + gj, acc[i][j]);
    }
  }
}

}  // namespace

void launch_box(int dtype, const DevCell* cells, const DevTerm* terms, const DevChunk* chunks, int nchunks, int vec,
                int max_rank, cudaStream_t s) {
  if (nchunks == 0) return;
  switch (dtype) {
    case DT_F32: box_dispatch<float>(cells, terms, chunks, nchunks, vec, max_rank, s); break;
    case DT_BF16: box_dispatch<__nv_bfloat16>(cells, terms, chunks, nchunks, vec, max_rank, s); break;
    case DT_I32: box_dispatch<int>(cells, terms, chunks, nchunks, vec, max_rank, s); break;
    default: throw std::runtime_error("box: bad dtype");
  }
  check_launch("box_kernel");
}

void launch_ew(int op, int dtype, const void* const* ins, int nin, void* out, std::int64_t count, cudaStream_t s) {
  if (nin > kMaxEwIn) throw std::runtime_error("ew: too many inputs per launch");
  if (count == 0) return;
#define PLANC_EW(T)                                                       \
  switch (op) {                                                           \
    case 0: ew_typed<T, 0>(ins, nin, out, count, s); break;               \
    case 1: ew_typed<T, 1>(ins, nin, out, count, s); break;               \
    default: ew_typed<T, 2>(ins, nin, out, count, s); break;              \
  }
  if (dtype == DT_F32) {
    PLANC_EW(float)
  } else if (dtype == DT_BF16) {
    PLANC_EW(__nv_bfloat16)
  } else {
    throw std::runtime_error("ew: unsupported dtype");
  }
#undef PLANC_EW
  check_launch("ew_kernel");
}

namespace {
bool aligned16(const void* p) { return reinterpret_cast<std::uintptr_t>(p) % 16 == 0; }

// Axis splits of a column reduction: one full wave of resident blocks
// (occupancy x SMs — a second, partial wave doubled the kernel's time:
// 512 blocks on 444 slots measured 61 us for 134 MB), at least 128 rows per
// split (the finishing pass reads S partials per column).
int reduce_resident_blocks(int vec) {
  static int cached[2] = {0, 0};
  int& c = cached[vec > 4 ? 1 : 0];
  if (c == 0) {
    int per_sm = 0;
    const cudaError_t e =
        vec > 4 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reduce_cols_kernel<__nv_bfloat16, 8>,
                                                                kRedWarps * 32, 0)
                : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reduce_cols_kernel<float, 4>, kRedWarps * 32, 0);
    if (e != cudaSuccess || per_sm <= 0) {
      (void)cudaGetLastError();
      per_sm = 3;
    }
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    c = per_sm * std::max(sms, 1);
  }
  return c;
}

int reduce_splits(std::int64_t outer, std::int64_t axis_len, std::int64_t inner, int vec) {
  const std::int64_t tiles = outer * ((inner + 32 * vec * kRedCV - 1) / (32 * vec * kRedCV));
  std::int64_t S = std::max<std::int64_t>(1, reduce_resident_blocks(vec) / tiles);
  S = std::min<std::int64_t>(S, std::max<std::int64_t>(1, axis_len / 128));
  return static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(S, 1024)));
}

template <typename T>
void reduce_typed(const void* in_, void* out_, void* scratch, std::int64_t outer, std::int64_t axis_len,
                  std::int64_t inner, cudaStream_t s) {
  constexpr int VV = 16 / sizeof(T);
  const T* in = static_cast<const T*>(in_);
  T* out = static_cast<T*>(out_);
  if (inner == 1) {
    if (aligned16(in) && axis_len % VV == 0)
      pdl_launch("reduce_rows_kernel", reduce_rows_kernel<T, VV>, dim3(grid_for(outer * 32, 256)), dim3(256), 0, s, in,
                 out, outer, axis_len);
    else
      pdl_launch("reduce_rows_kernel", reduce_rows_kernel<T, 1>, dim3(grid_for(outer * 32, 256)), dim3(256), 0, s, in,
                 out, outer, axis_len);
    return;
  }
  const bool vec = aligned16(in) && inner % VV == 0;
  const int v = vec ? VV : 1;
  const int S = scratch ? reduce_splits(outer, axis_len, inner, v) : 1;
  if (outer > 65535) throw std::runtime_error("reduce: more than 65535 outer rows with a column reduction");
  dim3 grid(static_cast<unsigned>((inner + 32 * v * kRedCV - 1) / (32 * v * kRedCV)), static_cast<unsigned>(outer),
            static_cast<unsigned>(S));
  float* part = static_cast<float*>(scratch);
  if (vec)
    pdl_launch("reduce_cols_kernel", reduce_cols_kernel<T, VV>, grid, dim3(kRedWarps * 32), 0, s, in, out, part,
               outer, axis_len, inner);
  else
    pdl_launch("reduce_cols_kernel", reduce_cols_kernel<T, 1>, grid, dim3(kRedWarps * 32), 0, s, in, out, part, outer,
               axis_len, inner);
  if (S > 1)
    pdl_launch("reduce_cols_finish", reduce_cols_finish<T>, dim3(grid_for(outer * inner, 256)), dim3(256), 0, s,
               static_cast<const float*>(part), out, outer, S, inner);
}
}  // namespace

std::int64_t reduce_scratch_bytes(std::int64_t outer, std::int64_t axis_len, std::int64_t inner, int dtype) {
  if (inner == 1) return 0;
  const int v = dtype == DT_BF16 ? 8 : 4;
  const int S = reduce_splits(outer, axis_len, inner, v);
  return S > 1 ? static_cast<std::int64_t>(S) * outer * inner * 4 : 0;
}

int reduce_launches(std::int64_t outer, std::int64_t axis_len, std::int64_t inner, int dtype) {
  return reduce_scratch_bytes(outer, axis_len, inner, dtype) > 0 ? 2 : 1;
}

void launch_reduce(int dtype, const void* in, void* out, void* scratch, std::int64_t outer, std::int64_t axis_len,
                   std::int64_t inner, cudaStream_t s) {
  if (dtype == DT_F32) reduce_typed<float>(in, out, scratch, outer, axis_len, inner, s);
  else if (dtype == DT_BF16) reduce_typed<__nv_bfloat16>(in, out, scratch, outer, axis_len, inner, s);
  else throw std::runtime_error("reduce: unsupported dtype");
  check_launch("reduce_kernel");
}

void launch_emb_lookup(int dtype, const int* idx, const void* table, void* out, std::int64_t n, std::int64_t rows,
                       std::int64_t h, std::int64_t lo, cudaStream_t s) {
  int g = grid_for(n * 32, 256);
  const bool vec = aligned16(table) && aligned16(out);
  if (dtype == DT_F32) {
    const float* t = static_cast<const float*>(table);
    float* o = static_cast<float*>(out);
    if (vec && h % 4 == 0)
      pdl_launch("emb_lookup_kernel", emb_lookup_kernel<float, 4>, dim3(g), dim3(256), 0, s, idx, t, o, n, rows, h, lo);
    else
      pdl_launch("emb_lookup_kernel", emb_lookup_kernel<float, 1>, dim3(g), dim3(256), 0, s, idx, t, o, n, rows, h, lo);
  } else if (dtype == DT_BF16) {
    using B = __nv_bfloat16;
    const B* t = static_cast<const B*>(table);
    B* o = static_cast<B*>(out);
    if (vec && h % 8 == 0)
      pdl_launch("emb_lookup_kernel", emb_lookup_kernel<B, 8>, dim3(g), dim3(256), 0, s, idx, t, o, n, rows, h, lo);
    else
      pdl_launch("emb_lookup_kernel", emb_lookup_kernel<B, 1>, dim3(g), dim3(256), 0, s, idx, t, o, n, rows, h, lo);
  } else {
    throw std::runtime_error("embedding: unsupported dtype");
  }
  check_launch("emb_lookup_kernel");
}

std::int64_t emb_grad_scratch_bytes(std::int64_t n, std::int64_t h) {
  const std::int64_t nb = (n + kEmbBlock - 1) / kEmbBlock;
  return nb * kEmbBlock * h * 4 + nb * kEmbBlock * 4 + nb * 4 + 256;
}

void launch_emb_grad(int dtype, const int* idx, const void* gout, void* out, void* scratch, std::int64_t n,
                     std::int64_t rows, std::int64_t h, std::int64_t lo, cudaStream_t s) {
  if (dtype != DT_F32 && dtype != DT_BF16) throw std::runtime_error("embedding-grad: unsupported dtype");
  const std::int64_t nb = (n + kEmbBlock - 1) / kEmbBlock;
  float* partial = static_cast<float*>(scratch);
  int* seg_row = reinterpret_cast<int*>(partial + nb * kEmbBlock * h);
  int* nseg = seg_row + nb * kEmbBlock;
  if (nb > 0) {
    if (dtype == DT_F32)
      pdl_launch("emb_grad_block_kernel", emb_grad_block_kernel<float>, dim3(static_cast<unsigned>(nb)), dim3(512), 0, s,
                 idx, static_cast<const float*>(gout), partial, seg_row, nseg, n, rows, h, lo);
    else
      pdl_launch("emb_grad_block_kernel", emb_grad_block_kernel<__nv_bfloat16>, dim3(static_cast<unsigned>(nb)),
                 dim3(512), 0, s, idx, static_cast<const __nv_bfloat16*>(gout), partial, seg_row, nseg, n, rows, h, lo);
  }
  const int g = grid_for(rows * 32, 256);
  if (dtype == DT_F32)
    pdl_launch("emb_grad_combine_kernel", emb_grad_combine_kernel<float>, dim3(g), dim3(256), 0, s, partial, seg_row,
               nseg, static_cast<float*>(out), static_cast<int>(nb), rows, h);
  else
    pdl_launch("emb_grad_combine_kernel", emb_grad_combine_kernel<__nv_bfloat16>, dim3(g), dim3(256), 0, s, partial,
               seg_row, nseg, static_cast<__nv_bfloat16*>(out), static_cast<int>(nb), rows, h);
  check_launch("emb_grad_kernel");
}

void launch_gemm_simt(const GemmArgs& a, cudaStream_t s) {
  if (a.m == 0 || a.n == 0) return;
  if (a.k == 0) {
    // Empty contraction: C = 0.
    std::int64_t cnt = a.m * a.n;
    if (a.dc == DT_F32) {
      pdl_launch("zero_kernel", zero_kernel, dim3(grid_for(cnt, 256)), dim3(256), 0, s, static_cast<float*>(a.C), cnt);
    } else {
      cudaMemsetAsync(a.C, 0, cnt * 2, s);
    }
    check_launch("gemm_zero");
    return;
  }
  dim3 grid(static_cast<unsigned>((a.n + kTN - 1) / kTN), static_cast<unsigned>((a.m + kTM - 1) / kTM));
  pdl_launch("gemm_simt_kernel", gemm_simt_kernel, dim3(grid), dim3(256), 0, s, a);
  check_launch("gemm_simt_kernel");
}

void launch_convert(int dtype_out, void* out, const float* in, std::int64_t count, cudaStream_t s) {
  pdl_launch("convert_kernel", convert_kernel, dim3(grid_for(count, 256)), dim3(256), 0, s, dtype_out, out, in, count);
  check_launch("convert_kernel");
}

void launch_fill_zero_f32(float* p, std::int64_t count, cudaStream_t s) {
  pdl_launch("zero_kernel", zero_kernel, dim3(grid_for(count, 256)), dim3(256), 0, s, p, count);
  check_launch("zero_kernel");
}

namespace {

// ---- schema extension: row-wise sub-operators and GELU ----------------------
// One warp per segment; every lane walks the segment in 16-byte vectors
// (V elements) with fp32 statistics merged by warp shuffles, then a second
// (and, for layernorm-grad, third) pass re-reads the segment — from L1/L2,
// the segment being a few KB — and writes. HBM traffic: inputs once, output
// once.

constexpr int kRowWarps = 8;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T, int OP, int V>
__global__ void __launch_bounds__(kRowWarps * 32) row_kernel(const T* __restrict__ a, const T* __restrict__ b,
                                                             T* __restrict__ out, long long nseg, int seg, float eps) {
  pdl_wait();  // launch.cuh: inputs of the previous kernel visible
  pdl_trigger();
  const int lane = threadIdx.x % 32;
  const long long sidx = blockIdx.x * static_cast<long long>(kRowWarps) + threadIdx.x / 32;
  if (sidx >= nseg) return;
  const long long base = sidx * seg;
  const T* x = a + base;
  const T* dy = b ? b + base : nullptr;
  T* o = out + base;
  const int nv = seg / V;  // vectors per segment
  float xv[V], gv[V], ov[V];
  if constexpr (OP == 0) {  // softmax: online max / sum, then write
    float m = -INFINITY, sm = 0.f;
    for (int i = lane; i < nv; i += 32) {
      load_vec<T, V>(x + i * V, xv);
#pragma unroll
      for (int e = 0; e < V; ++e) {
        if (xv[e] > m) {
          sm = sm * expf(m - xv[e]) + 1.f;
          m = xv[e];
        } else {
          sm += expf(xv[e] - m);
        }
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, off), s2 = __shfl_xor_sync(0xffffffffu, sm, off);
      const float mm = fmaxf(m, m2);
      sm = (sm > 0.f ? sm * expf(m - mm) : 0.f) + (s2 > 0.f ? s2 * expf(m2 - mm) : 0.f);
      m = mm;
    }
    const float inv = __fdividef(1.f, sm);
    for (int i = lane; i < nv; i += 32) {
      load_vec<T, V>(x + i * V, xv);
#pragma unroll
      for (int e = 0; e < V; ++e) ov[e] = expf(xv[e] - m) * inv;
      store_vec<T, V>(o + i * V, ov);
    }
  } else if constexpr (OP == 1) {  // softmax-grad: dx = y * (dy - sum(dy * y))
    float dot = 0.f;
    for (int i = lane; i < nv; i += 32) {
      load_vec<T, V>(x + i * V, xv);
      load_vec<T, V>(dy + i * V, gv);
#pragma unroll
      for (int e = 0; e < V; ++e) dot += xv[e] * gv[e];
    }
    dot = warp_sum(dot);
    for (int i = lane; i < nv; i += 32) {
      load_vec<T, V>(x + i * V, xv);
      load_vec<T, V>(dy + i * V, gv);
#pragma unroll
      for (int e = 0; e < V; ++e) ov[e] = xv[e] * (gv[e] - dot);
      store_vec<T, V>(o + i * V, ov);
    }
  } else {  // layernorm / layernorm-grad: Welford statistics (Chan merge across lanes)
    float cnt = 0.f, mean = 0.f, m2 = 0.f;
    for (int i = lane; i < nv; i += 32) {
      load_vec<T, V>(x + i * V, xv);
#pragma unroll
      for (int e = 0; e < V; ++e) {
        cnt += 1.f;
        const float d = xv[e] - mean;
        mean += d * __fdividef(1.f, cnt);
        m2 += d * (xv[e] - mean);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float c2 = __shfl_xor_sync(0xffffffffu, cnt, off), mn2 = __shfl_xor_sync(0xffffffffu, mean, off),
                  q2 = __shfl_xor_sync(0xffffffffu, m2, off);
      const float c = cnt + c2;
      if (c > 0.f) {
        const float d = mn2 - mean;
        mean += d * (c2 * __fdividef(1.f, c));
        m2 += q2 + d * d * (cnt * c2 * __fdividef(1.f, c));
      }
      cnt = c;
    }
    const float rstd = rsqrtf(m2 * __fdividef(1.f, static_cast<float>(seg)) + eps);
    if constexpr (OP == 2) {
      for (int i = lane; i < nv; i += 32) {
        load_vec<T, V>(x + i * V, xv);
#pragma unroll
        for (int e = 0; e < V; ++e) ov[e] = (xv[e] - mean) * rstd;
        store_vec<T, V>(o + i * V, ov);
      }
    } else {  // dx = rstd * (dy - mean(dy) - xhat * mean(dy * xhat))
      float sdy = 0.f, sdx = 0.f;
      for (int i = lane; i < nv; i += 32) {
        load_vec<T, V>(x + i * V, xv);
        load_vec<T, V>(dy + i * V, gv);
#pragma unroll
        for (int e = 0; e < V; ++e) {
          sdy += gv[e];
          sdx += gv[e] * (xv[e] - mean) * rstd;
        }
      }
      const float inv_n = __fdividef(1.f, static_cast<float>(seg));
      const float mdy = warp_sum(sdy) * inv_n, mdx = warp_sum(sdx) * inv_n;
      for (int i = lane; i < nv; i += 32) {
        load_vec<T, V>(x + i * V, xv);
        load_vec<T, V>(dy + i * V, gv);
#pragma unroll
        for (int e = 0; e < V; ++e) ov[e] = rstd * (gv[e] - mdy - (xv[e] - mean) * rstd * mdx);
        store_vec<T, V>(o + i * V, ov);
      }
    }
  }
}

// Register-resident variant: a segment of seg = LPS x R x V elements or
// fewer lives in the registers of an LPS-lane group (32 / LPS segments per
// warp): ONE global read per operand, exact two-pass statistics from
// registers, group-local shuffles. Taken whenever R <= 16 (softmax heads of
// 128, LayerNorm rows of 2048 bf16).
template <int LPS>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = LPS / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <int LPS>
__device__ __forceinline__ float group_max(float v) {
#pragma unroll
  for (int o = LPS / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <typename T, int OP, int V, int LPS, int R>
__global__ void __launch_bounds__(kRowWarps * 32) row_reg_kernel(const T* __restrict__ a, const T* __restrict__ b,
                                                                 T* __restrict__ out, long long nseg, int seg,
                                                                 float eps) {
  pdl_wait();  // launch.cuh: inputs of the previous kernel visible
  pdl_trigger();
  constexpr int G = 32 / LPS;  // segments per warp
  const int lane = threadIdx.x % 32, j = lane % LPS;
  const long long sidx = (blockIdx.x * static_cast<long long>(kRowWarps) + threadIdx.x / 32) * G + lane / LPS;
  const bool live_seg = sidx < nseg;  // whole groups retire together; shuffles stay warp-wide
  const int nv = seg / V;
  const long long base = (live_seg ? sidx : 0) * seg;
  float x[R][V], g[R][V];
  {
    uint4 ra[R], rb[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int vi = j + r * LPS;
      ra[r] = rb[r] = make_uint4(0, 0, 0, 0);
      if (live_seg && vi < nv) {
        ra[r] = ld16(a + base + vi * V);
        if constexpr (OP == 1 || OP == 3) rb[r] = ld16(b + base + vi * V);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      unpack16<T, V>(ra[r], x[r]);
      unpack16<T, V>(rb[r], g[r]);
    }
  }
  auto valid = [&](int r) { return live_seg && j + r * LPS < nv; };
  const float inv_n = __fdividef(1.f, static_cast<float>(seg));
  if constexpr (OP == 0) {  // softmax
    float m = -INFINITY;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (valid(r))
#pragma unroll
        for (int e = 0; e < V; ++e) m = fmaxf(m, x[r][e]);
    m = group_max<LPS>(m);
    float sm = 0.f;
    const float ml = m * 1.4426950408889634f;  // exp(x - m) = 2^(x log2 e - m log2 e)
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int e = 0; e < V; ++e) {
        x[r][e] = valid(r) ? ex2_ftz(fmaf(x[r][e], 1.4426950408889634f, -ml)) : 0.f;
        sm += x[r][e];
      }
    const float inv = __fdividef(1.f, group_sum<LPS>(sm));
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int e = 0; e < V; ++e) x[r][e] *= inv;
  } else if constexpr (OP == 1) {  // softmax-grad
    float dot = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int e = 0; e < V; ++e) dot += x[r][e] * g[r][e];
    dot = group_sum<LPS>(dot);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int e = 0; e < V; ++e) x[r][e] = x[r][e] * (g[r][e] - dot);
  } else {  // layernorm / layernorm-grad: two-pass mean / variance from registers
    float sx = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int e = 0; e < V; ++e) sx += x[r][e];
    const float mean = group_sum<LPS>(sx) * inv_n;
    float sq = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (valid(r))
#pragma unroll
        for (int e = 0; e < V; ++e) sq += (x[r][e] - mean) * (x[r][e] - mean);
    const float rstd = rsqrtf(group_sum<LPS>(sq) * inv_n + eps);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int e = 0; e < V; ++e) x[r][e] = (x[r][e] - mean) * rstd;  // xhat
    if constexpr (OP == 3) {
      float sdy = 0.f, sdx = 0.f;
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int e = 0; e < V; ++e) {
          sdy += g[r][e];
          sdx += g[r][e] * x[r][e];
        }
      const float mdy = group_sum<LPS>(sdy) * inv_n, mdx = group_sum<LPS>(sdx) * inv_n;
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int e = 0; e < V; ++e) x[r][e] = rstd * (g[r][e] - mdy - x[r][e] * mdx);
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (valid(r)) store_vec<T, V>(out + base + (j + r * LPS) * V, x[r]);
}

// Wide segments (more than one warp's registers hold): one CTA per segment,
// every thread R vectors of the segment in registers — one global read per
// operand, exact two-pass statistics, CTA-wide reductions through shared
// memory in warp order (the same bits every run).
template <bool MAX>
__device__ __forceinline__ float cta_reduce(float v, float* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float w = __shfl_xor_sync(0xffffffffu, v, o);
    v = MAX ? fmaxf(v, w) : v + w;
  }
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  __syncthreads();  // the previous reduction's readers are done with sh
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  float r = MAX ? -INFINITY : 0.f;
  for (int w = 0; w < nw; ++w) r = MAX ? fmaxf(r, sh[w]) : r + sh[w];
  return r;
}

template <typename T, int OP, int V, int R>
__global__ void __launch_bounds__(512) row_cta_kernel(const T* __restrict__ a, const T* __restrict__ b,
                                                       T* __restrict__ out, int seg, float eps) {
  pdl_wait();  // launch.cuh: inputs of the previous kernel visible
  pdl_trigger();
  __shared__ float sh[32];
  const int nv = seg / V;
  const long long base = static_cast<long long>(blockIdx.x) * seg;
  float x[R][V], g[R][V];
  {
    uint4 ra[R], rb[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int vi = threadIdx.x + r * blockDim.x;
      ra[r] = rb[r] = make_uint4(0, 0, 0, 0);
      if (vi < nv) {
        ra[r] = ld16(a + base + vi * V);
        if constexpr (OP == 1 || OP == 3) rb[r] = ld16(b + base + vi * V);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      unpack16<T, V>(ra[r], x[r]);
      unpack16<T, V>(rb[r], g[r]);
    }
  }
  auto valid = [&](int r) { return static_cast<int>(threadIdx.x + r * blockDim.x) < nv; };
  const float inv_n = __fdividef(1.f, static_cast<float>(seg));
  if constexpr (OP == 0) {  // softmax
    float m = -INFINITY;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (valid(r))
#pragma unroll
        for (int e = 0; e < V; ++e) m = fmaxf(m, x[r][e]);
    m = cta_reduce<true>(m, sh);
    float sm = 0.f;
    const float ml = m * 1.4426950408889634f;  // exp(x - m) = 2^(x log2 e - m log2 e)
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int e = 0; e < V; ++e) {
        x[r][e] = valid(r) ? ex2_ftz(fmaf(x[r][e], 1.4426950408889634f, -ml)) : 0.f;
        sm += x[r][e];
      }
    const float inv = __fdividef(1.f, cta_reduce<false>(sm, sh));
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int e = 0; e < V; ++e) x[r][e] *= inv;
  } else if constexpr (OP == 1) {  // softmax-grad
    float dot = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int e = 0; e < V; ++e) dot += x[r][e] * g[r][e];
    dot = cta_reduce<false>(dot, sh);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int e = 0; e < V; ++e) x[r][e] = x[r][e] * (g[r][e] - dot);
  } else {  // layernorm / layernorm-grad
    float sx = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int e = 0; e < V; ++e) sx += x[r][e];
    const float mean = cta_reduce<false>(sx, sh) * inv_n;
    float sq = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (valid(r))
#pragma unroll
        for (int e = 0; e < V; ++e) sq += (x[r][e] - mean) * (x[r][e] - mean);
    const float rstd = rsqrtf(cta_reduce<false>(sq, sh) * inv_n + eps);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int e = 0; e < V; ++e) x[r][e] = (x[r][e] - mean) * rstd;
    if constexpr (OP == 3) {
      float sdy = 0.f, sdx = 0.f;
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int e = 0; e < V; ++e) {
          sdy += g[r][e];
          sdx += g[r][e] * x[r][e];
        }
      const float mdy = cta_reduce<false>(sdy, sh) * inv_n, mdx = cta_reduce<false>(sdx, sh) * inv_n;
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int e = 0; e < V; ++e) x[r][e] = rstd * (g[r][e] - mdy - x[r][e] * mdx);
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (valid(r)) store_vec<T, V>(out + base + (threadIdx.x + r * blockDim.x) * V, x[r]);
}

template <typename T, int OP, int V>
__global__ void __launch_bounds__(256) act_kernel(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out,
                                                  long long count) {
  pdl_wait();  // launch.cuh: inputs of the previous kernel visible
  pdl_trigger();
  const long long nvec = count / V;
  float xv[V], gv[V], ov[V];
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < nvec;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    load_vec<T, V>(a + i * V, xv);
    if constexpr (OP == 5) load_vec<T, V>(b + i * V, gv);
#pragma unroll
    for (int e = 0; e < V; ++e) ov[e] = OP == 4 ? gelu_f(xv[e]) : gelu_grad_f(xv[e], OP == 5 ? gv[e] : 0.f);
    store_vec<T, V>(out + i * V, ov);
  }
  // scalar tail (count % V elements)
  const long long t = nvec * V + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x < count - nvec * V) {
    const float x0 = to_acc<T>(a[t]);
    out[t] = from_acc<T>(OP == 4 ? gelu_f(x0) : gelu_grad_f(x0, OP == 5 ? to_acc<T>(b[t]) : 0.f));
  }
}

template <typename T>
void rowwise_typed(int op, const void* a, const void* b, void* out, std::int64_t count, std::int64_t seg, float eps,
                   cudaStream_t s) {
  constexpr int VV = 16 / sizeof(T);
  const T* A = static_cast<const T*>(a);
  const T* B = static_cast<const T*>(b);
  T* O = static_cast<T*>(out);
  if (op == 4 || op == 5) {
    const long long nvec = count / VV;
    const dim3 g(grid_for(std::max<long long>(nvec, 1), 256 * 4));
    if (op == 4) pdl_launch("act_kernel", act_kernel<T, 4, VV>, g, dim3(256), 0, s, A, B, O, (long long)count);
    else pdl_launch("act_kernel", act_kernel<T, 5, VV>, g, dim3(256), 0, s, A, B, O, (long long)count);
    return;
  }
  if (seg <= 0 || count % seg != 0 || seg > (1 << 30)) throw std::runtime_error("rowwise: bad segment");
  const long long nseg = count / seg;
  const dim3 g(static_cast<unsigned>((nseg + kRowWarps - 1) / kRowWarps));
  const dim3 blk(kRowWarps * 32);
  const int sg = static_cast<int>(seg);
  const bool vec = seg % VV == 0;
  // Register-resident path: LPS lanes (power of two) x R vectors per segment.
  if (vec) {
    const long long nv = seg / VV;
    int lps = 1;
    while (lps < 32 && lps < nv) lps <<= 1;
    const long long r = (nv + lps - 1) / lps;
    if (r <= 64 / VV) {  // <= 64 fp32 registers per operand per lane
      const int R = r <= 1 ? 1 : r <= 2 ? 2 : r <= 4 ? 4 : r <= 8 ? 8 : 16;
      const long long per_block = static_cast<long long>(kRowWarps) * (32 / lps);
      const dim3 gr(static_cast<unsigned>((nseg + per_block - 1) / per_block));
#define PLANC_RR(OPV, L, RR)                                                                                       \
  return pdl_launch("row_reg_kernel", row_reg_kernel<T, OPV, VV, L, RR>, gr, blk, 0, s, A, B, O, nseg, sg, eps)
#define PLANC_RR_R(OPV, L)       \
  switch (R) {                   \
    case 1: PLANC_RR(OPV, L, 1); \
    case 2: PLANC_RR(OPV, L, 2); \
    case 4: PLANC_RR(OPV, L, 4); \
    case 8: PLANC_RR(OPV, L, 8); \
    default: PLANC_RR(OPV, L, (VV == 4 ? 16 : 8)); \
  }
#define PLANC_RR_L(OPV)                 \
  switch (lps) {                        \
    case 1: PLANC_RR(OPV, 1, 1);        \
    case 2: PLANC_RR(OPV, 2, 1);        \
    case 4: PLANC_RR(OPV, 4, 1);        \
    case 8: PLANC_RR(OPV, 8, 1);        \
    case 16: PLANC_RR(OPV, 16, 1);      \
    default: PLANC_RR_R(OPV, 32);       \
  }
      switch (op) {
        case 0: PLANC_RR_L(0);
        case 1: PLANC_RR_L(1);
        case 2: PLANC_RR_L(2);
        default: PLANC_RR_L(3);
      }
#undef PLANC_RR_L
#undef PLANC_RR_R
#undef PLANC_RR
    }
  }
  // CTA-per-segment path: up to 512 threads x R vectors (R = 8 only for the
  // one-operand kinds: two operands of 8 vectors would spill).
  if (vec && nseg <= 0x7fffffffLL) {
    const long long nv = seg / VV;
    const int R = nv <= 4 * 512 ? 4 : (nv <= 8 * 512 && (op == 0 || op == 2)) ? 8 : 0;
    if (R) {
      const long long th = std::max<long long>(64, ((nv + R - 1) / R + 31) / 32 * 32);
      const dim3 gc(static_cast<unsigned>(nseg)), bc(static_cast<unsigned>(th));
#define PLANC_RC(OPV, RR) \
  return pdl_launch("row_cta_kernel", row_cta_kernel<T, OPV, VV, RR>, gc, bc, 0, s, A, B, O, sg, eps)
      switch (op) {
        case 0: if (R == 4) PLANC_RC(0, 4); else PLANC_RC(0, 8);
        case 1: PLANC_RC(1, 4);
        case 2: if (R == 4) PLANC_RC(2, 4); else PLANC_RC(2, 8);
        default: PLANC_RC(3, 4);
      }
#undef PLANC_RC
    }
  }
#define PLANC_ROW(OPV, V) pdl_launch("row_kernel", row_kernel<T, OPV, V>, g, blk, 0, s, A, B, O, nseg, sg, eps)
  switch (op) {
    case 0: if (vec) PLANC_ROW(0, VV); else PLANC_ROW(0, 1); break;
    case 1: if (vec) PLANC_ROW(1, VV); else PLANC_ROW(1, 1); break;
    case 2: if (vec) PLANC_ROW(2, VV); else PLANC_ROW(2, 1); break;
    default: if (vec) PLANC_ROW(3, VV); else PLANC_ROW(3, 1); break;
  }
#undef PLANC_ROW
}

}  // namespace

void launch_rowwise(int op, int dtype, const void* a, const void* b, void* out, std::int64_t count, std::int64_t seg,
                    float eps, cudaStream_t s) {
  if (count == 0) return;
  if (dtype == DT_BF16) rowwise_typed<__nv_bfloat16>(op, a, b, out, count, seg, eps, s);
  else if (dtype == DT_F32) rowwise_typed<float>(op, a, b, out, count, seg, eps, s);
  else throw std::runtime_error("rowwise: element type must be fp32 or bf16");
}

__global__ void __launch_bounds__(256) copy_bytes_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                                         long long nvec, unsigned char* __restrict__ dtail,
                                                         const unsigned char* __restrict__ stail, int tail) {
  pdl_wait();  // launch.cuh: inputs of the previous kernel visible
  pdl_trigger();
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < nvec; i += stride)
    dst[i] = __ldcs(src + i);
  if (blockIdx.x == 0 && static_cast<int>(threadIdx.x) < tail) dtail[threadIdx.x] = stail[threadIdx.x];
}

void launch_copy_bytes(void* dst, const void* src, std::int64_t bytes, cudaStream_t s) {
  if (bytes <= 0) return;
  if ((reinterpret_cast<std::uintptr_t>(dst) | reinterpret_cast<std::uintptr_t>(src)) % 16 != 0) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) throw std::runtime_error(std::string("copy: ") + cudaGetErrorString(e));
    return;
  }
  const long long nvec = bytes / 16;
  const int tail = static_cast<int>(bytes - nvec * 16);
  pdl_launch("copy_bytes_kernel", copy_bytes_kernel, dim3(grid_for(std::max<long long>(nvec, 1), 256 * 4)), dim3(256),
             0, s, static_cast<uint4*>(dst), static_cast<const uint4*>(src), nvec,
             static_cast<unsigned char*>(dst) + nvec * 16, static_cast<const unsigned char*>(src) + nvec * 16, tail);
}

// ---- peer-memory flags ------------------------------------------------------

__global__ void peer_epoch_kernel(unsigned* epoch) {
  pdl_wait();
  pdl_trigger();
  *epoch += 1u;
}

__global__ void peer_flags_kernel(const unsigned* epoch, PeerFlags f, unsigned long long timeout_ns, unsigned* err) {
  pdl_wait();  // launch.cuh: inputs of the previous kernel visible
  // No early pdl_trigger here: a dependent launched while this kernel spins
  // (e.g. a persistent GEMM holding every SM's shared memory in
  // griddepcontrol.wait) could starve the streams whose progress the awaited
  // peers depend on. Dependents start when the wait is over (kernel exit).
  const unsigned e = *reinterpret_cast<const volatile unsigned*>(epoch);
  const int t = threadIdx.x;
  if (t < f.n_sig) {
    // Everything this stream wrote before this kernel is visible at system
    // scope to whoever acquires the flag.
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f.sig[t]), "r"(e) : "memory");
  }
  if (t < f.n_wait) {
    unsigned long long t0, now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      unsigned v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f.wait[t]) : "memory");
      if (static_cast<int>(v - e) >= 0) break;  // wrap-safe v >= e
      __nanosleep(256);
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > timeout_ns) {
        // err[0] code, [1] value seen, [2] epoch awaited, [3..4] flag address
        if (err && atomicCAS(err, 0u, f.code) == 0u) {
          const unsigned long long a = reinterpret_cast<unsigned long long>(f.wait[t]);
          err[1] = v;
          err[2] = e;
          err[3] = static_cast<unsigned>(a);
          err[4] = static_cast<unsigned>(a >> 32);
        }
        __threadfence_system();
        __trap();
      }
    }
  }
}

void launch_peer_epoch(unsigned* epoch, cudaStream_t s) {
  pdl_launch("peer_epoch_kernel", peer_epoch_kernel, dim3(1), dim3(1), 0, s, epoch);
  check_launch("peer_epoch_kernel");
}

void launch_peer_flags(const unsigned* epoch, const PeerFlags& f, unsigned long long timeout_ns, unsigned* err,
                       cudaStream_t s) {
  pdl_launch("peer_flags_kernel", peer_flags_kernel, dim3(1), dim3(32), 0, s, epoch, f, timeout_ns, err);
  check_launch("peer_flags_kernel");
}

// Host gate (profiling): holds a stream until the host sets *flag, so the
// instruction enqueued behind it starts right after the preceding event
// record instead of after the host's launch latency — per-instruction event
// times then measure the kernels, not the enqueue. Gives up after 2 s.
namespace {
__global__ void host_gate_kernel(const volatile unsigned* flag) {
  std::uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*flag == 0) {
    std::uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 2000000000ull) break;
    __nanosleep(200);
  }
}
}  // namespace

void launch_host_gate(const unsigned* flag, cudaStream_t s) {
  host_gate_kernel<<<1, 32, 0, s>>>(flag);
  check_launch("host_gate_kernel");
}

}  // namespace planc_b200
