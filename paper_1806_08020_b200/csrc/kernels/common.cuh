#pragma once
// Shared device helpers: streaming loads, warp sums and the deterministic
// two-stage grid reduction used by every dot-product kernel.

#include <cuda_runtime.h>

#include <cstdint>

namespace ppa {
namespace kern {

/// Largest dynamic shared memory a launch of `kernel` may request: the
/// device's opt-in per-block limit minus the kernel's static shared memory.
template <typename K>
inline int max_dynamic_smem(K kernel) {
  int dev = 0, optin = 0;
  cudaFuncAttributes fa{};
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess ||
      cudaFuncGetAttributes(&fa, kernel) != cudaSuccess) {
    return 48 * 1024;
  }
  return optin - static_cast<int>(fa.sharedSizeBytes);
}

}  // namespace kern

namespace dev {

constexpr unsigned kFull = 0xffffffffu;

/// Butterfly warp sum: every lane ends with the same, order-fixed value
/// (fp addition is commutative, so the xor tree is lane-symmetric).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Matrix streams (values / column indices) are read exactly once per SpMV:
// bypass L1 and mark them evict-first in L2 so the gathered x vector stays
// resident (x is 33 MB at config 3, L2 is 126 MB).
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.f64 {%0,%1}, [%2];"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p));
  return r;
}
__device__ __forceinline__ int2 ld_stream(const int2* p) {
  int2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.s32 {%0,%1}, [%2];"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p));
  return r;
}
__device__ __forceinline__ double ld_stream(const double* p) {
  double r;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}

/// Deterministic grid reduction of NV per-thread values (entries j with
/// j < cnt or j >= NV - tail are live; the rest are skipped).
///
/// Stage 1: warp butterfly + fixed-order sum over warps -> one partial row
/// per block in `partials` (compacted width cnt + tail).
/// Stage 2: the last block to arrive (ticket) sums the rows in block order
/// (lane-strided, then butterfly) and leaves the totals in s_final[]
/// (compacted index).  Returns true only in that last block, after a
/// __syncthreads, so the caller can run its finalisation.
template <int NV, int T>
__device__ __forceinline__ bool grid_reduce(double (&v)[NV], int cnt, int tail,
                                            double* __restrict__ partials,
                                            unsigned int* ticket, double* s_final) {
  constexpr int W = T / 32;
  __shared__ double s_red[W][NV];
  __shared__ unsigned int s_last;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int width = cnt + tail;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    if (j < cnt || j >= NV - tail) {
      const double s = warp_sum(v[j]);
      if (lane == 0) s_red[warp][j] = s;
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < width; k += T) {
    const int j = k < cnt ? k : NV - tail + (k - cnt);
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < W; ++w) s += s_red[w][j];
    partials[static_cast<size_t>(blockIdx.x) * width + k] = s;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int t = atomicAdd(ticket, 1u);
    s_last = (t == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  for (int k = warp; k < width; k += W) {
    double s = 0.0;
    for (int b = lane; b < static_cast<int>(gridDim.x); b += 32) {
      s += __ldcg(partials + static_cast<size_t>(b) * width + k);
    }
    s = warp_sum(s);
    if (lane == 0) s_final[k] = s;
  }
  if (threadIdx.x == 0) *ticket = 0u;  // ready for the next launch on this stream
  __syncthreads();
  return true;
}

}  // namespace dev
}  // namespace ppa
