// Does an L2 persisting access-policy window keep the pi(A)v ping-pong pair
// (2 x 32.8 MB at config 3) on chip?  Times a copy chain and a 7-point
// gather chain with and without the window.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a l2_persist.cu -o /tmp/l2p
#include <cstdio>
#include <utility>
#include <cuda_runtime.h>

constexpr int N = 160;
constexpr int NN = N * N * N;

__global__ void k_copy(const double* __restrict__ x, double* __restrict__ y, int n) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) y[r] = x[r];
}

__global__ void k_stencil(const double* __restrict__ x, double* __restrict__ y, int n, double c0) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int off[7] = {-N * N, -N, -1, 0, 1, N, N * N};
  double xv[7];
#pragma unroll
  for (int j = 0; j < 7; ++j) xv[j] = __ldg(x + min(max(r + off[j], 0), n - 1));
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 7; ++j) s = __dadd_rn(s, __dmul_rn(j == 3 ? 6.0 : -1.0, xv[j]));
  y[r] = __dadd_rn(xv[3], __dmul_rn(c0, s));
}

template <typename F>
float timeit(cudaStream_t st, F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 4; ++i) f();
  cudaEventRecord(a, st);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / reps;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  printf("l2 %d MB, persistingL2CacheMaxSize %.1f MB, accessPolicyMaxWindowSize %.1f MB\n",
         p.l2CacheSize >> 20, p.persistingL2CacheMaxSize / 1048576.0,
         p.accessPolicyMaxWindowSize / 1048576.0);
  cudaStream_t st;
  cudaStreamCreate(&st);
  double* buf;
  const size_t bytes = 2ull * NN * 8;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  double *x = buf, *y = buf + NN;
  const int bs = 512, g = (NN + bs - 1) / bs;
  auto run = [&](const char* tag) {
    float tc = timeit(st, [&] { k_copy<<<g, bs, 0, st>>>(x, y, NN); std::swap(x, y); }, 200);
    float ts = timeit(st, [&] { k_stencil<<<g, bs, 0, st>>>(x, y, NN, 0.5); std::swap(x, y); }, 200);
    printf("%-34s copy %.2f us (%.0f GB/s)  stencil %.2f us\n", tag, tc, 16.0 * NN / tc / 1e3, ts);
  };
  run("no window");
  for (double frac : {0.25, 0.5, 0.75, 1.0}) {
    size_t lim = static_cast<size_t>(p.persistingL2CacheMaxSize * frac);
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, lim);
    size_t got = 0;
    cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize);
    for (double hr : {0.5, 1.0}) {
      cudaStreamAttrValue a{};
      a.accessPolicyWindow.base_ptr = buf;
      a.accessPolicyWindow.num_bytes = std::min(bytes, static_cast<size_t>(p.accessPolicyMaxWindowSize));
      double fit = static_cast<double>(got) / a.accessPolicyWindow.num_bytes;
      a.accessPolicyWindow.hitRatio = static_cast<float>(hr * (fit < 1 ? fit : 1.0));
      a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a);
      char tag[96];
      snprintf(tag, sizeof tag, "persist %.0f MB window %.0f MB hit %.2f", got / 1048576.0,
               a.accessPolicyWindow.num_bytes / 1048576.0, a.accessPolicyWindow.hitRatio);
      run(tag);
      cudaCtxResetPersistingL2Cache();
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
