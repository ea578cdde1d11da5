// FP64 pipe of the B200: DADD / DMUL throughput per SM and the dependent
// latency, the two numbers that bound the two-factor stencil passes
// (spmv_grid2.cu).  CH independent chains per thread, W warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_rate fp64_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH, bool MUL>
__global__ void k_chain(double* out, double a, int iters) {
  double v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = MUL ? __dmul_rn(v[c], a) : __dadd_rn(v[c], a);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += v[c];
  if (s == 12345.678) out[0] = s;
}

// one chain per warp, clock64 around a dependent sequence: latency in cycles
__global__ void k_lat(double* out, double a, int iters, long long* cyc) {
  double v = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __dadd_rn(v, a);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  if (v == 12345.678) out[0] = v;
}

template <int CH, bool MUL>
void run(int warps_per_sm, int sms, double* out) {
  const int iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) k_chain<CH, MUL><<<sms, 32 * warps_per_sm>>>(out, 1.0000001, iters);
  cudaEventRecord(e0);
  k_chain<CH, MUL><<<sms, 32 * warps_per_sm>>>(out, 1.0000001, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = double(sms) * warps_per_sm * 32 * CH * iters;
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double per_clk_sm = ops / (ms * 1e-3) / sms / (clk * 1e3);
  printf("%s CH=%2d warps/SM=%2d: %.1f GFLOP/s, %.1f lane-ops/clk/SM (at %d MHz nominal)\n",
         MUL ? "DMUL" : "DADD", CH, warps_per_sm, ops / (ms * 1e-3) / 1e9, per_clk_sm, clk / 1000);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8);
  k_lat<<<1, 32>>>(out, 1.0000001, 1024, cyc);
  cudaDeviceSynchronize();
  long long c;
  k_lat<<<1, 32>>>(out, 1.0000001, 1024, cyc);
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DADD dependent latency: %.2f cycles\n", c / 1024.0);
  for (int w : {4, 8, 16, 32}) {
    run<1, false>(w, sms, out);
    run<4, false>(w, sms, out);
    run<8, false>(w, sms, out);
  }
  run<8, true>(16, sms, out);
  run<8, true>(32, sms, out);
  return 0;
}
