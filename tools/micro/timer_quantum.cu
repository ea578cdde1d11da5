// Is per-kernel time quantised?  Copy kernels of growing size, timed with
// events over 50 back-to-back launches and one launch at a time.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_copy(const double* __restrict__ x, double* __restrict__ y, int n) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) y[r] = x[r];
}
__global__ void k_empty() {}
int main() {
  const int NMAX = 8 << 20;
  double *x, *y;
  cudaMalloc(&x, NMAX * 8);
  cudaMalloc(&y, NMAX * 8);
  cudaMemset(x, 0, NMAX * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 5; ++i) k_empty<<<1, 32>>>();
  cudaEventRecord(a);
  for (int i = 0; i < 200; ++i) k_empty<<<1, 32>>>();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("empty kernel: %.3f us per launch\n", ms * 1000 / 200);
  for (int n = 1 << 19; n <= NMAX; n += 1 << 19) {
    int g = (n + 511) / 512;
    for (int i = 0; i < 3; ++i) k_copy<<<g, 512>>>(x, y, n);
    cudaEventRecord(a);
    for (int i = 0; i < 50; ++i) k_copy<<<g, 512>>>(x, y, n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    float per = ms * 1000 / 50;
    float single = 0;
    for (int i = 0; i < 5; ++i) {
      cudaEventRecord(a);
      k_copy<<<g, 512>>>(x, y, n);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float t;
      cudaEventElapsedTime(&t, a, b);
      single += t * 1000 / 5;
    }
    printf("n %8d  %.3f MB  chain %.3f us  single %.3f us  %.0f GB/s\n", n, 16.0 * n / 1e6, per,
           single, 16.0 * n / per / 1e3);
  }
}
