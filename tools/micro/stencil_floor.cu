// Floors for the diagonal-coded SpMV at config-3 size (n = 160^3):
//   copy     y = x                       (16 B/row)
//   stencil  y = sum_j c_j x[r + off_j]   (7 gathers, constants, no codes)
//   codes    y = sum_j tab[code] x[...]   (8 B of codes per row)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a stencil_floor.cu -o /tmp/sf
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 160;
constexpr int NN = N * N * N;
__constant__ int c_off[8];

__global__ void k_copy(const double* __restrict__ x, double* __restrict__ y, int n) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) y[r] = x[r];
}

__global__ void k_stencil(const double* __restrict__ x, double* __restrict__ y, int n) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 7; ++j) {
    int c = min(max(r + c_off[j], 0), n - 1);
    s = __dadd_rn(s, __dmul_rn(j == 3 ? 6.0 : -1.0, __ldg(x + c)));
  }
  y[r] = s;
}

__global__ void k_codes(const uint2* __restrict__ codes, const double* __restrict__ x,
                        double* __restrict__ y, int n) {
  __shared__ double tab[256];
  if (threadIdx.x < 2) tab[threadIdx.x] = threadIdx.x ? -1.0 : 6.0;
  __syncthreads();
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  uint2 w = __ldcs(codes + r);
  double xv[7];
#pragma unroll
  for (int j = 0; j < 7; ++j) xv[j] = __ldg(x + min(max(r + c_off[j], 0), n - 1));
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 7; ++j) {
    unsigned c = __byte_perm(j < 4 ? w.x : w.y, 0, 0x4440 | (j & 3));
    if (c != 0xff) s = __dadd_rn(s, __dmul_rn(tab[c], xv[j]));
  }
  y[r] = s;
}

__constant__ double c_tab[256];
// codes, values by select (no table)
__global__ void k_codes_sel(const uint2* __restrict__ codes, const double* __restrict__ x,
                            double* __restrict__ y, int n) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  uint2 w = __ldcs(codes + r);
  double xv[7];
#pragma unroll
  for (int j = 0; j < 7; ++j) xv[j] = __ldg(x + min(max(r + c_off[j], 0), n - 1));
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 7; ++j) {
    unsigned c = __byte_perm(j < 4 ? w.x : w.y, 0, 0x4440 | (j & 3));
    if (c != 0xff) s = __dadd_rn(s, __dmul_rn(c ? -1.0 : 6.0, xv[j]));
  }
  y[r] = s;
}
// codes, table in shared but no barrier-dependent init (static pattern), ldg codes
__global__ void k_codes_ldg(const uint2* __restrict__ codes, const double* __restrict__ x,
                            double* __restrict__ y, int n) {
  __shared__ double tab[256];
  if (threadIdx.x < 2) tab[threadIdx.x] = threadIdx.x ? -1.0 : 6.0;
  __syncthreads();
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  uint2 w = __ldg(codes + r);
  double xv[7];
#pragma unroll
  for (int j = 0; j < 7; ++j) xv[j] = __ldg(x + min(max(r + c_off[j], 0), n - 1));
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 7; ++j) {
    unsigned c = __byte_perm(j < 4 ? w.x : w.y, 0, 0x4440 | (j & 3));
    if (c != 0xff) s = __dadd_rn(s, __dmul_rn(tab[c], xv[j]));
  }
  y[r] = s;
}
// codes loaded, then ignored except for the absent test (constant values)
__global__ void k_codes_only(const uint2* __restrict__ codes, const double* __restrict__ x,
                             double* __restrict__ y, int n) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  uint2 w = __ldcs(codes + r);
  double xv[7];
#pragma unroll
  for (int j = 0; j < 7; ++j) xv[j] = __ldg(x + min(max(r + c_off[j], 0), n - 1));
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 7; ++j) s = __dadd_rn(s, __dmul_rn(j == 3 ? 6.0 : -1.0, xv[j]));
  y[r] = s + (w.x == 12345u ? 1.0 : 0.0);
}

// regular-row kernel ingredients, one at a time
template <int NG, bool MASK, bool EPI>
__global__ void k_var(const unsigned* __restrict__ mask, const double* __restrict__ x,
                      double* __restrict__ y, int n, double c0) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  unsigned m = MASK ? __ldg(mask + (r >> 5)) : 0xffffffffu;
  double xv[NG];
#pragma unroll
  for (int j = 0; j < NG; ++j) xv[j] = __ldg(x + min(max(r + c_off[j], 0), n - 1));
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 7; ++j) s = __dadd_rn(s, __dmul_rn(j == 3 ? 6.0 : -1.0, xv[j]));
  if (!((m >> (r & 31)) & 1u)) return;
  y[r] = EPI ? __dadd_rn(__ldg(x + r), __dmul_rn(c0, s)) : s;
}

// 2.5D march along the +-S diagonals (S = N*N): x[r+S] is loaded once and
// reused as the 0 and -S entries of the next two planes.
template <int T>
__global__ void k_march(const unsigned* __restrict__ mask, const double* __restrict__ x,
                        double* __restrict__ y, int n, double c0, int S, int G, int NQ) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int g = w % G, ch = w / G;
  const int p = g * 32 + lane;
  const int q0 = ch * T;
  if (q0 >= NQ) return;
  int r = q0 * S + p;
  double xm = __ldg(x + max(r - S, 0) ), x0 = __ldg(x + min(r, n - 1));
#pragma unroll 1
  for (int t = 0; t < T && q0 + t < NQ; ++t, r += S) {
    const double xp = __ldg(x + min(r + S, n - 1));
    const unsigned m = __ldg(mask + (min(r, n - 1) >> 5));
    double xv[7];
    xv[0] = xm;
    xv[1] = __ldg(x + min(max(r - N, 0), n - 1));
    xv[2] = __ldg(x + min(max(r - 1, 0), n - 1));
    xv[3] = x0;
    xv[4] = __ldg(x + min(r + 1, n - 1));
    xv[5] = __ldg(x + min(r + N, n - 1));
    xv[6] = xp;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 7; ++j) s = __dadd_rn(s, __dmul_rn(j == 3 ? 6.0 : -1.0, xv[j]));
    if (r < n && ((m >> (r & 31)) & 1u)) y[r] = __dadd_rn(x0, __dmul_rn(c0, s));
    xm = x0;
    x0 = xp;
  }
}

// the march with every load of the T planes issued up front
template <int T>
__global__ void k_march_u(const unsigned* __restrict__ mask, const double* __restrict__ x,
                          double* __restrict__ y, int n, double c0, int S, int G, int NQ) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int g = w % G, ch = w / G;
  const int p = g * 32 + lane;
  const int q0 = ch * T;
  if (q0 >= NQ) return;
  const int rb = q0 * S + p;
  double pl[T + 2], xv[T][4];
  unsigned m[T];
#pragma unroll
  for (int t = 0; t < T + 2; ++t) pl[t] = __ldg(x + min(max(rb + (t - 1) * S, 0), n - 1));
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int r = rb + t * S;
    m[t] = __ldg(mask + (min(r, n - 1) >> 5));
    xv[t][0] = __ldg(x + min(max(r - N, 0), n - 1));
    xv[t][1] = __ldg(x + min(max(r - 1, 0), n - 1));
    xv[t][2] = __ldg(x + min(r + 1, n - 1));
    xv[t][3] = __ldg(x + min(r + N, n - 1));
  }
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int r = rb + t * S;
    double s = 0.0;
    s = __dadd_rn(s, __dmul_rn(-1.0, pl[t]));
    s = __dadd_rn(s, __dmul_rn(-1.0, xv[t][0]));
    s = __dadd_rn(s, __dmul_rn(-1.0, xv[t][1]));
    s = __dadd_rn(s, __dmul_rn(6.0, pl[t + 1]));
    s = __dadd_rn(s, __dmul_rn(-1.0, xv[t][2]));
    s = __dadd_rn(s, __dmul_rn(-1.0, xv[t][3]));
    s = __dadd_rn(s, __dmul_rn(-1.0, pl[t + 2]));
    if (q0 + t < NQ && r < n && ((m[t] >> (r & 31)) & 1u)) y[r] = __dadd_rn(pl[t + 1], __dmul_rn(c0, s));
  }
}

template <typename F>
float timeit(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / reps;
}

int main() {
  int off[8] = {-N * N, -N, -1, 0, 1, N, N * N, 0};
  cudaMemcpyToSymbol(c_off, off, sizeof off);
  double *x, *y;
  uint2* codes;
  cudaMalloc(&x, NN * 8);
  cudaMalloc(&y, NN * 8);
  cudaMalloc(&codes, NN * 8);
  cudaMemset(x, 0, NN * 8);
  cudaMemset(codes, 0, NN * 8);
  for (int bs : {128, 256, 512}) {
    int g = (NN + bs - 1) / bs;
    float t0 = timeit([&] { k_copy<<<g, bs>>>(x, y, NN); }, 50);
    // ping-pong like pi(A)v so x is the previous output
    float t1 = timeit([&] { k_stencil<<<g, bs>>>(x, y, NN); std::swap(x, y); }, 50);
    float t2 = timeit([&] { k_codes<<<g, bs>>>(codes, x, y, NN); std::swap(x, y); }, 50);
    float t3 = timeit([&] { k_codes_sel<<<g, bs>>>(codes, x, y, NN); std::swap(x, y); }, 50);
    float t4 = timeit([&] { k_codes_ldg<<<g, bs>>>(codes, x, y, NN); std::swap(x, y); }, 50);
    float t5 = timeit([&] { k_codes_only<<<g, bs>>>(codes, x, y, NN); std::swap(x, y); }, 50);
    printf("bs %d: copy %.2f us (%.0f GB/s)  stencil %.2f us  codes %.2f  sel %.2f  ldg %.2f  only %.2f\n", bs, t0,
           16.0 * NN / t0 / 1e3, t1, t2, t3, t4, t5);
  }
  unsigned* mask;
  cudaMalloc(&mask, (NN / 32 + 1) * 4);
  cudaMemset(mask, 0xff, (NN / 32 + 1) * 4);
  {
    int bs = 512, g = (NN + bs - 1) / bs;
    float a = timeit([&] { k_var<7, false, false><<<g, bs>>>(mask, x, y, NN, 0.5); std::swap(x, y); }, 50);
    float b = timeit([&] { k_var<8, false, false><<<g, bs>>>(mask, x, y, NN, 0.5); std::swap(x, y); }, 50);
    float c = timeit([&] { k_var<7, true, false><<<g, bs>>>(mask, x, y, NN, 0.5); std::swap(x, y); }, 50);
    float d = timeit([&] { k_var<7, false, true><<<g, bs>>>(mask, x, y, NN, 0.5); std::swap(x, y); }, 50);
    float e = timeit([&] { k_var<8, true, true><<<g, bs>>>(mask, x, y, NN, 0.5); std::swap(x, y); }, 50);
    printf("var: base7 %.2f  gather8 %.2f  mask %.2f  epi %.2f  all %.2f us\n", a, b, c, d, e);
    const int S = N * N, G = S / 32, NQ = N;
    for (int T : {4, 8, 16}) {
      const int warps = G * ((NQ + T - 1) / T);
      const int blocks = (warps * 32 + 255) / 256;
      float tm = 0;
      if (T == 4) tm = timeit([&] { k_march<4><<<blocks, 256>>>(mask, x, y, NN, 0.5, S, G, NQ); std::swap(x, y); }, 50);
      if (T == 8) tm = timeit([&] { k_march<8><<<blocks, 256>>>(mask, x, y, NN, 0.5, S, G, NQ); std::swap(x, y); }, 50);
      if (T == 16) tm = timeit([&] { k_march<16><<<blocks, 256>>>(mask, x, y, NN, 0.5, S, G, NQ); std::swap(x, y); }, 50);
      printf("march T=%d: %.2f us\n", T, tm);
    }
    for (int T : {2, 4, 8}) {
      const int warps = G * ((NQ + T - 1) / T);
      for (int bs2 : {128, 256, 512}) {
        const int blocks = (warps * 32 + bs2 - 1) / bs2;
        float tm = 0;
        if (T == 2) tm = timeit([&] { k_march_u<2><<<blocks, bs2>>>(mask, x, y, NN, 0.5, S, G, NQ); std::swap(x, y); }, 50);
        if (T == 4) tm = timeit([&] { k_march_u<4><<<blocks, bs2>>>(mask, x, y, NN, 0.5, S, G, NQ); std::swap(x, y); }, 50);
        if (T == 8) tm = timeit([&] { k_march_u<8><<<blocks, bs2>>>(mask, x, y, NN, 0.5, S, G, NQ); std::swap(x, y); }, 50);
        printf("march_u T=%d bs=%d: %.2f us\n", T, bs2, tm);
      }
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
