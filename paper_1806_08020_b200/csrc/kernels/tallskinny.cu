// Tall-skinny basis kernels: CGS2 orthogonalisation (replacing the MGS2 of
// arnoldi_extend, src/arnoldi.cpp:129-150), basis recombination V*Q / V*G
// (thick_restart src/arnoldi.cpp:309-311, ritz_vector src/arnoldi.cpp:258),
// and the counted length-n kernels of inc/cost.hpp:51-76.
//
// V is column-major in HBM with a leading dimension padded to 32 doubles
// (256 B), so every column starts on an L2 sector boundary and a warp's
// load of 32 consecutive rows of one column is a single 256 B request.
// All reductions are deterministic: per-block partial rows + a fixed-order
// final sum in the last block (common.cuh grid_reduce), never fp64 atomics.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "common.cuh"
#include "ws_layout.cuh"
#include "ppa/kernels.hpp"

namespace ppa {
namespace kern {


void ensure_workspace(ReduceWorkspace& ws, int blocks, int width) {
  if (!ws.tickets.get()) {
    ws.tickets.resize(64);
    PPA_CUDA(cudaMemset(ws.tickets.get(), 0, 64 * sizeof(unsigned int)));
    ws.scalars.resize(kScalCount);
    PPA_CUDA(cudaMemset(ws.scalars.get(), 0, kScalCount * sizeof(double)));
  }
  if (blocks > ws.max_blocks || width > ws.max_width) {
    const int b = std::max(blocks, ws.max_blocks);
    const int w = std::max(width, ws.max_width);
    // Only resized between launches on the owning stream; a pending kernel
    // may still read the old buffer, so synchronise the device first.
    PPA_CUDA(cudaDeviceSynchronize());
    ws.partials.resize(static_cast<size_t>(b) * static_cast<size_t>(w));
    ws.max_blocks = b;
    ws.max_width = w;
  }
}

namespace {

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

// ------------------------------------------------------------------------
// Generic small reductions (NV outputs).
// ------------------------------------------------------------------------

template <int NV, int T, typename Op>
__global__ void __launch_bounds__(T) k_reduce(long long n, int rows_per_block, Op op,
                                               double* partials, unsigned int* ticket) {
  double acc[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) acc[j] = 0.0;
  const long long r0 = static_cast<long long>(blockIdx.x) * rows_per_block;
  const long long r1 = min(n, r0 + rows_per_block);
  for (long long i = r0 + threadIdx.x; i < r1; i += T) op.row(i, acc);
  __shared__ double s_final[NV];
  if (dev::grid_reduce<NV, T>(acc, NV, 0, partials, ticket, s_final)) {
    if (threadIdx.x == 0) op.finalize(s_final);
  }
}

struct OpDot {
  const double* __restrict__ x;
  const double* __restrict__ y;
  double* out;
  __device__ void row(long long i, double (&a)[1]) const { a[0] = fma(x[i], y[i], a[0]); }
  __device__ void finalize(const double* s) const { out[0] = s[0]; }
};

struct OpNrm2 {
  const double* __restrict__ x;
  double* out;
  __device__ void row(long long i, double (&a)[1]) const { a[0] = fma(x[i], x[i], a[0]); }
  __device__ void finalize(const double* s) const { out[0] = sqrt(s[0]); }
};

// Real Ritz check, pass 2: ||Ay - mu y||, mu already on device.
struct OpResidReal {
  const double* __restrict__ y;
  const double* __restrict__ ay;
  double* out;  // out[0] = mu (read), out[1] = residual (written)
  __device__ void row(long long i, double (&a)[1]) const {
    const double r = ay[i] - out[0] * y[i];
    a[0] = fma(r, r, a[0]);
  }
  __device__ void finalize(const double* s) const { out[1] = sqrt(s[0]); }
};

// Complex Ritz check, pass 1: the four real dots of y^H A y.
struct OpCplxDots {
  const double* __restrict__ yr;
  const double* __restrict__ yi;
  const double* __restrict__ ar;
  const double* __restrict__ ai;
  double* out;  // out[0] = mu_re, out[1] = mu_im
  __device__ void row(long long i, double (&a)[4]) const {
    const double r = yr[i], m = yi[i], p = ar[i], q = ai[i];
    a[0] = fma(r, p, a[0]);
    a[1] = fma(m, q, a[1]);
    a[2] = fma(r, q, a[2]);
    a[3] = fma(m, p, a[3]);
  }
  __device__ void finalize(const double* s) const {
    out[0] = s[0] + s[1];
    out[1] = s[2] - s[3];
  }
};

struct OpCplxResid {
  const double* __restrict__ yr;
  const double* __restrict__ yi;
  const double* __restrict__ ar;
  const double* __restrict__ ai;
  double* out;  // out[0..1] = mu (read), out[2] = residual (written)
  __device__ void row(long long i, double (&a)[1]) const {
    const double mr = out[0], mi = out[1];
    const double rr = ar[i] - (mr * yr[i] - mi * yi[i]);
    const double ri = ai[i] - (mr * yi[i] + mi * yr[i]);
    a[0] = fma(rr, rr, fma(ri, ri, a[0]));
  }
  __device__ void finalize(const double* s) const { out[2] = sqrt(s[0]); }
};

template <int NV, typename Op>
void run_reduce(long long n, const Op& op, ReduceWorkspace& ws, int sm_count, cudaStream_t st) {
  constexpr int T = 256;
  const int blocks = std::max(1, std::min(ceil_div(n, T), sm_count * 8));
  const int rpb = ceil_div(ceil_div(n, blocks), 32) * 32;
  const int grid = std::max(1, ceil_div(n, rpb));
  ensure_workspace(ws, grid, NV);
  k_reduce<NV, T, Op><<<grid, T, 0, st>>>(n, rpb, op, ws.partials.get(), ws.tickets.get());
  PPA_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------------
// blas1
// ------------------------------------------------------------------------

__global__ void k_axpy(double a, const double* __restrict__ x, double* __restrict__ y, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    y[i] = __dadd_rn(y[i], __dmul_rn(a, x[i]));
  }
}
__global__ void k_scale(double* x, double a, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    x[i] = __dmul_rn(x[i], a);
  }
}
__global__ void k_div_scale(double* x, const double* a, long long n) {
  const double d = *a;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    x[i] = __ddiv_rn(x[i], d);
  }
}
__global__ void k_div_value(double* x, double a, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    x[i] = __ddiv_rn(x[i], a);
  }
}
__global__ void k_sub(const double* __restrict__ x, const double* __restrict__ w, double* y,
                      long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    y[i] = __dsub_rn(x[i], w[i]);
  }
}
__global__ void k_fill(double* x, double v, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    x[i] = v;
  }
}

inline int ew_grid(long long n) { return std::max(1, std::min(ceil_div(n, 256), 148 * 16)); }

// Out[:,0:p] = V[:,0:d] * G.  RB rows per thread (rows r and r + CB of the
// CTA's 2 CB-row block when RB = 2) with their p accumulators in registers:
// each row's d values are streamed once (JU columns of loads in flight per
// row), G comes from shared memory, row-major with an even row length, two
// columns per broadcast 16-byte read that serves all RB rows (RB = 2 halves
// the shared-memory wavefronts per FMA, which bounded the one-row kernel:
// 0.63 ms for d = 40, p = 20 in place on config 3).  A row's outputs are
// written only after all of its d inputs were read, by the same thread, so
// Out may alias V (the in-place thick restart, p <= d).  Per output: fma
// over j = 0..d-1 in order.
constexpr int CB = 256;  // threads per CTA

template <int PB>
__global__ void __launch_bounds__(CB) k_ts_combine(const double* V, long long ldv, int n, int d,
                                                   const double* __restrict__ G, int p,
                                                   double* Out, long long ldo) {
  static_assert(PB % 2 == 0, "column pairs");
  extern __shared__ double2 gs2[];  // G row-major: row j = columns 0..PB-1 (zero-padded)
  double* gs = reinterpret_cast<double*>(gs2);
  for (int k = threadIdx.x; k < d * PB; k += CB) {
    const int j = k / PB, c = k - j * PB;
    gs[k] = c < p ? G[static_cast<long long>(c) * d + j] : 0.0;
  }
  __syncthreads();
  const long long i = static_cast<long long>(blockIdx.x) * CB + threadIdx.x;
  const bool live = i < n;
  const long long row = live ? i : n - 1;  // clamped loads, no store
  double acc[PB];
#pragma unroll
  for (int c = 0; c < PB; ++c) acc[c] = 0.0;
  // columns p..PB-1 of G are zero in shared memory: no per-column test
  auto step = [&](double v, const double2* g) {
#pragma unroll
    for (int c = 0; c < PB / 2; ++c) {
      const double2 gv = g[c];
      acc[2 * c] = fma(v, gv.x, acc[2 * c]);
      acc[2 * c + 1] = fma(v, gv.y, acc[2 * c + 1]);
    }
  };
  constexpr int JU = 8;
  const double* vr = V + row;
  int j0 = 0;
  for (; j0 + JU <= d; j0 += JU) {
    double v[JU];
#pragma unroll
    for (int jj = 0; jj < JU; ++jj) v[jj] = vr[static_cast<long long>(j0 + jj) * ldv];
    const double2* g = gs2 + j0 * (PB / 2);
#pragma unroll
    for (int jj = 0; jj < JU; ++jj) step(v[jj], g + jj * (PB / 2));
  }
  for (; j0 < d; ++j0) step(vr[static_cast<long long>(j0) * ldv], gs2 + j0 * (PB / 2));
  if (!live) return;
#pragma unroll
  for (int c = 0; c < PB; ++c) {
    if (c < p) Out[row + static_cast<long long>(c) * ldo] = acc[c];
  }
}

// Two rows per thread (the RB = 2 form described above).

template <int PB, int RB>
__global__ void __launch_bounds__(CB, RB) k_ts_combine_rb(const double* V, long long ldv, int n, int d,
                                                   const double* __restrict__ G, int p,
                                                   double* Out, long long ldo) {
  static_assert(PB % 2 == 0, "column pairs");
  extern __shared__ double2 gs2[];  // G row-major: row j = columns 0..PB-1 (zero-padded)
  double* gs = reinterpret_cast<double*>(gs2);
  for (int k = threadIdx.x; k < d * PB; k += CB) {
    const int j = k / PB, c = k - j * PB;
    gs[k] = c < p ? G[static_cast<long long>(c) * d + j] : 0.0;
  }
  __syncthreads();
  long long row[RB];
  bool live[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    const long long i = static_cast<long long>(blockIdx.x) * (CB * RB) + r * CB + threadIdx.x;
    live[r] = i < n;
    row[r] = live[r] ? i : n - 1;  // clamped loads, no store
  }
  double acc[RB][PB];
#pragma unroll
  for (int r = 0; r < RB; ++r)
#pragma unroll
    for (int c = 0; c < PB; ++c) acc[r][c] = 0.0;
  // columns p..PB-1 of G are zero in shared memory: no per-column test
  auto step = [&](const double (&v)[RB], const double2* g) {
#pragma unroll
    for (int c = 0; c < PB / 2; ++c) {
      const double2 gv = g[c];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        acc[r][2 * c] = fma(v[r], gv.x, acc[r][2 * c]);
        acc[r][2 * c + 1] = fma(v[r], gv.y, acc[r][2 * c + 1]);
      }
    }
  };
  constexpr int JU = RB == 1 ? 8 : 2;
  int j0 = 0;
  for (; j0 + JU <= d; j0 += JU) {
    double v[JU][RB];
#pragma unroll
    for (int jj = 0; jj < JU; ++jj)
#pragma unroll
      for (int r = 0; r < RB; ++r) v[jj][r] = V[row[r] + static_cast<long long>(j0 + jj) * ldv];
    const double2* g = gs2 + j0 * (PB / 2);
#pragma unroll
    for (int jj = 0; jj < JU; ++jj) step(v[jj], g + jj * (PB / 2));
  }
  for (; j0 < d; ++j0) {
    double v[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) v[r] = V[row[r] + static_cast<long long>(j0) * ldv];
    step(v, gs2 + j0 * (PB / 2));
  }
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    if (!live[r]) continue;
#pragma unroll
    for (int c = 0; c < PB; ++c) {
      if (c < p) Out[row[r] + static_cast<long long>(c) * ldo] = acc[r][c];
    }
  }
}

template <int PB>
void launch_combine(const double* V, long long ldv, int n, int d, const double* G, int p,
                    double* Out, long long ldo, size_t smem, cudaStream_t st) {
  // two rows per thread at PB = 20 (the k = 20 restarts of configs 2 and 3):
  // measured 0.55 ms vs 0.63 ms for d = 40 in place; for other widths the
  // one-row kernel keeps more warps resident and is faster
  // (tools/combine_bench.py)
  if constexpr (PB == 20) {
    static const bool capped = [] {
      PPA_CUDA(cudaFuncSetAttribute(k_ts_combine_rb<PB, 2>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    max_dynamic_smem(k_ts_combine_rb<PB, 2>)));
      return true;
    }();
    (void)capped;
    k_ts_combine_rb<PB, 2><<<ceil_div(n, CB * 2), CB, smem, st>>>(V, ldv, n, d, G, p, Out, ldo);
  } else {
    static const bool capped = [] {  // once per instantiation, thread-safe
      PPA_CUDA(cudaFuncSetAttribute(k_ts_combine<PB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    max_dynamic_smem(k_ts_combine<PB>)));
      return true;
    }();
    (void)capped;
    k_ts_combine<PB><<<ceil_div(n, CB), CB, smem, st>>>(V, ldv, n, d, G, p, Out, ldo);
  }
}

}  // namespace

void check_cols(int c, const char* who) {
  if (c < 1 || c > kMaxCols) {
    throw std::invalid_argument(std::string(who) + ": column count out of range [1,128]");
  }
}

// ------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------

void copy(const double* x, double* y, long long n, cudaStream_t st) {
  if (n > 0 && x != y) {
    PPA_CUDA(cudaMemcpyAsync(y, x, static_cast<size_t>(n) * sizeof(double),
                             cudaMemcpyDeviceToDevice, st));
  }
}
void axpy(double a, const double* x, double* y, long long n, cudaStream_t st) {
  if (n <= 0) return;
  k_axpy<<<ew_grid(n), 256, 0, st>>>(a, x, y, n);
  PPA_CUDA(cudaGetLastError());
}
void scale(double* x, double a, long long n, cudaStream_t st) {
  if (n <= 0) return;
  k_scale<<<ew_grid(n), 256, 0, st>>>(x, a, n);
  PPA_CUDA(cudaGetLastError());
}
void div_scale(double* x, const double* a, long long n, cudaStream_t st) {
  if (n <= 0) return;
  k_div_scale<<<ew_grid(n), 256, 0, st>>>(x, a, n);
  PPA_CUDA(cudaGetLastError());
}
void div_value(double* x, double a, long long n, cudaStream_t st) {
  if (n <= 0) return;
  k_div_value<<<ew_grid(n), 256, 0, st>>>(x, a, n);
  PPA_CUDA(cudaGetLastError());
}
void sub(const double* x, const double* w, double* y, long long n, cudaStream_t st) {
  if (n <= 0) return;
  k_sub<<<ew_grid(n), 256, 0, st>>>(x, w, y, n);
  PPA_CUDA(cudaGetLastError());
}
void fill(double* x, double v, long long n, cudaStream_t st) {
  if (n <= 0) return;
  k_fill<<<ew_grid(n), 256, 0, st>>>(x, v, n);
  PPA_CUDA(cudaGetLastError());
}

void dot(const double* x, const double* y, long long n, double* out, ReduceWorkspace& ws,
         int sm_count, cudaStream_t st) {
  run_reduce<1>(n, OpDot{x, y, out}, ws, sm_count, st);
}
void nrm2(const double* x, long long n, double* out, ReduceWorkspace& ws, int sm_count,
          cudaStream_t st) {
  run_reduce<1>(n, OpNrm2{x, out}, ws, sm_count, st);
}

void ritz_check_real(const double* y, const double* ay, long long n, double* out,
                     ReduceWorkspace& ws, int sm_count, cudaStream_t st) {
  run_reduce<1>(n, OpDot{y, ay, out}, ws, sm_count, st);
  run_reduce<1>(n, OpResidReal{y, ay, out}, ws, sm_count, st);
}

void ritz_check_complex(const double* yr, const double* yi, const double* ar, const double* ai,
                        long long n, double* out, ReduceWorkspace& ws, int sm_count,
                        cudaStream_t st) {
  run_reduce<4>(n, OpCplxDots{yr, yi, ar, ai, out}, ws, sm_count, st);
  run_reduce<1>(n, OpCplxResid{yr, yi, ar, ai, out}, ws, sm_count, st);
}

void ts_combine(const double* V, long long ldv, int n, int d, const double* G, int p, double* Out,
                long long ldo, cudaStream_t st) {
  if (n <= 0 || p <= 0) return;
  if (d < 1) throw std::invalid_argument("ts_combine: d < 1");
  if (Out == V && p > d) throw std::invalid_argument("ts_combine: in-place needs p <= d");
  if (static_cast<size_t>(d) * std::min(p, 32) * sizeof(double) > 200 * 1024) {
    throw std::invalid_argument("ts_combine: d too large");
  }
  if (Out == V && p > 32) {
    // wide in-place restart (k > 32): combine into a stream-ordered
    // temporary in 32-column passes, then copy back over V
    double* tmp = nullptr;
    const long long ldt = (static_cast<long long>(n) + 31) / 32 * 32;
    PPA_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tmp),
                             static_cast<size_t>(ldt) * p * sizeof(double), st));
    ts_combine(V, ldv, n, d, G, p, tmp, ldt, st);
    PPA_CUDA(cudaMemcpy2DAsync(Out, static_cast<size_t>(ldo) * sizeof(double), tmp,
                               static_cast<size_t>(ldt) * sizeof(double),
                               static_cast<size_t>(n) * sizeof(double), p,
                               cudaMemcpyDeviceToDevice, st));
    PPA_CUDA(cudaFreeAsync(tmp, st));
    return;
  }
  // accumulator count bucketed so registers stay <= ~128 per thread; the
  // passes only read V, so they are independent (in place: one pass)
  int sms = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) {
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
  }
  for (int c0 = 0; c0 < p; c0 += 32) {
    const int pc = std::min(32, p - c0);
    const double* g = G + static_cast<long long>(c0) * d;
    double* out = Out + static_cast<long long>(c0) * ldo;
    if (ts_combine_tma(V, ldv, n, d, g, pc, out, ldo, sms, st)) continue;
    auto sm = [&](int pb) { return static_cast<size_t>(d) * pb * sizeof(double); };
    switch ((pc + 3) / 4) {  // accumulators rounded up to a multiple of 4
      case 1: launch_combine<4>(V, ldv, n, d, g, pc, out, ldo, sm(4), st); break;
      case 2: launch_combine<8>(V, ldv, n, d, g, pc, out, ldo, sm(8), st); break;
      case 3: launch_combine<12>(V, ldv, n, d, g, pc, out, ldo, sm(12), st); break;
      case 4: launch_combine<16>(V, ldv, n, d, g, pc, out, ldo, sm(16), st); break;
      case 5: launch_combine<20>(V, ldv, n, d, g, pc, out, ldo, sm(20), st); break;
      case 6: launch_combine<24>(V, ldv, n, d, g, pc, out, ldo, sm(24), st); break;
      case 7: launch_combine<28>(V, ldv, n, d, g, pc, out, ldo, sm(28), st); break;
      default: launch_combine<32>(V, ldv, n, d, g, pc, out, ldo, sm(32), st); break;
    }
    PPA_CUDA(cudaGetLastError());
  }
}

}  // namespace kern
}  // namespace ppa
