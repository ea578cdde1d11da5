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
#include "ppa/kernels.hpp"

namespace ppa {
namespace kern {

// Layout of ReduceWorkspace::scalars (device doubles).
constexpr int kScalH1 = 0;
constexpr int kScalH2 = 256;
constexpr int kScalHsub = 512;
constexpr int kScalTmp = 520;   // ritz checks
constexpr int kScalCount = 1024;
constexpr int kMaxCols = 128;

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

// ------------------------------------------------------------------------
// CGS2 sweeps: "warp = column group" layout.
//
// A 256-thread CTA is 8 warps; column j of V belongs to warp j % 8 (slot
// j / 8, at most CPW columns per warp).  Lanes walk row PAIRS with 16-byte
// loads (a warp reads 512 contiguous bytes of one column per request), so
// per-thread state is CPW accumulators (+ the cached V tile in sweep 2):
// low registers, many resident warps, every HBM byte coalesced.  Row sums
// that need all columns (w - V h) are combined across the 8 warps through
// shared memory in a fixed order, so results are deterministic.
// ------------------------------------------------------------------------

constexpr int NW = 8;           // warps per CTA
constexpr int TS = NW * 32;     // threads per CTA

__device__ __forceinline__ double2 ld_pair(const double* p, int r, int n) {
  if (r + 1 < n) return __ldg(reinterpret_cast<const double2*>(p + r));
  if (r < n) return make_double2(__ldg(p + r), 0.0);
  return make_double2(0.0, 0.0);
}

// Per-column block partials already unique per column (s_col[0..width)):
// write the block's row, the last CTA sums rows in block order.
__device__ __forceinline__ bool grid_finish(const double* s_col, int width, double* partials,
                                            unsigned int* ticket, double* s_final) {
  __shared__ unsigned int s_last;
  for (int k = threadIdx.x; k < width; k += blockDim.x) {
    partials[static_cast<size_t>(blockIdx.x) * width + k] = s_col[k];
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
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  for (int k = warp; k < width; k += nwarp) {
    double acc = 0.0;
    for (int b = lane; b < static_cast<int>(gridDim.x); b += 32) {
      acc += __ldcg(partials + static_cast<size_t>(b) * width + k);
    }
    acc = dev::warp_sum(acc);
    if (lane == 0) s_final[k] = acc;
  }
  if (threadIdx.x == 0) *ticket = 0u;
  __syncthreads();
  return true;
}

// out[j] = sum_i V[i,j] * w[i]  (SQ: sum_i V[i,j]^2), j < c.
template <int CPW, int QP, bool SQ>
__global__ void __launch_bounds__(TS) k_mdot(const double* __restrict__ V, long long ld, int n,
                                             int c, const double* __restrict__ w, int rpb,
                                             double* partials, unsigned int* ticket,
                                             double* out) {
  __shared__ double s_col[NW * CPW];
  __shared__ double s_final[NW * CPW];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  double acc[CPW];
#pragma unroll
  for (int jj = 0; jj < CPW; ++jj) acc[jj] = 0.0;
  const int r0 = blockIdx.x * rpb;
  const int r1 = min(n, r0 + rpb);
  for (int t0 = r0; t0 < r1; t0 += 64 * QP) {
    double2 wv[QP];
#pragma unroll
    for (int q = 0; q < QP; ++q) {
      const int r = t0 + 64 * q + 2 * lane;
      wv[q] = SQ ? make_double2(0.0, 0.0) : (r < r1 ? ld_pair(w, r, r1) : make_double2(0.0, 0.0));
    }
#pragma unroll
    for (int jj = 0; jj < CPW; ++jj) {
      const int j = g + NW * jj;
      if (j < c) {
        const double* col = V + static_cast<long long>(j) * ld;
#pragma unroll
        for (int q = 0; q < QP; ++q) {
          const int r = t0 + 64 * q + 2 * lane;
          const double2 v = r < r1 ? ld_pair(col, r, r1) : make_double2(0.0, 0.0);
          if (SQ) {
            acc[jj] = fma(v.x, v.x, acc[jj]);
            acc[jj] = fma(v.y, v.y, acc[jj]);
          } else {
            acc[jj] = fma(v.x, wv[q].x, acc[jj]);
            acc[jj] = fma(v.y, wv[q].y, acc[jj]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int jj = 0; jj < CPW; ++jj) {
    const int j = g + NW * jj;
    if (j < c) {
      const double t = dev::warp_sum(acc[jj]);
      if (lane == 0) s_col[j] = t;
    }
  }
  __syncthreads();
  if (grid_finish(s_col, c, partials, ticket, s_final)) {
    for (int j = threadIdx.x; j < c; j += TS) out[j] = s_final[j];
  }
}

// w -= V h (h device); optionally h2 = V^T w and ||w||^2 (DOT); the CGS2
// finalisation (Hessenberg column, hsub, breakdown flag) runs in the last CTA.
// MODE 0: CGS2 sweep 2.  MODE 1: single-pass reorth (norm only).
template <int CPW, int QP, int MODE>
__global__ void __launch_bounds__(TS) k_cgs_update(const double* __restrict__ V, long long ld,
                                                   int n, int c, double* __restrict__ w,
                                                   const double* __restrict__ h1, int rpb,
                                                   double* partials, unsigned int* ticket,
                                                   double* scal, double* Hcol, int* flag,
                                                   double* out_norm) {
  __shared__ double s_h[NW * CPW];
  __shared__ __align__(16) double s_part[2][NW][64 * QP];
  __shared__ double s_col[NW * CPW + 1];
  __shared__ double s_final[NW * CPW + 1];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  for (int j = threadIdx.x; j < NW * CPW; j += TS) s_h[j] = j < c ? h1[j] : 0.0;
  __syncthreads();
  double acc[CPW];
#pragma unroll
  for (int jj = 0; jj < CPW; ++jj) acc[jj] = 0.0;
  double nrm = 0.0;
  const int r0 = blockIdx.x * rpb;
  const int r1 = min(n, r0 + rpb);
  int par = 0;
  for (int t0 = r0; t0 < r1; t0 += 64 * QP, par ^= 1) {
    double2 vr[QP][MODE == 0 ? CPW : 1];
    double2 part[QP];
#pragma unroll
    for (int q = 0; q < QP; ++q) part[q] = make_double2(0.0, 0.0);
#pragma unroll
    for (int jj = 0; jj < CPW; ++jj) {
      const int j = g + NW * jj;
      if (j < c) {
        const double* col = V + static_cast<long long>(j) * ld;
        const double hj = s_h[j];
#pragma unroll
        for (int q = 0; q < QP; ++q) {
          const int r = t0 + 64 * q + 2 * lane;
          const double2 v = r < r1 ? ld_pair(col, r, r1) : make_double2(0.0, 0.0);
          if (MODE == 0) vr[q][jj] = v;
          part[q].x = fma(v.x, hj, part[q].x);
          part[q].y = fma(v.y, hj, part[q].y);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < QP; ++q) {
      reinterpret_cast<double2*>(s_part[par][g])[32 * q + lane] = part[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < QP; ++q) {
      const int r = t0 + 64 * q + 2 * lane;
      if (r >= r1) continue;
      double2 sum = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < NW; ++k) {
        const double2 pk = reinterpret_cast<const double2*>(s_part[par][k])[32 * q + lane];
        sum.x += pk.x;
        sum.y += pk.y;
      }
      const double2 wo = ld_pair(w, r, r1);
      const double2 wn = make_double2(wo.x - sum.x, wo.y - sum.y);
      if (MODE == 0) {
#pragma unroll
        for (int jj = 0; jj < CPW; ++jj) {
          if (g + NW * jj < c) {
            acc[jj] = fma(vr[q][jj].x, wn.x, acc[jj]);
            acc[jj] = fma(vr[q][jj].y, wn.y, acc[jj]);
          }
        }
      }
      if (g == 0) {
        nrm = fma(wn.x, wn.x, nrm);
        if (r + 1 < r1) {
          nrm = fma(wn.y, wn.y, nrm);
          *reinterpret_cast<double2*>(w + r) = wn;
        } else {
          w[r] = wn.x;
        }
      }
    }
  }
  const int width = MODE == 0 ? c + 1 : 1;
  if (MODE == 0) {
#pragma unroll
    for (int jj = 0; jj < CPW; ++jj) {
      const int j = g + NW * jj;
      if (j < c) {
        const double t = dev::warp_sum(acc[jj]);
        if (lane == 0) s_col[j] = t;
      }
    }
  }
  if (g == 0) {
    const double t = dev::warp_sum(nrm);
    if (lane == 0) s_col[width - 1] = t;
  }
  __syncthreads();
  if (!grid_finish(s_col, width, partials, ticket, s_final)) return;
  if (MODE == 1) {
    if (threadIdx.x == 0) *out_norm = sqrt(s_final[0]);
    return;
  }
  for (int j = threadIdx.x; j < c; j += TS) scal[kScalH2 + j] = s_final[j];
  if (threadIdx.x == 0) {
    double sq = 0.0;
    for (int j = 0; j < c; ++j) sq += s_final[j] * s_final[j];
    const double d2 = s_final[c] - sq;
    const double hsub = d2 > 0.0 ? sqrt(d2) : 0.0;
    scal[kScalHsub] = hsub;
    scal[kScalHsub + 1] = sqrt(s_final[c]);
    double cn = 0.0;
    for (int j = 0; j < c; ++j) {
      const double hj = s_h[j] + s_final[j];
      Hcol[j] = hj;
      cn += hj * hj;
    }
    cn += hsub * hsub;
    const double colnorm = sqrt(cn);
    int bd = 0;
    if (!isfinite(hsub) || !isfinite(colnorm)) {
      bd = 2;
    } else if (hsub <= 1e-14 * colnorm) {
      bd = 1;
    }
    Hcol[c] = bd ? 0.0 : hsub;
    *flag = bd;
  }
}

// Sweep 3: V[:,c] = (w - V h2) / hsub, skipped on breakdown.
template <int CPW, int QP>
__global__ void __launch_bounds__(TS) k_cgs_store(double* V, long long ld, int n, int c,
                                                  const double* __restrict__ w, int rpb,
                                                  const double* __restrict__ scal,
                                                  const int* flag) {
  if (*flag) return;
  __shared__ double s_h[NW * CPW];
  __shared__ __align__(16) double s_part[2][NW][64 * QP];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  for (int j = threadIdx.x; j < NW * CPW; j += TS) s_h[j] = j < c ? scal[kScalH2 + j] : 0.0;
  const double hsub = scal[kScalHsub];
  __syncthreads();
  double* out = V + static_cast<long long>(c) * ld;
  const int r0 = blockIdx.x * rpb;
  const int r1 = min(n, r0 + rpb);
  int par = 0;
  for (int t0 = r0; t0 < r1; t0 += 64 * QP, par ^= 1) {
    double2 part[QP];
#pragma unroll
    for (int q = 0; q < QP; ++q) part[q] = make_double2(0.0, 0.0);
#pragma unroll
    for (int jj = 0; jj < CPW; ++jj) {
      const int j = g + NW * jj;
      if (j < c) {
        const double* col = V + static_cast<long long>(j) * ld;
        const double hj = s_h[j];
#pragma unroll
        for (int q = 0; q < QP; ++q) {
          const int r = t0 + 64 * q + 2 * lane;
          const double2 v = r < r1 ? ld_pair(col, r, r1) : make_double2(0.0, 0.0);
          part[q].x = fma(v.x, hj, part[q].x);
          part[q].y = fma(v.y, hj, part[q].y);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < QP; ++q) {
      reinterpret_cast<double2*>(s_part[par][g])[32 * q + lane] = part[q];
    }
    __syncthreads();
    if (g < QP) {
      const int q = g;
      const int r = t0 + 64 * q + 2 * lane;
      if (r < r1) {
        double2 sum = make_double2(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < NW; ++k) {
          const double2 pk = reinterpret_cast<const double2*>(s_part[par][k])[32 * q + lane];
          sum.x += pk.x;
          sum.y += pk.y;
        }
        const double2 wo = ld_pair(w, r, r1);
        const double a = (wo.x - sum.x) / hsub;
        if (r + 1 < r1) {
          *reinterpret_cast<double2*>(out + r) = make_double2(a, (wo.y - sum.y) / hsub);
        } else {
          out[r] = a;
        }
      }
    }
  }
}

// Out[:,0:p] = V[:,0:d] * G, one row per thread, the block's rows staged
// in shared memory first (so Out may alias V).
constexpr int kCombineRows = 128;

__global__ void __launch_bounds__(kCombineRows) k_ts_combine(const double* V, long long ldv, int n,
                                                             int d, const double* __restrict__ G,
                                                             int p, double* Out, long long ldo) {
  extern __shared__ double sm[];
  double* tile = sm;                       // [d][kCombineRows]
  double* gs = sm + d * kCombineRows;      // [d*p] column-major
  for (int k = threadIdx.x; k < d * p; k += kCombineRows) gs[k] = G[k];
  const int r0 = blockIdx.x * kCombineRows;
  const int i = r0 + threadIdx.x;
  const bool live = i < n;
  for (int j = 0; j < d; ++j) {
    tile[j * kCombineRows + threadIdx.x] = live ? V[i + static_cast<long long>(j) * ldv] : 0.0;
  }
  __syncthreads();
  if (!live) return;
  for (int col = 0; col < p; ++col) {
    const double* g = gs + col * d;
    double acc = 0.0;
    for (int j = 0; j < d; ++j) acc = fma(tile[j * kCombineRows + threadIdx.x], g[j], acc);
    Out[i + static_cast<long long>(col) * ldo] = acc;
  }
}

template <typename K>
int occupancy_of(K kernel) {
  int o = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kernel, TS, 0);
  return std::max(1, o);
}

// Row partition: `blocks` CTAs, each a contiguous range of whole 128-row tiles.
struct Part {
  int grid, rpb;
};
Part partition(int n, int sm_count, int occ) {
  const int tiles = ceil_div(n, 128);
  const int blocks = std::max(1, std::min(tiles, sm_count * occ));
  const int rpb = ceil_div(tiles, blocks) * 128;
  return {std::max(1, ceil_div(n, rpb)), rpb};
}

void check_aligned(const void* p, const char* who) {
  if (reinterpret_cast<uintptr_t>(p) % 16 != 0) {
    throw std::invalid_argument(std::string(who) + ": vectors must be 16-byte aligned");
  }
}

template <int CPW>
void launch_mdot(const double* V, long long ld, int n, int c, const double* w, double* out,
                 bool sq, ReduceWorkspace& ws, int sm_count, cudaStream_t st) {
  constexpr int QP = CPW <= 4 ? 4 : 2;
  auto kern = sq ? k_mdot<CPW, QP, true> : k_mdot<CPW, QP, false>;
  static const int occ_t = occupancy_of(k_mdot<CPW, QP, false>);
  const Part pt = partition(n, sm_count, occ_t);
  ensure_workspace(ws, pt.grid, NW * CPW + 1);
  kern<<<pt.grid, TS, 0, st>>>(V, ld, n, c, w, pt.rpb, ws.partials.get(), ws.tickets.get(), out);
  PPA_CUDA(cudaGetLastError());
}

template <int CPW>
void launch_cgs2(double* V, long long ld, int n, int c, double* w, double* Hcol, int* flag,
                 ReduceWorkspace& ws, int sm_count, cudaStream_t st) {
  constexpr int QP = CPW <= 4 ? 2 : 1;
  launch_mdot<CPW>(V, ld, n, c, w, ws.scalars.get() + kScalH1, false, ws, sm_count, st);
  static const int occ_u = occupancy_of(k_cgs_update<CPW, QP, 0>);
  const Part pu = partition(n, sm_count, occ_u);
  ensure_workspace(ws, pu.grid, NW * CPW + 1);
  double* scal = ws.scalars.get();
  k_cgs_update<CPW, QP, 0><<<pu.grid, TS, 0, st>>>(V, ld, n, c, w, scal + kScalH1, pu.rpb,
                                                   ws.partials.get(), ws.tickets.get(), scal,
                                                   Hcol, flag, nullptr);
  static const int occ_s = occupancy_of(k_cgs_store<CPW, QP>);
  const Part ps = partition(n, sm_count, occ_s);
  k_cgs_store<CPW, QP><<<ps.grid, TS, 0, st>>>(V, ld, n, c, w, ps.rpb, scal, flag);
  PPA_CUDA(cudaGetLastError());
}

template <int CPW>
void launch_cgs1(const double* V, long long ld, int n, int c, double* v, double* corr,
                 double* out_norm, ReduceWorkspace& ws, int sm_count, cudaStream_t st) {
  constexpr int QP = CPW <= 4 ? 2 : 1;
  launch_mdot<CPW>(V, ld, n, c, v, corr, false, ws, sm_count, st);
  static const int occ_u = occupancy_of(k_cgs_update<CPW, QP, 1>);
  const Part pu = partition(n, sm_count, occ_u);
  ensure_workspace(ws, pu.grid, NW * CPW + 1);
  k_cgs_update<CPW, QP, 1><<<pu.grid, TS, 0, st>>>(V, ld, n, c, v, corr, pu.rpb,
                                                   ws.partials.get(), ws.tickets.get(), nullptr,
                                                   nullptr, nullptr, out_norm);
  PPA_CUDA(cudaGetLastError());
}

void check_cols(int c, const char* who) {
  if (c < 1 || c > kMaxCols) {
    throw std::invalid_argument(std::string(who) + ": column count out of range [1,128]");
  }
}

}  // namespace

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

#define PPA_CPW_DISPATCH(c, CALL) \
  do {                                  \
    if ((c) <= 8) { CALL(1); }          \
    else if ((c) <= 16) { CALL(2); }    \
    else if ((c) <= 32) { CALL(4); }    \
    else if ((c) <= 64) { CALL(8); }    \
    else { CALL(16); }                  \
  } while (0)

void ts_dot(const double* V, long long ld, int n, int c, const double* w, double* out,
            ReduceWorkspace& ws, int sm_count, cudaStream_t st) {
  check_cols(c, "ts_dot");
  check_aligned(V, "ts_dot");
  check_aligned(w, "ts_dot");
#define CALL(K) launch_mdot<K>(V, ld, n, c, w, out, false, ws, sm_count, st)
  PPA_CPW_DISPATCH(c, CALL);
#undef CALL
}

void cgs2_step(double* V, long long ld, int n, int c, double* w, double* Hcol, int* flag,
               ReduceWorkspace& ws, int sm_count, cudaStream_t st) {
  check_cols(c, "cgs2_step");
  check_aligned(V, "cgs2_step");
  check_aligned(w, "cgs2_step");
  if (ld % 2) throw std::invalid_argument("cgs2_step: ld must be even");
#define CALL(K) launch_cgs2<K>(V, ld, n, c, w, Hcol, flag, ws, sm_count, st)
  PPA_CPW_DISPATCH(c, CALL);
#undef CALL
}

void cgs1_pass(const double* V, long long ld, int n, int c, double* v, double* corr,
               double* out_norm, ReduceWorkspace& ws, int sm_count, cudaStream_t st) {
  check_cols(c, "cgs1_pass");
  check_aligned(V, "cgs1_pass");
  check_aligned(v, "cgs1_pass");
#define CALL(K) launch_cgs1<K>(V, ld, n, c, v, corr, out_norm, ws, sm_count, st)
  PPA_CPW_DISPATCH(c, CALL);
#undef CALL
}

void col_sumsq(const double* Y, long long ld, int n, int p, double* out, ReduceWorkspace& ws,
               int sm_count, cudaStream_t st) {
  check_cols(p, "col_sumsq");
  check_aligned(Y, "col_sumsq");
#define CALL(K) launch_mdot<K>(Y, ld, n, p, nullptr, out, true, ws, sm_count, st)
  PPA_CPW_DISPATCH(p, CALL);
#undef CALL
}

void ts_combine(const double* V, long long ldv, int n, int d, const double* G, int p, double* Out,
                long long ldo, cudaStream_t st) {
  if (n <= 0 || p <= 0) return;
  if (d < 1) throw std::invalid_argument("ts_combine: d < 1");
  if (Out == V && p > d) throw std::invalid_argument("ts_combine: in-place needs p <= d");
  const size_t smem = (static_cast<size_t>(d) * kCombineRows + static_cast<size_t>(d) * p) *
                      sizeof(double);
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    PPA_CUDA(cudaFuncSetAttribute(k_ts_combine, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(std::min<size_t>(smem, 227 * 1024))));
    configured = smem;
  }
  if (smem > 227 * 1024) throw std::invalid_argument("ts_combine: d*p too large");
  k_ts_combine<<<ceil_div(n, kCombineRows), kCombineRows, smem, st>>>(V, ldv, n, d, G, p, Out,
                                                                      ldo);
  PPA_CUDA(cudaGetLastError());
}

}  // namespace kern
}  // namespace ppa
