// Streaming CSR SpMV with the polynomial-factor epilogues fused in.
//
// Replaces CsrMatrix::multiply (src/operators.cpp:39-48) and the axpys of
// apply_poly (src/gmres_poly.cpp:129-143) / PolyOperator complement
// (src/gmres_poly.cpp:306-308).
//
// Layout: plain CSR in HBM (int32 row_ptr/col_idx, fp64 values), plus a
// host-built row-block partition (<= 256 rows and <= 2048 nonzeros each).
// One 256-thread CTA per row block:
//   phase 1  the block's contiguous slice of (col_idx, values) is streamed
//            with 8-/16-byte vector loads that bypass L1 (every byte of the
//            matrix is read once per SpMV), x is gathered through the
//            read-only path (x stays L2-resident: 33 MB at config 3), and
//            the products are staged in shared memory;
//   phase 2  thread t sums row t's products sequentially - the same
//            left-to-right order, without FMA contraction, as the reference's
//            scalar loop, so the SpMV is bit-identical to the CPU oracle -
//            and applies the factor epilogue with one coalesced store.
// A row longer than 2048 nonzeros gets a block of its own and a block-wide
// reduction (not bit-identical; no BASELINE config has such rows).

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "pdl.cuh"
#include "spmv_epilogue.cuh"
#include "ppa/kernels.hpp"

namespace ppa {
namespace kern {
namespace {

constexpr int T = kSpmvThreads;
constexpr int MAXR = kSpmvMaxRows;
constexpr int MAXNNZ = kSpmvMaxNnz;
// Pairs a thread may own: the slice [p0 & ~1, p1) has <= MAXNNZ + 1 elements.
constexpr int KPAIRS = ((MAXNNZ + 2) / 2 + T - 1) / T;

template <int MODE, bool COMPL>
__global__ void __launch_bounds__(T) k_spmv_rowblock(
    const int* __restrict__ row_ptr, const int* __restrict__ col_idx,
    const double* __restrict__ vals, const int* __restrict__ blk_row,
    const double* __restrict__ x, double* y, const EpiDev e) {
  __shared__ __align__(16) double prod[MAXNNZ + 2];
  __shared__ int rp[MAXR + 1];
  __shared__ double s_warp[T / 32];

  const int r0 = blk_row[blockIdx.x];
  const int r1 = blk_row[blockIdx.x + 1];
  const int nr = r1 - r0;
  for (int t = threadIdx.x; t <= nr; t += T) rp[t] = row_ptr[r0 + t];
  __syncthreads();
  const int p0 = rp[0];
  const int p1 = rp[nr];

  if (p1 - p0 <= MAXNNZ) {
    const int q0 = p0 & ~1;
    const int npairs = (p1 - q0 + 1) >> 1;
    int2 c[KPAIRS];
    double2 v[KPAIRS];
#pragma unroll
    for (int k = 0; k < KPAIRS; ++k) {
      const int pi = threadIdx.x + k * T;
      if (pi < npairs) {
        c[k] = dev::ld_stream(reinterpret_cast<const int2*>(col_idx + q0) + pi);
        v[k] = dev::ld_stream(reinterpret_cast<const double2*>(vals + q0) + pi);
      }
    }
#pragma unroll
    for (int k = 0; k < KPAIRS; ++k) {
      const int pi = threadIdx.x + k * T;
      if (pi < npairs) {
        const int q = q0 + 2 * pi;
        double a = 0.0, b = 0.0;
        if (q >= p0) a = __dmul_rn(v[k].x, __ldg(x + c[k].x));
        if (q + 1 < p1) b = __dmul_rn(v[k].y, __ldg(x + c[k].y));
        reinterpret_cast<double2*>(prod)[pi] = make_double2(a, b);
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nr; t += T) {
      const int a = rp[t] - q0;
      const int b = rp[t + 1] - q0;
      double s = 0.0;
      for (int p = a; p < b; ++p) s = __dadd_rn(s, prod[p]);
      y[r0 + t] = epilogue<MODE, COMPL>(r0 + t, s, x, e);
    }
  } else {
    // One long row (nr == 1): block-strided partial sums + fixed-order tree.
    double s = 0.0;
    for (int p = p0 + threadIdx.x; p < p1; p += T) {
      s = __dadd_rn(s, __dmul_rn(dev::ld_stream(vals + p), __ldg(x + col_idx[p])));
    }
    s = dev::warp_sum(s);
    if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0.0;
#pragma unroll
      for (int w = 0; w < T / 32; ++w) tot += s_warp[w];
      y[r0] = epilogue<MODE, COMPL>(r0, tot, x, e);
    }
  }
}

// SELL-32(-sigma): one warp per 32-row slice.  Lane l owns slice row 32s+l
// (original row perm[32s+l] when the rows were sorted by length inside
// sigma-windows, else 32s+l itself); entry k of the slice is one coalesced
// 128 B (col) + 256 B (value) request per warp, and for stencil matrices the
// x gathers of a slice column are contiguous too.  No shared memory and no
// barriers: every warp is independent, so the SM keeps many more loads in
// flight than the row-block kernel.  Padding entries (col < 0) are skipped,
// so each row is still summed left to right in the CSR's own column order
// (bit-identical to the CPU loop).
constexpr int SELL_WARPS = 8;
constexpr int SELL_UNROLL = 8;

template <int MODE, bool COMPL, bool PERM>
__global__ void __launch_bounds__(SELL_WARPS * 32) k_spmv_sell32(
    const long long* __restrict__ slice_ptr, const int* __restrict__ scol,
    const double* __restrict__ sval, const int* __restrict__ perm, int n, int nslices,
    const double* __restrict__ x, double* y, const EpiDev e) {
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int s = blockIdx.x * SELL_WARPS + (threadIdx.x >> 5);
  if (s >= nslices) {
    pdl_wait();
    return;
  }
  const int idx = s * 32 + lane;
  const int r = (PERM && idx < n) ? __ldg(perm + idx) : idx;
  const long long b0 = slice_ptr[s];
  const int width = static_cast<int>((slice_ptr[s + 1] - b0) >> 5);
  const int* cp = scol + b0 + lane;
  const double* vp = sval + b0 + lane;
  double sum = 0.0;
  pdl_wait();  // x is the previous factor's output
  for (int k0 = 0; k0 < width; k0 += SELL_UNROLL) {
    int c[SELL_UNROLL];
    double v[SELL_UNROLL];
#pragma unroll
    for (int u = 0; u < SELL_UNROLL; ++u) {
      if (k0 + u < width) {
        c[u] = __ldcs(cp + (k0 + u) * 32);
        v[u] = __ldcs(vp + (k0 + u) * 32);
      }
    }
#pragma unroll
    for (int u = 0; u < SELL_UNROLL; ++u) {
      if (k0 + u < width && c[u] >= 0) sum = __dadd_rn(sum, __dmul_rn(v[u], __ldg(x + c[u])));
    }
  }
  if (idx < n) y[r] = epilogue<MODE, COMPL>(r, sum, x, e);
}

template <int MODE, bool COMPL>
void launch(const CsrDevice& a, const double* x, double* y, const EpiArgs& ep, cudaStream_t st) {
  if (a.sell_val) {
    const int grid = (a.nslices + SELL_WARPS - 1) / SELL_WARPS;
    if (a.sell_perm) {
      launch_pdl(k_spmv_sell32<MODE, COMPL, true>, dim3(grid), dim3(SELL_WARPS * 32), 0, st,
                 a.slice_ptr, a.sell_col, a.sell_val, a.sell_perm, a.n, a.nslices, x, y, epi_dev(ep));
    } else {
      launch_pdl(k_spmv_sell32<MODE, COMPL, false>, dim3(grid), dim3(SELL_WARPS * 32), 0, st,
                 a.slice_ptr, a.sell_col, a.sell_val, static_cast<const int*>(nullptr), a.n,
                 a.nslices, x, y, epi_dev(ep));
    }
    return;
  }
  k_spmv_rowblock<MODE, COMPL><<<a.nblocks, T, 0, st>>>(a.row_ptr, a.col_idx, a.values,
                                                       a.blk_row, x, y, epi_dev(ep));
}

}  // namespace

void spmv(const CsrDevice& a, const double* x, double* y, const EpiArgs& ep, cudaStream_t st) {
  if (a.n == 0 || a.nblocks == 0) return;
  if (a.dia_code) {
    spmv_dia(a, x, y, ep, st);
    return;
  }
  if (a.pk_ptr) {
    spmv_packed(a, x, y, ep, st);
    return;
  }
  const bool compl_ = ep.base != nullptr;
  switch (ep.mode) {
    case Epi::plain:
      compl_ ? launch<0, true>(a, x, y, ep, st) : launch<0, false>(a, x, y, ep, st);
      break;
    case Epi::real:
      compl_ ? launch<1, true>(a, x, y, ep, st) : launch<1, false>(a, x, y, ep, st);
      break;
    case Epi::pair:
      compl_ ? launch<2, true>(a, x, y, ep, st) : launch<2, false>(a, x, y, ep, st);
      break;
  }
  PPA_CUDA(cudaGetLastError());
}

namespace {

// Multi-RHS SELL-32 (convergence check): each slice entry is
// loaded once and applied to PB right-hand sides; per column the row sum is
// the same left-to-right sequence as k_spmv_sell32.
constexpr int SPMM_PB = 8;

template <bool PERM>
__global__ void __launch_bounds__(SELL_WARPS * 32) k_spmm_sell32(
    const long long* __restrict__ slice_ptr, const int* __restrict__ scol,
    const double* __restrict__ sval, const int* __restrict__ perm, int n, int nslices,
    const double* __restrict__ Y, long long ldy, int p, double* __restrict__ AY, long long ldo) {
  const int lane = threadIdx.x & 31;
  const int s = blockIdx.x * SELL_WARPS + (threadIdx.x >> 5);
  if (s >= nslices) return;
  const int idx = s * 32 + lane;
  const int r = (PERM && idx < n) ? __ldg(perm + idx) : idx;
  const long long b0 = slice_ptr[s];
  const int width = static_cast<int>((slice_ptr[s + 1] - b0) >> 5);
  double sum[SPMM_PB];
#pragma unroll
  for (int j = 0; j < SPMM_PB; ++j) sum[j] = 0.0;
  for (int k = 0; k < width; ++k) {
    const int c = __ldcs(scol + b0 + 32LL * k + lane);
    const double v = __ldcs(sval + b0 + 32LL * k + lane);
    if (c < 0) continue;
#pragma unroll
    for (int j = 0; j < SPMM_PB; ++j) {
      if (j < p) sum[j] = __dadd_rn(sum[j], __dmul_rn(v, __ldg(Y + c + j * ldy)));
    }
  }
  if (idx < n) {
#pragma unroll
    for (int j = 0; j < SPMM_PB; ++j) {
      if (j < p) AY[r + j * ldo] = sum[j];
    }
  }
}

}  // namespace

void spmm(const CsrDevice& a, const double* Y, long long ldy, int p, double* AY, long long ldo,
          cudaStream_t st) {
  if (a.n == 0 || p <= 0) return;
  if (a.dia_code) {
    spmm_dia(a, Y, ldy, p, AY, ldo, st);
    return;
  }
  if (a.pk_ptr) {
    spmm_packed(a, Y, ldy, p, AY, ldo, st);
    return;
  }
  if (!a.sell_val) {
    for (int j = 0; j < p; ++j) spmv(a, Y + j * ldy, AY + j * ldo, EpiArgs{}, st);
    return;
  }
  const int grid = (a.nslices + SELL_WARPS - 1) / SELL_WARPS;
  for (int j0 = 0; j0 < p; j0 += SPMM_PB) {
    const int pb = std::min(SPMM_PB, p - j0);
    if (a.sell_perm) {
      k_spmm_sell32<true><<<grid, SELL_WARPS * 32, 0, st>>>(a.slice_ptr, a.sell_col, a.sell_val,
                                                            a.sell_perm, a.n, a.nslices,
                                                            Y + j0 * ldy, ldy, pb, AY + j0 * ldo,
                                                            ldo);
    } else {
      k_spmm_sell32<false><<<grid, SELL_WARPS * 32, 0, st>>>(a.slice_ptr, a.sell_col, a.sell_val,
                                                             nullptr, a.n, a.nslices,
                                                             Y + j0 * ldy, ldy, pb,
                                                             AY + j0 * ldo, ldo);
    }
  }
  PPA_CUDA(cudaGetLastError());
}

void build_row_blocks(const int* row_ptr, int n, int max_rows, int max_nnz,
                      std::vector<int>& blk_row) {
  blk_row.clear();
  blk_row.reserve(static_cast<size_t>(n) / 64 + 2);
  blk_row.push_back(0);
  int r = 0;
  while (r < n) {
    const int start = r;
    const int base = row_ptr[start];
    int e = start;
    while (e < n && e - start < max_rows && row_ptr[e + 1] - base <= max_nnz) ++e;
    if (e == start) e = start + 1;  // a single row longer than max_nnz
    blk_row.push_back(e);
    r = e;
  }
}

}  // namespace kern
}  // namespace ppa
