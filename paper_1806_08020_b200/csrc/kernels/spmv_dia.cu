// Diagonal-coded SpMV / SpMM for stencil matrices: every nonzero lies on one
// of a few diagonals (col - row in a small fixed set) and the matrix has few
// distinct values.  Config 3's 7-point Laplacian has 7 diagonals and 2
// values; configs 2 and 5 (5-point convection-diffusion) have 5 and 4.
//
// Replaces CsrMatrix::multiply (src/operators.cpp:39-48) for such matrices.
// Coded form: one byte per (row, diagonal), a code into the value table or
// kDiaAbsent where the row has no entry on that diagonal.  Row r's codes are
// contiguous (stride 4/8/16/32 bytes), one vector load per lane.
// Regular-row form (default when at least half the rows qualify): rows whose
// diagonals all carry their per-diagonal default value stream no codes at
// all - one mask bit per row - and the remaining rows (matrix boundary,
// coefficient jumps) come from a compact list with their codes.  Config 3
// then streams 2.3 MB per SpMV instead of the CSR's 424 MB; what is left is
// the x gathers and the y store.
//
// The x gathers x[r + off_j] of a warp are 32 consecutive doubles per
// diagonal (coalesced).  Diagonals are visited in increasing offset, i.e.
// increasing column, and absent entries are skipped, so each row is summed in
// the CSR's own order without FMA: bit-identical to the CPU loop.

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "pdl.cuh"
#include "spmv_epilogue.cuh"
#include "ppa/kernels.hpp"

namespace ppa {
namespace kern {
namespace {

constexpr int DW = 8;  // warps per CTA

// Diagonal offsets (warp-uniform kernel parameters).
struct DiaOffsets {
  int off[kDiaMaxDiag];
};

// Code j of a row (byte j % 4 of word j / 4), one PRMT.
__device__ __forceinline__ unsigned code_of(unsigned w, int j) {
  return __byte_perm(w, 0u, 0x4440u | static_cast<unsigned>(j & 3));
}

// Codes of one row: NW 32-bit words (4 codes each).
template <int NW>
__device__ __forceinline__ void load_codes(unsigned (&w)[NW], const unsigned* __restrict__ p) {
  if (NW == 1) {
    w[0] = __ldcs(p);
  } else if (NW == 2) {
    const uint2 v = __ldcs(reinterpret_cast<const uint2*>(p));
    w[0] = v.x;
    w[1] = v.y;
  } else {
#pragma unroll
    for (int k = 0; k < NW / 4; ++k) {
      const uint4 v = __ldcs(reinterpret_cast<const uint4*>(p) + k);
      w[4 * k] = v.x;
      w[4 * k + 1] = v.y;
      w[4 * k + 2] = v.z;
      w[4 * k + 3] = v.w;
    }
  }
}

__device__ __forceinline__ void load_table(double* tab, const double* __restrict__ dict,
                                           int ndict) {
  // entries past ndict (including kDiaAbsent's slot) are read but never used
  for (int t = threadIdx.x; t < ndict; t += blockDim.x) tab[t] = dict[t];
  __syncthreads();
}

// Gathers of row r: x[r + off_j], clamped into [0, n) so the addresses do
// not depend on the codes (entries outside the matrix are absent and their
// values are never used).  The gathers can therefore issue together with the
// code load instead of after it.
template <int ND>
__device__ __forceinline__ void dia_gather(double (&xv)[ND], int r, int n, const DiaOffsets& off,
                                           const double* __restrict__ x) {
#pragma unroll
  for (int j = 0; j < ND; ++j) xv[j] = __ldg(x + min(max(r + off.off[j], 0), n - 1));
}

// Row sum from the codes and gathered values, diagonals in increasing offset
// (= increasing column), absent entries skipped.
template <int NW>
__device__ __forceinline__ double dia_sum(const unsigned (&w)[NW], const double (&xv)[4 * NW],
                                          const double* tab) {
  double sum = 0.0;
#pragma unroll
  for (int j = 0; j < 4 * NW; ++j) {
    const unsigned c = code_of(w[j / 4], j);
    if (c != kDiaAbsent) sum = __dadd_rn(sum, __dmul_rn(tab[c], xv[j]));
  }
  return sum;
}

// Persistent warps, grid-stride over 32-row slices (all warps sweep the rows
// together, so the x lines neighbouring slices share stay cached).  The
// value table is loaded once per CTA.  Software pipeline of depth 2: while
// slice s is summed, the codes and x gathers of slice s + W are already in
// flight (their addresses depend only on the row), so every warp keeps a
// full slice of loads outstanding through its arithmetic.
// Coded path: persistent warps, grid-stride over 32-row slices (all warps
// sweep the rows together, so x lines shared by neighbouring slices stay
// cached).  The value table is loaded once per CTA.  Two-deep software
// pipeline: while slice s is summed, the codes and x gathers of slice s + W
// are in flight (gather addresses depend only on the row).
template <int MODE, bool COMPL, int NW>
__global__ void __launch_bounds__(DW * 32, 4) k_spmv_dia(
    const unsigned* __restrict__ codes, const double* __restrict__ dict, int ndict,
    const DiaOffsets off, int n, int nslices, const double* __restrict__ x, double* y,
    const EpiDev e) {
  __shared__ double tab[kDiaMaxDict + 1];
  const int lane = threadIdx.x & 31;
  const int W = gridDim.x * DW;
  int s = blockIdx.x * DW + (threadIdx.x >> 5);
  unsigned w[NW];
  double xv[4 * NW];
  pdl_trigger();
  if (s < nslices) load_codes<NW>(w, codes + (static_cast<long long>(s) * 32 + lane) * NW);
  load_table(tab, dict, ndict);
  pdl_wait();  // x is the previous factor's output
  if (s < nslices) dia_gather<4 * NW>(xv, s * 32 + lane, n, off, x);
  for (; s < nslices; s += W) {
    const int sn = s + W;
    unsigned wn[NW];
    double xn[4 * NW];
    if (sn < nslices) {
      load_codes<NW>(wn, codes + (static_cast<long long>(sn) * 32 + lane) * NW);
      dia_gather<4 * NW>(xn, sn * 32 + lane, n, off, x);
    }
    const int r = s * 32 + lane;
    const double sum = dia_sum<NW>(w, xv, tab);
    if (r < n) y[r] = epilogue<MODE, COMPL>(r, sum, x, e);
#pragma unroll
    for (int k = 0; k < NW; ++k) w[k] = wn[k];
#pragma unroll
    for (int j = 0; j < 4 * NW; ++j) xv[j] = xn[j];
  }
}

template <typename K>
int resident_ctas(K kernel) {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, DW * 32, 0) != cudaSuccess) b = 1;
  return std::max(b, 1);
}

int device_sms() {
  static const int sms = [] {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
      v = 148;
    }
    return v;
  }();
  return sms;
}

template <int MODE, bool COMPL, int NW>
void launch_dia_nw(const CsrDevice& a, const double* x, double* y, const EpiArgs& ep,
                   cudaStream_t st) {
  DiaOffsets off{};
  for (int j = 0; j < a.dia_ndiag; ++j) off.off[j] = a.dia_off[j];
  auto kernel = k_spmv_dia<MODE, COMPL, NW>;
  static const int per_sm = resident_ctas(kernel);
  const int grid = std::min((a.nslices + DW - 1) / DW, device_sms() * per_sm);
  launch_pdl(kernel, dim3(grid), dim3(DW * 32), 0, st,
             reinterpret_cast<const unsigned*>(a.dia_code), a.dia_dict, a.dia_ndict, off, a.n,
             a.nslices, x, y, epi_dev(ep));
}

// ---- regular-row form -----------------------------------------------------
// Rows whose diagonals all carry their default values (the interior of a
// constant-coefficient stencil) stream no codes at all: per 32-row slice the
// kernel reads one {regular mask, exception index} pair, gathers x, and sums
// default_j * x[r + off_j] in diagonal order.  Irregular rows (boundaries,
// coefficient jumps) read their codes from the exception list.  The sums are
// the same products in the same order as the coded path.
struct DiaRParams {
  int off[kDiaRegularMaxDiag];
  double val[kDiaRegularMaxDiag];
};

// One launch, two kinds of CTAs, one thread per row, no shared memory:
//   CTAs [0, gx)      the irregular rows, from a compact list (row index +
//                     codes, values from the L1-resident table);
//   CTAs [gx, ...)    all rows of their 512-row block, storing only the
//                     regular ones (mask bit set): default values, no codes.
// The two sets of rows are disjoint and both only read x, so they need no
// ordering; the irregular CTAs go first so their longer load chain overlaps
// the regular sweep.
constexpr int RB = 512;

// One irregular row from the exception list: codes, gathers, sum in
// diagonal order (shared by the regular-row and marching sweeps).
template <int MODE, bool COMPL, int ND>
__device__ __forceinline__ void irregular_row(const int* __restrict__ irr_rows,
                                              const unsigned char* __restrict__ irr_codes,
                                              int k, const double* __restrict__ dict,
                                              const DiaRParams& P, const double* __restrict__ x,
                                              double* y, const EpiDev& e) {
  constexpr int NW = ND <= 4 ? 1 : ND <= 8 ? 2 : 4;
  const int r = __ldg(irr_rows + k);
  unsigned ec[NW];
  load_codes<NW>(ec, reinterpret_cast<const unsigned*>(irr_codes) + static_cast<long long>(k) * NW);
  pdl_wait();  // x is the previous factor's output
  double xv[ND];
#pragma unroll
  for (int j = 0; j < ND; ++j) {
    const unsigned c = code_of(ec[j / 4], j);
    xv[j] = __ldg(x + (c != kDiaAbsent ? r + P.off[j] : r));
  }
  double sum = 0.0;
#pragma unroll
  for (int j = 0; j < ND; ++j) {
    const unsigned c = code_of(ec[j / 4], j);
    if (c != kDiaAbsent) sum = __dadd_rn(sum, __dmul_rn(__ldg(dict + c), xv[j]));
  }
  y[r] = epilogue<MODE, COMPL>(r, sum, x, e);
}


template <int MODE, bool COMPL, int ND, int RPT>
__global__ void __launch_bounds__(RB) k_spmv_diar(
    const unsigned* __restrict__ mask, const int* __restrict__ irr_rows,
    const unsigned char* __restrict__ irr_codes, int n_irr, int gx,
    const double* __restrict__ dict, const DiaRParams P, int n, const double* __restrict__ x,
    double* y, const EpiDev e) {
  pdl_trigger();
  const int bx = blockIdx.x;
  if (bx < gx) {
    const int k = bx * RB + threadIdx.x;
    if (k >= n_irr) {
      pdl_wait();
      return;
    }
    irregular_row<MODE, COMPL, ND>(irr_rows, irr_codes, k, dict, P, x, y, e);
    return;
  }
  // regular rows: RPT rows per thread, RB apart, all gathers issued first
  const int r0 = (bx - gx) * (RB * RPT) + threadIdx.x;
  unsigned m[RPT];
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int r = r0 + u * RB;
    m[u] = r < n ? __ldg(mask + (r >> 5)) : 0u;
  }
  pdl_wait();  // x is the previous factor's output
  double xv[RPT][ND];
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int r = min(r0 + u * RB, n - 1);
#pragma unroll
    for (int j = 0; j < ND; ++j) xv[u][j] = __ldg(x + min(max(r + P.off[j], 0), n - 1));
  }
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int r = r0 + u * RB;
    double sum = 0.0;
#pragma unroll
    for (int j = 0; j < ND; ++j) sum = __dadd_rn(sum, __dmul_rn(P.val[j], xv[u][j]));
    if (r < n && ((m[u] >> (r & 31)) & 1u)) y[r] = epilogue<MODE, COMPL>(r, sum, x, e);
  }
}

template <int MODE, bool COMPL, int ND, int RPT>
void launch_diar_rpt(const CsrDevice& a, const double* x, double* y, const EpiArgs& ep,
                     cudaStream_t st) {
  DiaRParams P{};
  for (int j = 0; j < a.dia_ndiag; ++j) {
    P.off[j] = a.dia_off[j];
    P.val[j] = a.dia_dflt[j];
  }
  const int gx = static_cast<int>((a.dia_nirr + RB - 1) / RB);
  const int grid = gx + (a.n + RB * RPT - 1) / (RB * RPT);
  launch_pdl(k_spmv_diar<MODE, COMPL, ND, RPT>, dim3(grid), dim3(RB), 0, st, a.dia_mask,
             a.dia_irr_rows, a.dia_irr_codes, static_cast<int>(a.dia_nirr), gx, a.dia_dict, P,
             a.n, x, y, epi_dev(ep));
}

// ---- marching form ----------------------------------------------------------
// When the outermost diagonals are +-D (a stencil's +-plane, or +-row in 2D),
// row r needs x[r - D] and x[r + D], which are the centres of rows r - D and
// r + D.  A thread that owns column c of the "plane" [0, D) and walks T
// consecutive planes, rows r_t = (q0 + t) D + c, loads the T + 2 plane values
// once and uses each up to three times, so the two outer gathers per row
// shrink to one load per row plus two per T rows.  The middle diagonals are
// gathered as in k_spmv_diar; the row sum visits the diagonals in the same
// increasing-offset order (bit-identical).  For symmetric stencils the
// centre x[r] is the middle plane value, reused by the epilogue too.  In the
// 50-factor chain (tools/spmv_ab.py, PPA_DIA_MARCH=0 turns it off): config 3
// 15.4 -> 14.5 us, config 5 11.9 -> 10.6 us, config 2 5.0 -> 4.6 us.
constexpr int MB = 256;  // threads per CTA of the marching sweep

template <int MODE, bool COMPL, int ND, int T, bool HC>
__global__ void __launch_bounds__(MB) k_spmv_diam(
    const unsigned* __restrict__ mask, const int* __restrict__ irr_rows,
    const unsigned char* __restrict__ irr_codes, int n_irr, int gx,
    const double* __restrict__ dict, const DiaRParams P, int n, int D, int G,
    const double* __restrict__ x, double* y, const EpiDev e) {
  static_assert(ND >= 3, "marching needs two outer diagonals and a middle one");
  pdl_trigger();
  const int bx = blockIdx.x;
  if (bx < gx) {
    const int k = bx * MB + threadIdx.x;
    if (k >= n_irr) {
      pdl_wait();
      return;
    }
    irregular_row<MODE, COMPL, ND>(irr_rows, irr_codes, k, dict, P, x, y, e);
    return;
  }
  // 32-bit rows: the launcher guarantees n + (T + 1) D < 2^31
  const int w = (bx - gx) * (MB / 32) + (threadIdx.x >> 5);
  const int g = w / G;
  const int c = (w - g * G) * 32 + (threadIdx.x & 31);
  const int rb = g * T * D + c;
  const bool col = c < D;
  unsigned m[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int r = rb + t * D;
    m[t] = (col && r < n) ? __ldg(mask + (r >> 5)) : 0u;
  }
  pdl_wait();  // x is the previous factor's output
  double pl[T + 2];
  double xv[T][ND - 2];
#pragma unroll
  for (int t = 0; t < T + 2; ++t) pl[t] = __ldg(x + min(max(rb + (t - 1) * D, 0), n - 1));
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int r = min(rb + t * D, n - 1);
#pragma unroll
    for (int j = 1; j < ND - 1; ++j) {
      // HC: diagonal (ND - 1) / 2 is offset 0, i.e. this row's plane value
      xv[t][j - 1] = HC && j == (ND - 1) / 2 ? pl[t + 1]
                                             : __ldg(x + min(max(r + P.off[j], 0), n - 1));
    }
  }
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int r = rb + t * D;
    double sum = __dadd_rn(0.0, __dmul_rn(P.val[0], pl[t]));
#pragma unroll
    for (int j = 1; j < ND - 1; ++j) sum = __dadd_rn(sum, __dmul_rn(P.val[j], xv[t][j - 1]));
    sum = __dadd_rn(sum, __dmul_rn(P.val[ND - 1], pl[t + 2]));
    if ((m[t] >> (r & 31)) & 1u) {
      y[r] = HC ? epilogue_x<MODE, COMPL>(r, sum, pl[t + 1], e) : epilogue<MODE, COMPL>(r, sum, x, e);
    }
  }
}

constexpr int kMarchT = 4;  // minimum planes per thread

// Marching applies when the outer diagonals are a symmetric pair +-D with
// enough columns per plane to fill warps and enough planes to walk.
bool march_applies(const CsrDevice& a) {
  static const bool enabled = [] {
    const char* v = std::getenv("PPA_DIA_MARCH");
    return !(v && v[0] == '0');
  }();
  if (!enabled || a.dia_ndiag < 3) return false;
  const int D = a.dia_off[a.dia_ndiag - 1];
  return D >= 256 && a.dia_off[0] == -D && a.n / D >= 2 * kMarchT &&
         static_cast<long long>(a.n) + 10LL * D < (1LL << 31);
}

template <int MODE, bool COMPL, int ND, int T>
void launch_diam_t(const CsrDevice& a, const double* x, double* y, const EpiArgs& ep,
                   cudaStream_t st) {
  DiaRParams P{};
  for (int j = 0; j < a.dia_ndiag; ++j) {
    P.off[j] = a.dia_off[j];
    P.val[j] = a.dia_dflt[j];
  }
  const int D = a.dia_off[ND - 1];
  const int G = (D + 31) / 32;
  const int nq = (a.n + D - 1) / D;
  const long long warps = static_cast<long long>(G) * ((nq + T - 1) / T);
  const int gx = static_cast<int>((a.dia_nirr + MB - 1) / MB);
  const int grid = gx + static_cast<int>((warps + MB / 32 - 1) / (MB / 32));
  // symmetric stencils (odd ND, offset 0 in the middle) reuse the centre
  const bool hc = (ND % 2 == 1) && a.dia_off[(ND - 1) / 2] == 0;
  auto kernel = hc ? k_spmv_diam<MODE, COMPL, ND, T, true> : k_spmv_diam<MODE, COMPL, ND, T, false>;
  launch_pdl(kernel, dim3(grid), dim3(MB), 0, st, a.dia_mask, a.dia_irr_rows, a.dia_irr_codes,
             static_cast<int>(a.dia_nirr), gx, a.dia_dict, P, a.n, D, G, x, y, epi_dev(ep));
}

// Planes per thread: 8 (config 3: 14.7 -> 14.5 us, config 5: 11.0 -> 10.6)
// while that still leaves a full wave of warps (64 per SM), else 4 (config
// 2, n = 1e6: 4.6 us with 4, 5.8 with 8).  PPA_DIA_MARCH_T=2|4|8 overrides.
template <int MODE, bool COMPL, int ND>
void launch_diam(const CsrDevice& a, const double* x, double* y, const EpiArgs& ep,
                 cudaStream_t st) {
  static const int forced = [] {
    const char* v = std::getenv("PPA_DIA_MARCH_T");
    return v ? std::atoi(v) : 0;
  }();
  const int D = a.dia_off[ND - 1];
  const long long nq = (a.n + D - 1) / D;
  const long long warps8 = static_cast<long long>((D + 31) / 32) * ((nq + 7) / 8);
  const int t = forced ? forced : warps8 >= 64LL * device_sms() ? 8 : 4;
  if (t == 2) return launch_diam_t<MODE, COMPL, ND, 2>(a, x, y, ep, st);
  if (t == 8) return launch_diam_t<MODE, COMPL, ND, 8>(a, x, y, ep, st);
  launch_diam_t<MODE, COMPL, ND, 4>(a, x, y, ep, st);
}

// Rows per thread of the regular sweep: each thread keeps RPT rows' gathers
// in flight (the kernel is latency-bound: 17.6 -> 15.4 us on config 3 and
// 15.0 -> 11.9 us on config 5 going from 1 to 3 rows), for matrices large
// enough to still fill ~4 waves of CTAs (config 2, n = 1e6, keeps 1), and
// not for wide stencils (registers).
template <int MODE, bool COMPL, int ND>
void launch_diar(const CsrDevice& a, const double* x, double* y, const EpiArgs& ep,
                 cudaStream_t st) {
  constexpr long long kRowsFor3 = 3LL * RB * 148 * 4 * 4;  // 3 rows x 4 waves x 4 CTAs/SM
  if constexpr (ND >= 3 && ND <= 8) {
    if (march_applies(a)) return launch_diam<MODE, COMPL, ND>(a, x, y, ep, st);
  }
  if constexpr (ND <= 8) {
    if (a.n >= kRowsFor3) return launch_diar_rpt<MODE, COMPL, ND, 3>(a, x, y, ep, st);
  }
  launch_diar_rpt<MODE, COMPL, ND, 1>(a, x, y, ep, st);
}

// The regular-row kernel is instantiated per diagonal count so the row sum
// is straight-line code over exactly the matrix's diagonals.
template <int MODE, bool COMPL, int ND = 1>
void launch_diar_nd(const CsrDevice& a, const double* x, double* y, const EpiArgs& ep,
                    cudaStream_t st) {
  if constexpr (ND < kDiaRegularMaxDiag) {
    if (a.dia_ndiag != ND) return launch_diar_nd<MODE, COMPL, ND + 1>(a, x, y, ep, st);
  }
  launch_diar<MODE, COMPL, ND>(a, x, y, ep, st);
}

template <int MODE, bool COMPL>
void launch_dia(const CsrDevice& a, const double* x, double* y, const EpiArgs& ep,
                cudaStream_t st) {
  if (a.dia_mask) return launch_diar_nd<MODE, COMPL>(a, x, y, ep, st);
  switch (a.dia_stride) {
    case 4: return launch_dia_nw<MODE, COMPL, 1>(a, x, y, ep, st);
    case 8: return launch_dia_nw<MODE, COMPL, 2>(a, x, y, ep, st);
    case 16: return launch_dia_nw<MODE, COMPL, 4>(a, x, y, ep, st);
    default: return launch_dia_nw<MODE, COMPL, 8>(a, x, y, ep, st);
  }
}

// Multi-RHS: each code is decoded once and applied to up to DB columns.
constexpr int DB = 8;

// One thread per row, no shared memory: gathers are unconditional (absent
// entries read row r itself) so no parameter load is predicated; only the
// accumulation is.
template <int NW>
__global__ void __launch_bounds__(256) k_spmm_dia(
    const unsigned* __restrict__ codes, const double* __restrict__ dict, const DiaOffsets off,
    int n, const double* __restrict__ Y, long long ldy, int p, double* __restrict__ AY,
    long long ldo) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  unsigned w[NW];
  load_codes<NW>(w, codes + static_cast<long long>(r) * NW);
  double sum[DB];
#pragma unroll
  for (int k = 0; k < DB; ++k) sum[k] = 0.0;
#pragma unroll
  for (int j = 0; j < 4 * NW; ++j) {
    const unsigned c = code_of(w[j / 4], j);
    const bool present = c != kDiaAbsent;
    const double v = __ldg(dict + (present ? c : 0u));
    const double* yc = Y + (present ? r + off.off[j] : r);
    double yv[DB];
#pragma unroll
    for (int k = 0; k < DB; ++k) yv[k] = k < p ? __ldg(yc + k * ldy) : 0.0;
#pragma unroll
    for (int k = 0; k < DB; ++k) {
      if (present && k < p) sum[k] = __dadd_rn(sum[k], __dmul_rn(v, yv[k]));
    }
  }
#pragma unroll
  for (int k = 0; k < DB; ++k) {
    if (k < p) AY[r + k * ldo] = sum[k];
  }
}

template <int NW>
void launch_spmm_dia_nw(const CsrDevice& a, const double* Y, long long ldy, int p, double* AY,
                        long long ldo, cudaStream_t st) {
  DiaOffsets off{};
  for (int j = 0; j < a.dia_ndiag; ++j) off.off[j] = a.dia_off[j];
  const int grid = (a.n + 255) / 256;
  for (int j0 = 0; j0 < p; j0 += DB) {
    k_spmm_dia<NW><<<grid, 256, 0, st>>>(reinterpret_cast<const unsigned*>(a.dia_code),
                                         a.dia_dict, off, a.n, Y + j0 * ldy, ldy,
                                         std::min(DB, p - j0), AY + j0 * ldo, ldo);
  }
}

}  // namespace

void spmv_dia(const CsrDevice& a, const double* x, double* y, const EpiArgs& ep,
              cudaStream_t st) {
  const bool compl_ = ep.base != nullptr;
  switch (ep.mode) {
    case Epi::plain:
      compl_ ? launch_dia<0, true>(a, x, y, ep, st) : launch_dia<0, false>(a, x, y, ep, st);
      break;
    case Epi::real:
      compl_ ? launch_dia<1, true>(a, x, y, ep, st) : launch_dia<1, false>(a, x, y, ep, st);
      break;
    case Epi::pair:
      compl_ ? launch_dia<2, true>(a, x, y, ep, st) : launch_dia<2, false>(a, x, y, ep, st);
      break;
  }
  PPA_CUDA(cudaGetLastError());
}

void spmm_dia(const CsrDevice& a, const double* Y, long long ldy, int p, double* AY,
              long long ldo, cudaStream_t st) {
  switch (a.dia_stride) {
    case 4: launch_spmm_dia_nw<1>(a, Y, ldy, p, AY, ldo, st); break;
    case 8: launch_spmm_dia_nw<2>(a, Y, ldy, p, AY, ldo, st); break;
    case 16: launch_spmm_dia_nw<4>(a, Y, ldy, p, AY, ldo, st); break;
    default: launch_spmm_dia_nw<8>(a, Y, ldy, p, AY, ldo, st); break;
  }
  PPA_CUDA(cudaGetLastError());
}

}  // namespace kern
}  // namespace ppa
