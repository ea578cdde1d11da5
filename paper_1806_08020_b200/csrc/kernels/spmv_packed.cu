// Packed SELL-32 SpMV / SpMM: the same slices, row order and per-row
// summation order as k_spmv_sell32 (spmv.cu), with a smaller matrix stream.
//
// Replaces CsrMatrix::multiply (src/operators.cpp:39-48) for matrices whose
// column offsets |col - row| fit int16 - banded and stencil matrices, which
// is every BASELINE config but the random one (C4).  Each entry is
//   column  int16 offset from its row           2 B  (CSR: 4 B)
//   value   uint8 code into a <= 256-entry table 1 B  (CSR: 8 B)
//           or the fp64 value itself when the matrix has more distinct values
// so a 7-point stencil row streams 8 x 3 = 24 B (width rounded up to 8)
// instead of 7 x 12 = 84 B.  Values are looked up exactly (the table holds
// the matrix's own fp64 bit patterns) and every row is still summed left to
// right without FMA, so results stay bit-identical to the CPU loop.
//
// Layout: lane l of slice s owns kPackChunk consecutive entries per chunk,
// so one warp-wide load moves 32 x 8 B of columns (uint2 per lane) and
// 32 x 4 B of codes (one 32-bit word per lane), 256 B + 128 B contiguous.
// One warp per slice, 8 warps per CTA, no barriers after the table load.

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "pdl.cuh"
#include "spmv_epilogue.cuh"
#include "ppa/kernels.hpp"

namespace ppa {
namespace kern {
namespace {

constexpr int PW = 8;           // warps (slices) per CTA
constexpr int KC = kPackChunk;  // entries per lane per chunk
constexpr int PU = 2;           // chunks in flight per warp

static_assert(KC == 4, "the load paths below assume 4 entries per chunk");

struct PackedChunk {
  uint2 col;      // 4 x int16 offsets
  unsigned code;  // 4 x uint8 codes (dictionary)
  double2 v01, v23;  // values (no dictionary)
};

template <bool DICT>
__device__ __forceinline__ void load_chunk(PackedChunk& c, const short* __restrict__ pcol,
                                           const unsigned char* __restrict__ pcode,
                                           const double* __restrict__ pval, long long e) {
  c.col = __ldcs(reinterpret_cast<const uint2*>(pcol + e));
  if (DICT) {
    c.code = __ldcs(reinterpret_cast<const unsigned*>(pcode + e));
  } else {
    c.v01 = __ldcs(reinterpret_cast<const double2*>(pval + e));
    c.v23 = __ldcs(reinterpret_cast<const double2*>(pval + e + 2));
  }
}

__device__ __forceinline__ int chunk_offset(const PackedChunk& c, int q) {
  const unsigned w = q < 2 ? c.col.x : c.col.y;
  return static_cast<short>((q & 1) ? (w >> 16) : (w & 0xffffu));
}

template <bool DICT>
__device__ __forceinline__ double chunk_value(const PackedChunk& c, int q, const double* tab) {
  if (DICT) return tab[(c.code >> (8 * q)) & 0xffu];
  return q == 0 ? c.v01.x : q == 1 ? c.v01.y : q == 2 ? c.v23.x : c.v23.y;
}

template <bool DICT>
__device__ __forceinline__ void load_table(double* tab, const double* __restrict__ dict,
                                           int ndict) {
  if (DICT) {
    for (int t = threadIdx.x; t < ndict; t += blockDim.x) tab[t] = dict[t];
    __syncthreads();
  }
}

template <int MODE, bool COMPL, bool PERM, bool DICT>
__global__ void __launch_bounds__(PW * 32) k_spmv_sellp(
    const long long* __restrict__ pk_ptr, const short* __restrict__ pcol,
    const unsigned char* __restrict__ pcode, const double* __restrict__ pval,
    const double* __restrict__ dict, int ndict, const int* __restrict__ perm, int n,
    int nslices, const double* __restrict__ x, double* y, const EpiDev e) {
  __shared__ double tab[DICT ? kPackMaxDict : 1];
  pdl_trigger();
  load_table<DICT>(tab, dict, ndict);
  const int lane = threadIdx.x & 31;
  const int s = blockIdx.x * PW + (threadIdx.x >> 5);
  if (s >= nslices) {
    pdl_wait();
    return;
  }
  const int idx = s * 32 + lane;
  const int r = (PERM && idx < n) ? __ldg(perm + idx) : idx;
  const long long b0 = pk_ptr[s];
  const int nch = static_cast<int>((pk_ptr[s + 1] - b0) / (32 * KC));
  const long long lb = b0 + KC * lane;
  const double* xr = x + r;
  double sum = 0.0;
  pdl_wait();  // x is the previous factor's output
  for (int j0 = 0; j0 < nch; j0 += PU) {
    PackedChunk c[PU];
#pragma unroll
    for (int u = 0; u < PU; ++u) {
      if (j0 + u < nch) load_chunk<DICT>(c[u], pcol, pcode, pval, lb + 32LL * KC * (j0 + u));
    }
#pragma unroll
    for (int u = 0; u < PU; ++u) {
      if (j0 + u < nch) {
#pragma unroll
        for (int q = 0; q < KC; ++q) {
          const int d = chunk_offset(c[u], q);
          if (d != kPackPad) {
            sum = __dadd_rn(sum, __dmul_rn(chunk_value<DICT>(c[u], q, tab), __ldg(xr + d)));
          }
        }
      }
    }
  }
  if (idx < n) y[r] = epilogue<MODE, COMPL>(r, sum, x, e);
}

template <int MODE, bool COMPL, bool PERM, bool DICT>
void launch_sellp(const CsrDevice& a, const double* x, double* y, const EpiArgs& ep,
                  cudaStream_t st) {
  const int grid = (a.nslices + PW - 1) / PW;
  launch_pdl(k_spmv_sellp<MODE, COMPL, PERM, DICT>, dim3(grid), dim3(PW * 32), 0, st, a.pk_ptr,
             a.pk_col, a.pk_code, a.pk_val, a.pk_dict, a.pk_ndict, a.sell_perm, a.n, a.nslices,
             x, y, epi_dev(ep));
}

template <int MODE, bool COMPL>
void launch_packed(const CsrDevice& a, const double* x, double* y, const EpiArgs& ep,
                   cudaStream_t st) {
  const bool perm = a.sell_perm != nullptr;
  const bool dict = a.pk_ndict > 0;
  if (perm) {
    dict ? launch_sellp<MODE, COMPL, true, true>(a, x, y, ep, st)
         : launch_sellp<MODE, COMPL, true, false>(a, x, y, ep, st);
  } else {
    dict ? launch_sellp<MODE, COMPL, false, true>(a, x, y, ep, st)
         : launch_sellp<MODE, COMPL, false, false>(a, x, y, ep, st);
  }
}

// Multi-RHS variant (convergence check): each packed entry is decoded once
// and applied to up to PB right-hand sides, column sums in the same order.
constexpr int PB = 8;

template <bool PERM, bool DICT>
__global__ void __launch_bounds__(PW * 32) k_spmm_sellp(
    const long long* __restrict__ pk_ptr, const short* __restrict__ pcol,
    const unsigned char* __restrict__ pcode, const double* __restrict__ pval,
    const double* __restrict__ dict, int ndict, const int* __restrict__ perm, int n,
    int nslices, const double* __restrict__ Y, long long ldy, int p, double* __restrict__ AY,
    long long ldo) {
  __shared__ double tab[DICT ? kPackMaxDict : 1];
  load_table<DICT>(tab, dict, ndict);
  const int lane = threadIdx.x & 31;
  const int s = blockIdx.x * PW + (threadIdx.x >> 5);
  if (s >= nslices) return;
  const int idx = s * 32 + lane;
  const int r = (PERM && idx < n) ? __ldg(perm + idx) : idx;
  const long long b0 = pk_ptr[s];
  const int nch = static_cast<int>((pk_ptr[s + 1] - b0) / (32 * KC));
  double sum[PB];
#pragma unroll
  for (int j = 0; j < PB; ++j) sum[j] = 0.0;
  for (int ch = 0; ch < nch; ++ch) {
    PackedChunk c;
    load_chunk<DICT>(c, pcol, pcode, pval, b0 + KC * lane + 32LL * KC * ch);
#pragma unroll
    for (int q = 0; q < KC; ++q) {
      const int d = chunk_offset(c, q);
      if (d == kPackPad) continue;
      const double v = chunk_value<DICT>(c, q, tab);
      const double* yc = Y + r + d;
#pragma unroll
      for (int j = 0; j < PB; ++j) {
        if (j < p) sum[j] = __dadd_rn(sum[j], __dmul_rn(v, __ldg(yc + j * ldy)));
      }
    }
  }
  if (idx < n) {
#pragma unroll
    for (int j = 0; j < PB; ++j) {
      if (j < p) AY[r + j * ldo] = sum[j];
    }
  }
}

}  // namespace

void spmv_packed(const CsrDevice& a, const double* x, double* y, const EpiArgs& ep,
                 cudaStream_t st) {
  const bool compl_ = ep.base != nullptr;
  switch (ep.mode) {
    case Epi::plain:
      compl_ ? launch_packed<0, true>(a, x, y, ep, st) : launch_packed<0, false>(a, x, y, ep, st);
      break;
    case Epi::real:
      compl_ ? launch_packed<1, true>(a, x, y, ep, st) : launch_packed<1, false>(a, x, y, ep, st);
      break;
    case Epi::pair:
      compl_ ? launch_packed<2, true>(a, x, y, ep, st) : launch_packed<2, false>(a, x, y, ep, st);
      break;
  }
  PPA_CUDA(cudaGetLastError());
}

void spmm_packed(const CsrDevice& a, const double* Y, long long ldy, int p, double* AY,
                 long long ldo, cudaStream_t st) {
  const int grid = (a.nslices + PW - 1) / PW;
  const bool perm = a.sell_perm != nullptr;
  const bool dict = a.pk_ndict > 0;
  for (int j0 = 0; j0 < p; j0 += PB) {
    const int pb = std::min(PB, p - j0);
#define PPA_SPMMP(P, D)                                                                        \
  k_spmm_sellp<P, D><<<grid, PW * 32, 0, st>>>(a.pk_ptr, a.pk_col, a.pk_code, a.pk_val,        \
                                               a.pk_dict, a.pk_ndict, a.sell_perm, a.n,        \
                                               a.nslices, Y + j0 * ldy, ldy, pb,               \
                                               AY + j0 * ldo, ldo)
    if (perm) {
      dict ? PPA_SPMMP(true, true) : PPA_SPMMP(true, false);
    } else {
      dict ? PPA_SPMMP(false, true) : PPA_SPMMP(false, false);
    }
#undef PPA_SPMMP
  }
  PPA_CUDA(cudaGetLastError());
}

bool build_sell32_packed(const int* row_ptr, const int* col_idx, const double* values, int n,
                         const std::vector<int>& perm, long long sell_entries,
                         std::vector<long long>& pk_ptr, std::vector<short>& cols,
                         std::vector<unsigned char>& codes, std::vector<double>& vals,
                         std::vector<double>& dict) {
  pk_ptr.clear();
  cols.clear();
  codes.clear();
  vals.clear();
  dict.clear();
  const int ns = (n + 31) / 32;
  auto row_of = [&](int i) { return perm.empty() ? i : perm[i]; };
  auto len = [&](int r) { return row_ptr[r + 1] - row_ptr[r]; };
  // offsets must fit int16 (kPackPad is reserved for padding)
  for (int r = 0; r < n; ++r) {
    for (int p = row_ptr[r]; p < row_ptr[r + 1]; ++p) {
      const long long d = static_cast<long long>(col_idx[p]) - r;
      if (d < -32767 || d > 32767) return false;
    }
  }
  // value dictionary over exact bit patterns, in first-seen order
  std::unordered_map<uint64_t, int> index;
  const long long nnz = row_ptr[n];
  for (long long p = 0; p < nnz; ++p) {
    uint64_t bits;
    std::memcpy(&bits, values + p, sizeof bits);
    if (index.count(bits)) continue;
    if (static_cast<int>(index.size()) == kPackMaxDict) {
      index.clear();
      dict.clear();
      break;
    }
    index.emplace(bits, static_cast<int>(dict.size()));
    dict.push_back(values[p]);
  }
  const bool use_dict = !dict.empty();
  pk_ptr.assign(static_cast<size_t>(ns) + 1, 0);
  long long total = 0;
  for (int s = 0; s < ns; ++s) {
    int w = 0;
    for (int i = s * 32; i < std::min(n, s * 32 + 32); ++i) w = std::max(w, len(row_of(i)));
    w = (w + KC - 1) / KC * KC;
    total += 32LL * w;
    pk_ptr[s + 1] = total;
  }
  const double packed = static_cast<double>(total) * packed_entry_bytes(use_dict ? 1 : 0);
  if (packed >= 12.0 * static_cast<double>(sell_entries)) {
    pk_ptr.clear();
    dict.clear();
    return false;
  }
  cols.assign(static_cast<size_t>(total), kPackPad);
  if (use_dict) {
    codes.assign(static_cast<size_t>(total), 0);
  } else {
    vals.assign(static_cast<size_t>(total), 0.0);
  }
  for (int s = 0; s < ns; ++s) {
    const long long b0 = pk_ptr[s];
    for (int l = 0; l < 32; ++l) {
      const int i = s * 32 + l;
      if (i >= n) break;
      const int r = row_of(i);
      for (int p = row_ptr[r], k = 0; p < row_ptr[r + 1]; ++p, ++k) {
        const long long e = b0 + 32LL * KC * (k / KC) + KC * l + k % KC;
        cols[e] = static_cast<short>(col_idx[p] - r);
        if (use_dict) {
          uint64_t bits;
          std::memcpy(&bits, values + p, sizeof bits);
          codes[e] = static_cast<unsigned char>(index.at(bits));
        } else {
          vals[e] = values[p];
        }
      }
    }
  }
  return true;
}

}  // namespace kern
}  // namespace ppa
