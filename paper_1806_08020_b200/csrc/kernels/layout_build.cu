// Device-side construction of the SpMV layouts from the device CSR copy
// ("device CSR -> SELL-C-sigma conversion").  Replaces
// the host loops that built SELL-32 and the diagonal-coded form entry by
// entry (0.3 s and 0.7 s at config 3, 3.5x the solve itself); each layout
// here is a handful of O(nnz) kernels plus CUB scans / sorts / selects, and
// only table-sized results (offsets, distinct values, counts) visit the
// host.  The arrays are the ones the host builders produced: same slice
// order (stable length sort inside sigma windows), same padding, same code
// per (row, diagonal) up to the numbering of the value dictionary, which
// here is ascending by bit pattern (results do not depend on it).

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include "common.cuh"
#include "ppa/device.hpp"
#include "ppa/kernels.hpp"

namespace ppa {
namespace kern {
namespace {

// Stream-ordered temporary (CUB workspaces, flags).
struct Tmp {
  void* p = nullptr;
  cudaStream_t st;
  Tmp(size_t bytes, cudaStream_t s) : st(s) {
    if (bytes) PPA_CUDA(cudaMallocAsync(&p, bytes, st));
  }
  ~Tmp() {
    if (p) cudaFreeAsync(p, st);
  }
  Tmp(const Tmp&) = delete;
  Tmp& operator=(const Tmp&) = delete;
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

inline int blocks_for(long long n, int t) { return static_cast<int>(std::max(1LL, (n + t - 1) / t)); }

// ---------------------------------------------------------------- SELL-32 --
__global__ void k_row_len(const int* __restrict__ row_ptr, int n, int* __restrict__ len,
                          int* __restrict__ iota) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) {
    len[r] = row_ptr[r + 1] - row_ptr[r];
    if (iota) iota[r] = r;
  }
}

__global__ void k_window_offsets(int* __restrict__ off, int nwin, int sigma, int n) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w <= nwin) off[w] = static_cast<int>(min(static_cast<long long>(w) * sigma,
                                               static_cast<long long>(n)));
}

// one warp per slice: 32 * (longest row of the slice)
__global__ void k_slice_size(const int* __restrict__ row_ptr, const int* __restrict__ perm, int n,
                             int ns, long long* __restrict__ size) {
  const int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s > ns) return;
  int w = 0;
  const int i = s * 32 + lane;
  if (s < ns && i < n) {
    const int r = perm ? perm[i] : i;
    w = row_ptr[r + 1] - row_ptr[r];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) w = max(w, __shfl_xor_sync(0xffffffffu, w, o));
  if (lane == 0) size[s] = s < ns ? 32LL * w : 0LL;
}

// one thread per slice row: its entries (padding: col -1, value 0)
__global__ void k_sell_fill(const int* __restrict__ row_ptr, const int* __restrict__ col_idx,
                            const double* __restrict__ values, const int* __restrict__ perm,
                            int n, int ns, const long long* __restrict__ slice_ptr,
                            int* __restrict__ cols, double* __restrict__ vals) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int s = static_cast<int>(i >> 5), l = static_cast<int>(i & 31);
  if (s >= ns) return;
  const long long b0 = slice_ptr[s];
  const int width = static_cast<int>((slice_ptr[s + 1] - b0) >> 5);
  int p = 0, e = 0;
  if (i < n) {
    const int r = perm ? perm[i] : static_cast<int>(i);
    p = row_ptr[r];
    e = row_ptr[r + 1];
  }
  for (int k = 0; k < width; ++k, ++p) {
    const bool live = p < e;
    cols[b0 + 32LL * k + l] = live ? col_idx[p] : -1;
    vals[b0 + 32LL * k + l] = live ? values[p] : 0.0;
  }
}

// ---------------------------------------------------------- diagonal form --
constexpr int kOffSlots = 128;   // open-addressing table of diagonal offsets
constexpr int kValSlots = 1024;  // open-addressing table of value bit patterns
constexpr long long kEmptyOff = static_cast<long long>(0x8000000000000000ULL);
constexpr unsigned long long kEmptyVal = 0xfff8dead0000beefULL;  // a NaN payload no input uses

__device__ __forceinline__ unsigned hash64(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  return static_cast<unsigned>(k);
}

// Insert (or find) key; returns the slot or -1 when the table is full.
template <int SLOTS>
__device__ int table_insert(unsigned long long* keys, unsigned long long key,
                            unsigned long long empty) {
  unsigned h = hash64(key) & (SLOTS - 1);
  for (int probe = 0; probe < SLOTS; ++probe, h = (h + 1) & (SLOTS - 1)) {
    const unsigned long long cur = keys[h];
    if (cur == key) return static_cast<int>(h);
    if (cur == empty) {
      const unsigned long long old = atomicCAS(keys + h, empty, key);
      if (old == empty || old == key) return static_cast<int>(h);
    }
  }
  return -1;
}

template <int SLOTS>
__device__ int table_find(const unsigned long long* keys, unsigned long long key,
                          unsigned long long empty) {
  unsigned h = hash64(key) & (SLOTS - 1);
  for (int probe = 0; probe < SLOTS; ++probe, h = (h + 1) & (SLOTS - 1)) {
    const unsigned long long cur = keys[h];
    if (cur == key) return static_cast<int>(h);
    if (cur == empty) return -1;
  }
  return -1;
}

// Distinct diagonal offsets (with counts) and distinct value bit patterns:
// per-CTA shared tables merged into global ones; `full` flags overflow.
__global__ void __launch_bounds__(256) k_dia_scan(const int* __restrict__ row_ptr,
                                                  const int* __restrict__ col_idx,
                                                  const double* __restrict__ values, int n,
                                                  unsigned long long* g_off,
                                                  unsigned long long* g_cnt,
                                                  unsigned long long* g_val, int* full) {
  __shared__ unsigned long long s_off[kOffSlots];
  __shared__ unsigned long long s_cnt[kOffSlots];
  __shared__ unsigned long long s_val[kValSlots];
  __shared__ int s_full;
  for (int k = threadIdx.x; k < kOffSlots; k += blockDim.x) {
    s_off[k] = static_cast<unsigned long long>(kEmptyOff);
    s_cnt[k] = 0;
  }
  for (int k = threadIdx.x; k < kValSlots; k += blockDim.x) s_val[k] = kEmptyVal;
  if (threadIdx.x == 0) s_full = 0;
  __syncthreads();
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    for (int p = row_ptr[r]; p < row_ptr[r + 1]; ++p) {
      const long long off = static_cast<long long>(col_idx[p]) - r;
      const int so = table_insert<kOffSlots>(s_off, static_cast<unsigned long long>(off),
                                             static_cast<unsigned long long>(kEmptyOff));
      if (so < 0) {
        s_full = 1;
      } else {
        atomicAdd(s_cnt + so, 1ULL);
      }
      unsigned long long bits;
      const double v = values[p];
      memcpy(&bits, &v, sizeof bits);
      // the empty marker itself cannot be tabled: such a matrix is not coded
      if (bits == kEmptyVal || table_insert<kValSlots>(s_val, bits, kEmptyVal) < 0) s_full = 1;
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < kOffSlots; k += blockDim.x) {
    if (s_off[k] != static_cast<unsigned long long>(kEmptyOff)) {
      const int g = table_insert<kOffSlots>(g_off, s_off[k],
                                            static_cast<unsigned long long>(kEmptyOff));
      if (g < 0) {
        atomicExch(full, 1);
      } else {
        atomicAdd(g_cnt + g, s_cnt[k]);
      }
    }
  }
  for (int k = threadIdx.x; k < kValSlots; k += blockDim.x) {
    if (s_val[k] != kEmptyVal && table_insert<kValSlots>(g_val, s_val[k], kEmptyVal) < 0) {
      atomicExch(full, 1);
    }
  }
  if (threadIdx.x == 0 && s_full) atomicExch(full, 1);
}

struct DiaTables {
  int off[kDiaMaxDiag];
  int ndiag;
};

// codes[r*stride + j] for every entry (the array is pre-filled with
// kDiaAbsent); value codes from the global table's slot -> code map
__global__ void k_dia_codes(const int* __restrict__ row_ptr, const int* __restrict__ col_idx,
                            const double* __restrict__ values, int n, const DiaTables t,
                            const unsigned long long* __restrict__ g_val,
                            const unsigned char* __restrict__ slot_code, int stride,
                            unsigned char* __restrict__ codes) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int p = row_ptr[r]; p < row_ptr[r + 1]; ++p) {
    const int off = col_idx[p] - r;
    int j = 0;
    while (j < t.ndiag && t.off[j] != off) ++j;
    unsigned long long bits;
    const double v = values[p];
    memcpy(&bits, &v, sizeof bits);
    const int s = table_find<kValSlots>(g_val, bits, kEmptyVal);
    codes[static_cast<long long>(r) * stride + j] = slot_code[s];
  }
}

// per-diagonal histogram of codes (shared-memory bins, merged once per CTA)
__global__ void __launch_bounds__(256) k_dia_hist(const unsigned char* __restrict__ codes, int n,
                                                  int ndiag, int stride,
                                                  unsigned long long* __restrict__ hist) {
  __shared__ unsigned s_h[kDiaRegularMaxDiag * 256];
  for (int k = threadIdx.x; k < ndiag * 256; k += blockDim.x) s_h[k] = 0;
  __syncthreads();
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    for (int j = 0; j < ndiag; ++j) atomicAdd(s_h + j * 256 + codes[static_cast<long long>(r) * stride + j], 1u);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < ndiag * 256; k += blockDim.x) {
    if (s_h[k]) atomicAdd(hist + k, static_cast<unsigned long long>(s_h[k]));
  }
}

struct DiaDefaults {
  unsigned char code[kDiaRegularMaxDiag];
  int ndiag;
};

// regular flag per row, mask word per 32 rows (ballot), irregular flags
__global__ void k_dia_regular(const unsigned char* __restrict__ codes, int n, int stride,
                              const DiaDefaults d, unsigned* __restrict__ mask,
                              unsigned char* __restrict__ irregular) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int words = (n + 31) / 32;
  if ((i >> 5) >= words) return;
  bool reg = false;
  if (i < n) {
    reg = true;
    for (int j = 0; j < d.ndiag; ++j) reg = reg && codes[i * stride + j] == d.code[j];
    irregular[i] = reg ? 0 : 1;
  }
  const unsigned b = __ballot_sync(0xffffffffu, reg);
  if ((threadIdx.x & 31) == 0) mask[i >> 5] = b;
}

// presence byte per row (bit j: an entry on diagonal j); *bad set when a
// present entry differs from its diagonal's default code
__global__ void k_dia_presence(const unsigned char* __restrict__ codes, int n, int stride,
                               const DiaDefaults d, unsigned char* __restrict__ pres,
                               int* __restrict__ bad) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned b = 0;
  bool ok = true;
  for (int j = 0; j < d.ndiag; ++j) {
    const unsigned c = codes[i * stride + j];
    if (c != kDiaAbsent) {
      b |= 1u << j;
      ok = ok && c == d.code[j];
    }
  }
  pres[i] = static_cast<unsigned char>(b);
  if (!ok) atomicOr(bad, 1);
}

// Counts the rows whose presence byte differs from the geometric presence of
// a box-grid stencil: nd = 7: offsets (-nx ny, -nx, -1, 0, 1, nx, nx ny) on an
// nx x ny x nz grid; nd = 5: (-nx, -1, 0, 1, nx) on nx x nz.  Diagonal j is
// present exactly when its neighbour lies inside the box (Dirichlet cut).
__global__ void k_grid_check(const unsigned char* __restrict__ pres, int n, int nd, int nx,
                             int ny, int nz, int* __restrict__ bad) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int x = static_cast<int>(i % nx);
  const long long rest = i / nx;
  unsigned want;
  if (nd == 7) {
    const int y = static_cast<int>(rest % ny);
    const int z = static_cast<int>(rest / ny);
    want = (z > 0 ? 1u : 0u) | (y > 0 ? 2u : 0u) | (x > 0 ? 4u : 0u) | 8u |
           (x < nx - 1 ? 16u : 0u) | (y < ny - 1 ? 32u : 0u) | (z < nz - 1 ? 64u : 0u);
  } else {
    const int z = static_cast<int>(rest);
    want = (z > 0 ? 1u : 0u) | (x > 0 ? 2u : 0u) | 4u | (x < nx - 1 ? 8u : 0u) |
           (z < nz - 1 ? 16u : 0u);
  }
  if (pres[i] != want) atomicAdd(bad, 1);
}

__global__ void k_gather_codes(const unsigned char* __restrict__ codes, const int* __restrict__ rows,
                               long long nrows, int stride, unsigned char* __restrict__ out) {
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= nrows * stride) return;
  const long long row = k / stride, j = k - row * stride;
  out[k] = codes[static_cast<long long>(rows[row]) * stride + j];
}

}  // namespace

// ------------------------------------------------------------------ SELL --
bool build_sell32_device(const int* row_ptr, const int* col_idx, const double* values, int n,
                         long long nnz, int sigma, DevSell& out, cudaStream_t st) {
  const int ns = (n + 31) / 32;
  out.perm.release();
  Tmp len(static_cast<size_t>(std::max(n, 1)) * sizeof(int), st);
  if (sigma > 1) {
    // stable descending length sort inside sigma windows (radix sort is stable)
    Tmp iota(static_cast<size_t>(std::max(n, 1)) * sizeof(int), st);
    Tmp len_sorted(static_cast<size_t>(std::max(n, 1)) * sizeof(int), st);
    const int nwin = (n + sigma - 1) / sigma;
    Tmp woff(static_cast<size_t>(nwin + 1) * sizeof(int), st);
    out.perm.resize(static_cast<size_t>(n));
    k_row_len<<<blocks_for(n, 256), 256, 0, st>>>(row_ptr, n, len.as<int>(), iota.as<int>());
    k_window_offsets<<<blocks_for(nwin + 1, 256), 256, 0, st>>>(woff.as<int>(), nwin, sigma, n);
    size_t bytes = 0;
    PPA_CUDA(cub::DeviceSegmentedRadixSort::SortPairsDescending(
        nullptr, bytes, len.as<int>(), len_sorted.as<int>(), iota.as<int>(), out.perm.get(), n,
        nwin, woff.as<int>(), woff.as<int>() + 1, 0, 32, st));
    Tmp ws(bytes, st);
    PPA_CUDA(cub::DeviceSegmentedRadixSort::SortPairsDescending(
        ws.p, bytes, len.as<int>(), len_sorted.as<int>(), iota.as<int>(), out.perm.get(), n,
        nwin, woff.as<int>(), woff.as<int>() + 1, 0, 32, st));
  }
  const int* perm = sigma > 1 ? out.perm.get() : nullptr;
  Tmp size(static_cast<size_t>(ns + 1) * sizeof(long long), st);
  out.slice_ptr.resize(static_cast<size_t>(ns) + 1);
  k_slice_size<<<blocks_for(32LL * (ns + 1), 256), 256, 0, st>>>(row_ptr, perm, n, ns,
                                                                  size.as<long long>());
  size_t bytes = 0;
  PPA_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, size.as<long long>(),
                                         out.slice_ptr.get(), ns + 1, st));
  {
    Tmp ws(bytes, st);
    PPA_CUDA(cub::DeviceScan::ExclusiveSum(ws.p, bytes, size.as<long long>(),
                                           out.slice_ptr.get(), ns + 1, st));
  }
  long long total = 0;
  PPA_CUDA(cudaMemcpyAsync(&total, out.slice_ptr.get() + ns, sizeof total,
                           cudaMemcpyDeviceToHost, st));
  PPA_CUDA(cudaStreamSynchronize(st));
  if (static_cast<double>(total) > kSellMaxPadding * static_cast<double>(nnz) + 32.0 * 64) {
    out.slice_ptr.release();
    out.perm.release();
    return false;
  }
  out.total = total;
  out.nslices = ns;
  out.cols.resize(static_cast<size_t>(total) + 32);
  out.vals.resize(static_cast<size_t>(total) + 32);
  if (ns > 0) {
    k_sell_fill<<<blocks_for(32LL * ns, 256), 256, 0, st>>>(row_ptr, col_idx, values, perm, n, ns,
                                                            out.slice_ptr.get(), out.cols.get(),
                                                            out.vals.get());
    PPA_CUDA(cudaGetLastError());
  }
  return true;
}

// ------------------------------------------------------------- diagonals --
bool build_dia_device(const int* row_ptr, const int* col_idx, const double* values, int n,
                      long long nnz, bool want_regular, DevDia& out, cudaStream_t st) {
  if (n <= 0 || nnz <= 0) return false;
  // distinct offsets / values
  Tmp t_off(kOffSlots * sizeof(unsigned long long), st), t_cnt(kOffSlots * sizeof(unsigned long long), st);
  Tmp t_val(kValSlots * sizeof(unsigned long long), st), t_full(sizeof(int), st);
  {
    std::vector<unsigned long long> eo(kOffSlots, static_cast<unsigned long long>(kEmptyOff));
    std::vector<unsigned long long> ev(kValSlots, kEmptyVal);
    PPA_CUDA(cudaMemcpyAsync(t_off.p, eo.data(), eo.size() * 8, cudaMemcpyHostToDevice, st));
    PPA_CUDA(cudaMemcpyAsync(t_val.p, ev.data(), ev.size() * 8, cudaMemcpyHostToDevice, st));
    PPA_CUDA(cudaMemsetAsync(t_cnt.p, 0, kOffSlots * 8, st));
    PPA_CUDA(cudaMemsetAsync(t_full.p, 0, sizeof(int), st));
    const int grid = std::min(blocks_for(n, 256), 148 * 8);
    k_dia_scan<<<grid, 256, 0, st>>>(row_ptr, col_idx, values, n, t_off.as<unsigned long long>(),
                                     t_cnt.as<unsigned long long>(),
                                     t_val.as<unsigned long long>(), t_full.as<int>());
    PPA_CUDA(cudaGetLastError());
  }
  std::vector<unsigned long long> h_off(kOffSlots), h_cnt(kOffSlots), h_val(kValSlots);
  int full = 0;
  PPA_CUDA(cudaMemcpyAsync(h_off.data(), t_off.p, kOffSlots * 8, cudaMemcpyDeviceToHost, st));
  PPA_CUDA(cudaMemcpyAsync(h_cnt.data(), t_cnt.p, kOffSlots * 8, cudaMemcpyDeviceToHost, st));
  PPA_CUDA(cudaMemcpyAsync(h_val.data(), t_val.p, kValSlots * 8, cudaMemcpyDeviceToHost, st));
  PPA_CUDA(cudaMemcpyAsync(&full, t_full.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  PPA_CUDA(cudaStreamSynchronize(st));
  if (full) return false;
  std::vector<long long> offs;
  for (int k = 0; k < kOffSlots; ++k) {
    if (h_off[k] != static_cast<unsigned long long>(kEmptyOff)) offs.push_back(static_cast<long long>(h_off[k]));
  }
  std::vector<unsigned long long> vals;
  std::vector<int> val_slot;
  for (int k = 0; k < kValSlots; ++k) {
    if (h_val[k] != kEmptyVal) vals.push_back(h_val[k]);
  }
  const int nd = static_cast<int>(offs.size());
  if (nd > kDiaMaxDiag || static_cast<int>(vals.size()) > kDiaMaxDict) return false;
  // every diagonal must be well filled (absent entries still stream codes)
  if (static_cast<double>(nd) * n > kDiaMaxFill * static_cast<double>(nnz)) return false;
  std::sort(offs.begin(), offs.end());
  std::sort(vals.begin(), vals.end());
  std::vector<unsigned char> slot_code(kValSlots, 0);
  for (int k = 0; k < kValSlots; ++k) {
    if (h_val[k] == kEmptyVal) continue;
    slot_code[k] = static_cast<unsigned char>(
        std::lower_bound(vals.begin(), vals.end(), h_val[k]) - vals.begin());
  }
  const int stride = nd <= 4 ? 4 : nd <= 8 ? 8 : nd <= 16 ? 16 : 32;
  out.ndiag = nd;
  out.stride = stride;
  out.offsets.assign(offs.begin(), offs.end());
  out.dict.resize(vals.size());
  for (size_t k = 0; k < vals.size(); ++k) std::memcpy(&out.dict[k], &vals[k], sizeof(double));
  // codes
  const long long rows = (static_cast<long long>(n) + 31) / 32 * 32;
  out.codes.resize(static_cast<size_t>(rows * stride));
  PPA_CUDA(cudaMemsetAsync(out.codes.get(), static_cast<int>(kDiaAbsent),
                           static_cast<size_t>(rows * stride), st));
  {
    Tmp sc(kValSlots, st);
    PPA_CUDA(cudaMemcpyAsync(sc.p, slot_code.data(), kValSlots, cudaMemcpyHostToDevice, st));
    DiaTables t{};
    t.ndiag = nd;
    for (int j = 0; j < nd; ++j) t.off[j] = static_cast<int>(offs[j]);
    k_dia_codes<<<blocks_for(n, 256), 256, 0, st>>>(row_ptr, col_idx, values, n, t,
                                                    t_val.as<unsigned long long>(),
                                                    sc.as<unsigned char>(), stride,
                                                    out.codes.get());
    PPA_CUDA(cudaGetLastError());
    PPA_CUDA(cudaStreamSynchronize(st));  // slot_code lives on this frame
  }
  out.nirr = 0;
  out.regular = false;
  if (!want_regular || nd > kDiaRegularMaxDiag) return true;
  // default code of each diagonal: its most frequent present code
  std::vector<unsigned long long> hist(static_cast<size_t>(nd) * 256);
  {
    Tmp th(hist.size() * 8, st);
    PPA_CUDA(cudaMemsetAsync(th.p, 0, hist.size() * 8, st));
    k_dia_hist<<<std::min(blocks_for(n, 256), 148 * 8), 256, 0, st>>>(
        out.codes.get(), n, nd, stride, th.as<unsigned long long>());
    PPA_CUDA(cudaMemcpyAsync(hist.data(), th.p, hist.size() * 8, cudaMemcpyDeviceToHost, st));
    PPA_CUDA(cudaStreamSynchronize(st));
  }
  DiaDefaults d{};
  d.ndiag = nd;
  out.defaults.assign(nd, 0.0);
  for (int j = 0; j < nd; ++j) {
    unsigned long long best = 0;
    int code = -1;
    for (int c = 0; c < static_cast<int>(kDiaAbsent); ++c) {
      if (hist[static_cast<size_t>(j) * 256 + c] > best) {
        best = hist[static_cast<size_t>(j) * 256 + c];
        code = c;
      }
    }
    if (code < 0) return true;  // a diagonal with no entry at all
    d.code[j] = static_cast<unsigned char>(code);
    out.defaults[j] = out.dict[code];
  }
  const int words = (n + 31) / 32;
  out.mask.resize(static_cast<size_t>(words));
  Tmp irrflag(static_cast<size_t>(n), st);
  k_dia_regular<<<blocks_for(32LL * words, 256), 256, 0, st>>>(out.codes.get(), n, stride, d,
                                                               out.mask.get(),
                                                               irrflag.as<unsigned char>());
  PPA_CUDA(cudaGetLastError());
  Tmp sel(static_cast<size_t>(n) * sizeof(int), st), nsel(sizeof(long long), st);
  size_t bytes = 0;
  cub::CountingInputIterator<int> it(0);
  PPA_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, irrflag.as<unsigned char>(),
                                      sel.as<int>(), nsel.as<long long>(), n, st));
  {
    Tmp ws(bytes, st);
    PPA_CUDA(cub::DeviceSelect::Flagged(ws.p, bytes, it, irrflag.as<unsigned char>(),
                                        sel.as<int>(), nsel.as<long long>(), n, st));
  }
  long long nirr = 0;
  PPA_CUDA(cudaMemcpyAsync(&nirr, nsel.p, sizeof nirr, cudaMemcpyDeviceToHost, st));
  PPA_CUDA(cudaStreamSynchronize(st));
  if (2 * nirr > n) {
    out.mask.release();
    out.defaults.clear();
    return true;
  }
  // one row of slack: the irregular list may be empty
  out.irr_rows.resize(static_cast<size_t>(nirr) + 1);
  out.irr_codes.resize(static_cast<size_t>(nirr) * stride + stride);
  if (nirr) {
    PPA_CUDA(cudaMemcpyAsync(out.irr_rows.get(), sel.p, static_cast<size_t>(nirr) * sizeof(int),
                             cudaMemcpyDeviceToDevice, st));
    k_gather_codes<<<blocks_for(nirr * stride, 256), 256, 0, st>>>(
        out.codes.get(), out.irr_rows.get(), nirr, stride, out.irr_codes.get());
    PPA_CUDA(cudaGetLastError());
  }
  out.nirr = nirr;
  out.regular = true;
  out.pres.release();
  if (nd <= 8 && n > 0) {
    // zero padding of 5 D + 64 rows (a multiple of 16) on both sides (D = the
    // widest offset): the two-factor pass copies presence bytes of rows just
    // outside the matrix, from 16-byte aligned starts (its last chunk reaches
    // row n + 4 D + Dm + 15 at most, Dm <= D / 4)
    const long long D = std::max(std::abs(static_cast<long long>(out.offsets.front())),
                                 std::abs(static_cast<long long>(out.offsets.back())));
    out.pres_pad = (5 * D + 64 + 15) & ~15LL;
    const size_t total = static_cast<size_t>(n + 2 * out.pres_pad + 16);
    out.pres.resize(total);
    PPA_CUDA(cudaMemsetAsync(out.pres.get(), 0, total, st));
    Tmp bad(sizeof(int), st);
    PPA_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    k_dia_presence<<<blocks_for(n, 256), 256, 0, st>>>(out.codes.get(), n, stride, d,
                                                       out.pres.get() + out.pres_pad,
                                                       bad.as<int>());
    PPA_CUDA(cudaGetLastError());
    int hbad = 0;
    PPA_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof hbad, cudaMemcpyDeviceToHost, st));
    PPA_CUDA(cudaStreamSynchronize(st));
    if (hbad) out.pres.release();
    // Box-grid geometry (spmv_grid2.cu): a 7-point stencil with offsets
    // (-nx ny, -nx, -1, 0, 1, nx, nx ny) or a 5-point one with (-nx, -1, 0, 1,
    // nx) whose entries are cut exactly at the box faces.
    const std::vector<int>& o = out.offsets;
    int gx = 0, gy = 0, gz = 0;
    if (!hbad && nd == 7 && o[2] == -1 && o[3] == 0 && o[4] == 1 && o[1] == -o[5] &&
        o[0] == -o[6] && o[5] > 1 && o[6] % o[5] == 0 && n % o[6] == 0) {
      gx = o[5];
      gy = o[6] / o[5];
      gz = n / o[6];
    } else if (!hbad && nd == 5 && o[1] == -1 && o[2] == 0 && o[3] == 1 && o[0] == -o[4] &&
               o[4] > 1 && n % o[4] == 0) {
      gx = o[4];
      gy = 1;
      gz = n / o[4];
    }
    if (gx > 0) {
      PPA_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
      k_grid_check<<<blocks_for(n, 256), 256, 0, st>>>(out.pres.get() + out.pres_pad, n, nd, gx,
                                                       gy, gz, bad.as<int>());
      PPA_CUDA(cudaGetLastError());
      int gbad = 0;
      PPA_CUDA(cudaMemcpyAsync(&gbad, bad.p, sizeof gbad, cudaMemcpyDeviceToHost, st));
      PPA_CUDA(cudaStreamSynchronize(st));
      if (gbad == 0) {
        grid2_zeros();
        out.grid[0] = gx;
        out.grid[1] = gy;
        out.grid[2] = gz;
      }
    }
  }
  PPA_CUDA(cudaStreamSynchronize(st));
  return true;
}

}  // namespace kern
}  // namespace ppa
