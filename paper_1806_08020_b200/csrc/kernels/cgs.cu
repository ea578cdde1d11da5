// CGS2 orthogonalisation and the other tall-skinny reductions over the
// Krylov basis, as TMA-pipelined kernels.
//
// Replaces the MGS2 loop of arnoldi_extend (src/arnoldi.cpp:129-150), the
// reorthogonalisation of thick_restart (src/arnoldi.cpp:317-324) and the
// norms of ritz_vector (src/arnoldi.cpp:261).
//
// V is column-major in HBM (ld a multiple of 32 doubles) and is described to
// the TMA unit by a 2D tensor map {rows = n, cols = c}.  A persistent CTA
// (256 threads; 1-2 per SM by shared-memory footprint) walks a contiguous
// range of 128-row tiles.  Thread 0 is the producer: one
// cp.async.bulk.tensor.2d per tile moves the whole 128 x c block (rows past n
// are zero-filled by the TMA) plus one 1 KB bulk copy of w into a
// shared-memory stage, completing on the stage's mbarrier; `stages` tiles
// stay in flight, so HBM never waits on the consumers.  The consumers (all 8
// warps) read the tile from shared memory:
//   dot     warp g owns columns j = g, g+8, ...; lanes walk rows
//   update  row sums s = V h over two thread halves (fixed-order combine),
//           then w -= s and the pass-2 dots / the norm / the V[:,c] store
// Per-CTA partials are reduced in block order by the last CTA (ticket), so
// every result is deterministic.  HBM bytes per CGS2 step at basis size c:
// 3 sweeps over V[:,0:c] + w read 3x and written once + V[:,c] written once
// = 8n(3c + 5) (the north-star model charges 8n(3c + 7)).

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "common.cuh"
#include "tma.cuh"
#include "ppa/kernels.hpp"
#include "ws_layout.cuh"

namespace ppa {
namespace kern {
namespace {

constexpr int TR = 128;  // rows per tile
constexpr int NT = 256;  // threads per CTA
constexpr int NWARP = NT / 32;
constexpr size_t kSmemPerSm = 200 * 1024;

enum Mode : int { kDot = 0, kSumSq = 1, kUpd2 = 2, kUpd1 = 3, kStore = 4, kDot2 = 5, kUpdD = 6 };

struct PipeArgs {
  const double* V;
  long long ld;
  int n;
  int c;
  double* w;        // dot: read; update: read + write
  const double* h;  // update/store coefficients (device, c)
  double* out;      // dot/sumsq: c results; upd1: the norm
  int tiles_per_cta;
  int stages;
  double* partials;
  unsigned int* ticket;
  double* scal;  // upd2 finalisation / store hsub
  double* Hcol;     // kUpd2: the Hessenberg column; nullptr = raw local sums into out
  int* flag;        // kStore: skipped when *flag (breakdown); nullptr = never
  const double* hsub;  // kStore: divisor (nullptr: scal[kScalHsub])
};

__device__ __forceinline__ bool finish_grid(const double* s_col, int width, double* partials,
                                            unsigned int* ticket, double* s_final) {
  __shared__ unsigned int s_last;
  for (int k = threadIdx.x; k < width; k += NT) {
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
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = warp; k < width; k += NWARP) {
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

template <int MODE, int CPW>
__global__ void __launch_bounds__(NT) k_tspipe(const __grid_constant__ CUtensorMap vmap,
                                               PipeArgs a) {
  constexpr bool kNeedW = MODE != kSumSq;
  constexpr int MAXC = NWARP * CPW;
  constexpr int RQ = TR / 32;  // rows per lane in the column-owner mapping
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr bool kTwo = MODE == kDot2 || MODE == kUpdD;  // two vectors / two row sums
  __shared__ double s_h[kTwo ? 2 * MAXC + 2 : MAXC];
  __shared__ double s_part[kTwo ? 4 : 2][TR];
  __shared__ double s_col[kTwo ? 2 * MAXC + 1 : MAXC + 1];
  __shared__ double s_final[kTwo ? 2 * MAXC + 1 : MAXC + 1];
  __shared__ double s_red[NWARP];
  __shared__ double s_wn[MODE == kUpd2 ? TR : 1];

  if (MODE == kStore && a.flag && *a.flag) return;
  const int tid = threadIdx.x, lane = tid & 31, g = tid >> 5;
  const int c = a.c;
  const int ntiles = (a.n + TR - 1) / TR;
  const int t_begin = blockIdx.x * a.tiles_per_cta;
  const int count = max(0, min(ntiles, t_begin + a.tiles_per_cta) - t_begin);
  const int S = a.stages;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  double* stage0 = reinterpret_cast<double*>(smem + 128);
  // stage layout: V tile [c][TR] then w [TR]; 1 KB aligned
  const size_t stage_elems = static_cast<size_t>(c + 1) * TR;

  if (MODE == kUpd2 || MODE == kUpd1 || MODE == kStore) {
    for (int j = tid; j < MAXC; j += NT) s_h[j] = j < c ? a.h[j] : 0.0;
  }
  if (MODE == kUpdD) {
    // h = [s (c-1), d (c-1), e, rho]: column c-1 of the tile is the pending u
    for (int j = tid; j < 2 * (c - 1) + 2; j += NT) s_h[j] = a.h[j];
  }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const uint64_t policy = evict_first_policy();
  auto issue = [&](int i) {
    const int s = i % S;
    const int row0 = (t_begin + i) * TR;
    const bool wfull = kNeedW && row0 + TR <= a.n;
    double* st = stage0 + s * stage_elems;
    mbar_expect_tx(&bar[s], static_cast<uint32_t>(TR * c * 8 + (wfull ? TR * 8 : 0)));
    tma_load_2d(st, &vmap, row0, 0, &bar[s], policy);
    if (wfull) bulk_load(st + c * TR, a.w + row0, TR * 8, &bar[s], policy);
  };
  if (tid == 0) {
    for (int i = 0; i < min(S, count); ++i) issue(i);
  }

  double acc[CPW], acc2[kTwo ? CPW : 1];
#pragma unroll
  for (int jj = 0; jj < CPW; ++jj) acc[jj] = 0.0;
#pragma unroll
  for (int jj = 0; jj < (kTwo ? CPW : 1); ++jj) acc2[jj] = 0.0;
  double nrm = 0.0;
  const int half = tid >> 7;  // row-sum split over two halves of the columns
  const int hr = tid & (TR - 1);
  const int ch = (c + 1) >> 1;
  const int jlo = half ? ch : 0;
  const int jhi = half ? c : ch;
  double* dstcol = const_cast<double*>(a.V) + static_cast<long long>(c) * a.ld;

  for (int i = 0; i < count; ++i) {
    const int s = i % S;
    mbar_wait(&bar[s], (i / S) & 1);
    const double* T = stage0 + s * stage_elems;
    const int row0 = (t_begin + i) * TR;
    const int rows = min(TR, a.n - row0);
    const bool full = rows == TR;
    const double* W = T + c * TR;

    if (MODE == kDot2) {
      // V^T z and V^T u in one sweep; u is the tile's last column
      double wr[RQ], ur[RQ];
#pragma unroll
      for (int q = 0; q < RQ; ++q) {
        const int r = lane + 32 * q;
        wr[q] = full ? W[r] : (r < rows ? a.w[row0 + r] : 0.0);
        ur[q] = T[(c - 1) * TR + r];
      }
#pragma unroll
      for (int jj = 0; jj < CPW; ++jj) {
        const int j = g + NWARP * jj;
        if (j < c) {
          const double* col = T + j * TR + lane;
#pragma unroll
          for (int q = 0; q < RQ; ++q) {
            const double v = col[32 * q];
            acc[jj] = fma(v, wr[q], acc[jj]);
            acc2[jj] = fma(v, ur[q], acc2[jj]);
          }
        }
      }
    } else if (MODE == kUpdD) {
      // V[:,c-1] = (u - V s)/rho and w = z/rho - V d - e u over the c-1 final
      // columns; u = tile column c-1, z = w (read and overwritten in place)
      const int cf = c - 1;
      const int chf = (cf + 1) >> 1;
      const int lo = half ? chf : 0, hi = half ? cf : chf;
      double sp = 0.0, sd = 0.0;
      const double* col = T + hr;
      for (int j = lo; j < hi; ++j) {
        const double v = col[j * TR];
        sp = fma(v, s_h[j], sp);
        sd = fma(v, s_h[cf + j], sd);
      }
      s_part[half][hr] = sp;
      s_part[2 + half][hr] = sd;
      __syncthreads();
      if (tid < rows) {
        const double rho = s_h[2 * cf + 1], e = s_h[2 * cf];
        const double u = T[cf * TR + tid];
        const double z = full ? W[tid] : a.w[row0 + tid];
        const double vs = s_part[0][tid] + s_part[1][tid];
        const double vd = s_part[2][tid] + s_part[3][tid];
        dstcol[row0 + tid - a.ld] = (u - vs) / rho;  // V[:, c-1]
        a.w[row0 + tid] = (z / rho - vd) - e * u;
      }
    } else if (MODE == kDot || MODE == kSumSq) {
      // rows beyond n are zero in the tile (TMA OOB fill) and w is zeroed here
      double wr[RQ];
#pragma unroll
      for (int q = 0; q < RQ; ++q) {
        const int r = lane + 32 * q;
        wr[q] = MODE == kDot ? (full ? W[r] : (r < rows ? a.w[row0 + r] : 0.0)) : 0.0;
      }
#pragma unroll
      for (int jj = 0; jj < CPW; ++jj) {
        const int j = g + NWARP * jj;
        if (j < c) {
          const double* col = T + j * TR + lane;
#pragma unroll
          for (int q = 0; q < RQ; ++q) {
            const double v = col[32 * q];
            acc[jj] = MODE == kDot ? fma(v, wr[q], acc[jj]) : fma(v, v, acc[jj]);
          }
        }
      }
    } else {
      // phase A: partial row sums over this thread's half of the columns
      double sp = 0.0;
      const double* col = T + hr;
      for (int j = jlo; j < jhi; ++j) sp = fma(col[j * TR], s_h[j], sp);
      s_part[half][hr] = sp;
      __syncthreads();
      if (MODE == kUpd2) {
        // the updated rows once (first 128 threads), then every warp's
        // pass-2 dots read them from shared memory
        if (tid < TR) {
          double wn = 0.0;
          if (tid < rows) {
            const double wo = full ? W[tid] : a.w[row0 + tid];
            wn = wo - (s_part[0][tid] + s_part[1][tid]);
            a.w[row0 + tid] = wn;
          }
          s_wn[tid] = wn;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < RQ; ++q) {
          const int r = lane + 32 * q;
          const double wn = s_wn[r];
#pragma unroll
          for (int jj = 0; jj < CPW; ++jj) {
            const int j = g + NWARP * jj;
            if (j < c) acc[jj] = fma(T[j * TR + r], wn, acc[jj]);
          }
          // ||w||^2 in warp 0, rows lane + 32q (the reduction order the
          // Hessenberg subdiagonal has always used)
          if (g == 0 && r < rows) nrm = fma(wn, wn, nrm);
        }
      } else if (tid < rows) {
        const double wo = full ? W[tid] : a.w[row0 + tid];
        const double wn = wo - (s_part[0][tid] + s_part[1][tid]);
        if (MODE == kUpd1) {
          nrm = fma(wn, wn, nrm);
          a.w[row0 + tid] = wn;
        } else {  // kStore: V[:,c] = (w - V h2) / hsub
          dstcol[row0 + tid] = wn / (a.hsub ? *a.hsub : a.scal[kScalHsub]);
        }
      }
    }
    __syncthreads();  // stage s and s_part are free again
    if (tid == 0 && i + S < count) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(i + S);
    }
  }

  if (MODE == kStore || MODE == kUpdD) return;
  int width = 1;
  if (MODE == kDot2) {
#pragma unroll
    for (int jj = 0; jj < CPW; ++jj) {
      const int j = g + NWARP * jj;
      if (j < c) {
        const double t = dev::warp_sum(acc[jj]);
        const double t2 = dev::warp_sum(acc2[jj]);
        if (lane == 0) {
          s_col[j] = t;
          s_col[c + j] = t2;
        }
      }
    }
    width = 2 * c;
  }
  if (MODE == kDot || MODE == kSumSq || MODE == kUpd2) {
#pragma unroll
    for (int jj = 0; jj < CPW; ++jj) {
      const int j = g + NWARP * jj;
      if (j < c) {
        const double t = dev::warp_sum(acc[jj]);
        if (lane == 0) s_col[j] = t;
      }
    }
    width = MODE == kUpd2 ? c + 1 : c;
  }
  if (MODE == kUpd2 || MODE == kUpd1) {
    const double t = dev::warp_sum(nrm);
    if (lane == 0) s_red[g] = t;
    __syncthreads();
    if (tid == 0) {
      double tot = 0.0;
      for (int k = 0; k < NWARP; ++k) tot += s_red[k];
      s_col[width - 1] = tot;
    }
  }
  __syncthreads();
  if (!finish_grid(s_col, width, a.partials, a.ticket, s_final)) return;

  if (MODE == kDot || MODE == kSumSq || MODE == kDot2) {
    for (int j = tid; j < width; j += NT) a.out[j] = s_final[j];
    return;
  }
  if (MODE == kUpd1) {
    if (tid == 0) *a.out = sqrt(s_final[0]);
    return;
  }
  if (MODE == kUpd2 && a.Hcol == nullptr) {
    // rank-local sums for the row-sharded solve (dist.py): [V^T w, ||w||^2],
    // all-reduced by the caller before the store sweep
    for (int j = tid; j <= c; j += NT) a.out[j] = s_final[j];
    return;
  }
  // kUpd2: s_final[0..c) = h2, s_final[c] = ||w||^2 -> Hessenberg column,
  // hsub (Pythagoras: ||w - V h2||^2 = ||w||^2 - ||h2||^2 for orthonormal V)
  // and the breakdown test of src/arnoldi.cpp:143-148.
  for (int j = tid; j < c; j += NT) a.scal[kScalH2 + j] = s_final[j];
  if (tid == 0) {
    double sq = 0.0;
    for (int j = 0; j < c; ++j) sq += s_final[j] * s_final[j];
    const double d2 = s_final[c] - sq;
    const double hsub = d2 > 0.0 ? sqrt(d2) : 0.0;
    a.scal[kScalHsub] = hsub;
    a.scal[kScalHsub + 1] = sqrt(s_final[c]);
    double cn = 0.0;
    for (int j = 0; j < c; ++j) {
      const double hj = s_h[j] + s_final[j];
      a.Hcol[j] = hj;
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
    a.Hcol[c] = bd ? 0.0 : hsub;
    *a.flag = bd;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    PPA_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) {
      throw CudaError("cuTensorMapEncodeTiled entry point unavailable");
    }
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// 2D map of the first c columns of V: dim0 = rows (n, contiguous), dim1 =
// columns (stride ld); box = 128 rows x c columns.
CUtensorMap basis_map(const double* V, long long ld, int n, int c) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(c)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * sizeof(double)};
  const cuuint32_t box[2] = {TR, static_cast<cuuint32_t>(c)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(V),
                               dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}

template <int MODE, int CPW>
void launch_pipe(PipeArgs a, ReduceWorkspace& ws, int sm_count, cudaStream_t st) {
  const size_t stage_bytes = static_cast<size_t>(a.c + 1) * TR * sizeof(double);
  int per_sm, stages;
  if (8 * stage_bytes <= kSmemPerSm / 2) {
    // small bases (c < ~12): short tiles, so more resident CTAs (4 stages
    // each) keep enough rows in flight and enough warps issuing
    stages = 4;
    per_sm = static_cast<int>(
        std::max<size_t>(1, std::min<size_t>(6, kSmemPerSm / (stages * stage_bytes + 1024))));
  } else {
    // two CTAs per SM when two double-buffered CTAs fit, else one deeper CTA
    per_sm = 4 * stage_bytes <= kSmemPerSm ? 2 : 1;
    const size_t budget = kSmemPerSm / per_sm;
    stages = static_cast<int>(std::max<size_t>(2, std::min<size_t>(6, budget / stage_bytes)));
  }
  const size_t smem = 128 + stage_bytes * stages;
  // raise the dynamic shared-memory cap once per instantiation (thread-safe
  // static initialisation; the launch's own size sets the occupancy)
  static const bool capped = [] {
    PPA_CUDA(cudaFuncSetAttribute(k_tspipe<MODE, CPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  max_dynamic_smem(k_tspipe<MODE, CPW>)));
    return true;
  }();
  (void)capped;
  {
    // never more CTAs than can be resident: the kernel is persistent
    int fit = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit, k_tspipe<MODE, CPW>, NT, smem) ==
            cudaSuccess &&
        fit > 0) {
      per_sm = std::min(per_sm, fit);
    }
  }
  const int ntiles = (a.n + TR - 1) / TR;
  const int grid0 = std::max(1, std::min(ntiles, sm_count * per_sm));
  a.tiles_per_cta = (ntiles + grid0 - 1) / grid0;
  const int grid = (ntiles + a.tiles_per_cta - 1) / a.tiles_per_cta;
  a.stages = stages;
  ensure_workspace(ws, grid, 2 * NWARP * CPW + 1);
  a.partials = ws.partials.get();
  a.ticket = ws.tickets.get();
  const CUtensorMap map = basis_map(a.V, a.ld, a.n, a.c);
  k_tspipe<MODE, CPW><<<grid, NT, smem, st>>>(map, a);
  PPA_CUDA(cudaGetLastError());
}

template <int MODE>
void dispatch(const PipeArgs& a, ReduceWorkspace& ws, int sm_count, cudaStream_t st) {
  if (a.c <= 8) return launch_pipe<MODE, 1>(a, ws, sm_count, st);
  if (a.c <= 16) return launch_pipe<MODE, 2>(a, ws, sm_count, st);
  if (a.c <= 32) return launch_pipe<MODE, 4>(a, ws, sm_count, st);
  if (a.c <= 64) return launch_pipe<MODE, 8>(a, ws, sm_count, st);
  return launch_pipe<MODE, 16>(a, ws, sm_count, st);
}

// Out[:, 0:p] = V[:, 0:d] * G, the thick-restart recombination V*Q and the
// batched Ritz vectors (src/arnoldi.cpp:258, 306-309), on the same persistent
// tile pipeline as the sweeps above: 128-row tiles of V[:, 0:d] arrive by
// TMA in `stages` shared-memory stages.  Thread t owns row t & 127 of a tile
// and the HP output columns [h HP, h HP + HP) of half h = t >> 7; G sits
// row-major in shared memory and is read as 16-byte broadcasts.  Per output
// the FMAs run over j = 0..d-1 in order, exactly as the register kernel of
// tallskinny.cu, so both give the same bits.  A tile's outputs are written
// after the tile is in shared memory and other tiles' rows are disjoint, so
// Out may alias V[:, 0:p] (p <= d).
template <int HP>
__global__ void __launch_bounds__(NT) k_combine_tma(const __grid_constant__ CUtensorMap vmap, int n,
                                                    int d, const double* __restrict__ G, int p,
                                                    double* Out, long long ldo, int tiles_per_cta,
                                                    int S) {
  constexpr int PB = 2 * HP;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  double* gs = reinterpret_cast<double*>(smem + 128);
  const int gsz = (d * PB + 127) / 128 * 128;  // doubles, a multiple of 1 KB
  double* stage0 = gs + gsz;
  const size_t stage_elems = static_cast<size_t>(d) * TR;
  const int tid = threadIdx.x;
  const int ntiles = (n + TR - 1) / TR;
  const int t_begin = blockIdx.x * tiles_per_cta;
  const int count = max(0, min(ntiles, t_begin + tiles_per_cta) - t_begin);
  for (int k = tid; k < d * PB; k += NT) {
    const int j = k / PB, c = k - j * PB;
    gs[k] = c < p ? G[static_cast<long long>(c) * d + j] : 0.0;
  }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t policy = evict_first_policy();
  auto issue = [&](int i) {
    const int s = i % S;
    mbar_expect_tx(&bar[s], static_cast<uint32_t>(TR * d * 8));
    tma_load_2d(stage0 + s * stage_elems, &vmap, (t_begin + i) * TR, 0, &bar[s], policy);
  };
  if (tid == 0) {
    for (int i = 0; i < min(S, count); ++i) issue(i);
  }
  // the CTA's halves take alternate tiles (S is even); in a half, thread u
  // owns rows u & 63 and (u & 63) + 64 and output columns [h HP, h HP + HP)
  // of h = u >> 6: every broadcast of a G pair serves four FMAs
  const int half = tid >> 7, u = tid & 127;
  const int r = u & 63, h = u >> 6;
  const double* gh = gs + h * HP;
  for (int i0 = 0; i0 < count; i0 += 2) {
    const int i = i0 + half;
    if (i < count) {
      const int s = i % S;
      mbar_wait(&bar[s], (i / S) & 1);
      const double* T = stage0 + s * stage_elems + r;
      double acc[2][HP];
#pragma unroll
      for (int c = 0; c < HP; ++c) acc[0][c] = acc[1][c] = 0.0;
      auto fma_row = [&](double v0, double v1, int j) {
        const double2* g2 = reinterpret_cast<const double2*>(gh + j * PB);
#pragma unroll
        for (int q = 0; q < HP / 2; ++q) {
          const double2 gv = g2[q];
          acc[0][2 * q] = fma(v0, gv.x, acc[0][2 * q]);
          acc[0][2 * q + 1] = fma(v0, gv.y, acc[0][2 * q + 1]);
          acc[1][2 * q] = fma(v1, gv.x, acc[1][2 * q]);
          acc[1][2 * q + 1] = fma(v1, gv.y, acc[1][2 * q + 1]);
        }
      };
      int j = 0;
      for (; j + 2 <= d; j += 2) {
        const double a0 = T[j * TR], b0 = T[j * TR + 64];
        const double a1 = T[(j + 1) * TR], b1 = T[(j + 1) * TR + 64];
        fma_row(a0, b0, j);
        fma_row(a1, b1, j + 1);
      }
      for (; j < d; ++j) fma_row(T[j * TR], T[j * TR + 64], j);
      const long long row = static_cast<long long>(t_begin + i) * TR + r;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (row + 64 * k < n) {
#pragma unroll
          for (int c = 0; c < HP; ++c) {
            const int col = h * HP + c;
            if (col < p) Out[row + 64 * k + static_cast<long long>(col) * ldo] = acc[k][c];
          }
        }
      }
    }
    // both halves are done with their stages: refill them
    __syncthreads();
    if (tid == 0) {
      if (i0 + S < count) issue(i0 + S);
      if (i0 + 1 + S < count) issue(i0 + 1 + S);
    }
  }
}

template <int HP>
void launch_combine_tma(const double* V, long long ld, int n, int d, const double* G, int p,
                        double* Out, long long ldo, int sm_count, cudaStream_t st) {
  const size_t stage_bytes = static_cast<size_t>(d) * TR * sizeof(double);
  const size_t g_bytes = static_cast<size_t>((d * 2 * HP + 127) / 128 * 128) * sizeof(double);
  // an even number of stages (the CTA's two halves take alternate tiles),
  // at least four so that a pair of tiles is in flight while a pair is
  // consumed: two CTAs per SM when both get four stages, else one with up
  // to six
  int per_sm = 2 * (128 + g_bytes + 4 * stage_bytes) <= kSmemPerSm ? 2 : 1;
  const size_t budget = kSmemPerSm / per_sm - 128 - g_bytes;
  const int stages = static_cast<int>(std::max<size_t>(2, std::min<size_t>(6, budget / stage_bytes))) & ~1;
  const size_t smem = 128 + g_bytes + stages * stage_bytes;
  static const bool capped = [] {
    PPA_CUDA(cudaFuncSetAttribute(k_combine_tma<HP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  max_dynamic_smem(k_combine_tma<HP>)));
    return true;
  }();
  (void)capped;
  int fit = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit, k_combine_tma<HP>, NT, smem) ==
          cudaSuccess &&
      fit > 0) {
    per_sm = std::min(per_sm, fit);
  }
  const int ntiles = (n + TR - 1) / TR;
  const int grid0 = std::max(1, std::min(ntiles, sm_count * per_sm));
  const int tpc = (ntiles + grid0 - 1) / grid0;
  const int grid = (ntiles + tpc - 1) / tpc;
  const CUtensorMap map = basis_map(V, ld, n, d);
  k_combine_tma<HP><<<grid, NT, smem, st>>>(map, n, d, G, p, Out, ldo, tpc, stages);
  PPA_CUDA(cudaGetLastError());
}

void check_aligned(const void* p, const char* who) {
  if (reinterpret_cast<uintptr_t>(p) % 16 != 0) {
    throw std::invalid_argument(std::string(who) + ": vectors must be 16-byte aligned");
  }
}

void check_basis(const double* V, long long ld, int n, int c, const char* who) {
  check_cols(c, who);
  check_aligned(V, who);
  if (ld % 2 || ld < n) {
    throw std::invalid_argument(std::string(who) + ": leading dimension must be even and >= n");
  }
}

PipeArgs base_args(const double* V, long long ld, int n, int c) {
  PipeArgs a{};
  a.V = V;
  a.ld = ld;
  a.n = n;
  a.c = c;
  return a;
}

}  // namespace

bool ts_combine_tma(const double* V, long long ldv, int n, int d, const double* G, int p,
                    double* Out, long long ldo, int sm_count, cudaStream_t st) {
  // the tensor map needs a 16-byte aligned base and an even ld; tiles of
  // d <= 96 columns keep two stages within the shared-memory budget
  if (p < 1 || p > 32 || d < 1 || d > 96 || n < TR) return false;
  if (reinterpret_cast<uintptr_t>(V) % 16 || ldv % 2 || ldv < n) return false;
  const char* off = std::getenv("PPA_COMBINE_TMA");
  if (off && off[0] == '0') return false;
  switch ((p + 3) / 4) {  // outputs per thread: half the padded column count
    case 1: launch_combine_tma<2>(V, ldv, n, d, G, p, Out, ldo, sm_count, st); break;
    case 2: launch_combine_tma<4>(V, ldv, n, d, G, p, Out, ldo, sm_count, st); break;
    case 3: launch_combine_tma<6>(V, ldv, n, d, G, p, Out, ldo, sm_count, st); break;
    case 4: launch_combine_tma<8>(V, ldv, n, d, G, p, Out, ldo, sm_count, st); break;
    case 5: launch_combine_tma<10>(V, ldv, n, d, G, p, Out, ldo, sm_count, st); break;
    case 6: launch_combine_tma<12>(V, ldv, n, d, G, p, Out, ldo, sm_count, st); break;
    case 7: launch_combine_tma<14>(V, ldv, n, d, G, p, Out, ldo, sm_count, st); break;
    default: launch_combine_tma<16>(V, ldv, n, d, G, p, Out, ldo, sm_count, st); break;
  }
  return true;
}

void ts_dot(const double* V, long long ld, int n, int c, const double* w, double* out,
            ReduceWorkspace& ws, int sm_count, cudaStream_t st) {
  if (n <= 0) return;
  check_basis(V, ld, n, c, "ts_dot");
  check_aligned(w, "ts_dot");
  PipeArgs a = base_args(V, ld, n, c);
  a.w = const_cast<double*>(w);
  a.out = out;
  dispatch<kDot>(a, ws, sm_count, st);
}

void col_sumsq(const double* Y, long long ld, int n, int p, double* out, ReduceWorkspace& ws,
               int sm_count, cudaStream_t st) {
  if (n <= 0) return;
  check_basis(Y, ld, n, p, "col_sumsq");
  PipeArgs a = base_args(Y, ld, n, p);
  a.out = out;
  dispatch<kSumSq>(a, ws, sm_count, st);
}

void cgs2_step(double* V, long long ld, int n, int c, double* w, double* Hcol, int* flag,
               ReduceWorkspace& ws, int sm_count, cudaStream_t st) {
  check_basis(V, ld, n, c, "cgs2_step");
  check_aligned(w, "cgs2_step");
  double* scal = ws.scalars.get();
  ts_dot(V, ld, n, c, w, scal + kScalH1, ws, sm_count, st);
  PipeArgs a = base_args(V, ld, n, c);
  a.w = w;
  a.h = scal + kScalH1;
  a.scal = scal;
  a.Hcol = Hcol;
  a.flag = flag;
  dispatch<kUpd2>(a, ws, sm_count, st);
  PipeArgs b = base_args(V, ld, n, c);
  b.w = w;
  b.h = scal + kScalH2;
  b.scal = scal;
  b.flag = flag;
  dispatch<kStore>(b, ws, sm_count, st);
}

void dcgs2_dot(const double* V, long long ld, int n, int c, const double* z, double* out,
               ReduceWorkspace& ws, int sm_count, cudaStream_t st) {
  if (n <= 0) return;
  check_basis(V, ld, n, c, "dcgs2_dot");
  check_aligned(z, "dcgs2_dot");
  PipeArgs a = base_args(V, ld, n, c);
  a.w = const_cast<double*>(z);
  a.out = out;
  dispatch<kDot2>(a, ws, sm_count, st);
}

void dcgs2_update(double* V, long long ld, int n, int c, double* z, const double* coef,
                  ReduceWorkspace& ws, int sm_count, cudaStream_t st) {
  if (n <= 0) return;
  check_basis(V, ld, n, c, "dcgs2_update");
  check_aligned(z, "dcgs2_update");
  if (c < 2) throw std::invalid_argument("dcgs2_update: needs a final column and u");
  PipeArgs a = base_args(V, ld, n, c);
  a.w = z;
  a.h = coef;
  dispatch<kUpdD>(a, ws, sm_count, st);
}

void cgs_update_dot_local(const double* V, long long ld, int n, int c, double* w,
                          const double* h, double* out, ReduceWorkspace& ws, int sm_count,
                          cudaStream_t st) {
  if (n <= 0) return;
  check_basis(V, ld, n, c, "cgs_update_dot_local");
  check_aligned(w, "cgs_update_dot_local");
  PipeArgs a = base_args(V, ld, n, c);
  a.w = w;
  a.h = h;
  a.out = out;
  a.scal = ws.scalars.get();
  a.Hcol = nullptr;
  dispatch<kUpd2>(a, ws, sm_count, st);
}

void cgs_store_local(double* V, long long ld, int n, int c, const double* w, const double* h2,
                     const double* hsub, ReduceWorkspace& ws, int sm_count, cudaStream_t st) {
  if (n <= 0) return;
  check_basis(V, ld, n, c, "cgs_store_local");
  check_aligned(w, "cgs_store_local");
  PipeArgs a = base_args(V, ld, n, c);
  a.w = const_cast<double*>(w);
  a.h = h2;
  a.hsub = hsub;
  a.scal = ws.scalars.get();
  a.flag = nullptr;
  dispatch<kStore>(a, ws, sm_count, st);
}

void cgs1_pass(const double* V, long long ld, int n, int c, double* v, double* corr,
               double* out_norm, ReduceWorkspace& ws, int sm_count, cudaStream_t st) {
  check_basis(V, ld, n, c, "cgs1_pass");
  check_aligned(v, "cgs1_pass");
  ts_dot(V, ld, n, c, v, corr, ws, sm_count, st);
  PipeArgs a = base_args(V, ld, n, c);
  a.w = v;
  a.h = corr;
  a.out = out_norm;
  dispatch<kUpd1>(a, ws, sm_count, st);
}

}  // namespace kern
}  // namespace ppa
