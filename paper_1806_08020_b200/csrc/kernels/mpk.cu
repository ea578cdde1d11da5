// Matrix-powers fusion: two polynomial factors per pass over a banded
// SELL-32 matrix.
//
// pi(A)v applies eff_degree factors in sequence; each plain launch streams
// the whole matrix from HBM (424 MB at config 3, well over the 126 MB L2).
// For a matrix of bandwidth BW (|col - row| <= BW), level 2 of a fused pass
// on rows R needs level-1 results only for rows R +- BW.  One persistent
// cooperative kernel processes both levels: work items (level, chunk of 8
// slices = 256 rows) form a global order in which level 2 of chunk c trails
// level 1 of chunk c by `lag` chunks (lag > BW/chunk + half the CTAs), and
// CTA b takes items b, b + G, b + 2G, ...  Every CTA is co-resident
// (cooperative launch), so the smallest-index blocked item can always
// proceed: no deadlock.  Warps are independent: warp w owns slice w of
// every chunk, publishes a finished level-1 slice with a release-add on the
// chunk's monotone counter, and waits for a level-2 slice with acquire loads
// of the counters over [c - bwc, c + bwc].  The reuse distance (a few
// hundred chunks, ~40 MB of traffic at config 3) fits in L2, so level 2
// reads the matrix slice and the level-1 vector from L2: HBM streams the
// matrix once per TWO factors (ncu: 377 MB DRAM read per fused pass).
//
// Per row the arithmetic is exactly the single-factor kernels' (sequential
// row sums, no FMA contraction), so fused and unfused chains are
// bit-identical and both match the CPU oracle bit for bit.
//   real, real : y1 = x + a0 (A x);          y2 = y1 + b0 (A y1)
//   pair       : t  = A x;                   y2 = (x + a1 t) + a0 (A t)
//   complement (last pass of tau = I - pi): y2 = base - y2

#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "ppa/kernels.hpp"

namespace ppa {
namespace kern {
namespace {

constexpr int MP_WARPS = 8;
constexpr int MP_CH = MP_WARPS;  // slices per chunk: one per warp (256 rows)
constexpr int MP_UNROLL = 8;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct MpArgs {
  const long long* slice_ptr;
  const int* scol;
  const double* sval;
  int n, nslices, nchunks, bwc, lag;
  double a0, a1, b0;
  const double* x;
  double* y1;
  double* y2;
  const double* base;
  unsigned* done;   // per-chunk level-1 completion counters (monotone)
  unsigned target;  // done[c] == target <=> level 1 of chunk c finished this pass
};

// item k -> (level, chunk): L1(0..lag-1), then L2(j), L1(lag+j) alternating,
// then the remaining L2 items.
__device__ __forceinline__ void decode(int k, int nchunks, int lag, int& level, int& c) {
  if (k < lag) {
    level = 1;
    c = k;
    return;
  }
  const int r = k - lag;
  const int rest = nchunks - lag;  // L1 items still to interleave
  if (r < 2 * rest) {
    level = (r & 1) ? 1 : 2;
    c = (r & 1) ? lag + (r >> 1) : (r >> 1);
  } else {
    level = 2;
    c = rest + (r - 2 * rest);
  }
}

// Row sum of one slice; GATHER_CG reads the gathered vector through L2 only
// (it is being written by other CTAs of this kernel).
template <bool GATHER_CG>
__device__ __forceinline__ double slice_sum(const MpArgs& a, const double* g, int s, int lane) {
  double sum = 0.0;
  const long long b0 = a.slice_ptr[s];
  const int width = static_cast<int>((a.slice_ptr[s + 1] - b0) >> 5);
  const int* cp = a.scol + b0 + lane;
  const double* vp = a.sval + b0 + lane;
  for (int k0 = 0; k0 < width; k0 += MP_UNROLL) {
    int c[MP_UNROLL];
    double v[MP_UNROLL];
#pragma unroll
    for (int u = 0; u < MP_UNROLL; ++u) {
      if (k0 + u < width) {
        c[u] = __ldcg(cp + (k0 + u) * 32);
        v[u] = __ldcg(vp + (k0 + u) * 32);
      }
    }
#pragma unroll
    for (int u = 0; u < MP_UNROLL; ++u) {
      if (k0 + u < width && c[u] >= 0) {
        const double xv = GATHER_CG ? __ldcg(g + c[u]) : __ldg(g + c[u]);
        sum = __dadd_rn(sum, __dmul_rn(v[u], xv));
      }
    }
  }
  return sum;
}

template <bool PAIR, bool COMPL, bool TICKET>
__global__ void __launch_bounds__(MP_WARPS * 32, 4) k_spmv_mp2(MpArgs a, unsigned* ticket) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = 2 * a.nchunks;
  __shared__ int s_next[2];
  if (TICKET) {
    if (threadIdx.x == 0) s_next[0] = static_cast<int>(atomicAdd(ticket, 1u));
    __syncthreads();
  }
  for (int it = 0, k = TICKET ? s_next[0] : static_cast<int>(blockIdx.x); k < total;
       ++it, k = TICKET ? s_next[it & 1] : k + static_cast<int>(gridDim.x)) {
    // dynamic schedule: the next ticket is fetched while this item runs
    if (TICKET && threadIdx.x == 0) s_next[(it + 1) & 1] = static_cast<int>(atomicAdd(ticket, 1u));
    int level, c;
    decode(k, a.nchunks, a.lag, level, c);
    const int s = c * MP_CH + warp;
    const int r = s * 32 + lane;
    if (level == 1) {
      if (s < a.nslices) {
        const double sum = slice_sum<false>(a, a.x, s, lane);
        if (r < a.n) a.y1[r] = PAIR ? sum : __dadd_rn(__ldg(a.x + r), __dmul_rn(a.a0, sum));
      }
      __syncwarp();
      if (lane == 0) red_release_add(a.done + c, 1u);
    } else {
      const int lo = max(0, c - a.bwc), hi = min(a.nchunks - 1, c + a.bwc);
      for (int q = lo + lane; q <= hi; q += 32) {
        unsigned spins = 0;
        while (ld_acquire(a.done + q) < a.target) {
          __nanosleep(20);
          if (++spins > (1u << 26)) __trap();  // a lost dependency must fail loudly, not hang
        }
      }
      __syncwarp();
      if (s < a.nslices) {
        const double sum = slice_sum<true>(a, a.y1, s, lane);
        if (r < a.n) {
          double z;
          if (PAIR) {
            z = __dadd_rn(__dadd_rn(__ldg(a.x + r), __dmul_rn(a.a1, __ldcg(a.y1 + r))),
                          __dmul_rn(a.a0, sum));
          } else {
            z = __dadd_rn(__ldcg(a.y1 + r), __dmul_rn(a.b0, sum));
          }
          if (COMPL) z = __dsub_rn(a.base[r], z);
          a.y2[r] = z;
        }
      }
    }
    if (TICKET) __syncthreads();  // publishes s_next for the next iteration
  }
}

template <bool PAIR, bool COMPL>
int occupancy() {
  static int occ = [] {
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_spmv_mp2<PAIR, COMPL, false>,
                                                  MP_WARPS * 32, 0);
    return std::max(1, o);
  }();
  return occ;
}

template <bool PAIR, bool COMPL>
void launch_mp2(MpArgs& m, unsigned* ticket, int sm_count, cudaStream_t st) {
  static const double lag_rounds = [] {
    const char* e = std::getenv("PPA_MPK_LAG_ROUNDS");
    return e ? std::atof(e) : 1.0;
  }();
  static const int ctas_per_sm = [] {
    const char* e = std::getenv("PPA_MPK_CTAS_PER_SM");
    return e ? std::atoi(e) : 0;
  }();
  static const bool static_sched = [] {
    const char* e = std::getenv("PPA_MPK_SCHED");
    return e && std::string(e) == "static";
  }();
  const int occ = occupancy<PAIR, COMPL>();
  const int per_sm = ctas_per_sm > 0 ? std::min(ctas_per_sm, occ) : occ;
  int grid = std::max(1, std::min(2 * m.nchunks, sm_count * per_sm));
  if (!static_sched) {
    // dynamic tickets: items are handed out in order to running CTAs, so a
    // level-2 item's level-1 dependencies were always handed out first
    m.lag = std::min(m.nchunks, m.bwc + 1 + static_cast<int>(lag_rounds * grid));
    PPA_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned), st));
    k_spmv_mp2<PAIR, COMPL, true><<<grid, MP_WARPS * 32, 0, st>>>(m, ticket);
    PPA_CUDA(cudaGetLastError());
    return;
  }
  // static round-robin: needs every CTA co-resident (cooperative launch); an
  // odd grid makes each CTA alternate levels so none runs ahead on level 1
  if (grid > 1 && grid % 2 == 0) --grid;
  m.lag = std::min(m.nchunks, m.bwc + 1 + static_cast<int>(lag_rounds * grid));
  unsigned* none = nullptr;
  void* args[] = {&m, &none};
  PPA_CUDA(cudaLaunchCooperativeKernel(
      reinterpret_cast<const void*>(k_spmv_mp2<PAIR, COMPL, false>), dim3(grid),
      dim3(MP_WARPS * 32), args, 0, st));
}

}  // namespace

bool mp2_supported(const CsrDevice& a) {
  return a.sell_val != nullptr && a.sell_perm == nullptr && a.bandwidth >= 0 &&
         static_cast<long long>(a.bandwidth) * 8 <= a.n && a.n >= (1 << 16);
}

void spmv_mp2(const CsrDevice& a, const Mp2Pass& p, const double* x, double* y1, double* y2,
              const double* base, MpWork& w, int sm_count, cudaStream_t st) {
  const int nchunks = (a.nslices + MP_CH - 1) / MP_CH;
  if (w.capacity < nchunks) {
    PPA_CUDA(cudaStreamSynchronize(st));
    w.flags.resize(static_cast<size_t>(nchunks));
    PPA_CUDA(cudaMemset(w.flags.get(), 0, static_cast<size_t>(nchunks) * sizeof(int)));
    if (!w.counter.get()) w.counter.resize(1);
    w.capacity = nchunks;
    w.epoch = 0;
  }
  // fresh per-chunk completion counters for this pass (stream-ordered)
  PPA_CUDA(cudaMemsetAsync(w.flags.get(), 0, static_cast<size_t>(nchunks) * sizeof(int), st));
  ++w.epoch;
  const int rows_per_chunk = MP_CH * 32;
  MpArgs m;
  m.slice_ptr = a.slice_ptr;
  m.scol = a.sell_col;
  m.sval = a.sell_val;
  m.n = a.n;
  m.nslices = a.nslices;
  m.nchunks = nchunks;
  // +4 rows: every 32-byte sector a level-2 gather touches is fully written
  m.bwc = (a.bandwidth + 4 + rows_per_chunk - 1) / rows_per_chunk;
  m.lag = 0;
  m.a0 = p.a0;
  m.a1 = p.a1;
  m.b0 = p.b0;
  m.x = x;
  m.y1 = y1;
  m.y2 = y2;
  m.base = base;
  m.done = reinterpret_cast<unsigned*>(w.flags.get());
  m.target = MP_WARPS;
  const bool compl_ = base != nullptr;
  if (p.pair) {
    compl_ ? launch_mp2<true, true>(m, w.counter.get(), sm_count, st)
           : launch_mp2<true, false>(m, w.counter.get(), sm_count, st);
  } else {
    compl_ ? launch_mp2<false, true>(m, w.counter.get(), sm_count, st)
           : launch_mp2<false, false>(m, w.counter.get(), sm_count, st);
  }
}

}  // namespace kern
}  // namespace ppa
