// Kernel and launch templates of the box-grid two-factor pass (see
// spmv_grid2.cu for the description).  Included by spmv_grid2.cu (planner,
// public entry points) and by one translation unit per (stencil, cells per
// thread) pair, spmv_grid2_i*.cu, which instantiate the block sizes; the
// split only shortens the build (nvcc compiles the units in parallel).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <vector>

#include "common.cuh"
#include "pdl.cuh"
#include "tma.cuh"
#include "ppa/kernels.hpp"

namespace ppa {
namespace kern {
namespace g2 {

struct G2Params {
  double val[7];
  double a0, a1, b0;
  int nx, ny, nz, D;
  int ntx, nty, nchunks;
  int P;      // slot pitch (doubles) = widest tile + 4
  int SL;     // lines per x slot (3-D: tile lines + 4; 2-D: 1)
  int LL;     // lines per level-1 slot (3-D: tile lines + 2; 2-D: 1)
  int nslot;  // x slots
  int segs;   // 3-D: 32-column segments per line; 2-D: segments per level-1 line
  int cw;     // warps that own cells (the block may be rounded up)
  double* y_q;            // the output vector (the kernel's y)
  const double* base_q;   // the complement's base vector (COMPL)
  const double* zeros;  // >= one line of zeros: the copy source of planes outside the box
  // z-slab mode (the sharded pass, dist.py ShardedGridPoly): this rank owns
  // the global planes [zo0, zo1); x, y and base hold those planes only (local
  // plane 0 = global plane zo0).  The halo planes below / above come straight
  // from the neighbours' buffers xl / xr (their local plane 0 = global planes
  // zl0 / zo1) once the neighbours' epoch flags fl / fr reach `epoch`.
  // Unsharded: zo0 = 0, zo1 = nz, no neighbours.
  int zo0, zo1, zl0;
  const double* xl;
  const double* xr;
  const long long* fl;
  const long long* fr;
  long long epoch;
  int* err;  // set when a neighbour's flag does not arrive (~10 s)
  // this rank's flag (word 0) and pass ticket counter (word 1): the last
  // CTA of the pass publishes epoch + 1 (nullptr: no publish)
  long long* own;
};

struct G2Plan {
  int ok = 0;
  int nd = 0, ry = 0, nt = 0, ntx = 1, nty = 1, nchunks = 1, P = 0, SL = 0, LL = 0, nslot = 0,
      segs = 0, cw = 0;
  size_t smem = 0;
};

// One (stencil, cells per thread) pair each, defined in spmv_grid2_i*.cu.
#define PPA_G2_DECL(ND, RY)                                                                   \
  void launch_##ND##_##RY(const G2Params& P, const G2Plan& pl, bool pair, const double* x,    \
                          double* y, const double* base, cudaStream_t st, bool one, bool slab);
PPA_G2_DECL(7, 2) PPA_G2_DECL(7, 3) PPA_G2_DECL(7, 4)
PPA_G2_DECL(5, 1) PPA_G2_DECL(5, 2) PPA_G2_DECL(5, 3) PPA_G2_DECL(5, 4)
#undef PPA_G2_DECL

}  // namespace g2

namespace {

using g2::G2Params;
using g2::G2Plan;

constexpr int G2_BARS = 48;  // doubles reserved for mbarriers: x_full[12], l1_done[24]
constexpr int G2_MAXSLOT = 12;

// Most consumer threads per stencil and cells per thread that compile
// without register spills under __launch_bounds__(NT + 32, 1) (ptxas -v, sm_100a).
constexpr int g2_maxnt(int nd, int ry) {
  return nd == 7 ? (ry == 2 ? 768 : ry == 3 ? 640 : 512)
                 : (ry == 1 ? 960 : ry == 2 ? 896 : ry == 3 ? 640 : 448);
}

__device__ __forceinline__ void g2_bulk(uint32_t dst, const void* src, uint32_t bytes,
                                        uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void g2_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}

// Row sum in increasing offset.  3-D: t = (-D, -nx, -1, 0, +1, +nx, +D);
// 2-D: (-D, -1, 0, +1, +D).
template <int ND>
__device__ __forceinline__ double g2_sum(const double (&v)[7], const double (&t)[ND]) {
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < ND; ++j) s = __dadd_rn(s, __dmul_rn(v[j], t[j]));
  return s;
}


// Per-thread constants of the cells (byte offsets relative to a slot base).
template <int RY>
struct G2Cells {
  int aX[RY], aL[RY];  // cell r in an x slot / a level-1 slot
  int aXm, aXp;        // 3-D: x-slot offsets of the line above cell 0 / below cell RY-1
  int aLm, aLp;        // the same in a level-1 slot
  int row2[RY];        // row of the cell within its plane
  bool v1[RY];         // level-1 cell inside the box (else its value is 0)
  bool v2[RY];         // level-2 cell (in the tile): stored
  bool w2[RY];         // some lane of the warp has a level-2 cell r
};

// Slot rings: NS x slots (load index i in slot i % NS) and G2_LSLOT level-1
// slots (step t in slot t % 4); the level-1 barriers form a ring of 2 NS so
// that the producer, which may trail the consumers by up to NS - 2 steps,
// never waits on a barrier that has moved two phases on.  The step loop is
// unrolled three times so the +-D register triples rotate without moves
// (a 12-fold unroll that made every slot index constant needed ~150
// registers per thread).
constexpr int G2_LSLOT = 4;

struct G2Geo {
  int nsteps, za, nz, D, xs0, slot_x, ls0, slot_l;
};

// Block-uniform running state of the rings (advanced once per step).
struct G2Ring {
  uint32_t xq, xn;   // x slots of load indices t + 1 (plane q) and t + 2 (plane q + 1)
  uint32_t xbeg, xend, xstep;
  int sn, pn;        // x_full index and parity of load index t + 2
  uint32_t lw, lr;   // level-1 slots of steps t and t - 1
  uint32_t lbeg, lend, lstep;
  int bw, bwp;       // l1_done index / parity of step t
  int br, brp;       // the same for step t - 1
};

template <int OFF>
__device__ __forceinline__ double g2_lds(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(a), "n"(OFF) : "memory");
  return v;
}
__device__ __forceinline__ void g2_sts(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

// One consumer step t.  Shared memory is addressed with 32-bit shared-window
// addresses: a block-uniform slot address plus the cell's byte offset, with
// the +-1 neighbours at immediate offsets.
template <int ND, int RY, bool PAIR, bool COMPL, int NS, bool ONE>
__device__ __forceinline__ bool g2_step(
    int t, const G2Geo& G, const G2Cells<RY>& C, const G2Params& P, const double (&v)[7],
    G2Ring& R, uint64_t* x_full, uint64_t* l1_done, int lane, double*& yb, const double*& bb,
    int cs, double (&xm)[RY], double (&x0v)[RY], double (&xp)[RY],
    double (&lm)[RY], double (&lc)[RY], double (&ln)[RY]) {
  constexpr bool D3 = ND == 7;
  if (t >= G.nsteps) return false;
  const int q = G.za - 1 + t;
  // x plane q + 1 (load index t + 2); its in-plane neighbours (plane q) are
  // in the slot of load index t + 1
  const uint32_t xn = R.xn, xq = R.xq;
  // planes outside the box arrive as zeros (copied from P.zeros)
  mbar_wait(x_full + R.sn, R.pn);
#pragma unroll
  for (int r = 0; r < RY; ++r) xp[r] = g2_lds<0>(xn + C.aX[r]);
  if (!ONE && t >= 2 && q >= 0 && q < G.nz) {
    // steady state: wait for level 1 of step t - 1 first, then compute
    // level 1 at plane q and level 2 at plane q - 1 in one block, so the
    // 2 RY row-sum chains interleave (the DADD chains are the latency)
    mbar_wait(l1_done + R.br, R.brp);
    const uint32_t lw = R.lw, lr = R.lr;
    double u[RY], z[RY];
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      const uint32_t a = xq + C.aX[r];
      const uint32_t b = lr + C.aL[r];
      double s1, s2;
      if constexpr (D3) {
        const double ym = r > 0 ? x0v[r > 0 ? r - 1 : 0] : g2_lds<0>(xq + C.aXm);
        const double yp = r < RY - 1 ? x0v[r < RY - 1 ? r + 1 : 0] : g2_lds<0>(xq + C.aXp);
        const double t1[7] = {xm[r], ym, g2_lds<-8>(a), x0v[r], g2_lds<8>(a), yp, xp[r]};
        // (halo lines have no level 2: their outer neighbours lie outside
        // the level-1 slot, so those loads are skipped, warp-uniformly)
        const double lym = r > 0 ? lc[r > 0 ? r - 1 : 0] : (C.w2[r] ? g2_lds<0>(lr + C.aLm) : 0.0);
        const double lyp = r < RY - 1 ? lc[r < RY - 1 ? r + 1 : 0]
                                      : (C.w2[r] ? g2_lds<0>(lr + C.aLp) : 0.0);
        s1 = g2_sum<7>(v, t1);
        const double t2[7] = {lm[r], lym, g2_lds<-8>(b), lc[r], g2_lds<8>(b), lyp, 0.0};
        // the +D term of level 2 is level 1 of this step: summed last
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < 6; ++j) acc = __dadd_rn(acc, __dmul_rn(v[j], t2[j]));
        s2 = acc;
      } else {
        const double t1[5] = {xm[r], g2_lds<-8>(a), x0v[r], g2_lds<8>(a), xp[r]};
        s1 = g2_sum<5>(v, t1);
        double acc = 0.0;
        const double t2[4] = {lm[r], g2_lds<-8>(b), lc[r], g2_lds<8>(b)};
#pragma unroll
        for (int j = 0; j < 4; ++j) acc = __dadd_rn(acc, __dmul_rn(v[j], t2[j]));
        s2 = acc;
      }
      u[r] = PAIR ? s1 : __dadd_rn(x0v[r], __dmul_rn(P.a0, s1));
      ln[r] = C.v1[r] ? u[r] : 0.0;
      if (C.v1[r]) g2_sts(lw + C.aL[r], u[r]);
      // the level-2 sum's last term (+D: level 1 at plane q, own column)
      s2 = __dadd_rn(s2, __dmul_rn(v[ND - 1], ln[r]));
      z[r] = PAIR ? __dadd_rn(__dadd_rn(xm[r], __dmul_rn(P.a1, lc[r])), __dmul_rn(P.a0, s2))
                  : __dadd_rn(lc[r], __dmul_rn(P.b0, s2));
    }
    __syncwarp();
    if (lane == 0) g2_arrive(l1_done + R.bw);
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      if (C.v2[r]) {
        double zz = z[r];
        if (COMPL) zz = __dsub_rn(__ldg(bb + r * cs), zz);
        yb[r * cs] = zz;
      }
    }
  } else {
  // ---- level 1 at plane q into level-1 slot t % 4 (last read by level 2 of
  // step t - 3, which every warp finished before arriving at step t - 2, and
  // this warp waited for that barrier in step t - 1)
  if (q >= 0 && q < G.nz) {
    const uint32_t lw = R.lw;
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      const uint32_t a = xq + C.aX[r];
      double s;
      if constexpr (D3) {
        const double ym = r > 0 ? x0v[r > 0 ? r - 1 : 0] : g2_lds<0>(xq + C.aXm);
        const double yp = r < RY - 1 ? x0v[r < RY - 1 ? r + 1 : 0] : g2_lds<0>(xq + C.aXp);
        const double tt[7] = {xm[r], ym, g2_lds<-8>(a), x0v[r], g2_lds<8>(a), yp, xp[r]};
        s = g2_sum<7>(v, tt);
      } else {
        const double tt[5] = {xm[r], g2_lds<-8>(a), x0v[r], g2_lds<8>(a), xp[r]};
        s = g2_sum<5>(v, tt);
      }
      const double u = PAIR ? s : __dadd_rn(x0v[r], __dmul_rn(P.a0, s));
      if constexpr (ONE) {
        // one factor: level 1 of the tile's planes [za, zb) is the output
        // (yb points at plane q - 1)
        if (C.v2[r] && t >= 1 && t <= G.nsteps - 2) yb[G.D + r * cs] = u;
      } else {
        ln[r] = C.v1[r] ? u : 0.0;
        if (C.v1[r]) g2_sts(lw + C.aL[r], u);
      }
    }
  } else {
#pragma unroll
    for (int r = 0; r < RY; ++r) ln[r] = 0.0;
  }
  // one arrival per warp: __syncwarp orders the lanes' level-1 stores before
  // lane 0's (release) arrival; per-thread arrivals on one mbarrier
  // serialise in the SYNCS unit
  __syncwarp();
  if (lane == 0) g2_arrive(l1_done + R.bw);
  // ---- level 2 at plane q - 1: wait until every warp stored level 1 of
  // step t - 1 (this warp's own level-1 work of step t overlapped the wait)
  if (!ONE && t >= 2) {
    mbar_wait(l1_done + R.br, R.brp);
    const uint32_t lr = R.lr;
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      if (!C.w2[r]) continue;  // warp-uniform: a halo line
      const uint32_t a = lr + C.aL[r];
      double s;
      if constexpr (D3) {
        const double ym = r > 0 ? lc[r > 0 ? r - 1 : 0] : g2_lds<0>(lr + C.aLm);
        const double yp = r < RY - 1 ? lc[r < RY - 1 ? r + 1 : 0] : g2_lds<0>(lr + C.aLp);
        const double tt[7] = {lm[r], ym, g2_lds<-8>(a), lc[r], g2_lds<8>(a), yp, ln[r]};
        s = g2_sum<7>(v, tt);
      } else {
        const double tt[5] = {lm[r], g2_lds<-8>(a), lc[r], g2_lds<8>(a), ln[r]};
        s = g2_sum<5>(v, tt);
      }
      double z = PAIR ? __dadd_rn(__dadd_rn(xm[r], __dmul_rn(P.a1, lc[r])), __dmul_rn(P.a0, s))
                      : __dadd_rn(lc[r], __dmul_rn(P.b0, s));
      if (C.v2[r]) {
        if (COMPL) z = __dsub_rn(__ldg(bb + r * cs), z);
        yb[r * cs] = z;
      }
    }
  }
  }
  // ---- advance the output rows and the rings
  yb += G.D;
  if (COMPL) bb += G.D;
  R.xq = R.xn;
  R.xn += R.xstep;
  if (++R.sn == NS) {
    R.sn = 0;
    R.pn ^= 1;
    R.xn = R.xbeg;
  }
  R.lr = R.lw;
  R.lw += R.lstep;
  if (R.lw == R.lend) R.lw = R.lbeg;
  R.br = R.bw;
  R.brp = R.bwp;
  if (++R.bw == 2 * NS) {
    R.bw = 0;
    R.bwp ^= 1;
  }
  return true;
}

// The producer warp: refills the x slot of load index t with load index
// t + NS once every consumer warp has stored level 1 of step t - 1 (the last
// reader of that slot, x plane q - 1).
// Wait (all lanes of the producer warp, system scope) until a neighbour
// published the pass that wrote its buffer; then its halo planes may be
// copied through the async proxy.  Bounded: on timeout the error word is set
// and the copies go ahead with stale data rather than hanging the consumers.
__device__ __forceinline__ void g2_peer_wait(const long long* flag, long long epoch, int* err) {
  long long spins = 0, v;
  for (;;) {
    asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v >= epoch) break;
    __nanosleep(256);
    if (++spins > (1LL << 25)) {
      if (err) atomicExch(err, 1);
      break;
    }
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <bool D3, int NS, bool SLAB>
__device__ __forceinline__ void g2_produce(const G2Geo& G, const G2Params& P, char* sb,
                                           uint64_t* x_full, uint64_t* l1_done, int lane,
                                           const double* __restrict__ x, int x0, int xa, int y0,
                                           int ylo, int yhi, uint32_t line_bytes,
                                           uint32_t plane_bytes, int i0, int i1, int tstart) {
  const uint32_t sbase = smem_u32(sb);
  for (int i = i0; i < i1; ++i) {
    // the slot of load index i - NS was last read by level 1 of consumer
    // step i - NS - 1 (index 0: by the consumers' first loads, before step 0)
    const int t = i - NS;
    if (t >= tstart) {
      const int tp = t > 0 ? t - 1 : 0;
      mbar_wait(l1_done + tp % (2 * NS), (tp / (2 * NS)) & 1);
    }
    const int p = G.za - 2 + i;
    const bool pin = p >= 0 && p < G.nz;
    const int sl_i = i % NS;
    // the plane's source: this rank's x, a neighbour's buffer (slab mode:
    // the first halo plane of a pass waits for the neighbour's flag), or the
    // zero page outside the box
    const double* pb = P.zeros;
    if (!SLAB) {
      if (pin) pb = x + static_cast<long long>(p) * G.D;
    } else if (pin) {
      if (p < P.zo0) {
        if (i == 0 || p == 0) g2_peer_wait(P.fl, P.epoch, P.err);  // first halo plane
        pb = P.xl + static_cast<long long>(p - P.zl0) * G.D;
      } else if (p >= P.zo1) {
        if (p == P.zo1) g2_peer_wait(P.fr, P.epoch, P.err);
        pb = P.xr + static_cast<long long>(p - P.zo1) * G.D;
      } else {
        pb = x + static_cast<long long>(p - P.zo0) * G.D;
      }
    }
    if (lane == 0) mbar_expect_tx(x_full + sl_i, plane_bytes);
    __syncwarp();
    for (int yy = ylo + lane; yy < yhi; yy += 32) {
      const int sl = D3 ? yy - (y0 - 2) : 0;
      const uint32_t dst = sbase + 8u * static_cast<uint32_t>(G.xs0 + sl_i * G.slot_x +
                                                               sl * P.P + (xa - (x0 - 2)));
      const double* src =
          pin ? pb + (static_cast<long long>(yy) * P.nx + xa) : P.zeros;
      g2_bulk(dst, src, line_bytes, smem_u32(x_full + sl_i));
    }
  }
}

// NT consumer threads plus one producer warp.
template <int ND, int RY, bool PAIR, bool COMPL, int NT, bool ONE, bool SLAB>
__global__ void __launch_bounds__(NT + 32, 1)
    k_spmv_grid2(const double* __restrict__ x, double* y, const double* __restrict__ base,
                 G2Params P) {
  static_assert(ND == 5 || ND == 7, "5- or 7-point stencils");
  constexpr bool D3 = ND == 7;
  constexpr int NS = D3 ? 6 : 12;  // x slots
  P.y_q = y;
  P.base_q = base;
  extern __shared__ __align__(128) double g2_sm[];
  char* sb = reinterpret_cast<char*>(g2_sm);
  uint64_t* x_full = reinterpret_cast<uint64_t*>(g2_sm);
  uint64_t* l1_done = x_full + G2_MAXSLOT;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int nx = P.nx, ny = P.ny, nz = P.nz, Pt = P.P;

  // ---- tile and chunk
  const int ntile = P.ntx * P.nty;
  const int tile = blockIdx.x % ntile;
  const int chunk = blockIdx.x / ntile;
  const int tx = tile % P.ntx, ty = tile / P.ntx;
  const int x0 = (tx * nx / P.ntx) & ~1;
  const int x1 = tx + 1 == P.ntx ? nx : ((tx + 1) * nx / P.ntx) & ~1;
  const int y0 = D3 ? ty * ny / P.nty : 0;
  const int y1 = D3 ? (ty + 1) * ny / P.nty : 1;
  G2Geo G;
  // chunks of the owned planes [zo0, zo1) (all of [0, nz) unsharded)
  const int zo0 = SLAB ? P.zo0 : 0, nzo = SLAB ? P.zo1 - P.zo0 : nz;
  G.za = zo0 + static_cast<int>(static_cast<long long>(chunk) * nzo / P.nchunks);
  const int zb = zo0 + static_cast<int>(static_cast<long long>(chunk + 1) * nzo / P.nchunks);
  G.nsteps = zb - G.za + 2;  // level-1 planes za-1 .. zb
  G.nz = nz;
  G.D = P.D;
  G.xs0 = G2_BARS;
  G.slot_x = P.SL * Pt;
  G.ls0 = G.xs0 + NS * G.slot_x;
  G.slot_l = P.LL * Pt;
  const int nload = G.nsteps + 2;  // x planes za-2 .. zb+1

  // ---- init barriers; overlaps the previous pass (PDL)
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(x_full + s, 1);
    for (int s = 0; s < 2 * NS; ++s) mbar_init(l1_done + s, NT / 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();  // x is the previous pass's output

  const int xa = max(x0 - 2, 0), xb = min(x1 + 2, nx);
  const int ylo = D3 ? max(y0 - 2, 0) : 0, yhi = D3 ? min(y1 + 2, ny) : 1;
  const uint32_t line_bytes = static_cast<uint32_t>(xb - xa) * 8u;
  const uint32_t plane_bytes = line_bytes * static_cast<uint32_t>(yhi - ylo);

  if (warp == NT / 32) {
    // producer warp: the first NS loads at once, then one refill per step
    g2_produce<D3, NS, SLAB>(G, P, sb, x_full, l1_done, lane, x, x0, xa, y0, ylo, yhi,
                             line_bytes, plane_bytes, 0, min(NS, nload), 0);
    g2_produce<D3, NS, SLAB>(G, P, sb, x_full, l1_done, lane, x, x0, xa, y0, ylo, yhi,
                             line_bytes, plane_bytes, NS, nload, 0);
    return;
  }

  // ---- zero the slot cells that are read but never written - the pad
  // columns of each line and whole lines outside the box or the tile - while
  // the first planes are in flight (the copies and the level-1 stores write
  // the other cells before they are read; these cells are disjoint from the
  // copies, so no proxy fence is needed)
  {
    // x slots: copies write lines [xl0, xl1), columns [xw0, xw1)
    const int xw0 = xa - (x0 - 2), xw1 = xb - (x0 - 2);
    const int xl0 = D3 ? ylo - (y0 - 2) : 0, xl1 = D3 ? yhi - (y0 - 2) : 1;
    // level-1 slots: stores write lines [ll0, ll1), columns [lw0, lw1)
    int lw0, lw1, ll0, ll1;
    if (D3) {
      lw0 = 2;
      lw1 = nx + 2;
      ll0 = max(0, 1 - y0);
      ll1 = min(y1 - y0 + 2, ny - y0 + 1);
    } else {
      lw0 = max(x0 - 1, 0) - x0 + 2;
      lw1 = min(x1 + 1, nx) - x0 + 2;
      ll0 = 0;
      ll1 = 1;
    }
    const int nxl = NS * P.SL, nll = G2_LSLOT * P.LL;
    for (int k = tid; k < nxl + nll; k += NT) {
      const bool isx = k < nxl;
      const int kk = isx ? k : k - nxl;
      const int sl = kk / (isx ? P.SL : P.LL), line = kk % (isx ? P.SL : P.LL);
      double* row = g2_sm + (isx ? G.xs0 + sl * G.slot_x : G.ls0 + sl * G.slot_l) + line * Pt;
      const bool in = isx ? (line >= xl0 && line < xl1) : (line >= ll0 && line < ll1);
      const int c0 = in ? (isx ? xw0 : lw0) : Pt, c1 = in ? (isx ? xw1 : lw1) : Pt;
      for (int c = 0; c < c0; ++c) row[c] = 0.0;
      for (int c = c1; c < Pt; ++c) row[c] = 0.0;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");
  }

  // ---- cells of this (consumer) thread
  G2Cells<RY> C;
  if constexpr (D3) {
    // TX = nx: columns [0, nx); the cell's slot column is x + 2.  The planner
    // makes the line groups tile the level-1 slot exactly (LL = groups x RY).
    const bool wok = warp < P.cw;
    const int seg = warp % P.segs, g = wok ? warp / P.segs : 0;
    const int xc = seg * 32 + lane;
    const bool xin = wok && xc < nx;
    const int c = xin ? xc + 2 : 0;
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      const int yl = g * RY + r;  // level-1 slot line; grid line y0 - 1 + yl
      const int yy = y0 - 1 + yl;
      C.aL[r] = 8 * (yl * Pt + c);
      C.aX[r] = C.aL[r] + 8 * Pt;
      C.v1[r] = xin && yl < (y1 - y0) + 2 && yy >= 0 && yy < ny;
      C.v2[r] = xin && yl >= 1 && yl <= y1 - y0;
      C.row2[r] = yy * nx + xc;
    }
    C.aXm = C.aX[0] - 8 * Pt;
    C.aXp = C.aX[RY - 1] + 8 * Pt;
    C.aLm = C.aL[0] - 8 * Pt;
    C.aLp = C.aL[RY - 1] + 8 * Pt;
  } else {
    const int xl = max(x0 - 1, 0), xr = min(x1 + 1, nx);
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      const int xc = xl + (warp * RY + r) * 32 + lane;
      const bool in = xc < xr;
      C.aL[r] = C.aX[r] = 8 * (in ? xc - x0 + 2 : 1);
      C.v1[r] = in;
      C.v2[r] = in && xc >= x0 && xc < x1;
      C.row2[r] = xc;
    }
    C.aXm = C.aXp = C.aLm = C.aLp = 0;
  }
#pragma unroll
  for (int r = 0; r < RY; ++r) C.w2[r] = __any_sync(0xffffffffu, C.v2[r]);
  double v[7];
#pragma unroll
  for (int j = 0; j < 7; ++j) {
    v[j] = j < ND ? P.val[j] : 0.0;
    asm volatile("" : "+d"(v[j]));  // keep the coefficients in registers
  }
  const uint32_t sbase = smem_u32(g2_sm);
  // output rows of cell 0 at the level-2 plane of step 0 (za - 2; advanced
  // by one plane per step, dereferenced only for level-2 cells); cell r sits
  // cs rows further (3-D: the next grid line, 2-D: the next 32-column segment)
  const long long row0 = static_cast<long long>(G.za - 2 - zo0) * G.D + C.row2[0];
  double* yb = y + row0;
  const double* bb = COMPL ? base + row0 : nullptr;
  const int cs = D3 ? nx : 32;

  // registers: x and level-1 values of three consecutive planes per cell,
  // in rotating triples (a, b, c); x planes za-2 and za-1 first
  double xa_[RY], xb_[RY], xc_[RY], la[RY], lb[RY], lcc[RY];
  mbar_wait(x_full + 0, 0);
  mbar_wait(x_full + 1, 0);
  {
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      xa_[r] = g2_lds<0>(sbase + 8u * G.xs0 + C.aX[r]);
      xb_[r] = g2_lds<0>(sbase + 8u * (G.xs0 + G.slot_x) + C.aX[r]);
      xc_[r] = la[r] = lb[r] = lcc[r] = 0.0;
    }
  }
  G2Ring R;
  R.xstep = 8u * G.slot_x;
  R.xbeg = sbase + 8u * G.xs0;
  R.xend = R.xbeg + NS * R.xstep;
  R.xq = R.xbeg + R.xstep;
  R.xn = R.xbeg + 2 * R.xstep;
  R.sn = 2;
  R.pn = 0;
  R.lstep = 8u * G.slot_l;
  R.lbeg = sbase + 8u * G.ls0;
  R.lend = R.lbeg + G2_LSLOT * R.lstep;
  R.lw = R.lbeg;
  R.lr = R.lbeg + (G2_LSLOT - 1) * R.lstep;
  R.bw = 0;
  R.bwp = 0;
  R.br = 2 * NS - 1;
  R.brp = 1;
#define G2_STEP(XM, X0, XP, LM, LC, LN)                                                     \
  if (!g2_step<ND, RY, PAIR, COMPL, NS, ONE>(t++, G, C, P, v, R, x_full, l1_done, lane, yb, bb, cs, \
                                        XM, X0, XP, LM, LC, LN)) {                          \
    break;                                                                                  \
  }
  for (int t = 0;;) {
    G2_STEP(xa_, xb_, xc_, la, lb, lcc)
    G2_STEP(xb_, xc_, xa_, lb, lcc, la)
    G2_STEP(xc_, xa_, xb_, lcc, la, lb)
  }
#undef G2_STEP
  if constexpr (SLAB) {
    // publish the pass: every consumer's stores, then a device-scope fence
    // per CTA and a ticket; the CTA that completes the grid's count has
    // observed every CTA's stores through the tickets and releases epoch + 1
    // into this rank's flag at system scope (cumulative; no publish launch)
    // Only CTAs whose chunk reads a neighbour's planes or writes planes a
    // neighbour reads (within two planes of a shared slab face) take part;
    // the others exit at once (the next pass on this rank is stream-ordered).
    auto touches = [&](int a, int b) {
      return (P.zo0 > 0 && a < P.zo0 + 2) || (P.zo1 < nz && b > P.zo1 - 2);
    };
    if (P.own && touches(G.za, zb)) {
      int parts = 0;  // participating CTAs (every tile of a touching chunk)
      for (int c = 0; c < P.nchunks; ++c) {
        const int a = zo0 + static_cast<int>(static_cast<long long>(c) * nzo / P.nchunks);
        const int b = zo0 + static_cast<int>(static_cast<long long>(c + 1) * nzo / P.nchunks);
        parts += touches(a, b) ? P.ntx * P.nty : 0;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");
      if (tid == 0) {
        __threadfence();
        const unsigned long long tk =
            atomicAdd(reinterpret_cast<unsigned long long*>(P.own + 1), 1ull);
        if ((tk + 1) % static_cast<unsigned long long>(parts) == 0) {
          asm volatile("fence.acq_rel.sys;" ::: "memory");
          asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(P.own), "l"(P.epoch + 1)
                       : "memory");
        }
      }
    }
  }
}

template <int ND, int RY, bool PAIR, bool COMPL, int NT, bool ONE, bool SLAB>
void launch_g2(const G2Params& P, const G2Plan& pl, const double* x, double* y,
               const double* base, cudaStream_t st) {
  auto kernel = k_spmv_grid2<ND, RY, PAIR, COMPL, NT, ONE, SLAB>;
  // the attribute is per device: set it on every launch (cheap) rather than
  // once per process
  PPA_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(pl.smem)));
  launch_pdl(kernel, dim3(pl.ntx * pl.nty * pl.nchunks), dim3(NT + 32), pl.smem, st, x, y, base,
             P);
}

template <int ND, int RY, bool PAIR, bool COMPL, bool ONE = false, bool SLAB = false>
void launch_g2_nt(const G2Params& P, const G2Plan& pl, const double* x, double* y,
                  const double* base, cudaStream_t st) {
  // thread counts in steps of 32 lanes x segments: instantiate the multiples
  // of 64 up to 1024 and round the plan up (extra warps own no cells)
  switch ((pl.nt + 63) / 64) {
#define G2_NT(k)                                                     \
  case k:                                                            \
    if constexpr (64 * k <= g2_maxnt(ND, RY)) {                      \
      return launch_g2<ND, RY, PAIR, COMPL, 64 * k, ONE, SLAB>(P, pl, x, y, base, st); \
    }                                                                \
    break;
    G2_NT(1) G2_NT(2) G2_NT(3) G2_NT(4) G2_NT(5) G2_NT(6) G2_NT(7) G2_NT(8) G2_NT(9)
    G2_NT(10) G2_NT(11) G2_NT(12) G2_NT(13) G2_NT(14) G2_NT(15)
#undef G2_NT
    default: break;
  }
  throw std::runtime_error("spmv_grid2: unsupported thread count");
}

template <int ND, int RY>
void launch_g2_m(const G2Params& P, const G2Plan& pl, bool pair, const double* x, double* y,
                 const double* base, cudaStream_t st, bool one = false, bool slab = false) {
  // slab mode (neighbours' halo planes, owned plane range) and single real
  // factors have their own instantiations, so the unsharded pass's producer
  // keeps its plain source computation
  if (one) {  // a single real factor (the sharded pass's leftovers; no complement)
    launch_g2_nt<ND, RY, false, false, true, true>(P, pl, x, y, base, st);
  } else if (slab) {
    pair ? launch_g2_nt<ND, RY, true, false, false, true>(P, pl, x, y, base, st)
         : launch_g2_nt<ND, RY, false, false, false, true>(P, pl, x, y, base, st);
  } else if (pair) {
    base ? launch_g2_nt<ND, RY, true, true>(P, pl, x, y, base, st)
         : launch_g2_nt<ND, RY, true, false>(P, pl, x, y, base, st);
  } else {
    base ? launch_g2_nt<ND, RY, false, true>(P, pl, x, y, base, st)
         : launch_g2_nt<ND, RY, false, false>(P, pl, x, y, base, st);
  }
}

}  // namespace
}  // namespace kern
}  // namespace ppa

// The body of spmv_grid2_i<ND><RY>.cu.
#define PPA_G2_DEFINE(ND, RY)                                                                  \
  namespace ppa {                                                                              \
  namespace kern {                                                                             \
  namespace g2 {                                                                               \
  void launch_##ND##_##RY(const G2Params& P, const G2Plan& pl, bool pair, const double* x,     \
                          double* y, const double* base, cudaStream_t st, bool one, bool slab) { \
    launch_g2_m<ND, RY>(P, pl, pair, x, y, base, st, one, slab);                               \
  }                                                                                            \
  }                                                                                            \
  }                                                                                            \
  }
