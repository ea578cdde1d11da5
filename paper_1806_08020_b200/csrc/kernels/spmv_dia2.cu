// Two polynomial factors per pass over a stencil matrix (temporal blocking of
// the diagonal layout): the pass reads x once and writes only the second
// factor's output, so a pair of factors moves 16n bytes of vectors instead of
// 32n.  Replaces two consecutive launches of the factor chain
// (src/gmres_poly.cpp:129-143):
//   two real roots : u = x + a0 (A x),  y = u + b0 (A u)
//   conjugate pair : t = A x,           y = (x + a1 t) + a0 (A t)
// optionally followed by the complement y = base - y (src/gmres_poly.cpp:306-308).
// Every row sum visits the diagonals in increasing offset (= the CSR's column
// order) and skips absent entries, with __dmul_rn/__dadd_rn: bit-identical to
// the two single-factor launches and to the CPU loop.
//
// Applies to 3-, 5- and 7-point stencils in the regular-row diagonal layout
// (centre offset 0 in the middle, outer diagonals +-D: the plane offset of a
// 3-D stencil, the row offset of a 2-D one) when every present entry carries
// its diagonal's default value (stencils truncated at the boundary; presence
// is one byte per row, dia_pres).
//
// Geometry.  Row r = q D + c is column c of plane q.  A CTA owns a column tile
// [c0, c0 + TW) of a chunk of planes [qa, qb) and marches through the planes:
//   step q : level 1 (the first factor) at plane q over the extended tile
//            [c0 - Dm, c0 + TW + Dm)   (Dm = largest in-plane offset |off|)
//            level 2 (the second factor) at plane q - 1 over the tile.
// Level 1 at plane q reads x planes q-1, q, q+1; level 2 reads the level-1
// planes q-2, q-1, q.  Each thread owns columns e = tid + k*NT of the extended
// tile and keeps its own column's x and level-1 values of three consecutive
// planes in registers (the +-D and centre terms); the in-plane neighbours come
// from shared memory: x planes and their presence bytes arrive by
// cp.async.bulk into a ring of NSLOT slots (prefetched NSLOT-2 planes ahead),
// level-1 planes are stored into a ring of three.  One __syncthreads per
// step; the step loop is unrolled six times so the register triples and the
// slot indices are fixed per unrolled step.
//
// The halo rows (level 1 outside the tile, planes qa-1 and qb) are computed
// twice, by neighbouring CTAs; the host picks the tile width, chunk count
// and CTAs per SM that minimise the per-SM work (f2_plan).  Issue-bound on
// B200, not HBM-bound.

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "pdl.cuh"
#include "tma.cuh"
#include "ppa/kernels.hpp"

namespace ppa {
namespace kern {
namespace {

constexpr int F2_NSLOT = 6;   // x-plane slots (prefetch NSLOT - 2 planes ahead)
constexpr int F2_LSLOT = 3;   // level-1 plane slots
constexpr int F2_XS = 16;     // first double of the x slots (the mbarriers sit below)

// Most threads per CTA for KC owned columns per thread (registers: ~10 per
// column of state plus the step's temporaries).
constexpr int f2_max_nt(int kc) { return kc <= 2 ? 1024 : kc == 3 ? 768 : 512; }

struct F2Params {
  int off[8];
  double val[8];
  int n, D, Dm, E1, E2, TW, SH, ntiles, nq, nchunks;
  int ppad;  // zero rows of dia_pres on each side (a multiple of 16)
  double a0, a1, b0;
};

__device__ __forceinline__ void bulk_load_plain(uint32_t dst, const void* src, uint32_t bytes,
                                                uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// Row sum: diagonals in increasing offset.  xm / xp are the -D / +D terms,
// xc the centre (diagonal JC, offset 0), the other middle terms sm[c + off_j].
// CHECK: an absent term contributes val * (+0.0), which leaves the sum's bits
// unchanged (the sum starts at +0.0 and round-to-nearest never produces -0.0
// from it), i.e. exactly the reference's skipped entry, even for inf/nan x.
// Addresses are split into a per-thread byte offset tb and a warp-uniform
// one (ub + 8 off_j) so the loads use the [R + UR] form.
__device__ __forceinline__ double f2_lds(const char* smc, uint32_t tb, int ub) {
  return *reinterpret_cast<const double*>(smc + (tb + static_cast<uint32_t>(ub)));
}

// Row sum: diagonals in increasing offset.  xm / xp are the -D / +D terms,
// xc the centre (diagonal JC, offset 0), the other middle terms at byte
// tb + ub + 8 off_j.  CHECK: an absent term (bit j of pr clear) contributes
// val * (+0.0), which leaves the sum's bits unchanged (the sum starts at +0.0
// and round-to-nearest never produces -0.0 from it), i.e. exactly the
// reference's skipped entry, even for inf/nan x.
// UNIT: the diagonals next to the centre are offsets -1 and +1 (every 2-D
// and 3-D stencil), read at immediate offsets.
template <int ND, bool UNIT, bool CHECK>
__device__ __forceinline__ double f2_row(const F2Params& P, unsigned pr, double xm, double xc,
                                         double xp, const char* smc, uint32_t tb, int ub) {
  constexpr int JC = (ND - 1) / 2;
  double s = 0.0;
  s = __dadd_rn(s, __dmul_rn(P.val[0], CHECK && !(pr & 1u) ? 0.0 : xm));
#pragma unroll
  for (int j = 1; j < ND - 1; ++j) {
    const int o = UNIT && j == JC - 1 ? -1 : UNIT && j == JC + 1 ? 1 : P.off[j];
    double v = j == JC ? xc : f2_lds(smc, tb, ub + 8 * o);
    if (CHECK && !(pr & (1u << j))) v = 0.0;
    s = __dadd_rn(s, __dmul_rn(P.val[j], v));
  }
  s = __dadd_rn(s, __dmul_rn(P.val[ND - 1], CHECK && !(pr & (1u << (ND - 1))) ? 0.0 : xp));
  return s;
}

// Shared-memory map (doubles): [0, 16) mbarriers; x slots F2_XS + s E2;
// level-1 slots ls + s E1; presence slots (bytes) after them, PW bytes each.
// Per-thread constants of one CTA.
template <int KC>
struct F2Thread {
  int ee[KC];     // owned column (0 for lanes past E1)
  uint32_t eb[KC];  // 8 ee
  uint32_t cb[KC];  // 8 x (core ? ee : Dm): level-2 column (halo lanes read a valid one)
  bool own[KC];   // column inside the extended tile
  bool core[KC];  // column inside the tile (level 2 stores it)
  bool wcore[KC]; // some lane of the warp has a core column k
  int ls;         // first double of the level-1 slots
  int ps;         // first byte of the presence slots
  int pw;         // bytes per presence slot
  int qa, nsteps, c0, rbase;  // rbase = c0 - Dm - SH: the row of column e is q D + rbase + e
};

// One step of the march (t = 6 u + V): level 1 at plane q = qa - 1 + t,
// level 2 at plane q - 1.  The register triples rotate with period 3 and the
// slots with period 6, so the six unrolled steps use fixed registers and
// fixed slot indices.
template <int ND, bool UNIT, int KC, bool PAIR, bool COMPL, int V>
__device__ __forceinline__ bool f2_step(const F2Params& P, const F2Thread<KC>& T, int u,
                                        double* __restrict__ sm, uint64_t* bar,
                                        const double* __restrict__ x, double* y,
                                        const double* __restrict__ base, const unsigned char* pres,
                                        double (&xm)[KC], double (&x0)[KC], double (&xp)[KC],
                                        double (&l1m)[KC], double (&l1c)[KC], double (&l1n)[KC],
                                        const unsigned (&pr_prev)[KC], unsigned (&prc)[KC]) {
  const int t = 6 * u + V;
  if (t >= T.nsteps) return false;
  const int q = T.qa - 1 + t;
  const int D = P.D, Dm = P.Dm, E1 = P.E1, E2 = P.E2;
  constexpr int SQ = (V + 1) % F2_NSLOT, SP = (V + 2) % F2_NSLOT;
  mbar_wait(bar + SP, (u + (V >= 4 ? 1 : 0)) & 1);  // plane q + 1 (plane q: one step earlier)
  const int xq = F2_XS + SQ * E2 + Dm;  // column e of plane q at xq + e
  const int xn = F2_XS + SP * E2 + Dm;  // plane q + 1
  // presence slots hold rows from a 16-byte aligned start: plane p's row of
  // column e at byte ps + s pw + e + ((p D + rbase) & 15)
  const unsigned char* pb = reinterpret_cast<const unsigned char*>(sm);
  const char* smc = reinterpret_cast<const char*>(sm);
  const int pq = T.ps + SQ * T.pw + ((q * D + T.rbase) & 15);
  constexpr unsigned kAll = (1u << ND) - 1u;
  // presence of plane q - 1 (level 2) is the previous step's plane-q presence
  unsigned prp[KC];
  bool full = true;
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    xp[k] = f2_lds(smc, T.eb[k], 8 * xn);
    prc[k] = T.own[k] ? pb[static_cast<uint32_t>(T.ee[k]) + static_cast<uint32_t>(pq)] : kAll;
    prp[k] = T.core[k] ? pr_prev[k] : kAll;
    full = full && prc[k] == kAll;
  }
  // ---- level 1 at plane q (warp-uniform: interior warps skip the presence tests)
  if (__all_sync(0xffffffffu, full)) {
#pragma unroll
    for (int k = 0; k < KC; ++k) {
      const double s = f2_row<ND, UNIT, false>(P, kAll, xm[k], x0[k], xp[k], smc, T.eb[k], 8 * xq);
      l1n[k] = PAIR ? s : __dadd_rn(x0[k], __dmul_rn(P.a0, s));
    }
  } else {
#pragma unroll
    for (int k = 0; k < KC; ++k) {
      const double s = f2_row<ND, UNIT, true>(P, prc[k], xm[k], x0[k], xp[k], smc, T.eb[k], 8 * xq);
      l1n[k] = PAIR ? s : __dadd_rn(x0[k], __dmul_rn(P.a0, s));
    }
  }
  const int lw = T.ls + (V % F2_LSLOT) * E1;
  const int lr = T.ls + ((V + 2) % F2_LSLOT) * E1;
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    if (T.own[k]) {
      *reinterpret_cast<double*>(reinterpret_cast<char*>(sm) +
                                 (T.eb[k] + static_cast<uint32_t>(8 * lw))) = l1n[k];
    }
  }
  // level-1 plane q visible to the next step, whose refill of this step's
  // plane q - 1 slot relies on every thread having passed here
  __syncthreads();
  // ---- level 2 at plane q - 1
  if (t >= 2) {
    const int r2q = q * D + T.rbase - D;
    bool full2 = true;
#pragma unroll
    for (int k = 0; k < KC; ++k) full2 = full2 && prp[k] == kAll;
    const bool f2all = __all_sync(0xffffffffu, full2);
#pragma unroll
    for (int k = 0; k < KC; ++k) {
      if (!T.wcore[k]) continue;  // warp-uniform: the whole warp is in the halo
      const double s =
          f2all ? f2_row<ND, UNIT, false>(P, kAll, l1m[k], l1c[k], l1n[k], smc, T.cb[k], 8 * lr)
                : f2_row<ND, UNIT, true>(P, prp[k], l1m[k], l1c[k], l1n[k], smc, T.cb[k], 8 * lr);
      double z = PAIR ? __dadd_rn(__dadd_rn(xm[k], __dmul_rn(P.a1, l1c[k])), __dmul_rn(P.a0, s))
                      : __dadd_rn(l1c[k], __dmul_rn(P.b0, s));
      const int r2 = r2q + T.ee[k];
      if (T.core[k] && r2 < P.n) {
        if (COMPL) z = __dsub_rn(__ldg(base + r2), z);
        y[r2] = z;
      }
    }
  }
  return true;
}

template <int ND, bool UNIT, int KC, bool PAIR, bool COMPL>
__global__ void __launch_bounds__(f2_max_nt(KC), 1) k_spmv_dia2(
    const unsigned char* __restrict__ pres, const double* __restrict__ x, double* y,
    const double* __restrict__ base, const F2Params P) {
  extern __shared__ __align__(128) double f2_sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(f2_sm);
  const uint32_t sm_base = smem_u32(f2_sm);
  const int tid = threadIdx.x;
  const int NT = blockDim.x;
  const int tile = blockIdx.x % P.ntiles;
  const int chunk = blockIdx.x / P.ntiles;
  const int n = P.n, D = P.D, Dm = P.Dm, E1 = P.E1, E2 = P.E2;
  F2Thread<KC> T;
  T.c0 = tile * P.TW;
  T.rbase = T.c0 - Dm - P.SH;
  T.qa = static_cast<int>(static_cast<long long>(chunk) * P.nq / P.nchunks);
  const int qb = static_cast<int>(static_cast<long long>(chunk + 1) * P.nq / P.nchunks);
  T.nsteps = qb - T.qa + 2;  // q = qa-1 .. qb
  T.ls = F2_XS + F2_NSLOT * E2;
  T.ps = 8 * (T.ls + F2_LSLOT * E1);
  T.pw = (E1 + 31) & ~15;
  const int twe = min(P.TW, D - T.c0);  // columns of this tile inside the plane
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    const int e = tid + k * NT;
    T.own[k] = e < E1;
    T.ee[k] = T.own[k] ? e : 0;
    T.core[k] = T.own[k] && e >= Dm + P.SH && e < Dm + P.SH + twe;
    T.eb[k] = 8u * static_cast<uint32_t>(T.ee[k]);
    T.cb[k] = 8u * static_cast<uint32_t>(T.core[k] ? T.ee[k] : Dm);
    T.wcore[k] = __any_sync(0xffffffffu, T.core[k]);
  }

  if (tid == 0) {
    for (int s = 0; s < F2_NSLOT; ++s) mbar_init(bar + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();  // x is the previous pass's output

  // Plane p = qa - 2 + i lives in slot i % NSLOT: x rows p D + c0 - 2 Dm +
  // [0, E2) clipped to the matrix (32-bit rows: the host guarantees
  // n + 6 D < 2^31) and the presence bytes of rows p D + rbase + [0, E1)
  // from the 16-byte boundary below (pres is zero-padded by >= 5 D rows).
  const int pfirst = T.qa - 2;
  const int plast = qb + 1;
  auto issue = [&](int i) {
    const int p = pfirst + i;
    if (p > plast) return;
    const int lo = p * D + T.rbase - Dm;
    const int a = max(lo, 0), b = min(lo + E2, n);
    const uint32_t bytes = b > a ? static_cast<uint32_t>(b - a) * 8u : 0u;
    const int r1 = p * D + T.rbase;
    // clamped to the padded presence array (never binding for the planner's
    // geometries: rows stay within n + 4 D + Dm + 15 of a 5 D + 64 padding)
    const int pa = max(r1 & ~15, -P.ppad);
    const int pe = max(pa, min((r1 + E1 + 15) & ~15, (n + P.ppad + 15) & ~15));
    const uint32_t pbytes = static_cast<uint32_t>(pe - pa);
    const int sl = i % F2_NSLOT;
    mbar_expect_tx(bar + sl, bytes + pbytes);
    if (bytes) {
      bulk_load_plain(sm_base + 8u * static_cast<uint32_t>(F2_XS + sl * E2 + (a - lo)), x + a,
                      bytes, smem_u32(bar + sl));
    }
    if (pbytes) {
      bulk_load_plain(sm_base + static_cast<uint32_t>(T.ps + sl * T.pw + (pa - (r1 & ~15))),
                      pres + pa, pbytes, smem_u32(bar + sl));
    }
  };
  if (tid == 0) {
    for (int i = 0; i < F2_NSLOT; ++i) issue(i);
  }

  // registers: x planes and level-1 planes in rotating triples
  double xa[KC], xb[KC], xc[KC], la[KC], lb[KC], lc[KC];
  mbar_wait(bar + 0, 0);
  mbar_wait(bar + 1, 0);
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    xa[k] = f2_sm[F2_XS + Dm + T.ee[k]];       // plane qa - 2
    xb[k] = f2_sm[F2_XS + E2 + Dm + T.ee[k]];  // plane qa - 1
    xc[k] = la[k] = lb[k] = lc[k] = 0.0;
  }
  // presence of the previous step's plane, alternating between two arrays
  unsigned pr_a[KC], pr_b[KC];
#pragma unroll
  for (int k = 0; k < KC; ++k) pr_a[k] = pr_b[k] = (1u << ND) - 1u;
  __syncthreads();  // every thread has read slots 0 and 1 before they are refilled
  // Step t refills the slot of plane q - 1 (last read in step t - 1, whose
  // closing barrier every thread has passed) before it computes.
  for (int u = 0;; ++u) {
#define F2_STEP(V, XM, X0, XP, LM, LC, LN, PP, PC)                                              \
  if (tid == 0) issue(6 * u + V + F2_NSLOT);                                                    \
  if (!f2_step<ND, UNIT, KC, PAIR, COMPL, V>(P, T, u, f2_sm, bar, x, y, base, pres, XM, X0, XP, \
                                             LM, LC, LN, PP, PC)) {                             \
    break;                                                                                      \
  }
    F2_STEP(0, xa, xb, xc, la, lb, lc, pr_a, pr_b)
    F2_STEP(1, xb, xc, xa, lb, lc, la, pr_b, pr_a)
    F2_STEP(2, xc, xa, xb, lc, la, lb, pr_a, pr_b)
    F2_STEP(3, xa, xb, xc, la, lb, lc, pr_b, pr_a)
    F2_STEP(4, xb, xc, xa, lb, lc, la, pr_a, pr_b)
    F2_STEP(5, xc, xa, xb, lc, la, lb, pr_b, pr_a)
#undef F2_STEP
  }
}

struct F2Plan {
  int nt = 0, kc = 0, tw = 0, sh = 0, ntiles = 0, nchunks = 0;
  size_t smem = 0;
};

// Per-device queries (a process may drive several GPUs): not cached.
int f2_sms() {
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    v = 148;
  }
  return v;
}

int f2_smem_limit() { return max_dynamic_smem(k_spmv_dia2<7, true, 2, true, true>); }

size_t f2_smem_bytes(int e1, int dm) {
  return sizeof(double) * (static_cast<size_t>(F2_XS) +
                           static_cast<size_t>(F2_NSLOT) * (e1 + 2 * dm) +
                           static_cast<size_t>(F2_LSLOT) * e1) +
         static_cast<size_t>(F2_NSLOT) * ((e1 + 31) & ~15);
}

// Tile and chunk choice.  cps CTAs per SM; the dynamic shared memory request
// is raised so that no further CTA fits (a dependent launch of the next pass
// must not share an SM with this one).  The march is latency-bound per step,
// so at least 768 threads per SM are required; among those the plan with the
// fewest lane-steps per SM wins: waves x cps x (planes + 2) x NT x KC (both
// levels sweep KC columns of NT threads per plane; halo columns and the two
// warm-up planes are the overhead).  Measured on B200 (tools/spmv_ab.py):
// config 3 one 896-thread CTA per SM (18 tiles), config 5 one 768-thread CTA
// (the whole 2048-column plane), config 2 two 512-thread CTAs.
// PPA_DIA2_CPS / PPA_DIA2_NTMIN / PPA_DIA2_NTMAX override (A/B only).
int f2_env(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

F2Plan f2_plan_search(int n, int D, int Dm) {
  const int sms = f2_sms();
  // 3-D stencils: the boundary rows of a grid line (ix = N - 1 and the next
  // line's ix = 0) are neighbours.  With lines of a multiple of 32 rows,
  // tiles of a multiple of 32 columns and the extended tile starting 16
  // columns early, each such pair falls inside one warp, so one warp in
  // Dm / 32 takes the presence-tested path instead of two.
  const int sh = (Dm >= 64 && Dm % 32 == 0 && D % 32 == 0 && f2_env("PPA_DIA2_SHIFT", 1)) ? 16 : 0;
  const int nq = (n + D - 1) / D;
  const int force_cps = f2_env("PPA_DIA2_CPS", 0);
  const int ntmax = f2_env("PPA_DIA2_NTMAX", 1024);
  const int ntmin_env = f2_env("PPA_DIA2_NTMIN", 0);
  const int lim = f2_smem_limit();
  constexpr int kSmTotal = 228 * 1024;  // per SM, incl. 1 KB per CTA reserved by the driver
  F2Plan best;
  double best_cost = 1e300;
  for (int relax = 0; relax < 2 && best.nt == 0; ++relax) {
    for (int cps = 1; cps <= 2; ++cps) {
      if (force_cps && cps != force_cps) continue;
      const size_t floor_bytes = static_cast<size_t>(kSmTotal / (cps + 1));
      const int slots = sms * cps;
      const int ntmin = ntmin_env ? ntmin_env : relax ? 128 : (768 + cps - 1) / cps;
      for (int kc = 2; kc <= 4; ++kc) {
        // two CTAs per SM only where the register budget of
        // __launch_bounds__(f2_max_nt(KC), 1) leaves room for both (KC = 2:
        // 64 registers at up to 1024 threads; KC = 3 / 4 allow ~85 / 128)
        if (cps > 1 && kc > 2) continue;
        for (int nt = 128; nt <= std::min(ntmax, f2_max_nt(kc)); nt += 32) {
          if (nt < ntmin || nt * cps > 2048) continue;
          const int cap = nt * kc - 2 * Dm;
          if (cap < 64) continue;
          const int ntiles = (D + cap - 1) / cap;
          int tw = (D + ntiles - 1) / ntiles;
          tw += tw & 1;
          if (sh) tw = (tw + 31) & ~31;
          const int e1 = tw + 2 * Dm + sh;
          if (e1 > nt * kc) continue;
          size_t smem = f2_smem_bytes(e1, Dm);
          if ((smem + 1024) * cps > static_cast<size_t>(kSmTotal) ||
              smem > static_cast<size_t>(lim)) {
            continue;
          }
          smem = std::min(static_cast<size_t>(lim), std::max(smem, floor_bytes));
          const int nchunks = std::max(1, std::min(nq, slots / ntiles));
          const int tq = (nq + nchunks - 1) / nchunks;
          const long long ctas = static_cast<long long>(ntiles) * nchunks;
          const long long waves = (ctas + slots - 1) / slots;
          // measured, not modelled: two CTAs per SM on a plane split into
          // several tiles ran 1.4x slower than the model says (config 5:
          // 13.0 us per factor vs 9.4 with one 768-thread CTA per SM)
          const double penalty = (cps > 1 && ntiles > 1) ? 1.25 : 1.0;
          const double cost = penalty * static_cast<double>(waves) * cps * (tq + 2) *
                              (static_cast<double>(nt) * kc);
          if (cost < best_cost * 0.999) {
            best_cost = cost;
            best = F2Plan{nt, kc, tw, sh, ntiles, nchunks, smem};
          }
        }
      }
    }
  }
  return best;
}

// Plans are searched once per geometry (the search visits a few hundred
// candidates; a solve launches thousands of passes).  The A/B overrides
// (PPA_DIA2_*) apply to geometries planned after they are set.
F2Plan f2_plan(int n, int D, int Dm) {
  struct Entry {
    int dev, n, D, Dm;
    F2Plan plan;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  for (const Entry& e : cache) {
    if (e.dev == dev && e.n == n && e.D == D && e.Dm == Dm) return e.plan;
  }
  const F2Plan plan = f2_plan_search(n, D, Dm);
  if (cache.size() >= 64) cache.erase(cache.begin());
  cache.push_back({dev, n, D, Dm, plan});
  return plan;
}

template <int ND, bool UNIT, int KC, bool PAIR, bool COMPL>
void launch_f2(const CsrDevice& a, const F2Params& P, const F2Plan& pl, const double* x,
               double* y, const double* base, cudaStream_t st) {
  auto kernel = k_spmv_dia2<ND, UNIT, KC, PAIR, COMPL>;
  // the attribute is per device: set on every launch (a cheap host call)
  // rather than once per process
  PPA_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(pl.smem)));
  launch_pdl(kernel, dim3(pl.ntiles * pl.nchunks), dim3(pl.nt), pl.smem, st, a.dia_pres, x, y,
             base, P);
}

template <int ND, bool UNIT, int KC>
void launch_f2_k(const CsrDevice& a, const F2Params& P, const F2Plan& pl, bool pair,
                 const double* x, double* y, const double* base, cudaStream_t st) {
  if (pair) {
    base ? launch_f2<ND, UNIT, KC, true, true>(a, P, pl, x, y, base, st)
         : launch_f2<ND, UNIT, KC, true, false>(a, P, pl, x, y, base, st);
  } else {
    base ? launch_f2<ND, UNIT, KC, false, true>(a, P, pl, x, y, base, st)
         : launch_f2<ND, UNIT, KC, false, false>(a, P, pl, x, y, base, st);
  }
}

template <int ND, bool UNIT>
void launch_f2_u(const CsrDevice& a, const F2Params& P, const F2Plan& pl, bool pair,
                 const double* x, double* y, const double* base, cudaStream_t st) {
  switch (pl.kc) {
    case 2: return launch_f2_k<ND, UNIT, 2>(a, P, pl, pair, x, y, base, st);
    case 3: return launch_f2_k<ND, UNIT, 3>(a, P, pl, pair, x, y, base, st);
    default: return launch_f2_k<ND, UNIT, 4>(a, P, pl, pair, x, y, base, st);
  }
}

template <int ND>
void launch_f2_nd(const CsrDevice& a, const F2Params& P, const F2Plan& pl, bool pair,
                  const double* x, double* y, const double* base, cudaStream_t st) {
  if constexpr (ND >= 5) {
    constexpr int JC = (ND - 1) / 2;
    if (P.off[JC - 1] == -1 && P.off[JC + 1] == 1) {
      return launch_f2_u<ND, true>(a, P, pl, pair, x, y, base, st);
    }
  }
  launch_f2_u<ND, false>(a, P, pl, pair, x, y, base, st);
}

int f2_dm(const CsrDevice& a) {
  int dm = 0;
  for (int j = 1; j + 1 < a.dia_ndiag; ++j) dm = std::max(dm, std::abs(a.dia_off[j]));
  return dm;
}

}  // namespace

bool dia2_supported(const CsrDevice& a) {
  const char* off = std::getenv("PPA_DISABLE_DIA2");
  if (off && off[0] == '1') return false;
  if (grid2_supported(a)) return true;
  const int nd = a.dia_ndiag;
  // odd stencils with the centre (offset 0) in the middle: 3, 5 or 7 points
  if (!a.dia_pres || (nd != 3 && nd != 5 && nd != 7) || a.dia_off[(nd - 1) / 2] != 0) return false;
  const int D = a.dia_off[nd - 1];
  if (a.dia_off[0] != -D || D < 64 || (D & 1) || (a.n & 1)) return false;
  const int dm = f2_dm(a);
  if (4 * dm > D || a.n / D < 4) return false;
  // 32-bit rows: the kernel forms rows up to n + 4 D + Dm + 15
  if (static_cast<long long>(a.n) + 6LL * D >= (1LL << 31)) return false;
  return f2_plan(a.n, D, dm).nt > 0;
}

void spmv_dia2(const CsrDevice& a, const Mp2Pass& p, const double* x, double* y,
               const double* base, cudaStream_t st) {
  // box-grid stencils take the boundary-free form (spmv_grid2.cu)
  if (grid2_supported(a)) return spmv_grid2(a, p, x, y, base, st);
  const int ND = a.dia_ndiag;
  const int D = a.dia_off[ND - 1];
  const int dm = f2_dm(a);
  const F2Plan pl = f2_plan(a.n, D, dm);
  F2Params P{};
  for (int j = 0; j < ND; ++j) {
    P.off[j] = a.dia_off[j];
    P.val[j] = a.dia_dflt[j];
  }
  P.n = a.n;
  P.D = D;
  P.Dm = dm;
  P.TW = pl.tw;
  P.SH = pl.sh;
  P.ppad = static_cast<int>(a.dia_pres_pad);
  P.E1 = pl.tw + 2 * dm + pl.sh;
  P.E2 = P.E1 + 2 * dm;
  P.ntiles = pl.ntiles;
  P.nq = (a.n + D - 1) / D;
  P.nchunks = pl.nchunks;
  P.a0 = p.a0;
  P.a1 = p.a1;
  P.b0 = p.b0;
  switch (ND) {
    case 3: launch_f2_nd<3>(a, P, pl, p.pair, x, y, base, st); break;
    case 5: launch_f2_nd<5>(a, P, pl, p.pair, x, y, base, st); break;
    default: launch_f2_nd<7>(a, P, pl, p.pair, x, y, base, st); break;
  }
  PPA_CUDA(cudaGetLastError());
}

}  // namespace kern
}  // namespace ppa
