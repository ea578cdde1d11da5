// Two polynomial factors per pass over a box-grid stencil: the boundary-free
// form of the temporally blocked pass (spmv_dia2.cu).  Replaces two
// consecutive launches of the factor chain (src/gmres_poly.cpp:129-143):
//   two real roots : u = x + a0 (A x),  y = u + b0 (A u)
//   conjugate pair : t = A x,           y = (x + a1 t) + a0 (A t)
// optionally followed by the complement y = base - y (src/gmres_poly.cpp:306-308).
//
// Applies when the diagonal layout's presence form is exactly a 7-point
// stencil on an nx x ny x nz box (offsets -nx ny, -nx, -1, 0, 1, nx, nx ny) or
// a 5-point one on nx x nz (offsets -nx, -1, 0, 1, nx), cut at the box faces,
// with one value per diagonal (layout_build.cu k_grid_check): configs 2, 3, 5.
// Then "entry absent" means "neighbour outside the box", so the kernel needs
// no presence bytes and no per-row tests: the shared-memory copies of x and
// of the first factor carry zero cells around the box, an absent term
// contributes val * (+0.0) and the row sum keeps the reference's bits (the
// sum starts at +0.0 and round-to-nearest never turns it into -0.0; x's own
// inf/nan values never reach a zero cell).  Row sums visit the diagonals in
// increasing offset with __dmul_rn / __dadd_rn, as the CSR loop does.
//
// Geometry.  Row r = (z ny + y) nx + x.  A CTA owns the tile [x0, x1) x
// [y0, y1) of the (x, y) plane over the planes [za, zb) and marches in z:
//   step t: level 1 (first factor) at plane q = za - 1 + t over the tile
//           widened by one cell in x and y (cells outside the box stay 0);
//           level 2 (second factor) at plane q - 1 over the tile.
// x planes arrive by cp.async.bulk, one copy per grid line of the widened
// tile, into a ring of shared-memory slots laid out with pitch P = TX + 4
// (two zero columns on each side); level-1 planes go to a ring of three
// slots of the same pitch.  Each thread owns RY cells (3-D: RY consecutive
// lines of one column; 2-D: RY 32-column segments of the line) and keeps the
// x and level-1 values of three consecutive planes of its cells in
// registers: the +-D terms and (3-D) the +-nx terms between its own lines
// come from registers, the rest from shared memory.
//
// Synchronisation is split per plane, with no block-wide barrier in the
// loop: every warp arrives on l1_done[t % 3] after storing level 1 of step
// t and every thread waits on l1_done[(t - 1) % 3] at the start of step t, so warps drift
// freely within a step.  The wait at step t proves that all threads finished
// step t - 2 entirely (the level-1 slot of step t - 3 is free) and read the x
// plane of step t - 1 (its slot is refilled then, by warp 0's lanes).

#include "spmv_grid2_kernel.cuh"

namespace ppa {
namespace kern {
namespace {

int g2_env(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

struct DevInfo {
  int sms = 148;
  int smem_optin = 227 * 1024;
};

DevInfo g2_dev() {
  DevInfo d;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&d.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  return d;
}

size_t g2_smem(int P, int SL, int LL, int nslot) {
  return sizeof(double) * (static_cast<size_t>(G2_BARS) + static_cast<size_t>(nslot) * SL * P +
                           static_cast<size_t>(G2_LSLOT) * LL * P);
}

constexpr int kRY3[] = {2, 3, 4};

// Cost of a plan (one CTA per SM): steps x lane-slots of the CTA, with one
// cell's worth of per-step overhead per warp (barrier waits, ring
// bookkeeping; RY = 1 measured 1.25x slower than RY = 2 on config 5) and a
// latency penalty below 16 warps.  Fitted to B200 measurements of configs 2,
// 3 and 5 (tools/spmv_ab.py with PPA_GRID2_RY / _TY / _NTX).
double g2_cost(int lz, int warps, int ry) {
  const double pen = warps < 16 ? std::pow(16.0 / warps, 1.5) : 1.0;
  return static_cast<double>(lz + 2) * warps * 32.0 * (ry + 1) * pen;
}
constexpr int kRY2[] = {1, 2, 3, 4};

// Plan search.  One CTA per SM (the loop has no block barrier; warps of one
// CTA overlap each other); the level-1 work of a CTA is (tile + halo cells)
// x (planes + 2).  Cost = waves x (planes + 2) x lane-slots of the CTA,
// minimised over the tile shape, cells per thread and chunk count; at least
// 12 warps per CTA.  PPA_GRID2_TY / _RY / _NTX / _NSLOT override (A/B only).
G2Plan g2_plan_search(int nd, int nx, int ny, int nz) {
  const DevInfo dv = g2_dev();
  const int sms = dv.sms;
  // x slots: fixed per stencil (3-D 6, 2-D 12: the kernel's NS), level-1
  // slots G2_LSLOT
  auto slots_for = [&](size_t, size_t) { return nd == 7 ? 6 : 12; };
  const int want_ty = g2_env("PPA_GRID2_TY", 0), want_ry = g2_env("PPA_GRID2_RY", 0),
            want_ntx = g2_env("PPA_GRID2_NTX", 0);
  G2Plan best;
  double best_cost = 1e300;
  // at least 12 warps per CTA when the geometry allows; small grids relax it
  for (int minw : {12, 1}) {
    if (best.ok) break;
    if (nd == 7) {
      if (nx > 252 || nx < 2 || (nx & 1)) return best;
      const int segs = (nx + 31) / 32;
      for (int ry : kRY3) {
        if (want_ry && ry != want_ry) continue;
        for (int nty = 1; nty <= ny; ++nty) {
          const int ty = (ny + nty - 1) / nty;  // widest tile
          if (want_ty && ty != want_ty) continue;
          const int ll = ty + 2;
          if (ll % ry) continue;
          const int groups = ll / ry;
          const int warps = groups * segs;
          if ((warps * 32 + 63) / 64 * 64 > g2_maxnt(nd, ry) || warps < minw) continue;
          const int P = nx + 4, SL = ty + 4;
          const int nslot = slots_for(8u * SL * P, g2_smem(P, SL, ll, 0));
          const size_t smem = g2_smem(P, SL, ll, nslot);
          if (smem > static_cast<size_t>(dv.smem_optin)) continue;
          const int nch = std::max(1, std::min(nz, sms / nty));
          const int lz = (nz + nch - 1) / nch;
          const double cost = g2_cost(lz, warps, ry);
          if (cost < best_cost * 0.999) {
            best_cost = cost;
            best = G2Plan{1, nd, ry, warps * 32, 1, nty, nch, P, SL, ll, nslot, segs, warps, smem};
          }
        }
      }
    } else {
      if (nx < 2 || (nx & 1)) return best;
      for (int ry : kRY2) {
        if (want_ry && ry != want_ry) continue;
        for (int ntx = 1; ntx <= 64; ++ntx) {
          if (want_ntx && ntx != want_ntx) continue;
          const int tw = ((nx + ntx - 1) / ntx + 1) & ~1;  // widest tile (even)
          if (tw < 32 && ntx > 1) break;
          if ((tw + 4) * 8 > 64 * 1024) continue;  // a line must fit the zero page
          const int cells = tw + 2;
          const int segs = (cells + 31) / 32;
          const int warps = (segs + ry - 1) / ry;
          if ((warps * 32 + 63) / 64 * 64 > g2_maxnt(nd, ry) || warps < minw) continue;
          const int P = tw + 4;
          const int nslot = slots_for(8u * P, g2_smem(P, 1, 1, 0));
          const size_t smem = g2_smem(P, 1, 1, nslot);
          if (smem > static_cast<size_t>(dv.smem_optin)) continue;
          const int nch = std::max(1, std::min(nz, sms / ntx));
          const int lz = (nz + nch - 1) / nch;
          const double cost = g2_cost(lz, warps, ry);
          if (cost < best_cost * 0.999) {
            best_cost = cost;
            best = G2Plan{1, nd, ry, warps * 32, ntx, 1, nch, P, 1, 1, nslot, segs, warps, smem};
          }
        }
      }
    }
  }
  if (best.ok) {
    // one CTA per SM: ask for enough shared memory that no second CTA (e.g.
    // the next pass's, launched early by PDL) shares the SM
    constexpr size_t kSmTotal = 228 * 1024;
    best.smem = std::min(static_cast<size_t>(dv.smem_optin), std::max(best.smem, kSmTotal / 2));
  }
  return best;
}

G2Plan g2_plan(int nd, int nx, int ny, int nz) {
  struct Entry {
    int dev, nd, nx, ny, nz;
    G2Plan plan;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  for (const Entry& e : cache) {
    if (e.dev == dev && e.nd == nd && e.nx == nx && e.ny == ny && e.nz == nz) return e.plan;
  }
  const G2Plan plan = g2_plan_search(nd, nx, ny, nz);
  if (std::getenv("PPA_GRID2_DEBUG")) {
    std::fprintf(stderr,
                 "grid2 plan %dx%dx%d nd=%d: ok=%d ry=%d nt=%d ntx=%d nty=%d nchunks=%d P=%d SL=%d "
                 "LL=%d nslot=%d segs=%d cw=%d smem=%zu\n",
                 nx, ny, nz, nd, plan.ok, plan.ry, plan.nt, plan.ntx, plan.nty, plan.nchunks,
                 plan.P, plan.SL, plan.LL, plan.nslot, plan.segs, plan.cw, plan.smem);
  }
  if (cache.size() >= 64) cache.erase(cache.begin());
  cache.push_back({dev, nd, nx, ny, nz, plan});
  return plan;
}

}  // namespace

// 64 KB of zeros per device, the copy source of x planes outside the box.
// Allocated when a box-grid layout is built (never under stream capture),
// kept for the life of the process.
const double* grid2_zeros() {
  constexpr size_t kBytes = 64 * 1024;
  static std::mutex mu;
  static std::vector<std::pair<int, double*>> bufs;
  int dev = 0;
  PPA_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& b : bufs)
    if (b.first == dev) return b.second;
  void* p = nullptr;
  PPA_CUDA(cudaMalloc(&p, kBytes));
  PPA_CUDA(cudaMemset(p, 0, kBytes));
  bufs.emplace_back(dev, static_cast<double*>(p));
  return static_cast<double*>(p);
}

bool grid2_supported(const CsrDevice& a) {
  const char* off = std::getenv("PPA_DISABLE_GRID2");
  if (off && off[0] == '1') return false;
  if (a.grid_nx <= 0 || !a.dia_pres) return false;
  if (static_cast<long long>(a.n) + 4LL * a.grid_nx * a.grid_ny >= (1LL << 31)) return false;
  return g2_plan(a.dia_ndiag, a.grid_nx, a.grid_ny, a.grid_nz).ok != 0;
}

namespace {

// One pass over the owned planes [zo0, zo1) of an nx x ny x nz box (ny = 1:
// 5-point 2-D) with the diagonal values vals; plan for the owned planes.
void grid2_launch(int nd, int nx, int ny, int nz, const double* vals, const Mp2Pass& p,
                  const double* x, double* y, const double* base, int zo0, int zo1,
                  const double* xl, int zl0, const long long* fl, const double* xr,
                  const long long* fr, long long epoch, int* err, long long* own,
                  cudaStream_t st) {
  const G2Plan pl = g2_plan(nd, nx, ny, zo1 - zo0);
  if (!pl.ok) throw std::invalid_argument("spmv_grid2: no launch plan for this box");
  G2Params P{};
  for (int j = 0; j < nd; ++j) P.val[j] = vals[j];
  P.a0 = p.a0;
  P.a1 = p.a1;
  P.b0 = p.b0;
  P.nx = nx;
  P.ny = ny;
  P.nz = nz;
  P.D = nx * ny;
  P.ntx = pl.ntx;
  P.nty = pl.nty;
  P.nchunks = pl.nchunks;
  P.P = pl.P;
  P.SL = pl.SL;
  P.LL = pl.LL;
  P.nslot = pl.nslot;
  P.segs = pl.segs;
  P.zeros = grid2_zeros();
  P.cw = pl.cw;
  P.zo0 = zo0;
  P.zo1 = zo1;
  P.zl0 = zl0;
  P.xl = xl;
  P.xr = xr;
  P.fl = fl;
  P.fr = fr;
  P.epoch = epoch;
  P.err = err;
  P.own = own;
  const bool slab = zo0 != 0 || zo1 != nz || xl || xr || own;
  if (slab && base) throw std::invalid_argument("spmv_grid2: no complement in slab mode");
  if (nd == 7) {
    switch (pl.ry) {
      case 2: g2::launch_7_2(P, pl, p.pair, x, y, base, st, p.one, slab); break;
      case 3: g2::launch_7_3(P, pl, p.pair, x, y, base, st, p.one, slab); break;
      default: g2::launch_7_4(P, pl, p.pair, x, y, base, st, p.one, slab); break;
    }
  } else {
    switch (pl.ry) {
      case 1: g2::launch_5_1(P, pl, p.pair, x, y, base, st, p.one, slab); break;
      case 2: g2::launch_5_2(P, pl, p.pair, x, y, base, st, p.one, slab); break;
      case 3: g2::launch_5_3(P, pl, p.pair, x, y, base, st, p.one, slab); break;
      default: g2::launch_5_4(P, pl, p.pair, x, y, base, st, p.one, slab); break;
    }
  }
  PPA_CUDA(cudaGetLastError());
}

}  // namespace

void grid2_row_evals(const CsrDevice& a, long long* l1, long long* l2) {
  *l1 = *l2 = 0;
  if (!grid2_supported(a)) return;
  const int nd = a.dia_ndiag, nx = a.grid_nx, ny = a.grid_ny, nz = a.grid_nz;
  const G2Plan pl = g2_plan(nd, nx, ny, nz);
  // the kernel's tiles and chunks (k_spmv_grid2): level 1 runs on the tile
  // widened by one line (3-D) or column (2-D) each side and on one more
  // plane each side of the chunk, clipped to the box; level 2 on every row
  long long cells = 0;  // level-1 cells per plane, summed over tiles
  if (nd == 7) {
    for (int ty = 0; ty < pl.nty; ++ty) {
      const int y0 = ty * ny / pl.nty, y1 = (ty + 1) * ny / pl.nty;
      cells += static_cast<long long>(std::min(y1 + 1, ny) - std::max(y0 - 1, 0)) * nx;
    }
  } else {
    for (int tx = 0; tx < pl.ntx; ++tx) {
      const int x0 = (tx * nx / pl.ntx) & ~1;
      const int x1 = tx + 1 == pl.ntx ? nx : ((tx + 1) * nx / pl.ntx) & ~1;
      cells += std::min(x1 + 1, nx) - std::max(x0 - 1, 0);
    }
  }
  long long planes = 0;
  for (int c = 0; c < pl.nchunks; ++c) {
    const int za = static_cast<int>(static_cast<long long>(c) * nz / pl.nchunks);
    const int zb = static_cast<int>(static_cast<long long>(c + 1) * nz / pl.nchunks);
    planes += std::min(zb + 1, nz) - std::max(za - 1, 0);
  }
  *l1 = cells * planes;
  *l2 = static_cast<long long>(nx) * ny * nz;
}

void spmv_grid2(const CsrDevice& a, const Mp2Pass& p, const double* x, double* y,
                const double* base, cudaStream_t st) {
  grid2_launch(a.dia_ndiag, a.grid_nx, a.grid_ny, a.grid_nz, a.dia_dflt, p, x, y, base, 0,
               a.grid_nz, nullptr, 0, nullptr, nullptr, nullptr, 0, nullptr, nullptr, st);
}

void spmv_grid2_slab_check(int nd, int nx, int ny, int nz, int zo0, int zo1, const double* xl,
                           int zl0, const long long* fl, const double* xr,
                           const long long* fr) {
  if (nd != 5 && nd != 7) throw std::invalid_argument("spmv_grid2_slab: 5- or 7-point stencil");
  if ((nd == 5) != (ny == 1)) throw std::invalid_argument("spmv_grid2_slab: 2-D boxes have ny = 1");
  if (zo0 < 0 || zo1 > nz || zo1 - zo0 < 2) {
    throw std::invalid_argument("spmv_grid2_slab: a slab needs >= 2 planes inside the box");
  }
  if ((zo0 > 0 && (!xl || !fl || zo0 - zl0 < 2)) || (zo1 < nz && (!xr || !fr))) {
    throw std::invalid_argument("spmv_grid2_slab: missing neighbour buffer or flag");
  }
  if (nx < 2 || ny < 1) throw std::invalid_argument("spmv_grid2_slab: bad box");
  if (static_cast<long long>(nx) * ny * (zo1 - zo0) + 4LL * nx * ny >= (1LL << 31)) {
    throw std::invalid_argument("spmv_grid2_slab: slab too large");
  }
}

void spmv_grid2_slab(int nd, int nx, int ny, int nz, const double* vals, int zo0, int zo1,
                     const Mp2Pass& p, const double* x, double* y, const double* xl, int zl0,
                     const long long* fl, const double* xr, const long long* fr,
                     long long epoch, int* err, long long* own, cudaStream_t st) {
  spmv_grid2_slab_check(nd, nx, ny, nz, zo0, zo1, xl, zl0, fl, xr, fr);
  grid2_launch(nd, nx, ny, nz, vals, p, x, y, nullptr, zo0, zo1, xl, zl0, fl, xr, fr, epoch,
               err, own, st);
}

}  // namespace kern
}  // namespace ppa