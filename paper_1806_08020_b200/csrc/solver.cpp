// PP-Arnoldi driver: solve / solve_double / operator_norm_estimate.
// The reference declares these (inc/solver.hpp:57-116) without a body; the
// cycle structure follows SPEC.md [MODULE] solver and PAPER.md:563-575
// (Arnoldi(m,k) on pi(A), Ritz values ordered by |1 - nu|, convergence
// tested with Rayleigh quotients and true residuals against A).

#include "ppa/solver.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <future>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>

#include "ppa/kernels.hpp"
#include "ppa/rng.hpp"

namespace ppa {

namespace {

using cplx = std::complex<double>;
using Clock = std::chrono::steady_clock;

double seconds_since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

DBuffer<double> upload(const std::vector<double>& h) {
  DBuffer<double> d(h.size());
  PPA_CUDA(cudaMemcpy(d.get(), h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
  return d;
}

long long round_ld(int n) { return (static_cast<long long>(n) + 31) / 32 * 32; }

// The seeded start vectors of one solve,
// generated on a host thread in the order the solve consumes them, so that
// drawing the next vector overlaps the device work of the current phase
// (norm estimate, polynomial build).  take() waits for a stream's vector
// and returns a fresh device copy (a damping probe restarts from the same
// Arnoldi start vector).
// Pinned host buffers for the start vectors, kept across solves (page-locking
// 32 MB costs milliseconds; a pinned source makes the upload a DMA at full
// PCIe/C2C speed instead of a staged pageable copy).
class PinnedPool {
 public:
  static PinnedPool& get() {
    static PinnedPool p;
    return p;
  }
  double* acquire(size_t count) {
    std::lock_guard<std::mutex> g(mu_);
    // best fit: the smallest free buffer that holds `count`
    size_t best = free_.size();
    for (size_t i = 0; i < free_.size(); ++i) {
      if (free_[i].second >= count && (best == free_.size() || free_[i].second < free_[best].second))
        best = i;
    }
    if (best < free_.size()) {
      double* p = free_[best].first;
      free_.erase(free_.begin() + static_cast<long>(best));
      return p;
    }
    void* p = nullptr;
    if (cudaMallocHost(&p, count * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      throw std::runtime_error("StartVectors: pinned allocation failed");
    }
    size_[static_cast<double*>(p)] = count;
    return static_cast<double*>(p);
  }
  void release(double* p) {
    std::lock_guard<std::mutex> g(mu_);
    free_.emplace_back(p, size_[p]);
    // keep up to 16 buffers and 1 GiB (solves of different sizes in one
    // process must not page-lock fresh buffers each time: ~100 ms per
    // 130 MB); drop the smallest beyond that
    auto bytes = [&]() {
      size_t b = 0;
      for (const auto& f : free_) b += f.second * sizeof(double);
      return b;
    };
    while (free_.size() > 16 || (free_.size() > 1 && bytes() > (size_t{1} << 30))) {
      auto it = std::min_element(free_.begin(), free_.end(),
                                 [](const auto& a, const auto& b) { return a.second < b.second; });
      cudaFreeHost(it->first);
      size_.erase(it->first);
      free_.erase(it);
    }
  }

 private:
  std::mutex mu_;
  std::vector<std::pair<double*, size_t>> free_;
  std::map<double*, size_t> size_;
};

struct PinnedRelease {
  void operator()(double* p) const { PinnedPool::get().release(p); }
};

class StartVectors {
 public:
  StartVectors(int n, unsigned long long seed, std::vector<uint64_t> streams)
      : n_(n), streams_(std::move(streams)) {
    for (size_t i = 0; i < streams_.size(); ++i) {
      host_.emplace_back(PinnedPool::get().acquire(static_cast<size_t>(n)));
      ready_.emplace_back();
    }
    std::vector<std::promise<void>> done(streams_.size());
    for (size_t i = 0; i < streams_.size(); ++i) ready_[i] = done[i].get_future().share();
    worker_ = std::thread([this, seed, done = std::move(done)]() mutable {
      for (size_t i = 0; i < streams_.size(); ++i) {
        try {
          rng::fill_normal(host_[i].get(), n_, seed, streams_[i]);
          done[i].set_value();
        } catch (...) {
          done[i].set_exception(std::current_exception());
        }
      }
    });
  }
  StartVectors(const StartVectors&) = delete;
  StartVectors& operator=(const StartVectors&) = delete;
  ~StartVectors() {
    if (worker_.joinable()) worker_.join();
    cudaStreamSynchronize(current_context().stream());  // uploads from host_ done
  }

  PoolBuffer take(uint64_t stream) {
    for (size_t i = 0; i < streams_.size(); ++i) {
      if (streams_[i] != stream) continue;
      ready_[i].get();
      PoolBuffer d;
      d.resize(static_cast<size_t>(n_));
      PPA_CUDA(cudaMemcpyAsync(d.get(), host_[i].get(), static_cast<size_t>(n_) * sizeof(double),
                               cudaMemcpyHostToDevice, current_context().stream()));
      // the pinned source stays valid until the StartVectors dies, which
      // synchronises in its destructor
      return d;
    }
    throw std::logic_error("StartVectors: stream not scheduled");
  }

 private:
  int n_;
  std::vector<uint64_t> streams_;
  std::vector<std::unique_ptr<double, PinnedRelease>> host_;
  std::vector<std::shared_future<void>> ready_;
  std::thread worker_;
};

struct CheckOutcome {
  std::vector<cplx> mu;
  std::vector<double> res;
  int real_checks = 0;
  int pair_checks = 0;
};

// True-residual test of the first nev Ritz pairs against A (
// PAPER.md:569-571).  All Ritz vectors are formed by one V*G launch; each
// check is an SpMV plus two fused reductions; one read-back at the end.
// Counters per real check: ritz_vector's charge (src/arnoldi.cpp:260-263)
// + 1 mvp + 2 dots + 3 vops; per conjugate pair: + 2 mvps + 6 dots + 10 vops
// (DESIGN.md "Solver decisions").
CheckOutcome check_pairs(const ArnoldiState& st, const RitzSet& set, int nev,
                         const LinearOperator& a, CostRecord& rec) {
  Context& ctx = current_context();
  const cudaStream_t s = ctx.stream();
  const int d = set.vectors_h.rows;
  const int nchk = std::min(nev, set.count());
  // Plan: columns of G and which checks are pairs.
  struct Item {
    int j;
    bool pair;
    int col;
  };
  std::vector<Item> items;
  int p = 0;
  for (int j = 0; j < nchk;) {
    const bool pair = ritz_is_complex(set.values[j]) && j + 1 < set.count();
    items.push_back({j, pair, p});
    p += pair ? 2 : 1;
    j += pair ? 2 : 1;
  }
  std::vector<double> g(static_cast<size_t>(d) * p);
  for (const Item& it : items) {
    for (int r = 0; r < d; ++r) {
      g[static_cast<size_t>(it.col) * d + r] = set.vectors_h(r, it.j).real();
      if (it.pair) g[static_cast<size_t>(it.col + 1) * d + r] = set.vectors_h(r, it.j).imag();
    }
  }
  Scratch gdev(g.size());
  PPA_CUDA(cudaMemcpyAsync(gdev.get(), g.data(), g.size() * sizeof(double),
                           cudaMemcpyHostToDevice, s));
  const long long ldy = round_ld(st.n);
  Scratch Y(static_cast<size_t>(ldy) * p);
  kern::ts_combine(st.V.get(), st.ld, st.n, d, gdev.get(), p, Y.get(), ldy, s);
  Scratch sums(static_cast<size_t>(p) + 3 * items.size() + 8);
  kern::col_sumsq(Y.get(), ldy, st.n, p, sums.get(), ctx.ws(), ctx.sm_count(), s);
  std::vector<double> hs(p);
  PPA_CUDA(cudaMemcpyAsync(hs.data(), sums.get(), p * sizeof(double), cudaMemcpyDeviceToHost, s));
  ctx.sync();
  double* outs = sums.get() + p;
  // unit Ritz vectors (ritz_vector's counted normalisation, src/arnoldi.cpp:261-263)
  for (const Item& it : items) {
    double* yr = Y.get() + static_cast<long long>(it.col) * ldy;
    if (!it.pair) {
      kern::div_value(yr, std::sqrt(hs[it.col]), st.n, s);
      rec.vops += d;
      rec.dots += 1;
      rec.vops += 2;
    } else {
      const double nrm = std::sqrt(hs[it.col] + hs[it.col + 1]);
      kern::div_value(yr, nrm, st.n, s);
      kern::div_value(yr + ldy, nrm, st.n, s);
      rec.vops += 2LL * d;
      rec.dots += 2;
      rec.vops += 4;
    }
  }
  // A Y: one multi-RHS SpMM (the matrix is read once per 8 vectors) when A is
  // a CSR operator, otherwise one counted apply per column.
  const auto* csr = dynamic_cast<const CsrOperator*>(&a);
  Scratch AY(static_cast<size_t>(ldy) * (csr ? p : 2));
  if (csr) {
    kern::spmm(csr->device(), Y.get(), ldy, p, AY.get(), ldy, s);
    rec.mvps += p;
  }
  for (size_t t = 0; t < items.size(); ++t) {
    const Item& it = items[t];
    double* yr = Y.get() + static_cast<long long>(it.col) * ldy;
    double* ar = csr ? AY.get() + static_cast<long long>(it.col) * ldy : AY.get();
    if (!it.pair) {
      if (!csr) a.apply(yr, ar, rec);
      kern::ritz_check_real(yr, ar, st.n, outs + 3 * t, ctx.ws(), ctx.sm_count(), s);
      rec.dots += 2;
      rec.vops += 3;
    } else {
      double* yi = yr + ldy;
      double* ai = ar + ldy;
      if (!csr) {
        a.apply(yr, ar, rec);
        a.apply(yi, ai, rec);
      }
      kern::ritz_check_complex(yr, yi, ar, ai, st.n, outs + 3 * t, ctx.ws(), ctx.sm_count(), s);
      rec.dots += 6;
      rec.vops += 10;
    }
  }
  std::vector<double> ho(3 * items.size());
  PPA_CUDA(cudaMemcpyAsync(ho.data(), outs, ho.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  ctx.sync();
  CheckOutcome out;
  out.mu.assign(nchk, cplx(0.0, 0.0));
  out.res.assign(nchk, 0.0);
  for (size_t t = 0; t < items.size(); ++t) {
    const Item& it = items[t];
    if (!it.pair) {
      out.mu[it.j] = cplx(ho[3 * t], 0.0);
      out.res[it.j] = ho[3 * t + 1];
      ++out.real_checks;
    } else {
      const cplx mu(ho[3 * t], ho[3 * t + 1]);
      out.mu[it.j] = mu;
      out.res[it.j] = ho[3 * t + 2];
      if (it.j + 1 < nchk) {
        out.mu[it.j + 1] = std::conj(mu);
        out.res[it.j + 1] = ho[3 * t + 2];
      }
      ++out.pair_checks;
    }
  }
  return out;
}

// Unit eigenvector estimates y_j (j < nev) of the final cycle, kept on the
// device as (Re, Im) column pairs; conjugate partners share columns with the
// sign of Im flipped.  Output materialisation only: uncounted.
void keep_eigenvectors(const ArnoldiState& st, const RitzSet& set, int nev, EigResult& res) {
  Context& ctx = current_context();
  const cudaStream_t s = ctx.stream();
  const int d = set.vectors_h.rows;
  const int ne = std::min(nev, set.count());
  if (ne <= 0 || d <= 0) return;
  const long long ld = round_ld(st.n);
  std::vector<double> g(static_cast<size_t>(d) * 2 * ne, 0.0);
  for (int j = 0; j < ne; ++j) {
    for (int r = 0; r < d; ++r) {
      g[static_cast<size_t>(2 * j) * d + r] = set.vectors_h(r, j).real();
      g[static_cast<size_t>(2 * j + 1) * d + r] = set.vectors_h(r, j).imag();
    }
  }
  Scratch gdev(g.size());
  PPA_CUDA(cudaMemcpyAsync(gdev.get(), g.data(), g.size() * sizeof(double),
                           cudaMemcpyHostToDevice, s));
  res.eigenvectors.resize(static_cast<size_t>(ld) * 2 * ne);
  res.eigvec_ld = ld;
  kern::ts_combine(st.V.get(), st.ld, st.n, d, gdev.get(), 2 * ne, res.eigenvectors.get(), ld, s);
  Scratch sums(static_cast<size_t>(2 * ne));
  kern::col_sumsq(res.eigenvectors.get(), ld, st.n, 2 * ne, sums.get(), ctx.ws(), ctx.sm_count(),
                  s);
  std::vector<double> hs(2 * ne);
  PPA_CUDA(cudaMemcpyAsync(hs.data(), sums.get(), hs.size() * sizeof(double),
                           cudaMemcpyDeviceToHost, s));
  ctx.sync();
  for (int j = 0; j < ne; ++j) {
    const double nrm = std::sqrt(hs[2 * j] + hs[2 * j + 1]);
    kern::div_value(res.eigenvectors.get() + 2LL * j * ld, nrm, st.n, s);
    kern::div_value(res.eigenvectors.get() + (2LL * j + 1) * ld, nrm, st.n, s);
  }
  ctx.sync();
}

// One full first cycle (extend + Ritz pairs + checks of `nchk` pairs): the
// damping heuristic's probe, reusable as cycle 1 of the solve.
struct FirstCycle {
  ArnoldiState st;
  RitzSet set;
  CheckOutcome chk;
  int start_dim = 0;
};

RitzSet select_pairs(const ArnoldiState& st, const SolveConfig& cfg, RitzOrdering ordering) {
  return cfg.variant == RestartVariant::harmonic ? harmonic_restart_selection(st, ordering)
                                                 : ritz_pairs(st, ordering);
}

FirstCycle first_cycle(const LinearOperator& a, const LinearOperator& op, const SolveConfig& cfg,
                       RitzOrdering ordering, int nchk, CostRecord& rec, StartVectors& sv) {
  const int n = a.dim();
  PoolBuffer v0 = sv.take(rng::kArnoldiStart);
  FirstCycle f;
  f.st = arnoldi_init(v0.get(), n, cfg.m, rec);
  f.st.ortho = cfg.orthogonalization;
  f.start_dim = f.st.cur_dim;
  arnoldi_extend(f.st, op, cfg.m, rec);
  f.set = select_pairs(f.st, cfg, ordering);
  f.chk = check_pairs(f.st, f.set, nchk, a, rec);
  return f;
}

// Cycle loop shared by solve and solve_double.
void run_cycles(const LinearOperator& a, const LinearOperator& op, const SolveConfig& cfg,
                RitzOrdering ordering, EigResult& res, CostRecord& rec, StartVectors& sv,
                FirstCycle* probe = nullptr) {
  Context& ctx = current_context();
  const int n = a.dim();
  ArnoldiState st;
  if (probe) {
    st = std::move(probe->st);
  } else {
    PoolBuffer v0 = sv.take(rng::kArnoldiStart);
    st = arnoldi_init(v0.get(), n, cfg.m, rec);
    st.ortho = cfg.orthogonalization;
  }
  (void)ctx;
  std::vector<double> best;
  res.max_err = std::numeric_limits<double>::infinity();
  for (int cycle = 1; cycle <= cfg.max_cycles; ++cycle) {
    CycleStats cs;
    cs.cycle = cycle;
    RitzSet set;
    CheckOutcome chk;
    auto t0 = Clock::now();
    if (cycle == 1 && probe) {
      // the passing damping probe is this solve's first cycle (SPEC.md
      // solver design decisions): its checks cover the first k >= nev pairs
      cs.start_dim = probe->start_dim;
      cs.end_dim = st.cur_dim;
      set = std::move(probe->set);
      chk = std::move(probe->chk);
      const int keep = std::min<int>(cfg.nev, static_cast<int>(chk.mu.size()));
      chk.mu.resize(keep);
      chk.res.resize(keep);
    } else {
      cs.start_dim = st.cur_dim;
      bool checked = false;
      if (cfg.check_mid_cycle && cfg.mid_cycle_stride > 0) {
        // optional early exit inside a cycle (section 8 remark;
        // SPEC.md solver design decisions): every `stride` steps, test the
        // Ritz pairs of the partial factorisation against A
        while (st.cur_dim < cfg.m && !st.breakdown) {
          const int to = std::min(cfg.m, st.cur_dim + cfg.mid_cycle_stride);
          arnoldi_extend(st, op, to, rec);
          if (st.cur_dim >= cfg.m || st.breakdown || st.cur_dim < cfg.nev) continue;
          set = select_pairs(st, cfg, ordering);
          chk = check_pairs(st, set, cfg.nev, a, rec);
          bool ok = static_cast<int>(chk.res.size()) == cfg.nev;
          for (double r : chk.res) ok = ok && r <= res.rtol;
          if (ok) {
            checked = true;
            break;
          }
        }
      } else {
        arnoldi_extend(st, op, cfg.m, rec);
      }
      res.timing.extend += seconds_since(t0);
      cs.end_dim = st.cur_dim;
      if (!checked) {
        t0 = Clock::now();
        set = select_pairs(st, cfg, ordering);
        chk = check_pairs(st, set, cfg.nev, a, rec);
        res.timing.check += seconds_since(t0);
      }
    }
    cs.real_checks = chk.real_checks;
    cs.pair_checks = chk.pair_checks;
    double mx = 0.0;
    bool all = static_cast<int>(chk.res.size()) == cfg.nev;
    for (double r : chk.res) {
      mx = std::max(mx, r);
      all = all && r <= res.rtol;
    }
    cs.max_residual = mx;
    res.cycles = cycle;
    if (mx < res.max_err) res.max_err = mx;
    best.push_back(res.max_err);
    res.eigenvalues = chk.mu;
    res.residuals = chk.res;
    res.converged_flags.assign(chk.res.size(), false);
    for (size_t i = 0; i < chk.res.size(); ++i) res.converged_flags[i] = chk.res[i] <= res.rtol;
    // stagnation_stop: run until the best max-residual has not improved by
    // stagnation_rtol over stagnation_window cycles (inc/solver.hpp:48-52)
    const int w = cfg.stagnation_window;
    const bool stagnated = cfg.stagnation_stop && w > 0 && cycle > w &&
                           best.back() > (1.0 - cfg.stagnation_rtol) * best[cycle - 1 - w];
    const bool done = cfg.stagnation_stop ? stagnated : all;
    if (done || cycle == cfg.max_cycles || st.breakdown || st.cur_dim < cfg.m) {
      res.converged = all;
      res.history.push_back(cs);
      if (cfg.want_eigenvectors) keep_eigenvectors(st, set, cfg.nev, res);
      break;
    }
    t0 = Clock::now();
    cs.restart_k = set.harmonic ? harmonic_thick_restart(st, set, cfg.k, rec)
                                : thick_restart(st, set, cfg.k, rec);
    res.timing.restart += seconds_since(t0);
    res.history.push_back(cs);
  }
}

PolyPrecond stabilise(PolyPrecond p, const SolveConfig& cfg) {
  if (cfg.stability == StabilityMode::pof_auto && p.roots.size() >= 2) {
    return add_stability_roots(p);
  }
  return p;
}

// The damping heuristic of PAPER.md section 6.3: probe one
// Arnoldi(m,k) cycle on pi(A); if the Rayleigh quotients of the first k pairs
// fail the ideal order condition, rebuild pi from the damped start Ab, then
// keep halving the degree (rebuilding from Ab) until a probe passes or d = 1.
// A passing probe is handed back for reuse as the solve's first cycle;
// failed probes are logged as discarded cycles.  All probe costs count.
PolyPrecond damping_search(const OperatorPtr& a, const SolveConfig& cfg, CostRecord& rec,
                           std::vector<CycleStats>& history, std::optional<FirstCycle>& keep,
                           StartVectors& sv) {
  const int n = a->dim();
  PoolBuffer b = sv.take(rng::kPolyStart);
  DBuffer<double> ab;
  int d = cfg.degree;
  bool damped = false;
  for (;;) {
    const double* start = damped ? ab.get() : b.get();
    PolyPrecond p = stabilise(build_gmres_poly(*a, start, d, rec, cfg.orthogonalization), cfg);
    if (damped) {
      p.provenance = PolyProvenance::damped;
      p.damping_power = 1;
    }
    const OperatorPtr op = make_poly_operator(a, p);
    FirstCycle f = first_cycle(*a, *op, cfg, RitzOrdering::target_one, cfg.k, rec, sv);
    const bool pass = static_cast<int>(f.chk.mu.size()) >= cfg.nev &&
                      check_ideal_order(f.chk.mu, cfg.nev);
    if (pass || d <= 1) {
      if (pass) keep.emplace(std::move(f));
      if (!pass) {
        CycleStats cs;
        cs.discarded_probe = true;
        cs.start_dim = f.start_dim;
        cs.end_dim = f.st.cur_dim;
        history.push_back(cs);
      }
      return p;
    }
    CycleStats cs;
    cs.discarded_probe = true;
    cs.start_dim = f.start_dim;
    cs.end_dim = f.st.cur_dim;
    cs.real_checks = f.chk.real_checks;
    cs.pair_checks = f.chk.pair_checks;
    history.push_back(cs);
    if (!damped) {
      ab.resize(static_cast<size_t>(n));
      damped_start(*a, b.get(), 0.0, 1, ab.get(), rec);
      damped = true;
    } else {
      d /= 2;
    }
  }
}

}  // namespace

PolyPrecond damping_heuristic(const OperatorPtr& a, const SolveConfig& cfg, CostRecord& rec) {
  if (!a) throw std::invalid_argument("damping_heuristic: null operator");
  cfg.validate();
  if (cfg.degree < 1) throw std::invalid_argument("damping_heuristic: degree < 1");
  std::vector<CycleStats> history;
  std::optional<FirstCycle> probe;
  StartVectors sv(a->dim(), cfg.seed, {rng::kPolyStart, rng::kArnoldiStart});
  return damping_search(a, cfg, rec, history, probe, sv);
}

void SolveConfig::validate() const {
  if (m < 2) throw std::invalid_argument("SolveConfig: m must be >= 2");
  if (k <= 0 || k >= m) throw std::invalid_argument("SolveConfig: need 0 < k < m");
  if (nev <= 0) throw std::invalid_argument("SolveConfig: need nev > 0");
  if (!allow_nev_above_k && nev > k) throw std::invalid_argument("SolveConfig: need nev <= k");
  if (nev >= m) throw std::invalid_argument("SolveConfig: need nev < m");
  if (degree < 0) throw std::invalid_argument("SolveConfig: degree < 0");
  if (double_d1 < 0 || double_d2 < 0) throw std::invalid_argument("SolveConfig: double degree < 0");
  if (max_cycles < 1) throw std::invalid_argument("SolveConfig: max_cycles < 1");
  if (rtol_absolute && !(*rtol_absolute > 0.0)) {
    throw std::invalid_argument("SolveConfig: rtol_absolute must be > 0");
  }
  if (!(rtol_multiplier > 0.0)) throw std::invalid_argument("SolveConfig: rtol_multiplier <= 0");
}

int EigResult::count_correct(const std::vector<cplx>& reference, double rel_tol) const {
  int c = 0;
  for (size_t i = 0; i < eigenvalues.size(); ++i) {
    if (i < converged_flags.size() && !converged_flags[i]) continue;
    for (const cplx& r : reference) {
      if (std::abs(eigenvalues[i] - r) <= rel_tol * std::abs(r)) {
        ++c;
        break;
      }
    }
  }
  return c;
}

bool check_ideal_order(const std::vector<cplx>& mu, int nev) {
  if (nev < 1 || nev > static_cast<int>(mu.size())) {
    throw std::invalid_argument("check_ideal_order: need 1 <= nev <= size");
  }
  for (int j = 1; j < nev; ++j)
    if (std::abs(mu[j]) < std::abs(mu[j - 1])) return false;
  for (size_t j = nev; j < mu.size(); ++j)
    if (!(std::abs(mu[nev - 1]) < std::abs(mu[j]))) return false;
  return true;
}

namespace {

// Five counted power-iteration steps from the seeded N(0,1) vector x
// (SPEC.md "one cycle of power iteration (5 mvps)").
template <typename Buf>
double power_norm_estimate(const LinearOperator& a, Buf x, CostRecord& rec) {
  Context& ctx = current_context();
  const cudaStream_t s = ctx.stream();
  const int n = a.dim();
  DBuffer<double> y(static_cast<size_t>(n));
  double nx = ctx.nrm2_sync(x.get(), n);
  ++rec.dots;
  ++rec.vops;
  if (nx == 0.0) return 0.0;
  kern::scale(x.get(), 1.0 / nx, n, s);
  ++rec.vops;
  double est = 0.0;
  for (int it = 0; it < 5; ++it) {
    a.apply(x.get(), y.get(), rec);
    est = ctx.nrm2_sync(y.get(), n);
    ++rec.dots;
    ++rec.vops;
    if (est == 0.0) break;
    if (it + 1 < 5) {
      kern::copy(y.get(), x.get(), n, s);
      kern::scale(x.get(), 1.0 / est, n, s);
      ++rec.vops;
    }
  }
  ctx.sync();
  return est;
}

double diagonal_norm(const std::vector<double>& d) {
  double mx = 0.0;
  for (double v : d) mx = std::max(mx, std::abs(v));
  return mx;
}

double norm_estimate(const LinearOperator& a, CostRecord& rec, StartVectors& sv) {
  if (const std::vector<double>* d = a.diagonal()) return diagonal_norm(*d);
  return power_norm_estimate(a, sv.take(rng::kNormEstimate), rec);
}

// Streams a solve draws, in the order it draws them: the polynomial start
// vector(s) first, then the norm-estimate vector (the estimate only sets
// rtol, which the first convergence test needs, so it runs after the
// polynomial build while the host draws the remaining vectors), then the
// Arnoldi start vector.
std::vector<uint64_t> solve_streams(const LinearOperator& a, std::vector<uint64_t> poly) {
  std::vector<uint64_t> s = std::move(poly);
  if (!a.diagonal()) s.push_back(rng::kNormEstimate);
  s.push_back(rng::kArnoldiStart);
  return s;
}

}  // namespace

double operator_norm_estimate(const LinearOperator& a, unsigned long long seed, CostRecord& rec) {
  if (const std::vector<double>* d = a.diagonal()) return diagonal_norm(*d);
  DBuffer<double> x = upload(rng::normal_vector(a.dim(), seed, rng::kNormEstimate));
  return power_norm_estimate(a, std::move(x), rec);
}

EigResult solve(const OperatorPtr& a, const SolveConfig& cfg) {
  if (!a) throw std::invalid_argument("solve: null operator");
  cfg.validate();
  if (a->dim() < cfg.m + 1) throw std::invalid_argument("solve: dimension must be >= m+1");
  const auto t_all = Clock::now();
  EigResult res;
  CostRecord rec;
  rec.nnzr = a->nnzr();
  auto t0 = Clock::now();
  StartVectors sv(a->dim(), cfg.seed,
                  solve_streams(*a, cfg.degree > 0 ? std::vector<uint64_t>{rng::kPolyStart}
                                                   : std::vector<uint64_t>{}));
  OperatorPtr op = a;
  RitzOrdering ordering = RitzOrdering::smallest_magnitude;
  std::optional<FirstCycle> probe;
  if (cfg.degree > 0) {
    PolyPrecond p;
    if (cfg.damping == DampingMode::auto_heuristic) {
      p = damping_search(a, cfg, rec, res.history, probe, sv);
    } else {
      PoolBuffer b = sv.take(rng::kPolyStart);
      if (cfg.damping == DampingMode::forced) {
        // damped start A^power b + alpha b (section 6)
        DBuffer<double> bd(static_cast<size_t>(a->dim()));
        damped_start(*a, b.get(), cfg.damping_alpha, cfg.damping_power, bd.get(), rec);
        p = build_gmres_poly(*a, bd.get(), cfg.degree, rec, cfg.orthogonalization);
        p.provenance = PolyProvenance::damped;
        p.damping_alpha = cfg.damping_alpha;
        p.damping_power = cfg.damping_power;
      } else {
        p = build_gmres_poly(*a, b.get(), cfg.degree, rec, cfg.orthogonalization);
      }
      p = stabilise(p, cfg);
    }
    res.composite_degree = p.effective_degree();
    op = make_poly_operator(a, p);
    res.poly = p;
    ordering = RitzOrdering::target_one;
  }
  res.norm_estimate = norm_estimate(*a, rec, sv);
  res.rtol = cfg.rtol_absolute ? *cfg.rtol_absolute : cfg.rtol_multiplier * res.norm_estimate;
  current_context().sync();
  res.timing.setup = seconds_since(t0);
  run_cycles(*a, *op, cfg, ordering, res, rec, sv, probe ? &*probe : nullptr);
  current_context().sync();
  res.timing.total = seconds_since(t_all);
  rec.wall_seconds = res.timing.total;
  res.cost = rec;
  if (!cfg.reference.empty()) res.correct_count = res.count_correct(cfg.reference);
  return res;
}

EigResult solve_double(const OperatorPtr& a, const SolveConfig& cfg) {
  if (!a) throw std::invalid_argument("solve_double: null operator");
  cfg.validate();
  if (cfg.double_d1 < 1 || cfg.double_d2 < 1) {
    throw std::invalid_argument("solve_double: d1, d2 must be >= 1");
  }
  if (a->dim() < cfg.m + 1) throw std::invalid_argument("solve_double: dimension must be >= m+1");
  const auto t_all = Clock::now();
  EigResult res;
  CostRecord rec;
  rec.nnzr = a->nnzr();
  auto t0 = Clock::now();
  StartVectors sv(a->dim(), cfg.seed, solve_streams(*a, {rng::kPolyStart, rng::kPoly2Start}));
  PoolBuffer b1 = sv.take(rng::kPolyStart);
  PolyPrecond p1 = build_gmres_poly(*a, b1.get(), cfg.double_d1, rec, cfg.orthogonalization);
  p1.provenance = PolyProvenance::composite_stage;
  OperatorPtr tau = make_poly_complement_operator(a, p1);
  PoolBuffer b2 = sv.take(rng::kPoly2Start);
  PolyPrecond p2 = build_gmres_poly(*tau, b2.get(), cfg.double_d2, rec, cfg.orthogonalization);
  if (cfg.stability == StabilityMode::pof_auto && p2.roots.size() >= 2) {
    p2 = add_stability_roots(p2);
  }
  res.composite_degree = p1.effective_degree() * p2.effective_degree();
  OperatorPtr op = make_poly_operator(tau, p2);
  res.inner_poly = p1;
  res.poly = p2;
  res.norm_estimate = norm_estimate(*a, rec, sv);
  res.rtol = cfg.rtol_absolute ? *cfg.rtol_absolute : cfg.rtol_multiplier * res.norm_estimate;
  current_context().sync();
  res.timing.setup = seconds_since(t0);
  run_cycles(*a, *op, cfg, RitzOrdering::target_one, res, rec, sv);
  current_context().sync();
  res.timing.total = seconds_since(t_all);
  rec.wall_seconds = res.timing.total;
  res.cost = rec;
  if (!cfg.reference.empty()) res.correct_count = res.count_correct(cfg.reference);
  return res;
}

}  // namespace ppa
