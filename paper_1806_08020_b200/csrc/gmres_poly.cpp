// GMRES polynomial: host-side root management + device pi(A)v.
// Reference: src/gmres_poly.cpp (line numbers cited per function).

#include "ppa/gmres_poly.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <map>
#include <mutex>
#include <optional>
#include <unordered_map>
#include <stdexcept>

namespace ppa {

namespace {

using cplx = std::complex<double>;

// src/gmres_poly.cpp:13-18: relative tolerance below which a root counts as real.
constexpr double kRootImagTol = 1e-13;
constexpr double kLnFloor = -690.0;  // ln(1e-300), src/gmres_poly.cpp:14

bool poly_root_complex(const cplx& z) { return std::abs(z.imag()) > kRootImagTol * std::abs(z); }

bool conj_match(const cplx& a, const cplx& b) {
  return std::abs(a - std::conj(b)) <= 1e-10 * std::abs(b);
}

// First-occurrence distinct roots (src/gmres_poly.cpp:20-26).
std::vector<cplx> unique_in_order(const std::vector<cplx>& roots) {
  std::vector<cplx> u;
  for (const cplx& r : roots)
    if (std::find(u.begin(), u.end(), r) == u.end()) u.push_back(r);
  return u;
}

void recount(PolyPrecond& p) {  // src/gmres_poly.cpp:28-34
  p.multiplicity.resize(p.roots.size());
  for (size_t i = 0; i < p.roots.size(); ++i)
    p.multiplicity[i] = static_cast<int>(std::count(p.roots.begin(), p.roots.end(), p.roots[i]));
}

}  // namespace

double PofReport::max_pof() const { return std::pow(10.0, max_log10_pof); }

std::vector<cplx> leja_order(const std::vector<cplx>& roots) {
  const int d = static_cast<int>(roots.size());
  if (d == 0) throw std::invalid_argument("leja_order: empty root list");
  for (const cplx& r : roots)
    if (r == cplx(0.0, 0.0)) throw std::invalid_argument("leja_order: zero root");

  std::vector<char> taken(d, 0);
  std::vector<cplx> order;
  order.reserve(d);
  auto push = [&](int i) {
    taken[i] = 1;
    order.push_back(roots[i]);
    if (!poly_root_complex(roots[i])) return;
    // A chosen complex root drags its conjugate along (first match wins;
    // an unmatched root is tolerated, src/gmres_poly.cpp:52-63).
    for (int k = 0; k < d; ++k) {
      if (!taken[k] && k != i &&
          std::abs(roots[k] - std::conj(roots[i])) <= 1e-10 * std::abs(roots[i])) {
        taken[k] = 1;
        order.push_back(roots[k]);
        return;
      }
    }
  };

  int first = 0;  // maximal modulus, first index on ties
  for (int i = 1; i < d; ++i)
    if (std::abs(roots[i]) > std::abs(roots[first])) first = i;
  push(first);

  while (static_cast<int>(order.size()) < d) {
    int pick = -1;
    double best = -std::numeric_limits<double>::infinity();
    for (int i = 0; i < d; ++i) {
      if (taken[i]) continue;
      double score = 0.0;
      for (const cplx& c : order) {
        const double dist = std::abs(roots[i] - c);
        score += dist > 0.0 ? std::log(dist) : kLnFloor;
      }
      if (score > best) {
        best = score;
        pick = i;
      }
    }
    push(pick);
  }
  return order;
}

PolyPrecond build_gmres_poly(const LinearOperator& a, const double* b, int degree,
                             CostRecord& rec, Orthogonalization ortho) {
  if (degree < 1) throw std::invalid_argument("build_gmres_poly: degree < 1");
  if (b == nullptr) throw std::invalid_argument("build_gmres_poly: dimension mismatch");
  // Uncounted, like the reference's b.norm() guard (src/gmres_poly.cpp:101).
  if (current_context().nrm2_sync(b, a.dim()) == 0.0) {
    throw std::invalid_argument("build_gmres_poly: zero starting vector");
  }
  const int d = std::min(degree, a.dim());
  ArnoldiState st = arnoldi_init(b, a.dim(), d, rec);
  // delayed CGS2 by default (two sweeps over the basis per step instead of
  // three; the reference's MGS2 counters are charged either way, arnoldi.cpp)
  st.ortho = ortho;
  arnoldi_extend(st, a, d, rec);

  PolyPrecond p;
  p.roots = leja_order(harmonic_ritz_values(st));
  p.base_degree = static_cast<int>(p.roots.size());
  p.truncated = p.base_degree < degree;
  recount(p);
  return p;
}

PolyPrecond build_two_vector_poly(const OperatorPtr& a, const double* b1, const double* b2,
                                  int degree, CostRecord& rec) {
  if (!a || !b1 || !b2) throw std::invalid_argument("build_two_vector_poly: dimension mismatch");
  Context& ctx = current_context();
  const long long n = a->dim();
  const double n1 = ctx.nrm2_sync(b1, n);
  const double n2 = ctx.nrm2_sync(b2, n);
  rec.dots += 2;
  rec.vops += 2;
  if (n1 == 0.0 || n2 == 0.0) {
    throw std::invalid_argument("build_two_vector_poly: zero starting vector");
  }
  Scratch bhat(static_cast<size_t>(2 * n));
  kern::copy(b1, bhat.get(), n, ctx.stream());
  kern::copy(b2, bhat.get() + n, n, ctx.stream());
  kern::div_value(bhat.get(), n1 * std::sqrt(2.0), n, ctx.stream());
  kern::div_value(bhat.get() + n, n2 * std::sqrt(2.0), n, ctx.stream());
  rec.vops += 2;  // the two rescalings
  const OperatorPtr block = make_block2(a);
  PolyPrecond p = build_gmres_poly(*block, bhat.get(), degree, rec);
  p.provenance = PolyProvenance::two_vector;
  return p;
}

void damped_start(const LinearOperator& a, const double* b, double alpha, int power, double* out,
                  CostRecord& rec) {
  if (power != 1 && power != 2) throw std::invalid_argument("damped_start: power must be 1 or 2");
  if (alpha < 0.0) throw std::invalid_argument("damped_start: alpha < 0");
  Context& ctx = current_context();
  const long long n = a.dim();
  if (power == 2) {
    Scratch w(static_cast<size_t>(n));
    a.apply(b, w.get(), rec);
    a.apply(w.get(), out, rec);
  } else {
    a.apply(b, out, rec);
    if (alpha != 0.0) {
      kern::axpy(alpha, b, out, n, ctx.stream());
      ++rec.vops;
    }
  }
  const double nw = ctx.nrm2_sync(out, n);
  ++rec.dots;
  ++rec.vops;
  if (nw == 0.0) throw std::runtime_error("damped_start: damped vector vanished");
  kern::scale(out, 1.0 / nw, n, ctx.stream());
  ++rec.vops;
}

std::vector<PolyFactor> factor_plan(const PolyPrecond& p) {
  std::vector<PolyFactor> plan;
  const size_t nr = p.roots.size();
  for (size_t i = 0; i < nr;) {
    const cplx th = p.roots[i];
    PolyFactor f;
    if (!poly_root_complex(th)) {
      f.c0 = -1.0 / th.real();  // src/gmres_poly.cpp:130 (imaginary part dropped)
      i += 1;
    } else {
      if (i + 1 >= nr || std::abs(p.roots[i + 1] - std::conj(th)) > 1e-10 * std::abs(th)) {
        throw std::logic_error("apply_poly: complex root without adjacent conjugate");
      }
      const double inv_mod2 = 1.0 / std::norm(th);  // src/gmres_poly.cpp:138-139
      const double two_re_inv = 2.0 * th.real() * inv_mod2;
      f.pair = true;
      f.c0 = inv_mod2;
      f.c1 = -two_re_inv;
      i += 2;
    }
    plan.push_back(f);
  }
  return plan;
}

namespace {

// Fused chain for a CSR base operator.  The factors are grouped into passes:
//   single real root : one SpMV launch, y = x + c0 (A x)
//   conjugate pair   : t1 = A x, then y = (x + c1 t1) + c0 (A t1)
//   two real roots   : on stencils, one temporally blocked pass applies both
//                      (kernels/spmv_grid2.cu, spmv_dia2.cu); a pair too
// Every pass maps the current vector to a new buffer; buffers are assigned
// backwards from the end so the last pass writes `dst` directly, and
// `complement_base`, when set, is folded into that last pass (tau = I - pi,
// y = base - pi(A) x).  Counters charge the reference's per-factor
// increments (src/gmres_poly.cpp:129-143).
// Work vectors of one chain, supplied by the caller when the chain is
// captured into a CUDA graph (the graph must not own stream-ordered scratch).
struct ChainBuffers {
  double* other = nullptr;  // ping-pong partner of dst
  double* t1 = nullptr;     // a pair's A x
};

void apply_poly_csr(const std::vector<PolyFactor>& plan, const CsrOperator& a, const double* v,
                    double* dst, const double* complement_base, CostRecord& rec,
                    const kern::EpiArgs* outer_fold = nullptr,
                    const ChainBuffers* cb = nullptr) {
  Context& ctx = current_context();
  const cudaStream_t st = ctx.stream();
  const long long n = a.dim();
  const int K = static_cast<int>(plan.size());
  if (K == 0) {
    if (outer_fold) throw std::logic_error("apply_poly_csr: outer fold needs an inner factor");
    if (complement_base) {
      kern::sub(complement_base, v, dst, n, st);
    } else {
      kern::copy(v, dst, n, st);
    }
    return;
  }
  std::optional<Scratch> s_other, s_t1;
  double* other = cb ? cb->other : (s_other.emplace(static_cast<size_t>(n)), s_other->get());
  // Temporal blocking over stencils (kernels/spmv_dia2.cu): two real roots or
  // one pair per pass, x read once.  Its bulk copies need 16-byte aligned
  // sources (the chain's inputs: v and the ping-pong pair).
  auto aligned = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  const bool d2 = kern::dia2_supported(a.device()) && aligned(v) && aligned(dst) &&
                  aligned(other);
  struct Pass {
    int first;
    int count;  // factors in the pass (1 or 2 real roots, or 1 pair)
  };
  std::vector<Pass> passes;
  bool any_two = false;
  for (int k = 0; k < K;) {
    if (plan[k].pair) {
      passes.push_back({k, 1});
      any_two = true;
      k += 1;
    } else if (d2 && k + 1 < K && !plan[k + 1].pair) {
      passes.push_back({k, 2});
      any_two = true;
      k += 2;
    } else {
      passes.push_back({k, 1});
      k += 1;
    }
  }
  // the outer fold of a nested polynomial rides on a single-factor launch
  if (d2 && outer_fold && passes.back().count == 2) {
    const int k = passes.back().first;
    passes.back().count = 1;
    passes.push_back({k + 1, 1});
  }
  const int P = static_cast<int>(passes.size());
  double* t1p = cb ? cb->t1
                   : (s_t1.emplace(any_two ? static_cast<size_t>(n) : 1), s_t1->get());
  double* bufs[2] = {dst, other};
  const double* cur = v;
  for (int q = 0; q < P; ++q) {
    const Pass& ps = passes[q];
    double* out = bufs[(P - 1 - q) & 1];  // the last pass lands in dst
    const double* base = (q == P - 1) ? complement_base : nullptr;
    const PolyFactor& f = plan[ps.first];
    const bool fold_here = base && outer_fold;
    if (d2 && !fold_here && (ps.count == 2 || f.pair)) {
      kern::Mp2Pass m;
      m.pair = f.pair;
      m.a0 = f.c0;
      if (f.pair) {
        m.a1 = f.c1;
      } else {
        m.b0 = plan[ps.first + 1].c0;
      }
      kern::spmv_dia2(a.device(), m, cur, out, base, st);
    } else {
      kern::EpiArgs ep;
      ep.base = base;
      if (base && outer_fold) {
        ep.outer = outer_fold->outer;
        ep.oc0 = outer_fold->oc0;
        ep.oc1 = outer_fold->oc1;
        ep.oo = outer_fold->oo;
      }
      if (!f.pair) {
        ep.mode = kern::Epi::real;
        ep.c0 = f.c0;
        kern::spmv(a.device(), cur, out, ep, st);
      } else {
        kern::spmv(a.device(), cur, t1p, kern::EpiArgs{}, st);
        ep.mode = kern::Epi::pair;
        ep.c0 = f.c0;
        ep.c1 = f.c1;
        ep.o = cur;
        kern::spmv(a.device(), t1p, out, ep, st);
      }
    }
    const int mv = f.pair ? 2 : ps.count;
    rec.mvps += mv;
    rec.vops += mv;
    cur = out;
  }
}

// Reference operation sequence over an arbitrary operator.
void apply_poly_generic(const std::vector<PolyFactor>& plan, const LinearOperator& a,
                        const double* v, double* out, CostRecord& rec) {
  const cudaStream_t st = current_context().stream();
  const long long n = a.dim();
  kern::copy(v, out, n, st);
  bool any_pair = false;
  for (const PolyFactor& f : plan) any_pair |= f.pair;
  Scratch t1(static_cast<size_t>(n));
  Scratch t2(any_pair ? static_cast<size_t>(n) : 1);
  for (const PolyFactor& f : plan) {
    if (!f.pair) {
      a.apply(out, t1.get(), rec);
      kern::axpy(f.c0, t1.get(), out, n, st);
      rec.vops += 1;
    } else {
      a.apply(out, t1.get(), rec);
      a.apply(t1.get(), t2.get(), rec);
      kern::axpy(f.c1, t1.get(), out, n, st);
      kern::axpy(f.c0, t2.get(), out, n, st);
      rec.vops += 2;
    }
  }
}

// phi(tau(A)) v with tau = I - pi_1 over a CSR matrix (solve_double's
// operator): the same operation sequence as apply_poly_generic over the tau
// operator, but each outer factor's axpy is folded into the epilogue of the
// last inner launch (K4), so an outer real factor costs the
// inner chain only and no copy of v is made.  Outer factors ping-pong
// between `out` and one scratch vector, assigned backwards so the last one
// lands in `out`; counters are those of the generic path.
void apply_nested_csr(const std::vector<PolyFactor>& outer, const std::vector<PolyFactor>& inner,
                      const CsrOperator& a, const double* v, double* out, CostRecord& rec,
                      const ChainBuffers* ob = nullptr, const ChainBuffers* ib = nullptr) {
  const long long n = a.dim();
  const int Q = static_cast<int>(outer.size());
  if (Q == 0) {
    kern::copy(v, out, n, current_context().stream());
    return;
  }
  bool any_pair = false;
  for (const PolyFactor& f : outer) any_pair |= f.pair;
  std::optional<Scratch> s_other, s_t1;
  double* other = ob ? ob->other : (s_other.emplace(static_cast<size_t>(n)), s_other->get());
  double* t1 = ob ? ob->t1 : (s_t1.emplace(any_pair ? static_cast<size_t>(n) : 1), s_t1->get());
  double* bufs[2] = {out, other};
  const double* cur = v;
  for (int q = 0; q < Q; ++q) {
    const PolyFactor& f = outer[q];
    double* next = bufs[(Q - 1 - q) & 1];
    kern::EpiArgs fold;
    fold.oo = cur;
    fold.oc0 = f.c0;
    if (!f.pair) {
      fold.outer = 1;
      apply_poly_csr(inner, a, cur, next, cur, rec, &fold, ib);
      rec.vops += 2;  // tau's complement + the outer axpy
    } else {
      apply_poly_csr(inner, a, cur, t1, cur, rec, nullptr, ib);
      fold.outer = 2;
      fold.oc1 = f.c1;
      apply_poly_csr(inner, a, t1, next, t1, rec, &fold, ib);
      rec.vops += 4;  // two complements + two outer axpys
    }
    cur = next;
  }
}

}  // namespace

void apply_poly(const PolyPrecond& p, const LinearOperator& a, const double* v, double* out,
                CostRecord& rec) {
  if (v == nullptr || out == nullptr) throw std::invalid_argument("apply_poly: dimension mismatch");
  if (v == out) throw std::invalid_argument("apply_poly: input and output alias");
  const std::vector<PolyFactor> plan = factor_plan(p);
  if (const auto* csr = dynamic_cast<const CsrOperator*>(&a)) {
    apply_poly_csr(plan, *csr, v, out, nullptr, rec);
  } else {
    apply_poly_generic(plan, a, v, out, rec);
  }
}

std::complex<double> eval_poly(const PolyPrecond& p, std::complex<double> z) {
  cplx val(1.0, 0.0);
  for (const cplx& th : p.roots) val *= (1.0 - z / th);
  return val;
}

PofReport compute_pof(const PolyPrecond& p) {
  const std::vector<cplx> base = unique_in_order(p.roots);
  const int d = static_cast<int>(base.size());
  if (d < 2) throw std::invalid_argument("compute_pof: needs at least two roots");
  PofReport rep;
  rep.log10_pof.assign(d, 0.0);
  rep.copies_needed.assign(d, 0);
  rep.max_log10_pof = -std::numeric_limits<double>::infinity();
  for (int j = 0; j < d; ++j) {
    double lg = 0.0;
    for (int i = 0; i < d; ++i) {
      if (i == j) continue;
      const double f = std::abs(1.0 - base[j] / base[i]);
      lg += f > 0.0 ? std::log10(f) : kLnFloor;
    }
    rep.log10_pof[j] = lg;
    rep.copies_needed[j] = lg > 4.0 ? static_cast<int>(std::ceil((lg - 4.0) / 14.0)) : 0;
    rep.total_copies += rep.copies_needed[j];
    rep.max_log10_pof = std::max(rep.max_log10_pof, lg);
  }
  return rep;
}

PolyPrecond add_stability_roots(const PolyPrecond& p, int max_copies_per_root) {
  const PofReport rep = compute_pof(p);
  const std::vector<cplx> base = unique_in_order(p.roots);
  PolyPrecond out = p;
  std::vector<char> done(base.size(), 0);
  for (size_t j = 0; j < base.size(); ++j) {
    if (done[j]) continue;
    done[j] = 1;
    const int copies = std::min(rep.copies_needed[j], max_copies_per_root);
    if (copies <= 0) continue;
    const cplx th = base[j];
    std::vector<cplx> group{th};
    if (poly_root_complex(th)) {
      for (size_t k = 0; k < base.size(); ++k) {
        if (!done[k] && std::abs(base[k] - std::conj(th)) <= 1e-10 * std::abs(th)) {
          done[k] = 1;
          group.push_back(base[k]);
          break;
        }
      }
    }
    // src/gmres_poly.cpp:207-222: first copy appended; copies r = 1..c-1 at
    // jpos + round(r (L - jpos) / c), inserted from the back.
    const long long L = static_cast<long long>(out.roots.size());
    const long long jpos = std::find(out.roots.begin(), out.roots.end(), th) - out.roots.begin();
    std::vector<long long> at;
    for (int r = 1; r < copies; ++r)
      at.push_back(jpos + static_cast<long long>(
                              std::llround(double(r) * double(L - jpos) / double(copies))));
    std::sort(at.begin(), at.end(), std::greater<long long>());
    out.roots.insert(out.roots.end(), group.begin(), group.end());
    for (long long pos : at) out.roots.insert(out.roots.begin() + pos, group.begin(), group.end());
  }
  recount(out);
  return out;
}

namespace {

// CUDA-graph launch of the fused factor chain (opt-in: PPA_CHAIN_GRAPHS=1).
// Each apply records its chain (d launches, or d1*d2 for the nested
// operator) on a private capture stream - recording costs 5-130 us of host
// time, nothing runs - and updates one instantiated graph per (operator,
// stream) in place with cudaGraphExecUpdate (same topology, new x / y), then
// launches it; only the first apply pays for instantiation.  The chain's
// work vectors belong to the per-stream cache (a graph must not own
// stream-ordered scratch); the counters are those the recorded chain
// charged; results are bit-identical to direct launches.  In an isolated
// 50-factor chain the kernels run back to back without per-launch gaps
// (config 3: 14.5 -> 13.9 us per factor, config 1: 4.3 -> 1.7 us), but
// inside a solve the gain is 1-5 % of the extend phase (configs 1, 3, 5) or
// negative (config 2: the graph boundary stops PDL overlap with the CGS2
// kernels around it), within run-to-run noise (tools/graph_ab.py) - so
// chains launch directly by default.
bool graphs_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("PPA_CHAIN_GRAPHS");
    return v && v[0] == '1';
  }();
  return on;
}

struct ChainGraph {
  cudaStream_t capture = nullptr;
  cudaGraphExec_t exec = nullptr;
  DBuffer<double> buf[4];
  double t_capture = 0.0, t_update = 0.0;  // host microseconds (PPA_GRAPH_DEBUG)
  long long launches = 0, instantiations = 0;

  ~ChainGraph() {
    if (exec) cudaGraphExecDestroy(exec);
    if (capture) cudaStreamDestroy(capture);
  }
};

class PolyOperator final : public LinearOperator {
 public:
  PolyOperator(OperatorPtr a, PolyPrecond p, bool complement)
      : a_(std::move(a)), p_(std::move(p)), complement_(complement), plan_(factor_plan(p_)) {}
  ~PolyOperator() override {
    if (graphs_.empty()) return;
    cudaDeviceSynchronize();  // no launched chain still reads the buffers
    static const bool dbg = std::getenv("PPA_GRAPH_DEBUG") != nullptr;
    for (const auto& kv : graphs_) {
      const ChainGraph& g = *kv.second;
      if (dbg && g.launches) {
        std::fprintf(stderr, "chain graph: %lld launches, %lld instantiations, capture %.1f us, "
                     "update %.1f us per launch\n", g.launches, g.instantiations,
                     g.t_capture / g.launches, g.t_update / g.launches);
      }
    }
  }
  int dim() const override { return a_->dim(); }
  OperatorKind kind() const override {
    return complement_ ? OperatorKind::composite : OperatorKind::poly;
  }
  int mvps_per_apply() const override { return p_.effective_degree() * a_->mvps_per_apply(); }
  double nnzr() const override { return a_->nnzr(); }

  void apply(const double* x, double* y, CostRecord& rec) const override {
    if (x == y) throw std::invalid_argument("PolyOperator::apply: x and y alias");
    const auto* csr = dynamic_cast<const CsrOperator*>(a_.get());
    const PolyOperator* tau = nested_tau();
    if ((csr || tau) && graphs_enabled()) {
      apply_graphed(x, y, rec);
      return;
    }
    if (csr || tau) {
      run_chain(x, y, rec, nullptr);
      return;
    }
    if (!complement_) {
      apply_poly_generic(plan_, *a_, x, y, rec);
      return;
    }
    Scratch w(static_cast<size_t>(dim()));
    apply_poly_generic(plan_, *a_, x, w.get(), rec);
    kern::sub(x, w.get(), y, dim(), current_context().stream());
    rec.vops += 1;
  }

 private:
  // phi(tau(A)) with tau = I - pi_1 over a CSR matrix: the nested fold.
  const PolyOperator* nested_tau() const {
    if (complement_) return nullptr;
    const auto* tau = dynamic_cast<const PolyOperator*>(a_.get());
    const auto* base_csr = tau ? dynamic_cast<const CsrOperator*>(tau->a_.get()) : nullptr;
    if (tau && tau->complement_ && base_csr && !tau->plan_.empty()) {
      return tau;
    }
    return nullptr;
  }

  // The fused chain on the context's stream; `g` supplies its work vectors.
  void run_chain(const double* x, double* y, CostRecord& rec, ChainGraph* g) const {
    if (const auto* csr = dynamic_cast<const CsrOperator*>(a_.get())) {
      ChainBuffers cb;
      if (g) cb = ChainBuffers{g->buf[0].get(), g->buf[1].get()};
      // The complement y = x - w folds into the last fused launch.
      apply_poly_csr(plan_, *csr, x, y, complement_ ? x : nullptr, rec, nullptr, g ? &cb : nullptr);
      if (complement_) rec.vops += 1;
      return;
    }
    const PolyOperator* tau = nested_tau();
    const auto& base_csr = dynamic_cast<const CsrOperator&>(*tau->a_);
    ChainBuffers ob, ib;
    if (g) {
      ob = ChainBuffers{g->buf[0].get(), g->buf[1].get()};
      ib = ChainBuffers{g->buf[2].get(), g->buf[3].get()};
    }
    apply_nested_csr(plan_, tau->plan_, base_csr, x, y, rec, g ? &ob : nullptr,
                     g ? &ib : nullptr);
  }

  void apply_graphed(const double* x, double* y, CostRecord& rec) const {
    Context& ctx = current_context();
    const cudaStream_t st = ctx.stream();
    ChainGraph* g;
    {
      std::lock_guard<std::mutex> lock(gmu_);
      std::unique_ptr<ChainGraph>& slot = graphs_[st];
      if (!slot) slot = std::make_unique<ChainGraph>();
      g = slot.get();
    }
    if (!g->capture) {
      PPA_CUDA(cudaStreamCreateWithFlags(&g->capture, cudaStreamNonBlocking));
      for (auto& b : g->buf) b.resize(static_cast<size_t>(dim()));
    }
    const auto t0 = std::chrono::steady_clock::now();
    cudaGraph_t graph = nullptr;
    CostRecord d;
    const cudaStream_t prev = ctx.swap_stream(g->capture);
    PPA_CUDA(cudaStreamBeginCapture(g->capture, cudaStreamCaptureModeThreadLocal));
    try {
      run_chain(x, y, d, g);
    } catch (...) {
      cudaStreamEndCapture(g->capture, &graph);
      if (graph) cudaGraphDestroy(graph);
      ctx.swap_stream(prev);
      throw;
    }
    const cudaError_t ce = cudaStreamEndCapture(g->capture, &graph);
    ctx.swap_stream(prev);
    PPA_CUDA(ce);
    const auto t1 = std::chrono::steady_clock::now();
    bool updated = false;
    if (g->exec) {
      cudaGraphExecUpdateResultInfo info;
      updated = cudaGraphExecUpdate(g->exec, graph, &info) == cudaSuccess;
      if (!updated) {
        cudaGetLastError();
        cudaGraphExecDestroy(g->exec);
        g->exec = nullptr;
      }
    }
    if (!updated) {
      const cudaError_t ie = cudaGraphInstantiate(&g->exec, graph, 0);
      if (ie != cudaSuccess) cudaGraphDestroy(graph);
      PPA_CUDA(ie);
      ++g->instantiations;
    }
    cudaGraphDestroy(graph);
    const auto t2 = std::chrono::steady_clock::now();
    // replays on one stream are ordered, so they can share g->buf
    PPA_CUDA(cudaGraphLaunch(g->exec, st));
    ++g->launches;
    g->t_capture += std::chrono::duration<double, std::micro>(t1 - t0).count();
    g->t_update += std::chrono::duration<double, std::micro>(t2 - t1).count();
    rec.mvps += d.mvps;
    rec.dots += d.dots;
    rec.vops += d.vops;
  }

  OperatorPtr a_;
  PolyPrecond p_;
  bool complement_;
  std::vector<PolyFactor> plan_;
  mutable std::mutex gmu_;
  mutable std::map<cudaStream_t, std::unique_ptr<ChainGraph>> graphs_;
};

}  // namespace

OperatorPtr make_poly_operator(OperatorPtr a, PolyPrecond p) {
  return std::make_shared<PolyOperator>(std::move(a), std::move(p), false);
}

OperatorPtr make_poly_complement_operator(OperatorPtr a, PolyPrecond p) {
  return std::make_shared<PolyOperator>(std::move(a), std::move(p), true);
}

std::string poly_dump_csv(const PolyPrecond& p) {
  std::string s = "index,re,im,multiplicity,pof\n";
  const std::vector<cplx> base = unique_in_order(p.roots);
  std::vector<double> lg(base.size(), 0.0);
  if (base.size() >= 2) lg = compute_pof(p).log10_pof;
  char line[160];
  for (size_t i = 0; i < base.size(); ++i) {
    const int mult = static_cast<int>(std::count(p.roots.begin(), p.roots.end(), base[i]));
    std::snprintf(line, sizeof(line), "%zu,%.17g,%.17g,%d,%.17g\n", i, base[i].real(),
                  base[i].imag(), mult, std::pow(10.0, lg[i]));
    s += line;
  }
  return s;
}

}  // namespace ppa
