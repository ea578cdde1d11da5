// Thick-restarted Arnoldi with the basis on the device.
// Reference: src/arnoldi.cpp (cited per function).

#include "ppa/arnoldi.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>

#include "ppa/kernels.hpp"

namespace ppa {

namespace {

using cplx = std::complex<double>;

constexpr double kPairTol = 1e-10;  // src/arnoldi.cpp:16

bool conj_pair(const cplx& a, const cplx& b) {
  return std::abs(a - std::conj(b)) <= kPairTol * std::max(1.0, std::abs(a));
}

double sort_key(const cplx& z, RitzOrdering ord) {
  switch (ord) {
    case RitzOrdering::smallest_magnitude: return std::abs(z);
    case RitzOrdering::largest_magnitude: return -std::abs(z);
    case RitzOrdering::target_one: return std::abs(1.0 - z);
  }
  return std::abs(z);
}

// Stable sort by key with conjugate mates pulled adjacent, +imag first
// (src/arnoldi.cpp:40-95).
void arrange_pairs(RitzSet& s) {
  const int d = s.count();
  std::vector<int> idx(d);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
    return sort_key(s.values[a], s.ordering) < sort_key(s.values[b], s.ordering);
  });
  std::vector<int> out;
  out.reserve(d);
  std::vector<char> used(d, 0);
  for (int r = 0; r < d; ++r) {
    const int i = idx[r];
    if (used[i]) continue;
    used[i] = 1;
    if (!ritz_is_complex(s.values[i])) {
      out.push_back(i);
      continue;
    }
    int mate = -1;
    for (int q = 0; q < d && mate < 0; ++q) {
      const int j = idx[q];
      if (!used[j] && conj_pair(s.values[i], s.values[j])) mate = j;
    }
    if (mate < 0) {
      out.push_back(i);
      continue;
    }
    used[mate] = 1;
    if (s.values[i].imag() >= 0.0) {
      out.push_back(i);
      out.push_back(mate);
    } else {
      out.push_back(mate);
      out.push_back(i);
    }
  }
  std::vector<cplx> v(d);
  std::vector<double> res(d);
  dense::CMat g(s.vectors_h.rows, d);
  for (int r = 0; r < d; ++r) {
    v[r] = s.values[out[r]];
    res[r] = s.residuals[out[r]];
    for (int i = 0; i < g.rows; ++i) g(i, r) = s.vectors_h(i, out[r]);
  }
  s.values = std::move(v);
  s.residuals = std::move(res);
  s.vectors_h = std::move(g);
}

dense::Mat leading_block(const ArnoldiState& st, int d) {
  dense::Mat M(d, d);
  for (int j = 0; j < d; ++j)
    for (int i = 0; i < d; ++i) M(i, j) = st.h(i, j);
  return M;
}

// M + hsub^2 f e_d^T with f = Hd^{-T} e_d (src/arnoldi.cpp:183-198).
dense::Mat harmonic_matrix(const ArnoldiState& st, const char* who) {
  const int d = st.cur_dim;
  dense::Mat M = leading_block(st, d);
  const double hsub = st.h(d, d - 1);
  if (hsub != 0.0) {
    std::vector<double> ed(d, 0.0), f;
    ed[d - 1] = 1.0;
    if (!dense::solve_transpose_full_pivot(M, ed, f)) {
      // message texts of src/arnoldi.cpp:189-192 and 217-221
      const bool sel = std::string(who) == "harmonic_restart_selection";
      throw std::runtime_error(std::string(who) +
                               (sel ? ": singular projection; "
                                    : ": singular projection (GMRES stagnation); ") +
                               "try a different starting vector");
    }
    for (int i = 0; i < d; ++i) M(i, d - 1) += (hsub * hsub) * f[i];
  }
  return M;
}

long long round_ld(int n) { return (static_cast<long long>(n) + 31) / 32 * 32; }

}  // namespace

bool ritz_is_complex(const cplx& z) {
  return std::abs(z.imag()) > kPairTol * std::max(1.0, std::abs(z));
}

ArnoldiState arnoldi_init(const double* v0, int n, int m, CostRecord& rec) {
  if (m < 1) throw std::invalid_argument("arnoldi_init: m < 1");
  if (n < m + 1) throw std::invalid_argument("arnoldi_init: m+1 exceeds dimension");
  Context& ctx = current_context();
  ArnoldiState st;
  st.max_dim = m;
  st.n = n;
  st.ld = round_ld(n);
  st.V.resize(static_cast<size_t>(st.ld) * (m + 1));
  PPA_CUDA(cudaMemsetAsync(st.V.get(), 0, st.V.size() * sizeof(double), ctx.stream()));
  st.H.assign(static_cast<size_t>(m + 1) * m, 0.0);
  const double nb = ctx.nrm2_sync(v0, n);
  ++rec.dots;
  ++rec.vops;
  if (nb == 0.0) throw std::invalid_argument("arnoldi_init: zero start");
  kern::copy(v0, st.col(0), n, ctx.stream());
  kern::scale(st.col(0), 1.0 / nb, n, ctx.stream());
  ++rec.vops;
  return st;
}

namespace {

// Classic CGS2: three sweeps per step (kernels/cgs.cu).  The host needs each
// step's Hessenberg column and breakdown flag, but the device does not need
// the host to start the next step (its input V[:,j+1] is written by the
// store sweep), so step j+1 is enqueued before the host waits for step j:
// the device never idles on the round trip.  If step j breaks down, step
// j+1 ran on an unwritten column; its results are ignored (columns past
// cur_dim are never read) and its operator application is un-charged.
void extend_cgs2(ArnoldiState& st, const LinearOperator& op, int to_dim, CostRecord& rec) {
  Context& ctx = current_context();
  const cudaStream_t s = ctx.stream();
  Scratch w(static_cast<size_t>(st.n));
  const size_t slot = static_cast<size_t>(st.max_dim) + 4;
  Scratch hdev(slot);
  double* Hcol = hdev.get();
  int* flag = reinterpret_cast<int*>(hdev.get() + st.max_dim + 2);
  double* host = ctx.pinned_aux(2 * slot);
  cudaEvent_t ev[2];
  PPA_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  PPA_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  struct EventGuard {
    cudaEvent_t* e;
    ~EventGuard() {
      cudaEventDestroy(e[0]);
      cudaEventDestroy(e[1]);
    }
  } guard{ev};
  const int j0 = st.cur_dim;
  auto issue = [&](int j) {
    op.apply(st.col(j), w.get(), rec);
    kern::cgs2_step(st.V.get(), st.ld, st.n, j + 1, w.get(), Hcol, flag, ctx.ws(),
                    ctx.sm_count(), s);
    const int b = (j - j0) & 1;
    PPA_CUDA(cudaMemcpyAsync(host + b * slot, hdev.get(), slot * sizeof(double),
                             cudaMemcpyDeviceToHost, s));
    PPA_CUDA(cudaEventRecord(ev[b], s));
  };
  issue(j0);
  for (int j = j0; j < to_dim; ++j) {
    const CostRecord before_next = rec;
    if (j + 1 < to_dim) issue(j + 1);
    const int b = (j - j0) & 1;
    PPA_CUDA(cudaEventSynchronize(ev[b]));
    const double* hc = host + b * slot;
    const int c = j + 1;
    for (int i = 0; i <= c; ++i) st.h(i, j) = hc[i];
    const int bd = *reinterpret_cast<const int*>(hc + st.max_dim + 2);
    st.cur_dim = j + 1;
    if (bd == 2) {
      ctx.sync();
      throw std::runtime_error("arnoldi_extend: non-finite basis vector");
    }
    // MGS2 charges (src/arnoldi.cpp:130-140): 2c dots+axpys, one norm.
    if (bd == 1) {
      ctx.sync();
      rec = before_next;  // the speculative next step does not count
      rec.dots += 2LL * c + 1;
      rec.vops += 4LL * c + 1;
      st.h(j + 1, j) = 0.0;
      st.breakdown = true;
      return;
    }
    rec.dots += 2LL * c + 1;
    rec.vops += 4LL * c + 2;  // + the scaling (src/arnoldi.cpp:149-150)
  }
}

// Column j-1 of H gets its reorthogonalisation coefficients s and its
// subdiagonal rho; returns false (and records the breakdown) when rho fails
// the test of src/arnoldi.cpp:143-148.
bool finish_column(ArnoldiState& st, int col, const double* s, double rho) {
  double cn = 0.0;
  for (int k = 0; k <= col; ++k) {
    st.h(k, col) += s[k];
    cn += st.h(k, col) * st.h(k, col);
  }
  cn += rho * rho;
  const double colnorm = std::sqrt(cn);
  if (!std::isfinite(rho) || !std::isfinite(colnorm)) {
    throw std::runtime_error("arnoldi_extend: non-finite basis vector");
  }
  if (rho <= 1e-14 * colnorm) {
    st.h(col + 1, col) = 0.0;
    st.breakdown = true;
    st.cur_dim = col + 1;
    return false;
  }
  st.h(col + 1, col) = rho;
  st.cur_dim = col + 1;
  return true;
}

// Delayed CGS2 (DCGS2): the second (reorthogonalisation) pass of v_j and
// its normalisation are deferred to step j+1 and share its two sweeps over
// V, so a step reads V twice instead of three times.  Step j applies the
// operator to the pending first-pass vector u = V[:,j]: z = op(u), then
//   sweep 1 (dcgs2_dot): t = Q^T z, beta = u.z, s = Q^T u, nu = u.u
//   host: rho = sqrt(nu - |s|^2) completes column j-1 of H (+= s, rho);
//         A q_j = (z - Q_{j+1} g)/rho with g = H(0:j,0:j-1) s (Arnoldi
//         relation), so its first-pass coefficients are
//         h = [(t - g[:j])/rho ; ((beta - s.t)/rho - g[j])/rho]
//   sweep 2 (dcgs2_update): V[:,j] = (u - Q s)/rho (final q_j) and the next
//         pending vector z/rho - Q_{j+1}(g/rho + h), written over z.
// The first step of an extend is a plain first pass, the last pending vector
// is flushed with one more CGS pass.  Counters are charged exactly as the
// reference's MGS2 (src/arnoldi.cpp:130-150); a breakdown found one step
// late un-charges the extra operator application.
void extend_dcgs2(ArnoldiState& st, const LinearOperator& op, int to_dim, CostRecord& rec) {
  Context& ctx = current_context();
  const cudaStream_t str = ctx.stream();
  const int M = st.max_dim;
  Scratch dbuf(static_cast<size_t>(4 * M + 8));
  double* dout = dbuf.get();               // 2c reductions (or c + norm)
  double* dcoef = dbuf.get() + 2 * M + 4;  // 2j + 2 coefficients
  double* host = ctx.pinned_aux(static_cast<size_t>(4 * M + 8));
  double* hout = host;
  double* hcoef = host + 2 * M + 4;
  double* V = st.V.get();
  const int j0 = st.cur_dim;

  // step j0: first pass only; the pending vector lands in V[:, j0+1]
  op.apply(st.col(j0), st.col(j0 + 1), rec);
  {
    const int c = j0 + 1;
    kern::cgs1_pass(V, st.ld, st.n, c, st.col(j0 + 1), dout, dout + c, ctx.ws(), ctx.sm_count(),
                    str);
    PPA_CUDA(cudaMemcpyAsync(hout, dout, c * sizeof(double), cudaMemcpyDeviceToHost, str));
    ctx.sync();
    for (int i = 0; i < c; ++i) st.h(i, j0) = hout[i];
    rec.dots += 2LL * c + 1;
    rec.vops += 4LL * c + 1;
  }
  std::vector<double> g, hcol;
  for (int j = j0 + 1; j < to_dim; ++j) {
    const CostRecord before = rec;
    op.apply(st.col(j), st.col(j + 1), rec);  // z = op(u)
    const int c = j + 1;
    kern::dcgs2_dot(V, st.ld, st.n, c, st.col(j + 1), dout, ctx.ws(), ctx.sm_count(), str);
    PPA_CUDA(cudaMemcpyAsync(hout, dout, 2 * c * sizeof(double), cudaMemcpyDeviceToHost, str));
    ctx.sync();
    const double* t = hout;
    const double beta = hout[j];
    const double* sv = hout + c;
    const double nu = hout[c + j];
    double ss = 0.0, st_dot = 0.0;
    for (int k = 0; k < j; ++k) {
      ss += sv[k] * sv[k];
      st_dot += sv[k] * t[k];
    }
    const double d2 = nu - ss;
    const double rho = d2 > 0.0 ? std::sqrt(d2) : 0.0;
    if (!finish_column(st, j - 1, sv, rho)) {
      rec = before;  // the application to the dependent vector does not count
      return;
    }
    ++rec.vops;  // the scaling of v_j (src/arnoldi.cpp:149-150)
    // g = H(0:j, 0:j-1) s over every row: after thick_restart the leading
    // restart_k columns are full (rows 0..restart_k), so H is not upper
    // Hessenberg there (src/arnoldi.cpp:326-333).
    g.assign(static_cast<size_t>(j) + 1, 0.0);
    for (int k = 0; k < j; ++k) {
      const int last = std::min(j, std::max(k + 1, st.restart_k));
      for (int i = 0; i <= last; ++i) g[i] += st.h(i, k) * sv[k];
    }
    hcol.assign(static_cast<size_t>(j) + 1, 0.0);
    for (int k = 0; k < j; ++k) hcol[k] = (t[k] - g[k]) / rho;
    hcol[j] = ((beta - st_dot) / rho - g[j]) / rho;
    const double cj = g[j] / rho + hcol[j];
    const double e = cj / rho;
    for (int k = 0; k < j; ++k) {
      hcoef[k] = sv[k];
      hcoef[j + k] = (g[k] / rho + hcol[k]) - e * sv[k];
    }
    hcoef[2 * j] = e;
    hcoef[2 * j + 1] = rho;
    for (int i = 0; i <= j; ++i) st.h(i, j) = hcol[i];
    PPA_CUDA(cudaMemcpyAsync(dcoef, hcoef, (2 * j + 2) * sizeof(double), cudaMemcpyHostToDevice,
                             str));
    kern::dcgs2_update(V, st.ld, st.n, c, st.col(j + 1), dcoef, ctx.ws(), ctx.sm_count(), str);
    rec.dots += 2LL * c + 1;
    rec.vops += 4LL * c + 1;
  }
  // flush the pending V[:, to_dim]: second pass, then normalise
  const int c = to_dim;
  kern::cgs1_pass(V, st.ld, st.n, c, st.col(to_dim), dout, dout + c, ctx.ws(), ctx.sm_count(),
                  str);
  PPA_CUDA(cudaMemcpyAsync(hout, dout, (c + 1) * sizeof(double), cudaMemcpyDeviceToHost, str));
  ctx.sync();
  if (!finish_column(st, to_dim - 1, hout, hout[c])) return;
  kern::div_value(st.col(to_dim), hout[c], st.n, str);
  ++rec.vops;
}

// Delayed CGS2 is the solver's default (SolveConfig::orthogonalization,
// DESIGN.md 3.2); a bare ArnoldiState starts in CGS2.  Its roundoff differs
// from CGS2's, so matvec-count parity with the oracle is a property of the
// current kernels, not a guarantee.  A single-step extend keeps CGS2 (the
// delayed form would need a flush pass as well).
bool use_dcgs2(const ArnoldiState& st, int steps) {
  return st.ortho == Orthogonalization::dcgs2 && steps >= 2;
}

}  // namespace

void arnoldi_extend(ArnoldiState& st, const LinearOperator& op, int to_dim, CostRecord& rec) {
  if (to_dim > st.max_dim) throw std::invalid_argument("arnoldi_extend: to_dim > max_dim");
  if (to_dim <= st.cur_dim) throw std::invalid_argument("arnoldi_extend: to_dim <= cur_dim");
  if (op.dim() != st.n) throw std::invalid_argument("arnoldi_extend: dimension mismatch");
  if (use_dcgs2(st, to_dim - st.cur_dim)) {
    extend_dcgs2(st, op, to_dim, rec);
  } else {
    extend_cgs2(st, op, to_dim, rec);
  }
}

RitzSet ritz_pairs(const ArnoldiState& st, RitzOrdering ordering) {
  const int d = st.cur_dim;
  if (d < 1) throw std::invalid_argument("ritz_pairs: empty state");
  RitzSet set;
  set.ordering = ordering;
  if (!dense::eig(leading_block(st, d), set.values, &set.vectors_h)) {
    throw std::runtime_error("ritz_pairs: Hessenberg eigensolver failed");
  }
  set.residuals.resize(d);
  const double hsub = st.h(d, d - 1);
  for (int i = 0; i < d; ++i) {
    double nn = 0.0;
    for (int r = 0; r < d; ++r) nn += std::norm(set.vectors_h(r, i));
    const double nrm = std::sqrt(nn);
    for (int r = 0; r < d; ++r) set.vectors_h(r, i) /= nrm;
    set.residuals[i] = std::abs(hsub) * std::abs(set.vectors_h(d - 1, i));
  }
  arrange_pairs(set);
  return set;
}

std::vector<cplx> harmonic_ritz_values(const ArnoldiState& st) {
  if (st.cur_dim < 1) throw std::invalid_argument("harmonic_ritz_values: empty state");
  const dense::Mat M = harmonic_matrix(st, "harmonic_ritz_values");
  std::vector<cplx> vals;
  if (!dense::eig(M, vals, nullptr)) {
    throw std::runtime_error("harmonic_ritz_values: eigensolver failed");
  }
  return vals;
}

RitzSet harmonic_restart_selection(const ArnoldiState& st, RitzOrdering ordering) {
  const int d = st.cur_dim;
  if (d < 1) throw std::invalid_argument("harmonic_restart_selection: empty");
  const dense::Mat M = harmonic_matrix(st, "harmonic_restart_selection");
  const dense::Mat Hd = leading_block(st, d);
  const double hsub = st.h(d, d - 1);
  RitzSet set;
  set.ordering = ordering;
  set.harmonic = true;
  if (!dense::eig(M, set.values, &set.vectors_h)) {
    throw std::runtime_error("harmonic_restart_selection: eigensolver failed");
  }
  set.residuals.resize(d);
  for (int i = 0; i < d; ++i) {
    double nn = 0.0;
    for (int r = 0; r < d; ++r) nn += std::norm(set.vectors_h(r, i));
    const double nrm = std::sqrt(nn);
    for (int r = 0; r < d; ++r) set.vectors_h(r, i) /= nrm;
    // ||Hd g - theta g||^2 + |hsub g_d|^2 (src/arnoldi.cpp:242-246)
    double top = 0.0;
    for (int r = 0; r < d; ++r) {
      cplx acc(0.0, 0.0);
      for (int c = 0; c < d; ++c) acc += Hd(r, c) * set.vectors_h(c, i);
      top += std::norm(acc - set.values[i] * set.vectors_h(r, i));
    }
    set.residuals[i] = std::sqrt(top + std::norm(hsub * set.vectors_h(d - 1, i)));
  }
  arrange_pairs(set);
  return set;
}

DeviceComplexVector ritz_vector(const ArnoldiState& st, const RitzSet& set, int j,
                                CostRecord& rec) {
  const int d = set.vectors_h.rows;
  if (j < 0 || j >= set.count()) throw std::invalid_argument("ritz_vector: index out of range");
  Context& ctx = current_context();
  const cudaStream_t s = ctx.stream();
  double imn = 0.0;
  for (int r = 0; r < d; ++r) imn += set.vectors_h(r, j).imag() * set.vectors_h(r, j).imag();
  const bool cplx_vec = std::sqrt(imn) > 0.0;
  const int p = cplx_vec ? 2 : 1;
  std::vector<double> g(static_cast<size_t>(d) * p);
  for (int r = 0; r < d; ++r) {
    g[r] = set.vectors_h(r, j).real();
    if (cplx_vec) g[d + r] = set.vectors_h(r, j).imag();
  }
  Scratch gdev(g.size());
  PPA_CUDA(cudaMemcpyAsync(gdev.get(), g.data(), g.size() * sizeof(double),
                           cudaMemcpyHostToDevice, s));
  DeviceComplexVector y;
  y.complex = cplx_vec;
  const long long ldy = round_ld(st.n);
  Scratch tmp(static_cast<size_t>(ldy) * p);
  kern::ts_combine(st.V.get(), st.ld, st.n, d, gdev.get(), p, tmp.get(), ldy, s);
  rec.vops += static_cast<long long>(p) * d;
  double* sums = ctx.results();
  kern::col_sumsq(tmp.get(), ldy, st.n, p, sums, ctx.ws(), ctx.sm_count(), s);
  double* h = ctx.pinned(2);
  PPA_CUDA(cudaMemcpyAsync(h, sums, p * sizeof(double), cudaMemcpyDeviceToHost, s));
  ctx.sync();
  const double nrm = std::sqrt(h[0] + (cplx_vec ? h[1] : 0.0));
  y.re.resize(st.n);
  kern::copy(tmp.get(), y.re.get(), st.n, s);
  kern::div_value(y.re.get(), nrm, st.n, s);
  if (cplx_vec) {
    y.im.resize(st.n);
    kern::copy(tmp.get() + ldy, y.im.get(), st.n, s);
    kern::div_value(y.im.get(), nrm, st.n, s);
  }
  rec.dots += cplx_vec ? 2 : 1;
  rec.vops += cplx_vec ? 4 : 2;
  ctx.sync();  // gdev / tmp are released on return
  return y;
}

int thick_restart(ArnoldiState& st, const RitzSet& keep, int k, CostRecord& rec) {
  const int m = st.cur_dim;
  if (m != st.max_dim) throw std::invalid_argument("thick_restart: cycle not at full dimension");
  if (k <= 0 || k >= m) throw std::invalid_argument("thick_restart: bad k");
  if (keep.count() < k) throw std::invalid_argument("thick_restart: selection smaller than k");
  if (st.h(m, m - 1) == 0.0) {
    throw std::runtime_error("thick_restart: no residual vector (breakdown)");
  }
  // Real basis of the kept span (src/arnoldi.cpp:285-299).
  dense::Mat G(m, k);
  int col = 0, j = 0;
  while (col < k && j < keep.count()) {
    if (!ritz_is_complex(keep.values[j])) {
      for (int r = 0; r < m; ++r) G(r, col) = keep.vectors_h(r, j).real();
      ++col;
      j += 1;
    } else {
      if (col + 2 > k) break;
      for (int r = 0; r < m; ++r) {
        G(r, col) = keep.vectors_h(r, j).real();
        G(r, col + 1) = keep.vectors_h(r, j).imag();
      }
      col += 2;
      j += 2;
    }
  }
  const int kk = col;
  if (kk == 0) throw std::invalid_argument("thick_restart: k too small");
  dense::Mat Gk(m, kk);
  std::copy(G.a.begin(), G.a.begin() + static_cast<long>(m) * kk, Gk.a.begin());
  const dense::Mat Q = dense::householder_q(Gk);
  const dense::Mat Hm = leading_block(st, m);
  dense::Mat Hk = dense::matmul_tn(Q, dense::matmul(Hm, Q));
  std::vector<double> hrow(kk);
  for (int c = 0; c < kk; ++c) hrow[c] = st.h(m, m - 1) * Q(m - 1, c);

  Context& ctx = current_context();
  const cudaStream_t s = ctx.stream();
  Scratch qdev(Q.a.size());
  PPA_CUDA(cudaMemcpyAsync(qdev.get(), Q.a.data(), Q.a.size() * sizeof(double),
                           cudaMemcpyHostToDevice, s));
  kern::ts_combine(st.V.get(), st.ld, st.n, m, qdev.get(), kk, st.V.get(), st.ld, s);
  rec.vops += static_cast<long long>(m) * kk;
  kern::copy(st.col(m), st.col(kk), st.n, s);

  // Reorthogonalise the carried residual vector (one pass) and fold the
  // corrections into H (src/arnoldi.cpp:313-333).
  double* dres = ctx.results();
  Scratch corr(static_cast<size_t>(kk) + 1);
  kern::cgs1_pass(st.V.get(), st.ld, st.n, kk, st.col(kk), corr.get(), dres, ctx.ws(),
                  ctx.sm_count(), s);
  double* h = ctx.pinned(static_cast<size_t>(kk) + 1);
  PPA_CUDA(cudaMemcpyAsync(h, corr.get(), kk * sizeof(double), cudaMemcpyDeviceToHost, s));
  PPA_CUDA(cudaMemcpyAsync(h + kk, dres, sizeof(double), cudaMemcpyDeviceToHost, s));
  ctx.sync();
  std::vector<double> cvec(h, h + kk);
  const double rn = h[kk];
  rec.dots += kk;
  rec.vops += 2LL * kk;
  ++rec.dots;
  ++rec.vops;
  kern::scale(st.col(kk), 1.0 / rn, st.n, s);
  ++rec.vops;
  for (int c = 0; c < kk; ++c)
    for (int r = 0; r < kk; ++r) Hk(r, c) += cvec[r] * hrow[c];

  std::fill(st.H.begin(), st.H.end(), 0.0);
  for (int c = 0; c < kk; ++c) {
    for (int r = 0; r < kk; ++r) st.h(r, c) = Hk(r, c);
    st.h(kk, c) = rn * hrow[c];
  }
  st.cur_dim = kk;
  st.restart_k = kk;
  ++st.cycle_count;
  ctx.sync();  // qdev is released on return
  return kk;
}

// Harmonic thick restart (the solve's RestartVariant::harmonic).  The
// reference solve would pass harmonic_restart_selection's vectors to
// thick_restart (src/arnoldi.cpp:267-334), which keeps v_{m+1} as the
// residual direction - correct for Ritz vectors only: for harmonic pairs
// Hbar g - theta [g; 0] is parallel to p = [-h f; 1] (f = H^{-T} e_m), not to
// e_{m+1}, so the compressed factorisation stops being an Arnoldi relation
// and the iteration stalls (diag(1..1000): max residual stuck at 15.25 for
// 300 cycles in both implementations).  SPEC.md:178 requires the Krylov
// property to survive the restart, so the harmonic variant keeps
// span{[G; 0], p} instead (Morgan's GMRES-DR construction): with Qh the
// orthonormal basis of [[G; 0], p], A V_m Q = V_{m+1} Qh (Qh^T Hbar Q)
// exactly.  Counters follow thick_restart's (basis compression, one
// reorthogonalisation pass of the carried vector).
int harmonic_thick_restart(ArnoldiState& st, const RitzSet& keep, int k, CostRecord& rec) {
  const int m = st.cur_dim;
  if (m != st.max_dim) throw std::invalid_argument("thick_restart: cycle not at full dimension");
  if (k <= 0 || k >= m) throw std::invalid_argument("thick_restart: bad k");
  if (keep.count() < k) throw std::invalid_argument("thick_restart: selection smaller than k");
  const double hm = st.h(m, m - 1);
  if (hm == 0.0) throw std::runtime_error("thick_restart: no residual vector (breakdown)");
  dense::Mat G(m, k);
  int col = 0, j = 0;
  while (col < k && j < keep.count()) {
    if (!ritz_is_complex(keep.values[j])) {
      for (int r = 0; r < m; ++r) G(r, col) = keep.vectors_h(r, j).real();
      ++col;
      j += 1;
    } else {
      if (col + 2 > k) break;
      for (int r = 0; r < m; ++r) {
        G(r, col) = keep.vectors_h(r, j).real();
        G(r, col + 1) = keep.vectors_h(r, j).imag();
      }
      col += 2;
      j += 2;
    }
  }
  const int kk = col;
  if (kk == 0) throw std::invalid_argument("thick_restart: k too small");
  // p = [-h f; 1], H_m^T f = e_m
  const dense::Mat Hm = leading_block(st, m);
  std::vector<double> em(m, 0.0), f;
  em[m - 1] = 1.0;
  if (!dense::solve_transpose_full_pivot(Hm, em, f)) {
    throw std::runtime_error("harmonic_restart_selection: singular projection; "
                             "try a different starting vector");
  }
  dense::Mat P(m + 1, kk + 1);
  for (int c = 0; c < kk; ++c)
    for (int r = 0; r < m; ++r) P(r, c) = G(r, c);
  for (int r = 0; r < m; ++r) P(r, kk) = -hm * f[r];
  P(m, kk) = 1.0;
  const dense::Mat Qh = dense::householder_q(P);  // (m+1) x (kk+1)
  dense::Mat Hbar(m + 1, m);
  for (int c = 0; c < m; ++c)
    for (int r = 0; r <= m; ++r) Hbar(r, c) = st.h(r, c);
  dense::Mat Qm(m, kk);
  for (int c = 0; c < kk; ++c)
    for (int r = 0; r < m; ++r) Qm(r, c) = Qh(r, c);
  const dense::Mat Hn = dense::matmul_tn(Qh, dense::matmul(Hbar, Qm));  // (kk+1) x kk

  Context& ctx = current_context();
  const cudaStream_t s = ctx.stream();
  Scratch qdev(Qh.a.size());
  PPA_CUDA(cudaMemcpyAsync(qdev.get(), Qh.a.data(), Qh.a.size() * sizeof(double),
                           cudaMemcpyHostToDevice, s));
  kern::ts_combine(st.V.get(), st.ld, st.n, m + 1, qdev.get(), kk + 1, st.V.get(), st.ld, s);
  rec.vops += static_cast<long long>(m + 1) * (kk + 1);

  // one reorthogonalisation pass of the new column kk; corrections folded
  // into H as in thick_restart (v = rn v_new + V_k c)
  double* dres = ctx.results();
  Scratch corr(static_cast<size_t>(kk) + 1);
  kern::cgs1_pass(st.V.get(), st.ld, st.n, kk, st.col(kk), corr.get(), dres, ctx.ws(),
                  ctx.sm_count(), s);
  double* h = ctx.pinned(static_cast<size_t>(kk) + 1);
  PPA_CUDA(cudaMemcpyAsync(h, corr.get(), kk * sizeof(double), cudaMemcpyDeviceToHost, s));
  PPA_CUDA(cudaMemcpyAsync(h + kk, dres, sizeof(double), cudaMemcpyDeviceToHost, s));
  ctx.sync();
  const double rn = h[kk];
  rec.dots += kk + 1;
  rec.vops += 2LL * kk + 2;
  kern::scale(st.col(kk), 1.0 / rn, st.n, s);
  std::fill(st.H.begin(), st.H.end(), 0.0);
  for (int c = 0; c < kk; ++c) {
    for (int r = 0; r < kk; ++r) st.h(r, c) = Hn(r, c) + h[r] * Hn(kk, c);
    st.h(kk, c) = rn * Hn(kk, c);
  }
  st.cur_dim = kk;
  st.restart_k = kk;
  ++st.cycle_count;
  ctx.sync();  // qdev is released on return
  return kk;
}

}  // namespace ppa
