// extern "C" boundary (include/ppa_b200.h).  Every entry catches and maps
// the C++ exceptions of the ppa namespace to status codes.

#include "ppa_b200.h"

#include <algorithm>
#include <cstring>
#include <string>

#include "ppa/arnoldi.hpp"
#include "ppa/gmres_poly.hpp"
#include "ppa/kernels.hpp"
#include "ppa/operators.hpp"
#include "ppa/rng.hpp"
#include "ppa/solver.hpp"

struct ppa_host_csr {
  ppa::CsrMatrix m;
};
struct ppa_op {
  ppa::OperatorPtr p;
};
struct ppa_arnoldi {
  ppa::ArnoldiState s;
};

namespace {

thread_local std::string t_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return PPA_OK;
  } catch (const std::invalid_argument& e) {
    t_err = e.what();
    return PPA_INVALID_ARGUMENT;
  } catch (const std::logic_error& e) {
    t_err = e.what();
    return PPA_LOGIC_ERROR;
  } catch (const ppa::CudaError& e) {
    t_err = e.what();
    return PPA_CUDA_ERROR;
  } catch (const std::runtime_error& e) {
    t_err = e.what();
    return PPA_RUNTIME_ERROR;
  } catch (const std::exception& e) {
    t_err = e.what();
    return PPA_INTERNAL_ERROR;
  } catch (...) {
    t_err = "unknown error";
    return PPA_INTERNAL_ERROR;
  }
}

void add_cost(ppa_cost* c, const ppa::CostRecord& r) {
  if (!c) return;
  c->mvps += r.mvps;
  c->dots += r.dots;
  c->vops += r.vops;
  if (r.nnzr > 0) c->nnzr = r.nnzr;
  c->wall_seconds += r.wall_seconds;
}

std::vector<std::complex<double>> roots_of(const double* re, const double* im, int n) {
  if (n < 0) throw std::invalid_argument("root list: negative length");
  if (n > 0 && (!re || !im)) throw std::invalid_argument("root list: null pointer");
  std::vector<std::complex<double>> r(n);
  for (int i = 0; i < n; ++i) r[i] = {re[i], im[i]};
  return r;
}

ppa::PolyPrecond poly_of(const double* re, const double* im, int n, int base_degree) {
  ppa::PolyPrecond p;
  p.roots = roots_of(re, im, n);
  p.base_degree = base_degree > 0 ? base_degree : n;
  p.multiplicity.resize(p.roots.size());
  for (size_t i = 0; i < p.roots.size(); ++i)
    p.multiplicity[i] = static_cast<int>(std::count(p.roots.begin(), p.roots.end(), p.roots[i]));
  return p;
}

ppa_host_csr* wrap(ppa::CsrMatrix&& m) {
  auto* h = new ppa_host_csr;
  h->m = std::move(m);
  return h;
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string(what) + ": null pointer");
}

ppa::SolveConfig to_config(const ppa_solve_config& c) {
  ppa::SolveConfig cfg;
  cfg.m = c.m;
  cfg.k = c.k;
  cfg.nev = c.nev;
  cfg.degree = c.degree;
  cfg.rtol_multiplier = c.rtol_multiplier;
  if (c.rtol_absolute > 0) cfg.rtol_absolute = c.rtol_absolute;
  cfg.variant = c.variant ? ppa::RestartVariant::harmonic : ppa::RestartVariant::ritz;
  cfg.stability = c.stability ? ppa::StabilityMode::pof_auto : ppa::StabilityMode::off;
  cfg.double_d1 = c.double_d1;
  cfg.double_d2 = c.double_d2;
  cfg.max_cycles = c.max_cycles;
  cfg.seed = c.seed;
  cfg.allow_nev_above_k = c.allow_nev_above_k != 0;
  cfg.damping = c.damping == 1   ? ppa::DampingMode::auto_heuristic
                : c.damping == 2 ? ppa::DampingMode::forced
                                 : ppa::DampingMode::off;
  cfg.damping_alpha = c.damping_alpha;
  cfg.damping_power = c.damping_power > 0 ? c.damping_power : 1;
  cfg.check_mid_cycle = c.check_mid_cycle != 0;
  if (c.mid_cycle_stride > 0) cfg.mid_cycle_stride = c.mid_cycle_stride;
  cfg.stagnation_stop = c.stagnation_stop != 0;
  if (c.stagnation_window > 0) cfg.stagnation_window = c.stagnation_window;
  if (c.stagnation_rtol > 0) cfg.stagnation_rtol = c.stagnation_rtol;
  cfg.want_eigenvectors = c.want_eigenvectors != 0;
  if (c.orthogonalization < 0 || c.orthogonalization > 1) {
    throw std::invalid_argument("SolveConfig: orthogonalization must be 0 or 1");
  }
  cfg.orthogonalization = static_cast<ppa::Orthogonalization>(c.orthogonalization);
  return cfg;
}

ppa_op* wrap_op(ppa::OperatorPtr p) {
  auto* o = new ppa_op;
  o->p = std::move(p);
  return o;
}

void roots_out(const ppa::PolyPrecond& p, double* re, double* im, int cap, int* nroots) {
  if (p.effective_degree() > cap) throw std::invalid_argument("root output capacity too small");
  for (int i = 0; i < p.effective_degree(); ++i) {
    re[i] = p.roots[i].real();
    im[i] = p.roots[i].imag();
  }
  if (nroots) *nroots = p.effective_degree();
}

}  // namespace

extern "C" {

const char* ppa_last_error(void) { return t_err.c_str(); }
int ppa_abi_version(void) { return 3; }

int ppa_device_info(int* sm_count, double* l2_bytes) {
  return guard([&] {
    int dev = 0, sms = 0, l2 = 0;
    PPA_CUDA(cudaGetDevice(&dev));
    PPA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    PPA_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    if (sm_count) *sm_count = sms;
    if (l2_bytes) *l2_bytes = l2;
  });
}

int ppa_set_stream(void* s) {
  return guard([&] { ppa::set_current_stream(static_cast<cudaStream_t>(s)); });
}

int ppa_synchronize(void) {
  return guard([&] { ppa::current_context().sync(); });
}

int ppa_host_csr_create(int n, long long nnz, const int* row_ptr, const int* col_idx,
                        const double* values, ppa_host_csr** out) {
  return guard([&] {
    need(out, "ppa_host_csr_create");
    if (n < 0 || nnz < 0) throw std::invalid_argument("CsrMatrix: negative dimension");
    need(row_ptr, "ppa_host_csr_create");
    if (nnz > 0) {
      need(col_idx, "ppa_host_csr_create");
      need(values, "ppa_host_csr_create");
    }
    ppa::CsrMatrix m;
    m.n = n;
    m.row_ptr.assign(row_ptr, row_ptr + n + 1);
    m.col_idx.assign(col_idx, col_idx + nnz);
    m.values.assign(values, values + nnz);
    m.validate();
    *out = wrap(std::move(m));
  });
}

int ppa_host_csr_from_triplets(int n, long long count, const int* rows, const int* cols,
                               const double* vals, ppa_host_csr** out) {
  return guard([&] {
    need(out, "ppa_host_csr_from_triplets");
    std::vector<std::tuple<int, int, double>> t;
    t.reserve(static_cast<size_t>(count));
    for (long long i = 0; i < count; ++i) t.emplace_back(rows[i], cols[i], vals[i]);
    *out = wrap(ppa::CsrMatrix::from_triplets(n, std::move(t)));
  });
}

int ppa_gen_convdiff_ref(int grid_n, ppa_host_csr** out) {
  return guard([&] { need(out, "gen"); *out = wrap(ppa::make_convection_diffusion(grid_n)); });
}
int ppa_gen_config(int config, ppa_host_csr** out) {
  return guard([&] { need(out, "gen"); *out = wrap(ppa::make_config_matrix(config)); });
}
int ppa_gen_bidiagonal(int n, ppa_host_csr** out) {
  return guard([&] { need(out, "gen"); *out = wrap(ppa::make_bidiagonal(n)); });
}
int ppa_gen_convdiff_const(int grid_n, double peclet, ppa_host_csr** out) {
  return guard([&] {
    need(out, "gen");
    *out = wrap(ppa::make_convection_diffusion_const(grid_n, peclet));
  });
}
int ppa_gen_laplacian_3d(int grid_n, ppa_host_csr** out) {
  return guard([&] { need(out, "gen"); *out = wrap(ppa::make_laplacian_3d(grid_n)); });
}
int ppa_gen_random_poisson(int n, double lambda, unsigned long long seed, ppa_host_csr** out) {
  return guard([&] { need(out, "gen"); *out = wrap(ppa::make_random_poisson(n, lambda, seed)); });
}

int ppa_host_csr_info(const ppa_host_csr* m, int* n, long long* nnz,
                      unsigned long long* fingerprint) {
  return guard([&] {
    need(m, "ppa_host_csr_info");
    if (n) *n = m->m.n;
    if (nnz) *nnz = m->m.nnz();
    if (fingerprint) *fingerprint = ppa::csr_fingerprint(m->m);
  });
}

int ppa_host_csr_arrays(const ppa_host_csr* m, const int** row_ptr, const int** col_idx,
                        const double** values) {
  return guard([&] {
    need(m, "ppa_host_csr_arrays");
    if (row_ptr) *row_ptr = m->m.row_ptr.data();
    if (col_idx) *col_idx = m->m.col_idx.data();
    if (values) *values = m->m.values.data();
  });
}

void ppa_host_csr_free(ppa_host_csr* m) { delete m; }

int ppa_normal_vector(long long n, unsigned long long seed, unsigned long long stream,
                      double* out) {
  return guard([&] {
    need(out, "ppa_normal_vector");
    const std::vector<double> v = ppa::rng::normal_vector(n, seed, stream);
    std::copy(v.begin(), v.end(), out);
  });
}

int ppa_host_csr_multiply(const ppa_host_csr* m, const double* x, double* y) {
  return guard([&] {
    need(m, "ppa_host_csr_multiply");
    need(x, "ppa_host_csr_multiply");
    need(y, "ppa_host_csr_multiply");
    m->m.multiply(x, y);
  });
}

int ppa_csr_operator_layout(const ppa_host_csr* m, int layout, ppa_op** out) {
  return guard([&] {
    need(m, "ppa_csr_operator_layout");
    need(out, "ppa_csr_operator_layout");
    if (layout < 0 || layout > 4) throw std::invalid_argument("ppa_csr_operator_layout: layout");
    *out = wrap_op(ppa::make_csr_operator(m->m, static_cast<ppa::CsrLayout>(layout)));
  });
}

int ppa_csr_operator(const ppa_host_csr* m, ppa_op** out) {
  return guard([&] {
    need(m, "ppa_csr_operator");
    need(out, "ppa_csr_operator");
    auto* o = new ppa_op;
    try {
      o->p = ppa::make_csr_operator(m->m);
    } catch (...) {
      delete o;
      throw;
    }
    *out = o;
  });
}

int ppa_diagonal_operator(int n, const double* diag, ppa_op** out) {
  return guard([&] {
    need(out, "ppa_diagonal_operator");
    if (n > 0) need(diag, "ppa_diagonal_operator");
    std::vector<double> d(diag, diag + std::max(0, n));
    auto* o = new ppa_op;
    try {
      o->p = ppa::make_diagonal(std::move(d));
    } catch (...) {
      delete o;
      throw;
    }
    *out = o;
  });
}

int ppa_poly_operator(const ppa_op* base, const double* re, const double* im, int nroots,
                      int base_degree, int complement, ppa_op** out) {
  return guard([&] {
    need(base, "ppa_poly_operator");
    need(out, "ppa_poly_operator");
    ppa::PolyPrecond p = poly_of(re, im, nroots, base_degree);
    auto* o = new ppa_op;
    try {
      o->p = complement ? ppa::make_poly_complement_operator(base->p, std::move(p))
                        : ppa::make_poly_operator(base->p, std::move(p));
    } catch (...) {
      delete o;
      throw;
    }
    *out = o;
  });
}

int ppa_op_create_callback(int dim, int mvps_per_apply, double nnzr, ppa_apply_fn apply,
                           void* ctx, ppa_op** out) {
  return guard([&] {
    need(out, "ppa_op_create_callback");
    if (!apply) throw std::invalid_argument("make_callback_operator: null apply");
    *out = wrap_op(ppa::make_callback_operator(
        dim, mvps_per_apply, nnzr,
        [apply, ctx](const double* x, double* y, cudaStream_t s) {
          return apply(ctx, x, y, static_cast<void*>(s));
        }));
  });
}

void ppa_op_free(ppa_op* op) { delete op; }

int ppa_op_info(const ppa_op* op, int* dim, int* mvps, double* nnzr, int* kind) {
  return guard([&] {
    need(op, "ppa_op_info");
    if (dim) *dim = op->p->dim();
    if (mvps) *mvps = op->p->mvps_per_apply();
    if (nnzr) *nnzr = op->p->nnzr();
    if (kind) *kind = static_cast<int>(op->p->kind());
  });
}

int ppa_op_apply(const ppa_op* op, const double* x, double* y, ppa_cost* cost) {
  return guard([&] {
    need(op, "ppa_op_apply");
    ppa::CostRecord r;
    op->p->apply(x, y, r);
    add_cost(cost, r);
  });
}

int ppa_op_apply_host(const ppa_op* op, const double* x, double* y, ppa_cost* cost) {
  return guard([&] {
    need(op, "ppa_op_apply_host");
    need(x, "ppa_op_apply_host");
    need(y, "ppa_op_apply_host");
    ppa::Context& ctx = ppa::current_context();
    const size_t bytes = static_cast<size_t>(op->p->dim()) * sizeof(double);
    ppa::Scratch dx(op->p->dim()), dy(op->p->dim());
    PPA_CUDA(cudaMemcpyAsync(dx.get(), x, bytes, cudaMemcpyHostToDevice, ctx.stream()));
    ppa::CostRecord r;
    op->p->apply(dx.get(), dy.get(), r);
    PPA_CUDA(cudaMemcpyAsync(y, dy.get(), bytes, cudaMemcpyDeviceToHost, ctx.stream()));
    ctx.sync();
    add_cost(cost, r);
  });
}

int ppa_op_apply_host_batch(const ppa_op* op, int count, const double* X, double* Y,
                            ppa_cost* cost) {
  return guard([&] {
    need(op, "ppa_op_apply_host_batch");
    if (count < 0) throw std::invalid_argument("ppa_op_apply_host_batch: negative count");
    if (count == 0) return;
    need(X, "ppa_op_apply_host_batch");
    need(Y, "ppa_op_apply_host_batch");
    ppa::Context& ctx = ppa::current_context();
    const cudaStream_t cs = ctx.stream();
    const long long n = op->p->dim();
    const size_t bytes = static_cast<size_t>(n) * sizeof(double);
    // Double-buffered pipeline: H2D of vector i+1 and D2H of vector i-1 run on
    // their own streams (PCIe copy engines) while the SMs apply the operator
    // to vector i; events order the buffer reuse.
    static thread_local cudaStream_t hin = nullptr, hout = nullptr;
    if (!hin) {
      PPA_CUDA(cudaStreamCreateWithFlags(&hin, cudaStreamNonBlocking));
      PPA_CUDA(cudaStreamCreateWithFlags(&hout, cudaStreamNonBlocking));
    }
    ppa::Scratch din0(n), din1(n), dout0(n), dout1(n);
    double* din[2] = {din0.get(), din1.get()};
    double* dout[2] = {dout0.get(), dout1.get()};
    cudaEvent_t ev[3][2];
    for (auto& row : ev)
      for (auto& e : row) PPA_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    enum { kIn = 0, kComp = 1, kOut = 2 };
    // buffers come from the stream-ordered pool of `cs`: make the copy streams wait
    cudaEvent_t ready;
    PPA_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    PPA_CUDA(cudaEventRecord(ready, cs));
    PPA_CUDA(cudaStreamWaitEvent(hin, ready, 0));
    PPA_CUDA(cudaStreamWaitEvent(hout, ready, 0));
    ppa::CostRecord r;
    for (int i = 0; i < count; ++i) {
      const int b = i & 1;
      if (i >= 2) PPA_CUDA(cudaStreamWaitEvent(hin, ev[kComp][b], 0));
      PPA_CUDA(cudaMemcpyAsync(din[b], X + static_cast<size_t>(i) * n, bytes,
                               cudaMemcpyHostToDevice, hin));
      PPA_CUDA(cudaEventRecord(ev[kIn][b], hin));
      PPA_CUDA(cudaStreamWaitEvent(cs, ev[kIn][b], 0));
      if (i >= 2) PPA_CUDA(cudaStreamWaitEvent(cs, ev[kOut][b], 0));
      op->p->apply(din[b], dout[b], r);
      PPA_CUDA(cudaEventRecord(ev[kComp][b], cs));
      PPA_CUDA(cudaStreamWaitEvent(hout, ev[kComp][b], 0));
      PPA_CUDA(cudaMemcpyAsync(Y + static_cast<size_t>(i) * n, dout[b], bytes,
                               cudaMemcpyDeviceToHost, hout));
      PPA_CUDA(cudaEventRecord(ev[kOut][b], hout));
    }
    PPA_CUDA(cudaStreamSynchronize(hin));
    PPA_CUDA(cudaStreamSynchronize(hout));
    // the scratch buffers are released on `cs`: order that after the copies
    PPA_CUDA(cudaEventRecord(ready, hout));
    PPA_CUDA(cudaStreamWaitEvent(cs, ready, 0));
    ctx.sync();
    for (auto& row : ev)
      for (auto& e : row) cudaEventDestroy(e);
    cudaEventDestroy(ready);
    add_cost(cost, r);
  });
}

int ppa_csr_model_bytes(const ppa_op* op, double* bytes, long long* nnz) {
  return guard([&] {
    need(op, "ppa_csr_model_bytes");
    const auto* c = dynamic_cast<const ppa::CsrOperator*>(op->p.get());
    if (!c) throw std::invalid_argument("ppa_csr_model_bytes: not a CSR operator");
    if (bytes) *bytes = c->model_bytes();
    if (nnz) *nnz = c->nnz();
  });
}

int ppa_csr_layout(const ppa_op* op, int* layout, double* stream_bytes, int* sigma,
                   int* dict_size) {
  return guard([&] {
    need(op, "ppa_csr_layout");
    const auto* c = dynamic_cast<const ppa::CsrOperator*>(op->p.get());
    if (!c) throw std::invalid_argument("ppa_csr_layout: not a CSR operator");
    if (layout) *layout = c->uses_dia() ? 3 : c->uses_packed() ? 2 : c->uses_sell() ? 1 : 0;
    if (stream_bytes) *stream_bytes = c->stream_bytes();
    if (sigma) *sigma = c->uses_sell() ? c->sell_sigma() : 0;
    if (dict_size) *dict_size = c->uses_dia() ? c->device().dia_ndict : c->device().pk_ndict;
  });
}

int ppa_csr_two_factor_pass(const ppa_op* op, int* supported) {
  return guard([&] {
    need(op, "ppa_csr_two_factor_pass");
    need(supported, "ppa_csr_two_factor_pass");
    const auto* c = dynamic_cast<const ppa::CsrOperator*>(op->p.get());
    if (!c) throw std::invalid_argument("ppa_csr_two_factor_pass: not a CSR operator");
    *supported = ppa::kern::dia2_supported(c->device()) ? 1 : 0;
  });
}

int ppa_csr_grid_form(const ppa_op* op, int* nx, int* ny, int* nz, int* supported) {
  return guard([&] {
    need(op, "ppa_csr_grid_form");
    const auto* c = dynamic_cast<const ppa::CsrOperator*>(op->p.get());
    if (!c) throw std::invalid_argument("ppa_csr_grid_form: not a CSR operator");
    const ppa::kern::CsrDevice& d = c->device();
    if (nx) *nx = d.grid_nx;
    if (ny) *ny = d.grid_ny;
    if (nz) *nz = d.grid_nz;
    if (supported) *supported = ppa::kern::grid2_supported(d) ? 1 : 0;
  });
}

int ppa_csr_grid_work(const ppa_op* op, long long* l1_rows, long long* l2_rows) {
  return guard([&] {
    need(op, "ppa_csr_grid_work");
    need(l1_rows, "ppa_csr_grid_work");
    need(l2_rows, "ppa_csr_grid_work");
    const auto* c = dynamic_cast<const ppa::CsrOperator*>(op->p.get());
    if (!c) throw std::invalid_argument("ppa_csr_grid_work: not a CSR operator");
    ppa::kern::grid2_row_evals(c->device(), l1_rows, l2_rows);
  });
}

int ppa_apply_poly(const double* re, const double* im, int nroots, const ppa_op* a,
                   const double* v, double* out, ppa_cost* cost) {
  return guard([&] {
    need(a, "ppa_apply_poly");
    ppa::PolyPrecond p = poly_of(re, im, nroots, nroots);
    ppa::CostRecord r;
    ppa::apply_poly(p, *a->p, v, out, r);
    add_cost(cost, r);
  });
}

int ppa_build_gmres_poly_ortho(const ppa_op* a, const double* b, int degree, int ortho,
                               double* re, double* im, int* nroots, int* truncated,
                               ppa_cost* cost) {
  return guard([&] {
    need(a, "ppa_build_gmres_poly");
    need(re, "ppa_build_gmres_poly");
    need(im, "ppa_build_gmres_poly");
    if (ortho != PPA_ORTHO_CGS2 && ortho != PPA_ORTHO_DCGS2) {
      throw std::invalid_argument("build_gmres_poly: orthogonalization must be 0 or 1");
    }
    ppa::CostRecord r;
    const ppa::PolyPrecond p =
        ppa::build_gmres_poly(*a->p, b, degree, r, static_cast<ppa::Orthogonalization>(ortho));
    for (size_t i = 0; i < p.roots.size(); ++i) {
      re[i] = p.roots[i].real();
      im[i] = p.roots[i].imag();
    }
    if (nroots) *nroots = p.effective_degree();
    if (truncated) *truncated = p.truncated ? 1 : 0;
    add_cost(cost, r);
  });
}

int ppa_build_gmres_poly(const ppa_op* a, const double* b, int degree, double* re, double* im,
                         int* nroots, int* truncated, ppa_cost* cost) {
  return ppa_build_gmres_poly_ortho(a, b, degree, PPA_ORTHO_DCGS2, re, im, nroots, truncated,
                                    cost);
}

int ppa_leja_order(const double* re, const double* im, int n, double* out_re, double* out_im) {
  return guard([&] {
    need(out_re, "ppa_leja_order");
    need(out_im, "ppa_leja_order");
    const auto o = ppa::leja_order(roots_of(re, im, n));
    for (size_t i = 0; i < o.size(); ++i) {
      out_re[i] = o[i].real();
      out_im[i] = o[i].imag();
    }
  });
}

int ppa_compute_pof(const double* re, const double* im, int n, double* log10_pof, int* copies,
                    int* ndistinct, double* max_log10, int* total) {
  return guard([&] {
    const ppa::PofReport rep = ppa::compute_pof(poly_of(re, im, n, n));
    for (size_t i = 0; i < rep.log10_pof.size(); ++i) {
      if (log10_pof) log10_pof[i] = rep.log10_pof[i];
      if (copies) copies[i] = rep.copies_needed[i];
    }
    if (ndistinct) *ndistinct = static_cast<int>(rep.log10_pof.size());
    if (max_log10) *max_log10 = rep.max_log10_pof;
    if (total) *total = rep.total_copies;
  });
}

int ppa_add_stability_roots(const double* re, const double* im, int n, int base_degree,
                            int max_copies, int cap, double* out_re, double* out_im,
                            int* out_n) {
  return guard([&] {
    need(out_re, "ppa_add_stability_roots");
    need(out_im, "ppa_add_stability_roots");
    const ppa::PolyPrecond p =
        ppa::add_stability_roots(poly_of(re, im, n, base_degree), max_copies);
    if (static_cast<int>(p.roots.size()) > cap) {
      throw std::invalid_argument("ppa_add_stability_roots: output capacity too small");
    }
    for (size_t i = 0; i < p.roots.size(); ++i) {
      out_re[i] = p.roots[i].real();
      out_im[i] = p.roots[i].imag();
    }
    if (out_n) *out_n = p.effective_degree();
  });
}

int ppa_eval_poly(const double* re, const double* im, int n, double zr, double zi, double* o_re,
                  double* o_im) {
  return guard([&] {
    const std::complex<double> v = ppa::eval_poly(poly_of(re, im, n, n), {zr, zi});
    if (o_re) *o_re = v.real();
    if (o_im) *o_im = v.imag();
  });
}

int ppa_arnoldi_init(const double* v0, int n, int m, ppa_cost* cost, ppa_arnoldi** out) {
  return guard([&] {
    need(out, "ppa_arnoldi_init");
    need(v0, "ppa_arnoldi_init");
    ppa::CostRecord r;
    auto* st = new ppa_arnoldi;
    try {
      st->s = ppa::arnoldi_init(v0, n, m, r);
    } catch (...) {
      delete st;
      throw;
    }
    *out = st;
    add_cost(cost, r);
  });
}

int ppa_arnoldi_extend(ppa_arnoldi* st, const ppa_op* op, int to_dim, ppa_cost* cost) {
  return guard([&] {
    need(st, "ppa_arnoldi_extend");
    need(op, "ppa_arnoldi_extend");
    ppa::CostRecord r;
    try {
      ppa::arnoldi_extend(st->s, *op->p, to_dim, r);
    } catch (...) {
      add_cost(cost, r);
      throw;
    }
    add_cost(cost, r);
  });
}

int ppa_arnoldi_set_orthogonalization(ppa_arnoldi* st, int mode) {
  return guard([&] {
    need(st, "ppa_arnoldi_set_orthogonalization");
    if (mode < 0 || mode > 1) throw std::invalid_argument("orthogonalization must be 0 or 1");
    st->s.ortho = static_cast<ppa::Orthogonalization>(mode);
  });
}

int ppa_arnoldi_info(const ppa_arnoldi* st, int* cur, int* maxd, int* bd, long long* ld,
                     double** V) {
  return guard([&] {
    need(st, "ppa_arnoldi_info");
    if (cur) *cur = st->s.cur_dim;
    if (maxd) *maxd = st->s.max_dim;
    if (bd) *bd = st->s.breakdown ? 1 : 0;
    if (ld) *ld = st->s.ld;
    if (V) *V = st->s.V.get();
  });
}

int ppa_arnoldi_get_H(const ppa_arnoldi* st, double* H) {
  return guard([&] {
    need(st, "ppa_arnoldi_get_H");
    need(H, "ppa_arnoldi_get_H");
    std::memcpy(H, st->s.H.data(), st->s.H.size() * sizeof(double));
  });
}

int ppa_arnoldi_ritz(const ppa_arnoldi* st, int ordering, double* re, double* im,
                     double* resid) {
  return guard([&] {
    need(st, "ppa_arnoldi_ritz");
    const ppa::RitzSet s = ppa::ritz_pairs(st->s, static_cast<ppa::RitzOrdering>(ordering));
    for (int i = 0; i < s.count(); ++i) {
      if (re) re[i] = s.values[i].real();
      if (im) im[i] = s.values[i].imag();
      if (resid) resid[i] = s.residuals[i];
    }
  });
}

int ppa_arnoldi_harmonic(const ppa_arnoldi* st, double* re, double* im) {
  return guard([&] {
    need(st, "ppa_arnoldi_harmonic");
    const auto v = ppa::harmonic_ritz_values(st->s);
    for (size_t i = 0; i < v.size(); ++i) {
      if (re) re[i] = v[i].real();
      if (im) im[i] = v[i].imag();
    }
  });
}

int ppa_arnoldi_ritz_vector(const ppa_arnoldi* st, int ordering, int j, double* yr, double* yi,
                            int* is_complex, ppa_cost* cost) {
  return guard([&] {
    need(st, "ppa_arnoldi_ritz_vector");
    need(yr, "ppa_arnoldi_ritz_vector");
    const ppa::RitzSet s = ppa::ritz_pairs(st->s, static_cast<ppa::RitzOrdering>(ordering));
    ppa::CostRecord r;
    ppa::DeviceComplexVector y = ppa::ritz_vector(st->s, s, j, r);
    const cudaStream_t str = ppa::current_context().stream();
    ppa::kern::copy(y.re.get(), yr, st->s.n, str);
    if (y.complex && yi) ppa::kern::copy(y.im.get(), yi, st->s.n, str);
    ppa::current_context().sync();
    if (is_complex) *is_complex = y.complex ? 1 : 0;
    add_cost(cost, r);
  });
}

namespace {
void ritz_out(const ppa::RitzSet& s, double* re, double* im, double* resid, double* vre,
              double* vim) {
  const int d = s.vectors_h.rows;
  for (int i = 0; i < s.count(); ++i) {
    if (re) re[i] = s.values[i].real();
    if (im) im[i] = s.values[i].imag();
    if (resid) resid[i] = s.residuals[i];
    for (int r = 0; r < d; ++r) {
      if (vre) vre[static_cast<size_t>(i) * d + r] = s.vectors_h(r, i).real();
      if (vim) vim[static_cast<size_t>(i) * d + r] = s.vectors_h(r, i).imag();
    }
  }
}
}  // namespace

int ppa_arnoldi_ritz_vectors(const ppa_arnoldi* st, int ordering, double* re, double* im,
                             double* resid, double* vec_re, double* vec_im) {
  return guard([&] {
    need(st, "ppa_arnoldi_ritz_vectors");
    ritz_out(ppa::ritz_pairs(st->s, static_cast<ppa::RitzOrdering>(ordering)), re, im, resid,
             vec_re, vec_im);
  });
}

int ppa_arnoldi_harmonic_selection(const ppa_arnoldi* st, int ordering, double* re, double* im,
                                   double* resid, double* vec_re, double* vec_im) {
  return guard([&] {
    need(st, "ppa_arnoldi_harmonic_selection");
    ritz_out(ppa::harmonic_restart_selection(st->s, static_cast<ppa::RitzOrdering>(ordering)),
             re, im, resid, vec_re, vec_im);
  });
}

int ppa_arnoldi_restart_keep(ppa_arnoldi* st, int count, const double* re, const double* im,
                             const double* vec_re, const double* vec_im, int k, ppa_cost* cost,
                             int* kk) {
  return guard([&] {
    need(st, "ppa_arnoldi_restart_keep");
    need(re, "ppa_arnoldi_restart_keep");
    need(vec_re, "ppa_arnoldi_restart_keep");
    if (count < 0) throw std::invalid_argument("thick_restart: selection smaller than k");
    const int d = st->s.cur_dim;
    ppa::RitzSet s;
    s.values.resize(count);
    s.residuals.assign(count, 0.0);
    s.vectors_h = ppa::dense::CMat(d, count);
    for (int i = 0; i < count; ++i) {
      s.values[i] = {re[i], im ? im[i] : 0.0};
      for (int r = 0; r < d; ++r) {
        const size_t at = static_cast<size_t>(i) * d + r;
        s.vectors_h(r, i) = {vec_re[at], vec_im ? vec_im[at] : 0.0};
      }
    }
    ppa::CostRecord r;
    const int got = ppa::thick_restart(st->s, s, k, r);
    if (kk) *kk = got;
    add_cost(cost, r);
  });
}

int ppa_arnoldi_restart(ppa_arnoldi* st, int ordering, int k, ppa_cost* cost, int* kk) {
  return guard([&] {
    need(st, "ppa_arnoldi_restart");
    const ppa::RitzSet s = ppa::ritz_pairs(st->s, static_cast<ppa::RitzOrdering>(ordering));
    ppa::CostRecord r;
    const int got = ppa::thick_restart(st->s, s, k, r);
    if (kk) *kk = got;
    add_cost(cost, r);
  });
}

void ppa_arnoldi_free(ppa_arnoldi* st) { delete st; }

int ppa_spmv(const ppa_op* a, const double* x, double* y) {
  return guard([&] {
    need(a, "ppa_spmv");
    const auto* c = dynamic_cast<const ppa::CsrOperator*>(a->p.get());
    if (!c) throw std::invalid_argument("ppa_spmv: not a CSR operator");
    ppa::kern::spmv(c->device(), x, y, ppa::kern::EpiArgs{}, ppa::current_context().stream());
  });
}

int ppa_spmv_factor(const ppa_op* a, const double* x, double* y, int mode, double c0, double c1,
                    const double* o, const double* base) {
  return guard([&] {
    need(a, "ppa_spmv_factor");
    const auto* c = dynamic_cast<const ppa::CsrOperator*>(a->p.get());
    if (!c) throw std::invalid_argument("ppa_spmv_factor: not a CSR operator");
    if (mode < 0 || mode > 2) throw std::invalid_argument("ppa_spmv_factor: mode");
    if (mode == 2 && !o) throw std::invalid_argument("ppa_spmv_factor: pair needs o");
    if (x == y) throw std::invalid_argument("ppa_spmv_factor: x and y alias");
    ppa::kern::EpiArgs ep;
    ep.mode = static_cast<ppa::kern::Epi>(mode);
    ep.c0 = c0;
    ep.c1 = c1;
    ep.o = o;
    ep.base = base;
    ppa::kern::spmv(c->device(), x, y, ep, ppa::current_context().stream());
  });
}

int ppa_factor_plan(const double* re, const double* im, int nroots, int* pair, double* c0,
                    double* c1, int* nfactors) {
  return guard([&] {
    need(nfactors, "ppa_factor_plan");
    const std::vector<ppa::PolyFactor> plan = ppa::factor_plan(poly_of(re, im, nroots, nroots));
    for (size_t i = 0; i < plan.size(); ++i) {
      if (pair) pair[i] = plan[i].pair ? 1 : 0;
      if (c0) c0[i] = plan[i].c0;
      if (c1) c1[i] = plan[i].c1;
    }
    *nfactors = static_cast<int>(plan.size());
  });
}

int ppa_spmm(const ppa_op* a, const double* Y, long long ldy, int p, double* AY, long long ldo) {
  return guard([&] {
    need(a, "ppa_spmm");
    const auto* c = dynamic_cast<const ppa::CsrOperator*>(a->p.get());
    if (!c) throw std::invalid_argument("ppa_spmm: not a CSR operator");
    ppa::kern::spmm(c->device(), Y, ldy, p, AY, ldo, ppa::current_context().stream());
  });
}

int ppa_cgs2_step(double* V, long long ld, int n, int c, double* w, double* Hcol, int* flag) {
  return guard([&] {
    ppa::Context& ctx = ppa::current_context();
    ppa::kern::cgs2_step(V, ld, n, c, w, Hcol, flag, ctx.ws(), ctx.sm_count(), ctx.stream());
  });
}

int ppa_dev_alloc(size_t bytes, void** out) {
  return guard([&] {
    need(out, "ppa_dev_alloc");
    void* p = nullptr;
    PPA_CUDA(cudaMalloc(&p, bytes ? bytes : 16));
    PPA_CUDA(cudaMemset(p, 0, bytes ? bytes : 16));
    *out = p;
  });
}

int ppa_dev_free(void* p) {
  return guard([&] {
    if (p) PPA_CUDA(cudaFree(p));
  });
}

int ppa_ipc_get_handle(const void* dev_ptr, unsigned char* handle) {
  return guard([&] {
    need(dev_ptr, "ppa_ipc_get_handle");
    need(handle, "ppa_ipc_get_handle");
    cudaIpcMemHandle_t h;
    PPA_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
    static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
    std::memcpy(handle, &h, sizeof(h));
  });
}

int ppa_ipc_open(const unsigned char* handle, void** peer_ptr) {
  return guard([&] {
    need(handle, "ppa_ipc_open");
    need(peer_ptr, "ppa_ipc_open");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    PPA_CUDA(cudaIpcOpenMemHandle(peer_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

int ppa_ipc_close(void* peer_ptr) {
  return guard([&] {
    if (peer_ptr) PPA_CUDA(cudaIpcCloseMemHandle(peer_ptr));
  });
}

int ppa_halo_publish(long long* flag_dev, long long epoch) {
  return guard([&] {
    need(flag_dev, "ppa_halo_publish");
    ppa::kern::publish(flag_dev, epoch, ppa::current_context().stream());
  });
}

int ppa_halo_pull(const ppa_peer_halo* peers_dev, int npeers, long long max_count,
                  double* x_ext_dev, long long epoch, int* error_dev) {
  return guard([&] {
    if (npeers <= 0) return;
    need(peers_dev, "ppa_halo_pull");
    need(error_dev, "ppa_halo_pull");
    static_assert(sizeof(ppa_peer_halo) == sizeof(ppa::kern::PeerHaloDesc), "layout");
    ppa::kern::halo_pull(reinterpret_cast<const ppa::kern::PeerHaloDesc*>(peers_dev), npeers,
                         max_count, x_ext_dev, epoch, error_dev,
                         ppa::current_context().stream());
  });
}

int ppa_grid2_slab_pass(int nd, int nx, int ny, int nz, const double* vals, int zo0, int zo1,
                        int kind, double a0, double a1, double b0, const double* x, double* y,
                        const double* xl, int zl0, const long long* fl, const double* xr,
                        const long long* fr, long long epoch, int* err, long long* own) {
  return guard([&] {
    need(vals, "ppa_grid2_slab_pass");
    need(x, "ppa_grid2_slab_pass");
    need(y, "ppa_grid2_slab_pass");
    if (x == y) throw std::invalid_argument("ppa_grid2_slab_pass: x and y must differ");
    if (kind < 0 || kind > 2) throw std::invalid_argument("ppa_grid2_slab_pass: kind must be 0, 1 or 2");
    ppa::kern::spmv_grid2_slab_check(nd, nx, ny, nz, zo0, zo1, xl, zl0, fl, xr, fr);
    ppa::kern::Mp2Pass m;
    m.pair = kind == 1;
    m.one = kind == 2;
    m.a0 = a0;
    m.a1 = a1;
    m.b0 = b0;
    ppa::kern::spmv_grid2_slab(nd, nx, ny, nz, vals, zo0, zo1, m, x, y, xl, zl0, fl, xr, fr, epoch,
                               err, own, ppa::current_context().stream());
  });
}

int ppa_grid2_slab_chain(int nd, int nx, int ny, int nz, const double* vals, int zo0, int zo1,
                         int npass, const int* kinds, const double* a0, const double* a1,
                         const double* b0, double* buf0, double* buf1, const double* xl0,
                         const double* xl1, int zl0, const long long* fl, const double* xr0,
                         const double* xr1, const long long* fr, long long epoch0, int* err,
                         long long* own, int* out_role) {
  return guard([&] {
    need(vals, "ppa_grid2_slab_chain");
    need(buf0, "ppa_grid2_slab_chain");
    need(buf1, "ppa_grid2_slab_chain");
    need(out_role, "ppa_grid2_slab_chain");
    if (npass < 0) throw std::invalid_argument("ppa_grid2_slab_chain: negative pass count");
    if (npass > 0) {
      need(kinds, "ppa_grid2_slab_chain");
      need(a0, "ppa_grid2_slab_chain");
      need(a1, "ppa_grid2_slab_chain");
      need(b0, "ppa_grid2_slab_chain");
    }
    double* buf[2] = {buf0, buf1};
    const double* xl[2] = {xl0, xl1};
    const double* xr[2] = {xr0, xr1};
    for (int k = 0; k < npass; ++k) {
      if (kinds[k] < 0 || kinds[k] > 2) {
        throw std::invalid_argument("ppa_grid2_slab_chain: kind must be 0, 1 or 2");
      }
    }
    ppa::kern::spmv_grid2_slab_check(nd, nx, ny, nz, zo0, zo1, xl0, zl0, fl, xr0, fr);
    if ((zo0 > 0 && !xl1) || (zo1 < nz && !xr1)) {
      throw std::invalid_argument("ppa_grid2_slab_chain: missing neighbour buffer (role 1)");
    }
    const cudaStream_t st = ppa::current_context().stream();
    for (int k = 0; k < npass; ++k) {
      ppa::kern::Mp2Pass m;
      m.pair = kinds[k] == 1;
      m.one = kinds[k] == 2;
      m.a0 = a0[k];
      m.a1 = a1[k];
      m.b0 = b0[k];
      const int r = k & 1;
      ppa::kern::spmv_grid2_slab(nd, nx, ny, nz, vals, zo0, zo1, m, buf[r], buf[r ^ 1], xl[r], zl0,
                                 fl, xr[r], fr, epoch0 + k, err, own, st);
    }
    *out_role = npass & 1;
  });
}

int ppa_cgs_dot_local(const double* V, long long ld, int n, int c, const double* w,
                      double* out) {
  return guard([&] {
    need(V, "ppa_cgs_dot_local");
    ppa::Context& ctx = ppa::current_context();
    ppa::kern::ts_dot(V, ld, n, c, w, out, ctx.ws(), ctx.sm_count(), ctx.stream());
  });
}

int ppa_cgs_update_dot_local(const double* V, long long ld, int n, int c, double* w,
                             const double* h, double* out) {
  return guard([&] {
    need(V, "ppa_cgs_update_dot_local");
    ppa::Context& ctx = ppa::current_context();
    ppa::kern::cgs_update_dot_local(V, ld, n, c, w, h, out, ctx.ws(), ctx.sm_count(),
                                    ctx.stream());
  });
}

int ppa_cgs_store_local(double* V, long long ld, int n, int c, const double* w, const double* h2,
                        const double* hsub) {
  return guard([&] {
    need(V, "ppa_cgs_store_local");
    need(hsub, "ppa_cgs_store_local");
    ppa::Context& ctx = ppa::current_context();
    ppa::kern::cgs_store_local(V, ld, n, c, w, h2, hsub, ctx.ws(), ctx.sm_count(), ctx.stream());
  });
}

int ppa_dot_local(const double* x, const double* y, long long n, double* out) {
  return guard([&] {
    need(out, "ppa_dot_local");
    ppa::Context& ctx = ppa::current_context();
    ppa::kern::dot(x, y, n, out, ctx.ws(), ctx.sm_count(), ctx.stream());
  });
}

int ppa_ts_combine(const double* V, long long ldv, int n, int d, const double* G, int p,
                   double* Out, long long ldo) {
  return guard([&] {
    ppa::kern::ts_combine(V, ldv, n, d, G, p, Out, ldo, ppa::current_context().stream());
  });
}

int ppa_solve_config_default(ppa_solve_config* c) {
  return guard([&] {
    need(c, "ppa_solve_config_default");
    const ppa::SolveConfig d;
    *c = ppa_solve_config{};
    c->m = d.m;
    c->k = d.k;
    c->nev = d.nev;
    c->degree = d.degree;
    c->rtol_multiplier = d.rtol_multiplier;
    c->rtol_absolute = 0.0;
    c->variant = 0;
    c->stability = 0;
    c->max_cycles = d.max_cycles;
    c->seed = d.seed;
    c->damping_alpha = d.damping_alpha;
    c->damping_power = d.damping_power;
    c->check_mid_cycle = d.check_mid_cycle ? 1 : 0;
    c->mid_cycle_stride = d.mid_cycle_stride;
    c->stagnation_stop = d.stagnation_stop ? 1 : 0;
    c->stagnation_window = d.stagnation_window;
    c->stagnation_rtol = d.stagnation_rtol;
    c->want_eigenvectors = d.want_eigenvectors ? 1 : 0;
    c->orthogonalization = static_cast<int>(d.orthogonalization);
  });
}

int ppa_solve(const ppa_op* a, const ppa_solve_config* c, ppa_solve_result* res) {
  return guard([&] {
    need(a, "ppa_solve");
    need(c, "ppa_solve");
    need(res, "ppa_solve");
    const ppa::SolveConfig cfg = to_config(*c);
    const ppa::EigResult r = c->use_double ? ppa::solve_double(a->p, cfg) : ppa::solve(a->p, cfg);
    res->discarded_probes = 0;
    for (const ppa::CycleStats& h : r.history) res->discarded_probes += h.discarded_probe ? 1 : 0;
    res->n_eig = static_cast<int>(r.eigenvalues.size());
    for (int i = 0; i < res->n_eig && i < res->cap_nev; ++i) {
      if (res->eig_re) res->eig_re[i] = r.eigenvalues[i].real();
      if (res->eig_im) res->eig_im[i] = r.eigenvalues[i].imag();
      if (res->residuals) res->residuals[i] = r.residuals[i];
      if (res->converged_flags) res->converged_flags[i] = r.converged_flags[i] ? 1 : 0;
    }
    res->n_poly = r.poly ? r.poly->effective_degree() : 0;
    res->poly_base_degree = r.poly ? r.poly->base_degree : 0;
    for (int i = 0; i < res->n_poly && i < res->cap_roots; ++i) {
      if (res->poly_re) res->poly_re[i] = r.poly->roots[i].real();
      if (res->poly_im) res->poly_im[i] = r.poly->roots[i].imag();
    }
    res->n_inner = r.inner_poly ? r.inner_poly->effective_degree() : 0;
    for (int i = 0; i < res->n_inner && i < res->cap_roots; ++i) {
      if (res->inner_re) res->inner_re[i] = r.inner_poly->roots[i].real();
      if (res->inner_im) res->inner_im[i] = r.inner_poly->roots[i].imag();
    }
    res->n_cycles = static_cast<int>(r.history.size());
    for (int i = 0; i < res->n_cycles && i < res->cap_cycles; ++i) {
      if (res->cycle_max_residual) res->cycle_max_residual[i] = r.history[i].max_residual;
    }
    if (r.eigenvectors.get() && (res->evec_re || res->evec_im)) {
      const int ne = std::min<int>(res->n_eig, res->cap_nev);
      const long long n = a->p->dim();
      if (res->evec_ld < n) throw std::invalid_argument("ppa_solve: evec_ld < n");
      for (int j = 0; j < ne && 2LL * j + 1 < static_cast<long long>(r.eigenvectors.size() / r.eigvec_ld); ++j) {
        const double* col = r.eigenvectors.get() + 2LL * j * r.eigvec_ld;
        if (res->evec_re)
          PPA_CUDA(cudaMemcpy(res->evec_re + j * res->evec_ld, col, n * sizeof(double),
                              cudaMemcpyDeviceToHost));
        if (res->evec_im)
          PPA_CUDA(cudaMemcpy(res->evec_im + j * res->evec_ld, col + r.eigvec_ld,
                              n * sizeof(double), cudaMemcpyDeviceToHost));
      }
    }
    res->converged = r.converged ? 1 : 0;
    res->cycles = r.cycles;
    res->composite_degree = r.composite_degree;
    res->rtol = r.rtol;
    res->max_err = r.max_err;
    res->norm_estimate = r.norm_estimate;
    res->cost = ppa_cost{r.cost.mvps, r.cost.dots, r.cost.vops, r.cost.nnzr, r.cost.wall_seconds};
    res->t_total = r.timing.total;
    res->t_setup = r.timing.setup;
    res->t_extend = r.timing.extend;
    res->t_check = r.timing.check;
    res->t_restart = r.timing.restart;
  });
}

int ppa_check_ideal_order(const double* re, const double* im, int count, int nev, int* holds) {
  return guard([&] {
    need(holds, "ppa_check_ideal_order");
    *holds = ppa::check_ideal_order(roots_of(re, im, count), nev) ? 1 : 0;
  });
}

int ppa_damping_heuristic(const ppa_op* a, const ppa_solve_config* c, double* re, double* im,
                          int cap, int* nroots, ppa_cost* cost) {
  return guard([&] {
    need(a, "ppa_damping_heuristic");
    need(c, "ppa_damping_heuristic");
    ppa::CostRecord r;
    const ppa::PolyPrecond p = ppa::damping_heuristic(a->p, to_config(*c), r);
    roots_out(p, re, im, cap, nroots);
    add_cost(cost, r);
  });
}

int ppa_block2_operator(const ppa_op* a, ppa_op** out) {
  return guard([&] {
    need(a, "ppa_block2_operator");
    need(out, "ppa_block2_operator");
    *out = wrap_op(ppa::make_block2(a->p));
  });
}

int ppa_shifted_operator(const ppa_op* a, double mu, ppa_op** out) {
  return guard([&] {
    need(a, "ppa_shifted_operator");
    need(out, "ppa_shifted_operator");
    *out = wrap_op(ppa::make_shifted(a->p, mu));
  });
}

int ppa_build_two_vector_poly(const ppa_op* a, const double* b1, const double* b2, int degree,
                              double* re, double* im, int* nroots, ppa_cost* cost) {
  return guard([&] {
    need(a, "ppa_build_two_vector_poly");
    ppa::CostRecord r;
    const ppa::PolyPrecond p = ppa::build_two_vector_poly(a->p, b1, b2, degree, r);
    roots_out(p, re, im, std::max(degree, 1), nroots);
    add_cost(cost, r);
  });
}

int ppa_damped_start(const ppa_op* a, const double* b, double alpha, int power, double* out,
                     ppa_cost* cost) {
  return guard([&] {
    need(a, "ppa_damped_start");
    ppa::CostRecord r;
    ppa::damped_start(*a->p, b, alpha, power, out, r);
    add_cost(cost, r);
  });
}

int ppa_read_matrix_market(const char* path, ppa_host_csr** out) {
  return guard([&] {
    need(path, "ppa_read_matrix_market");
    need(out, "ppa_read_matrix_market");
    *out = wrap(ppa::read_matrix_market(path));
  });
}

}  // extern "C"
