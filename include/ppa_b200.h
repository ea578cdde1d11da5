/*
 * ppa_b200.h - C-ABI of the B200-native polynomial-preconditioned Arnoldi
 * hot path (libppa_b200.so).
 *
 * The reference (arxiv/paper_1806_08020, /root/reference/proj) is a C++/Eigen
 * library with no foreign-function layer; these entry points are what a
 * binding to its hot path would expose.  Each one names the reference
 * interface it replaces (file:line under /root/reference/proj).
 *
 * Conventions
 *  - Every function returns a status (PPA_OK = 0); on failure
 *    ppa_last_error() returns the thread-local message, worded as the
 *    reference's exception text.  No C++ exception crosses the ABI.
 *      PPA_INVALID_ARGUMENT  <- std::invalid_argument
 *      PPA_RUNTIME_ERROR     <- std::runtime_error
 *      PPA_LOGIC_ERROR       <- std::logic_error (malformed root list)
 *      PPA_CUDA_ERROR        <- CUDA failure
 *  - "_dev" pointers are device pointers (HBM); everything else is host.
 *  - Kernels run on the calling thread's stream (ppa_set_stream; default
 *    stream otherwise).  Calls that return host results synchronise it.
 *  - ppa_cost mirrors CostRecord (inc/cost.hpp:17-23); calls add the
 *    reference's counter increments to *cost (may be NULL).
 */
#ifndef PPA_B200_H
#define PPA_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PPA_OK = 0,
  PPA_INVALID_ARGUMENT = 1,
  PPA_RUNTIME_ERROR = 2,
  PPA_LOGIC_ERROR = 3,
  PPA_CUDA_ERROR = 4,
  PPA_INTERNAL_ERROR = 5
};

/* OperatorKind (inc/operators.hpp:43) */
enum { PPA_KIND_CSR = 0, PPA_KIND_DIAGONAL = 1, PPA_KIND_SHIFTED = 2, PPA_KIND_BLOCK2 = 3,
       PPA_KIND_POLY = 4, PPA_KIND_COMPOSITE = 5,
       PPA_KIND_EXTERNAL = 6 /* ours: ppa_op_create_callback */ };
/* Orthogonalization of the device Arnoldi (ours).  The C++
   and Python SolveConfig default is PPA_ORTHO_DCGS2; a zero-filled
   ppa_solve_config is not a default configuration (m = 0 is invalid), use
   ppa_solve_config_default. */
enum { PPA_ORTHO_CGS2 = 0, PPA_ORTHO_DCGS2 = 1 };
/* RitzOrdering (inc/arnoldi.hpp:40) */
enum { PPA_SMALLEST_MAGNITUDE = 0, PPA_LARGEST_MAGNITUDE = 1, PPA_TARGET_ONE = 2 };

typedef struct ppa_cost {
  long long mvps;
  long long dots;
  long long vops;
  double nnzr;
  double wall_seconds;
} ppa_cost;

typedef struct ppa_host_csr ppa_host_csr; /* CsrMatrix (inc/operators.hpp:15-33) */
typedef struct ppa_op ppa_op;             /* OperatorPtr (inc/operators.hpp:78) */
typedef struct ppa_arnoldi ppa_arnoldi;   /* ArnoldiState (inc/arnoldi.hpp:18-26) */

const char* ppa_last_error(void);
int ppa_abi_version(void);
int ppa_device_info(int* sm_count, double* l2_bytes);
int ppa_set_stream(void* cuda_stream);
int ppa_synchronize(void);

/* ---- host CSR and generators ------------------------------------------ */
/* CsrMatrix + validate() (src/operators.cpp:12-37) */
int ppa_host_csr_create(int n, long long nnz, const int* row_ptr, const int* col_idx,
                        const double* values, ppa_host_csr** out);
/* CsrMatrix::from_triplets (src/operators.cpp:50-78) */
int ppa_host_csr_from_triplets(int n, long long count, const int* rows, const int* cols,
                               const double* vals, ppa_host_csr** out);
/* make_convection_diffusion (src/operators.cpp:190-244) */
int ppa_gen_convdiff_ref(int grid_n, ppa_host_csr** out);
/* BASELINE.json configs 1..5 and their parametric generators */
int ppa_gen_config(int config, ppa_host_csr** out);
int ppa_gen_bidiagonal(int n, ppa_host_csr** out);
int ppa_gen_convdiff_const(int grid_n, double peclet, ppa_host_csr** out);
int ppa_gen_laplacian_3d(int grid_n, ppa_host_csr** out);
int ppa_gen_random_poisson(int n, double lambda, unsigned long long seed, ppa_host_csr** out);
int ppa_host_csr_info(const ppa_host_csr* m, int* n, long long* nnz,
                      unsigned long long* fingerprint);
int ppa_host_csr_arrays(const ppa_host_csr* m, const int** row_ptr, const int** col_idx,
                        const double** values);
void ppa_host_csr_free(ppa_host_csr* m);
/* CsrMatrix::multiply (inc/operators.hpp:27-28): y = A x, uncounted, device
   vectors (a device copy of the matrix is built per call) */
int ppa_host_csr_multiply(const ppa_host_csr* m, const double* x_dev, double* y_dev);
/* Seeded N(0,1) vector (host), stream ids as in DESIGN.md */
int ppa_normal_vector(long long n, unsigned long long seed, unsigned long long stream,
                      double* out);

/* ---- operators --------------------------------------------------------- */
/* make_csr_operator (inc/operators.hpp:83): validates, uploads to HBM */
int ppa_csr_operator(const ppa_host_csr* m, ppa_op** out);
/* make_csr_operator with a device-layout cap: 0 automatic, 1 CSR row blocks,
   2 SELL-32 (fp64 values, int32 columns: the north-star byte model),
   3 packed SELL-32, 4 diagonal-coded.  Results are bit-identical. */
int ppa_csr_operator_layout(const ppa_host_csr* m, int layout, ppa_op** out);
/* make_diagonal (inc/operators.hpp:81) */
int ppa_diagonal_operator(int n, const double* diag, ppa_op** out);
/* make_poly_operator / make_poly_complement_operator (inc/gmres_poly.hpp:91,95) */
int ppa_poly_operator(const ppa_op* base, const double* re, const double* im, int nroots,
                      int base_degree, int complement, ppa_op** out);
/* A caller-defined operator: the reference's plugin mechanism, an abstract
   LinearOperator (inc/operators.hpp:49-76) that arnoldi_extend, build_gmres_poly,
   apply_poly and solve accept whatever its implementation.  apply(ctx, x_dev,
   y_dev, stream) must enqueue y = Op x (device vectors of length dim) on
   `stream` (a cudaStream_t: the library's current stream) and return 0; any
   other value fails the calling entry point with PPA_RUNTIME_ERROR.  Every
   apply charges mvps_per_apply matrix-vector products (mvps_per_apply(),
   inc/operators.hpp:53); nnzr is reported by ppa_op_info.  ctx must outlive
   the operator. */
typedef int (*ppa_apply_fn)(void* ctx, const double* x_dev, double* y_dev, void* cuda_stream);
int ppa_op_create_callback(int dim, int mvps_per_apply, double nnzr, ppa_apply_fn apply,
                           void* ctx, ppa_op** out);
void ppa_op_free(ppa_op* op);
/* dim(), mvps_per_apply(), nnzr(), kind() (inc/operators.hpp:53-68) */
int ppa_op_info(const ppa_op* op, int* dim, int* mvps_per_apply, double* nnzr, int* kind);
/* LinearOperator::apply (inc/operators.hpp:58-59), device vectors */
int ppa_op_apply(const ppa_op* op, const double* x_dev, double* y_dev, ppa_cost* cost);
/* Same with host vectors: H2D of x, apply, D2H of y (the end-to-end call) */
int ppa_op_apply_host(const ppa_op* op, const double* x, double* y, ppa_cost* cost);
/* Batch of `count` host vectors (X, Y: count x dim, vector i at X + i*dim).
   H2D of vector i+1 and D2H of vector i-1 overlap the apply of vector i
   (double-buffered, three streams).  Pinned X/Y give full PCIe bandwidth. */
int ppa_op_apply_host_batch(const ppa_op* op, int count, const double* X, double* Y,
                            ppa_cost* cost);
/* CSR operators: bytes of one SpMV under the north-star byte model */
int ppa_csr_model_bytes(const ppa_op* op, double* bytes, long long* nnz);
/* Device layout of a CSR operator: 0 CSR row blocks, 1 SELL-32, 2 packed
   SELL-32, 3 diagonal-coded; stream_bytes = matrix bytes one SpMV streams in that layout;
   dict_size = value-table size (0: fp64 values) */
int ppa_csr_layout(const ppa_op* op, int* layout, double* stream_bytes, int* sigma,
                   int* dict_size);
/* CSR operators: *supported = 1 when consecutive polynomial factors (two real
   roots, or a conjugate pair) run as one temporally blocked pass over the
   diagonal layout (stencils).  No reference
   counterpart: an introspection hook next to ppa_csr_layout. */
int ppa_csr_two_factor_pass(const ppa_op* op, int* supported);
/* CSR operators: the box-grid form of the two-factor pass (spmv_grid2.cu):
   nx, ny, nz of the 7-point (3-D) or 5-point (2-D, ny = 1) stencil the matrix
   is, or nx = 0; *supported = 1 when that form runs.  Introspection only. */
int ppa_csr_grid_form(const ppa_op* op, int* nx, int* ny, int* nz, int* supported);
/* Row evaluations one box-grid pass performs (the bench's FP64 roofline):
   level 1 over the widened tiles and the chunks' extra planes, level 2 over
   the n rows; both 0 when the form does not run.  Introspection only. */
int ppa_csr_grid_work(const ppa_op* op, long long* l1_rows, long long* l2_rows);

/* ---- polynomial -------------------------------------------------------- */
/* apply_poly (src/gmres_poly.cpp:117-147): out_dev = pi(A) v_dev */
int ppa_apply_poly(const double* re, const double* im, int nroots, const ppa_op* a,
                   const double* v_dev, double* out_dev, ppa_cost* cost);
/* build_gmres_poly (src/gmres_poly.cpp:95-115); re/im capacity >= degree.
   Delayed CGS2 (PPA_ORTHO_DCGS2), the solver's default. */
int ppa_build_gmres_poly(const ppa_op* a, const double* b_dev, int degree, double* re,
                         double* im, int* nroots, int* truncated, ppa_cost* cost);
/* Same with the orthogonalisation chosen (PPA_ORTHO_CGS2 / PPA_ORTHO_DCGS2);
   ppa_solve passes its config's orthogonalization to every polynomial build */
int ppa_build_gmres_poly_ortho(const ppa_op* a, const double* b_dev, int degree, int ortho,
                               double* re, double* im, int* nroots, int* truncated,
                               ppa_cost* cost);
/* leja_order (src/gmres_poly.cpp:38-93) */
int ppa_leja_order(const double* re, const double* im, int n, double* out_re, double* out_im);
/* compute_pof (src/gmres_poly.cpp:155-179); arrays sized >= n */
int ppa_compute_pof(const double* re, const double* im, int n, double* log10_pof, int* copies,
                    int* ndistinct, double* max_log10_pof, int* total_copies);
/* add_stability_roots (src/gmres_poly.cpp:181-226); out capacity `cap` */
int ppa_add_stability_roots(const double* re, const double* im, int n, int base_degree,
                            int max_copies_per_root, int cap, double* out_re, double* out_im,
                            int* out_n);
/* eval_poly (src/gmres_poly.cpp:149-153) */
int ppa_eval_poly(const double* re, const double* im, int n, double z_re, double z_im,
                  double* out_re, double* out_im);

/* ---- Arnoldi ----------------------------------------------------------- */
/* arnoldi_init (src/arnoldi.cpp:99-113) */
int ppa_arnoldi_init(const double* v0_dev, int n, int m, ppa_cost* cost, ppa_arnoldi** out);
/* arnoldi_extend (src/arnoldi.cpp:115-152), CGS2 on device */
int ppa_arnoldi_extend(ppa_arnoldi* st, const ppa_op* op, int to_dim, ppa_cost* cost);
/* orthogonalisation of later extends: 0 CGS2 (default), 1 delayed CGS2 */
int ppa_arnoldi_set_orthogonalization(ppa_arnoldi* st, int mode);
int ppa_arnoldi_info(const ppa_arnoldi* st, int* cur_dim, int* max_dim, int* breakdown,
                     long long* ld, double** V_dev);
/* H, (m+1) x m column-major */
int ppa_arnoldi_get_H(const ppa_arnoldi* st, double* H);
/* ritz_pairs (src/arnoldi.cpp:154-176): cur_dim values + residual estimates */
int ppa_arnoldi_ritz(const ppa_arnoldi* st, int ordering, double* re, double* im, double* resid);
/* harmonic_ritz_values (src/arnoldi.cpp:178-206) */
int ppa_arnoldi_harmonic(const ppa_arnoldi* st, double* re, double* im);
/* ritz_vector (src/arnoldi.cpp:252-265): unit vector j into y_re/y_im (device, n each;
   y_im untouched and *is_complex = 0 for a real pair) */
int ppa_arnoldi_ritz_vector(const ppa_arnoldi* st, int ordering, int j, double* y_re_dev,
                            double* y_im_dev, int* is_complex, ppa_cost* cost);
/* thick_restart with ritz_pairs(ordering) as keep set (src/arnoldi.cpp:267-334) */
int ppa_arnoldi_restart(ppa_arnoldi* st, int ordering, int k, ppa_cost* cost, int* kk);
/* ritz_pairs (src/arnoldi.cpp:154-176) with the eigenvectors of H: pair i's
   vector g_i (cur_dim entries) at vec_re/vec_im[i * cur_dim + r]; NULL skips */
int ppa_arnoldi_ritz_vectors(const ppa_arnoldi* st, int ordering, double* re, double* im,
                             double* resid, double* vec_re, double* vec_im);
/* harmonic_restart_selection (inc/arnoldi.hpp:68-69; src/arnoldi.cpp:208-246),
   same layout as ppa_arnoldi_ritz_vectors */
int ppa_arnoldi_harmonic_selection(const ppa_arnoldi* st, int ordering, double* re, double* im,
                                   double* resid, double* vec_re, double* vec_im);
/* thick_restart(state, keep, k) (inc/arnoldi.hpp:79-80) with a caller-built
   keep set: `count` values (re, im) and vectors g_i of H (vec layout as
   above; im / vec_im may be NULL for real sets), taken in the given order,
   conjugate pairs adjacent (+imag first) as ritz_pairs returns them */
int ppa_arnoldi_restart_keep(ppa_arnoldi* st, int count, const double* re, const double* im,
                             const double* vec_re, const double* vec_im, int k, ppa_cost* cost,
                             int* kk);
void ppa_arnoldi_free(ppa_arnoldi* st);

/* ---- raw device kernels -------------------------------------------------- */
/* y = A x with a CSR operator (src/operators.cpp:39-48) */
int ppa_spmv(const ppa_op* a, const double* x_dev, double* y_dev);
/* One fused polynomial factor (the epilogues of apply_poly,
   src/gmres_poly.cpp:129-143, 306-308): mode 0 y = Ax, 1 y = x + c0 Ax,
   2 y = (o + c1 x) + c0 Ax; base != NULL then y = base - y.  The building
   block of the row-sharded pi(A)v (paper_1806_08020_b200/dist.py). */
int ppa_spmv_factor(const ppa_op* a, const double* x_dev, double* y_dev, int mode, double c0,
                    double c1, const double* o_dev, const double* base_dev);
/* apply_poly's factor plan (src/gmres_poly.cpp:126-143): per factor pair flag
   and coefficients (real root: c0 = -1/Re theta; pair: c0 = 1/|theta|^2,
   c1 = -2 Re theta/|theta|^2); capacity >= nroots */
int ppa_factor_plan(const double* re, const double* im, int nroots, int* pair, double* c0,
                    double* c1, int* nfactors);
/* AY = A Y for p column-major device vectors (multi-RHS SELL SpMM; each column
   bit-identical to ppa_spmv); the solver's batched convergence check */
int ppa_spmm(const ppa_op* a, const double* Y_dev, long long ldy, int p, double* AY_dev,
             long long ldo);
/* One CGS2 step (replaces MGS2 of src/arnoldi.cpp:129-150); Hcol_dev c+1, flag_dev int */
int ppa_cgs2_step(double* V_dev, long long ld, int n, int c, double* w_dev, double* Hcol_dev,
                  int* flag_dev);
/* Row-sharded CGS2 building blocks (the three sweeps of ppa_cgs2_step with
   rank-local sums, for a c-wide all-reduce between sweeps; dist.py
   ShardedSolver over NCCL): out = V[:,0:c]^T w (c values);
   w -= V h then out = [V^T w, ||w||^2] (c + 1 values);
   V[:,c] = (w - V h2) / *hsub.  All pointers device, results deterministic. */
int ppa_cgs_dot_local(const double* V_dev, long long ld, int n, int c, const double* w_dev,
                      double* out_dev);
int ppa_cgs_update_dot_local(const double* V_dev, long long ld, int n, int c, double* w_dev,
                             const double* h_dev, double* out_dev);
int ppa_cgs_store_local(double* V_dev, long long ld, int n, int c, const double* w_dev,
                        const double* h2_dev, const double* hsub_dev);
/* Row-sharded pi(A)v halo over peer memory, without NCCL (dist.py PeerHalo;
   DESIGN.md 7).  Buffers that peers map come from ppa_dev_alloc (cudaMalloc,
   zeroed); handles are exchanged out of band (torch.distributed) and opened
   with ppa_ipc_open.  ppa_halo_publish enqueues a system-scope release store
   of `epoch` into the caller's flag; ppa_halo_pull enqueues, for each peer
   descriptor, a bounded acquire wait for *flag >= epoch (*error_dev = 1 on
   timeout instead of a hang) and the gather
   x_ext[dst_offset + i] = src[src_index[i]] (i < count); x_ext_dev = NULL
   waits only (a fence before a rank rewrites buffers its peers read). */
typedef struct ppa_peer_halo {
  const double* src;          /* the owner's vector (IPC pointer) */
  const long long* src_index; /* device, on the reader */
  long long count;
  long long dst_offset;
  const long long* flag;      /* the owner's epoch flag (IPC pointer) */
} ppa_peer_halo;
int ppa_dev_alloc(size_t bytes, void** out_dev);
int ppa_dev_free(void* dev_ptr);
int ppa_ipc_get_handle(const void* dev_ptr, unsigned char* handle64);
int ppa_ipc_open(const unsigned char* handle64, void** peer_ptr);
int ppa_ipc_close(void* peer_ptr);
int ppa_halo_publish(long long* flag_dev, long long epoch);
int ppa_halo_pull(const ppa_peer_halo* peers_dev, int npeers, long long max_count,
                  double* x_ext_dev, long long epoch, int* error_dev);
/* Sharded box-grid pass with the halo exchange fused in (dist.py
   ShardedGridPoly): polynomial factors of the chain of
   src/gmres_poly.cpp:129-143 - kind 0: two real roots (a0 = -1/theta1,
   b0 = -1/theta2), kind 1: a conjugate pair (a0 = 1/|theta|^2,
   a1 = -2 Re theta/|theta|^2), kind 2: one real root (a0) - over the planes
   [zo0, zo1) of an nx x ny x nz box stencil (nd = 7; nd = 5 with ny = 1: the
   2-D 5-point form) with the nd diagonal values vals (host, increasing
   offset).  x_dev / y_dev hold the owned planes only.  The kernel's copy
   engine reads the two halo planes below from xl_dev (a neighbour's vector,
   its local plane 0 = global plane zl0) and the two above from xr_dev (local
   plane 0 = global plane zo1) once the neighbours' flags (fl_dev, fr_dev,
   IPC pointers from ppa_halo_publish's protocol) reach `epoch`; *err_dev = 1
   if a flag never arrives (~10 s).  Pointers of absent neighbours (zo0 = 0,
   zo1 = nz) may be NULL.  own_dev (the caller's flag: two zero-initialised
   64-bit words, flag and ticket counter) non-NULL: the pass's last CTA
   publishes epoch + 1 into it (system-scope release; no ppa_halo_publish
   launch per pass).  Bit-identical to the unsharded pass. */
int ppa_grid2_slab_pass(int nd, int nx, int ny, int nz, const double* vals, int zo0, int zo1,
                        int kind, double a0, double a1, double b0, const double* x_dev,
                        double* y_dev, const double* xl_dev, int zl0, const long long* fl_dev,
                        const double* xr_dev, const long long* fr_dev, long long epoch,
                        int* err_dev, long long* own_dev);
/* The whole chain of one sharded pi(A)v in one call: pass k runs
   ppa_grid2_slab_pass(kinds[k], a0[k], a1[k], b0[k]) from role k % 2 to role
   (k + 1) % 2 of the caller's two buffers (buf0, buf1), reading the
   neighbours' buffers of the same role (xl0/xl1, xr0/xr1), waiting for
   epoch0 + k and publishing epoch0 + k + 1 into own_dev.  *out_role = the
   role holding the result. */
int ppa_grid2_slab_chain(int nd, int nx, int ny, int nz, const double* vals, int zo0, int zo1,
                         int npass, const int* kinds, const double* a0, const double* a1,
                         const double* b0, double* buf0_dev, double* buf1_dev,
                         const double* xl0_dev, const double* xl1_dev, int zl0,
                         const long long* fl_dev, const double* xr0_dev, const double* xr1_dev,
                         const long long* fr_dev, long long epoch0, int* err_dev,
                         long long* own_dev, int* out_role);
/* out_dev[0] = x . y, deterministic (dot, inc/cost.hpp:51-57) */
int ppa_dot_local(const double* x_dev, const double* y_dev, long long n, double* out_dev);
/* Out = V[:,0:d] G (G d x p col-major, device); in place allowed for p <= d
   (src/arnoldi.cpp:258, 309) */
int ppa_ts_combine(const double* V_dev, long long ldv, int n, int d, const double* G_dev, int p,
                   double* Out_dev, long long ldo);

/* ---- solver ------------------------------------------------------------ */
/* SolveConfig (inc/solver.hpp:21-58) */
typedef struct ppa_solve_config {
  int m, k, nev, degree;
  double rtol_multiplier;
  double rtol_absolute;      /* <= 0: unset */
  int variant;               /* 0 ritz, 1 harmonic */
  int stability;             /* 0 off, 1 pof_auto */
  int double_d1, double_d2;  /* solve_double stages when use_double */
  int use_double;
  int max_cycles;
  unsigned long long seed;
  int allow_nev_above_k;
  int damping;               /* 0 off, 1 auto_heuristic, 2 forced (DampingMode) */
  double damping_alpha;      /* forced: start A^power b + alpha b */
  int damping_power;
  /* SolveConfig::check_mid_cycle / mid_cycle_stride (inc/solver.hpp:40-41) */
  int check_mid_cycle, mid_cycle_stride;
  /* SolveConfig::stagnation_stop / _window / _rtol (inc/solver.hpp:43-45) */
  int stagnation_stop, stagnation_window;
  double stagnation_rtol;
  int want_eigenvectors;     /* keep unit eigenvectors for evec_re/evec_im */
  int orthogonalization;     /* PPA_ORTHO_CGS2 or PPA_ORTHO_DCGS2 (the default of
                                ppa_solve_config_default, C++ and Python); also used by
                                every polynomial build of the solve */
} ppa_solve_config;

/* EigResult (inc/solver.hpp:71-89); arrays supplied by the caller */
typedef struct ppa_solve_result {
  /* capacities (in) */
  int cap_nev, cap_roots, cap_cycles;
  /* per wanted pair */
  double* eig_re;
  double* eig_im;
  double* residuals;
  int* converged_flags;
  /* polynomial(s) in effect */
  double* poly_re;
  double* poly_im;
  double* inner_re;
  double* inner_im;
  /* per-cycle max residual */
  double* cycle_max_residual;
  /* scalars (out) */
  int n_eig, n_poly, n_inner, n_cycles;
  int converged, cycles, composite_degree, poly_base_degree;
  int discarded_probes;      /* damping probes whose basis was dropped */
  double rtol, max_err, norm_estimate;
  ppa_cost cost;
  double t_total, t_setup, t_extend, t_check, t_restart;
  /* optional eigenvector output (EigResult::eigenvectors, inc/solver.hpp:73):
     unit y_j with Re at evec_re[j*evec_ld + i], Im at evec_im[...]; NULL skips */
  double* evec_re;
  double* evec_im;
  long long evec_ld;
} ppa_solve_result;

/* Fill *cfg with the defaults of SolveConfig (inc/solver.hpp:21-58) */
int ppa_solve_config_default(ppa_solve_config* cfg);
/* solve (inc/solver.hpp:94) or solve_double (inc/solver.hpp:111) */
int ppa_solve(const ppa_op* a, const ppa_solve_config* cfg, ppa_solve_result* res);
/* check_ideal_order (inc/solver.hpp:99): 1 if the condition holds */
int ppa_check_ideal_order(const double* re, const double* im, int count, int nev, int* holds);
/* damping_heuristic (inc/solver.hpp:105-106): the polynomial it settles on */
int ppa_damping_heuristic(const ppa_op* a, const ppa_solve_config* cfg, double* re, double* im,
                          int cap, int* nroots, ppa_cost* cost);

/* ---- construction variants and ingest ------------------------ */
/* make_block2 (inc/operators.hpp:87) and make_shifted (inc/operators.hpp:90) */
int ppa_block2_operator(const ppa_op* a, ppa_op** out);
int ppa_shifted_operator(const ppa_op* a, double mu, ppa_op** out);
/* build_two_vector_poly (src/gmres_poly.cpp:228-264); b1/b2 device, length n */
int ppa_build_two_vector_poly(const ppa_op* a, const double* b1_dev, const double* b2_dev,
                              int degree, double* re, double* im, int* nroots, ppa_cost* cost);
/* damped_start (src/gmres_poly.cpp:266-283): out_dev = (A^p b + alpha b)/||.|| */
int ppa_damped_start(const ppa_op* a, const double* b_dev, double alpha, int power,
                     double* out_dev, ppa_cost* cost);
/* read_matrix_market (src/operators.cpp:246-305) */
int ppa_read_matrix_market(const char* path, ppa_host_csr** out);

#ifdef __cplusplus
}
#endif

#endif /* PPA_B200_H */
