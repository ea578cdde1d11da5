#pragma once
// GMRES residual polynomial as a preconditioner (drop-in for the reference's
// inc/gmres_poly.hpp entry points).
//
//   host   : root bookkeeping - Leja ordering, pof, stability copies - kept
//            bit-exact with the reference for identical root inputs
//   device : the product form pi(A) v, one fused SpMV launch per real root
//            and two per conjugate pair (kernels/spmv.cu)

#include <complex>
#include <string>
#include <vector>

#include "ppa/arnoldi.hpp"
#include "ppa/cost.hpp"
#include "ppa/operators.hpp"

namespace ppa {

using Root = std::complex<double>;
using RootList = std::vector<Root>;

/// How a polynomial was obtained (reference enum, same members).
enum class PolyProvenance { single, damped, two_vector, composite_stage };

/// The factored polynomial prod_i (1 - z/theta_i).  `roots` is the order the
/// factors are applied in; copies added for stability are visible through
/// `multiplicity` and added_roots().
struct PolyPrecond {
  RootList roots;
  std::vector<int> multiplicity;
  int base_degree = 0;
  PolyProvenance provenance = PolyProvenance::single;
  double damping_alpha = 0.0;
  int damping_power = 0;
  bool truncated = false;  // the Krylov space closed before `degree` steps

  int effective_degree() const { return static_cast<int>(roots.size()); }
  int added_roots() const { return effective_degree() - base_degree; }
};

/// Product-of-other-factors diagnostic over the distinct roots, in log10.
struct PofReport {
  std::vector<double> log10_pof;
  std::vector<int> copies_needed;
  double max_log10_pof = 0.0;
  int total_copies = 0;
  double max_pof() const;
};

// ---- construction --------------------------------------------------------
// GMRES(d) from the device start vector b: d = min(degree, n) Arnoldi steps
// (device CGS2), harmonic Ritz values on the host, then Leja order
// (reference src/gmres_poly.cpp:95-115).  `ortho` selects the device
// orthogonalisation of that Arnoldi run (the reference's MGS2 counters are
// charged either way); the solver passes SolveConfig::orthogonalization.
PolyPrecond build_gmres_poly(const LinearOperator& a, const double* b, int degree,
                             CostRecord& rec,
                             Orthogonalization ortho = Orthogonalization::dcgs2);
// Two start vectors: GMRES on diag(A, A) from [b1; b2] with each half scaled
// to norm 1/sqrt(2) (src/gmres_poly.cpp:228-264).
PolyPrecond build_two_vector_poly(const OperatorPtr& a, const double* b1, const double* b2,
                                  int degree, CostRecord& rec);
// Damped start (A^power b + alpha b) / norm written to `out`
// (src/gmres_poly.cpp:266-283); alpha is used with power 1 only.
void damped_start(const LinearOperator& a, const double* b, double alpha, int power, double* out,
                  CostRecord& rec);

// ---- root management (host) ----------------------------------------------
RootList leja_order(const RootList& roots);                       // src/gmres_poly.cpp:38-93
Root eval_poly(const PolyPrecond& p, Root z);                     // src/gmres_poly.cpp:149-153
PofReport compute_pof(const PolyPrecond& p);                      // src/gmres_poly.cpp:155-179
PolyPrecond add_stability_roots(const PolyPrecond& p,             // src/gmres_poly.cpp:181-226
                                int max_copies_per_root = 1 << 20);
std::string poly_dump_csv(const PolyPrecond& p);                  // src/gmres_poly.cpp:330-348

// ---- application ---------------------------------------------------------
// out = pi(A) v (device vectors).  A CSR operator gets the fused launch
// chain; any other operator (e.g. tau = I - pi1 in the double polynomial)
// gets the reference's apply/axpy sequence.  Counters follow the reference
// exactly (src/gmres_poly.cpp:117-147).
void apply_poly(const PolyPrecond& p, const LinearOperator& a, const double* v, double* out,
                CostRecord& rec);
// pi(A) and tau(A) = I - pi(A) as operators (src/gmres_poly.cpp:287-328).
OperatorPtr make_poly_operator(OperatorPtr a, PolyPrecond p);
OperatorPtr make_poly_complement_operator(OperatorPtr a, PolyPrecond p);

/// One real-arithmetic factor of the chain: a real root uses c0 = -1/theta;
/// a conjugate pair uses c0 = 1/|theta|^2 and c1 = -2 Re(theta)/|theta|^2.
/// factor_plan() rejects a complex root without its adjacent conjugate
/// (std::logic_error, as the reference's apply_poly does).
struct PolyFactor {
  bool pair = false;
  double c0 = 0.0;
  double c1 = 0.0;
};
std::vector<PolyFactor> factor_plan(const PolyPrecond& p);

}  // namespace ppa
