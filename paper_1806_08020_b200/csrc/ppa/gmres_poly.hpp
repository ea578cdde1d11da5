#pragma once
// GMRES-polynomial preconditioner (reference inc/gmres_poly.hpp).
// Root management (Leja order, pof, stability copies) stays on the host and
// is bit-exact with the reference given identical inputs; pi(A)v runs as a
// chain of fused SpMV-factor kernels on the device.

#include <complex>
#include <string>
#include <vector>

#include "ppa/arnoldi.hpp"
#include "ppa/cost.hpp"
#include "ppa/operators.hpp"

namespace ppa {

enum class PolyProvenance { single, damped, two_vector, composite_stage };

/// pi(z) = prod_i (1 - z/theta_i), roots in application order
/// (inc/gmres_poly.hpp:19-30).
struct PolyPrecond {
  std::vector<std::complex<double>> roots;
  std::vector<int> multiplicity;
  int base_degree = 0;
  PolyProvenance provenance = PolyProvenance::single;
  double damping_alpha = 0.0;
  int damping_power = 0;
  bool truncated = false;

  int effective_degree() const { return static_cast<int>(roots.size()); }
  int added_roots() const { return effective_degree() - base_degree; }
};

/// inc/gmres_poly.hpp:34-41.
struct PofReport {
  std::vector<double> log10_pof;
  std::vector<int> copies_needed;
  double max_log10_pof = 0.0;
  int total_copies = 0;
  double max_pof() const;
};

/// d = min(degree, n) Arnoldi steps on A from b (device vector), harmonic
/// Ritz values, Leja order (src/gmres_poly.cpp:95-115).
PolyPrecond build_gmres_poly(const LinearOperator& a, const double* b, int degree,
                             CostRecord& rec);

/// Modified Leja ordering (src/gmres_poly.cpp:38-93).
std::vector<std::complex<double>> leja_order(const std::vector<std::complex<double>>& roots);

/// out = pi(A) v on the device (src/gmres_poly.cpp:117-147).  When A is a
/// CSR operator every factor is one fused SpMV launch;
/// otherwise (A itself composite) the reference's apply/axpy sequence is
/// issued.  Counters charge exactly the reference's increments.
void apply_poly(const PolyPrecond& p, const LinearOperator& a, const double* v, double* out,
                CostRecord& rec);

std::complex<double> eval_poly(const PolyPrecond& p, std::complex<double> z);
PofReport compute_pof(const PolyPrecond& p);
PolyPrecond add_stability_roots(const PolyPrecond& p, int max_copies_per_root = 1 << 20);

/// One polynomial from two start vectors: GMRES on diag(A, A) with the
/// stacked start [b1; b2], halves rescaled to norm 1/sqrt(2)
/// (src/gmres_poly.cpp:228-264).  b1, b2: device vectors of length n.
PolyPrecond build_two_vector_poly(const OperatorPtr& a, const double* b1, const double* b2,
                                  int degree, CostRecord& rec);

/// Damped GMRES start A^power b + alpha b (alpha with power 1), normalised,
/// into `out` (device, length n) (src/gmres_poly.cpp:266-283).
void damped_start(const LinearOperator& a, const double* b, double alpha, int power, double* out,
                  CostRecord& rec);

/// pi(A) (or tau(A) = I - pi(A)) as an operator (src/gmres_poly.cpp:287-328).
OperatorPtr make_poly_operator(OperatorPtr a, PolyPrecond p);
OperatorPtr make_poly_complement_operator(OperatorPtr a, PolyPrecond p);

/// CSV dump of the distinct roots (src/gmres_poly.cpp:330-348).
std::string poly_dump_csv(const PolyPrecond& p);

/// Real-arithmetic factor plan of a root list: what each fused launch
/// computes (validates conjugate adjacency like the reference, throwing
/// std::logic_error).
struct PolyFactor {
  bool pair = false;
  double c0 = 0.0;  // real: -1/theta;  pair: 1/|theta|^2
  double c1 = 0.0;  // pair: -2 Re(theta)/|theta|^2
};
std::vector<PolyFactor> factor_plan(const PolyPrecond& p);

}  // namespace ppa
