// Drives the INTEGRATION.md level-1 binding (B200PolyOperator, compiled from
// the document itself by build_level1.py) the way the reference's callers
// do: LinearOperator::apply with host Eigen vectors.  Prints n, mvps, vops
// and pi(A)v so tests/test_integration_level1.py can compare it with the
// oracle.  TEST INFRASTRUCTURE ONLY.
#include <cstdio>
#include <vector>

#include "ppa/gmres_poly.hpp"
#include "ppa/operators.hpp"

namespace ppa {
OperatorPtr make_b200_poly_operator(const CsrMatrix& a, PolyPrecond p);
}

int main() {
  // the reference's 4x4 example family: an upper bidiagonal matrix a_ii = i,
  // a_i,i+1 = 1 (BASELINE config 1 at n = 300)
  const int n = 300;
  ppa::CsrMatrix A;
  A.n = n;
  A.row_ptr.push_back(0);
  for (int i = 0; i < n; ++i) {
    A.col_idx.push_back(i);
    A.values.push_back(i + 1.0);
    if (i + 1 < n) {
      A.col_idx.push_back(i + 1);
      A.values.push_back(1.0);
    }
    A.row_ptr.push_back(static_cast<int>(A.values.size()));
  }
  ppa::PolyPrecond p;
  p.roots = {{250.0, 0.0}, {120.0, 30.0}, {120.0, -30.0}, {40.0, 0.0}, {3.0, 0.0}};
  p.multiplicity = {1, 1, 1, 1, 1};
  p.base_degree = 5;
  try {
    const ppa::OperatorPtr op = ppa::make_b200_poly_operator(A, p);
    Eigen::VectorXd x(n), y(n);
    for (int i = 0; i < n; ++i) x[i] = 1.0 + 0.01 * i;
    ppa::CostRecord rec;
    op->apply(x, y, rec);
    std::printf("%d %lld %lld %d\n", op->dim(), rec.mvps, rec.vops, op->mvps_per_apply());
    for (int i = 0; i < n; ++i) std::printf("%.17g\n", y[i]);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "level1: %s\n", e.what());
    return 1;
  }
  return 0;
}
