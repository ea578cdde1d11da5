#pragma once
// Small dense linear algebra on the host (m <= 100): the only part of the
// solver that stays on the CPU (BASELINE.json north_star).  Replaces the
// reference's Eigen::EigenSolver / FullPivLU / HouseholderQR
// (src/arnoldi.cpp:158, 188, 199, 301-303) with LAPACK (dgeevx with
// BALANC='N', i.e. the same unbalanced Hessenberg-QR eigensolver class as
// Eigen's RealSchur; dgetc2/dgesc2 complete-pivoting LU; dgeqrf/dorgqr).

#include <complex>
#include <vector>

namespace ppa {
namespace dense {

using cplx = std::complex<double>;

/// Column-major real matrix.
struct Mat {
  int rows = 0, cols = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int r, int c) : rows(r), cols(c), a(static_cast<size_t>(r) * c, 0.0) {}
  double& operator()(int i, int j) { return a[static_cast<size_t>(j) * rows + i]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(j) * rows + i]; }
  double* data() { return a.data(); }
  const double* data() const { return a.data(); }
};

/// Column-major complex matrix.
struct CMat {
  int rows = 0, cols = 0;
  std::vector<cplx> a;
  CMat() = default;
  CMat(int r, int c) : rows(r), cols(c), a(static_cast<size_t>(r) * c) {}
  cplx& operator()(int i, int j) { return a[static_cast<size_t>(j) * rows + i]; }
  const cplx& operator()(int i, int j) const { return a[static_cast<size_t>(j) * rows + i]; }
};

/// Eigenvalues (and optionally unit-norm right eigenvectors) of a real
/// square matrix.  Conjugate pairs come out adjacent, +imag first.
/// Returns false if the QR iteration failed to converge.
bool eig(const Mat& A, std::vector<cplx>& values, CMat* vectors);

/// Solves A^T f = rhs with complete-pivoting LU of A^T.  Returns false when
/// A^T is not invertible under Eigen's FullPivLU rank rule
/// (|u_ii| > eps * d * max|u_jj| for all i).
bool solve_transpose_full_pivot(const Mat& A, const std::vector<double>& rhs,
                                std::vector<double>& f);

/// Thin orthogonal factor Q (m x k) of the Householder QR of G (m x k).
Mat householder_q(const Mat& G);

/// C = A^T B and C = A B (naive, small sizes).
Mat matmul(const Mat& A, const Mat& B);
Mat matmul_tn(const Mat& A, const Mat& B);

}  // namespace dense
}  // namespace ppa
