// LAPACK-backed small dense kernels (see ppa/dense.hpp).  LAPACK comes
// from the OpenBLAS build bundled with scipy in this image (LP64, symbols
// prefixed "scipy_"); the build script links it with an rpath.

#include "ppa/dense.hpp"

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <limits>
#include <stdexcept>

extern "C" {
void scipy_dgeevx_(const char* balanc, const char* jobvl, const char* jobvr, const char* sense,
                   const int* n, double* a, const int* lda, double* wr, double* wi, double* vl,
                   const int* ldvl, double* vr, const int* ldvr, int* ilo, int* ihi,
                   double* scale, double* abnrm, double* rconde, double* rcondv, double* work,
                   const int* lwork, int* iwork, int* info, size_t, size_t, size_t, size_t);
void scipy_dgetc2_(const int* n, double* a, const int* lda, int* ipiv, int* jpiv, int* info);
void scipy_dgesc2_(const int* n, const double* a, const int* lda, double* rhs, const int* ipiv,
                   const int* jpiv, double* scale);
void scipy_dgeqrf_(const int* m, const int* n, double* a, const int* lda, double* tau,
                   double* work, const int* lwork, int* info);
void scipy_dorgqr_(const int* m, const int* n, const int* k, double* a, const int* lda,
                   const double* tau, double* work, const int* lwork, int* info);
}

namespace ppa {
namespace dense {

bool eig(const Mat& A, std::vector<cplx>& values, CMat* vectors) {
  const int n = A.rows;
  if (A.cols != n) throw std::invalid_argument("eig: matrix not square");
  values.assign(n, cplx(0.0, 0.0));
  if (n == 0) return true;
  Mat a = A;
  std::vector<double> wr(n), wi(n), vr(vectors ? static_cast<size_t>(n) * n : 1), scale(n),
      rconde(n), rcondv(n);
  std::vector<int> iwork(std::max(1, 2 * n - 2));
  int ilo = 0, ihi = 0, info = 0, ldvl = 1, ldvr = vectors ? n : 1, lda = n;
  double abnrm = 0.0, wq = 0.0, vl = 0.0;
  const char* jobvr = vectors ? "V" : "N";
  int lwork = -1;
  scipy_dgeevx_("N", "N", jobvr, "N", &n, a.data(), &lda, wr.data(), wi.data(), &vl, &ldvl,
                vr.data(), &ldvr, &ilo, &ihi, scale.data(), &abnrm, rconde.data(), rcondv.data(),
                &wq, &lwork, iwork.data(), &info, 1, 1, 1, 1);
  lwork = std::max(1, static_cast<int>(wq));
  std::vector<double> work(lwork);
  scipy_dgeevx_("N", "N", jobvr, "N", &n, a.data(), &lda, wr.data(), wi.data(), &vl, &ldvl,
                vr.data(), &ldvr, &ilo, &ihi, scale.data(), &abnrm, rconde.data(), rcondv.data(),
                work.data(), &lwork, iwork.data(), &info, 1, 1, 1, 1);
  if (info != 0) return false;
  for (int i = 0; i < n; ++i) values[i] = cplx(wr[i], wi[i]);
  if (vectors) {
    *vectors = CMat(n, n);
    for (int j = 0; j < n; ++j) {
      if (wi[j] == 0.0) {
        for (int i = 0; i < n; ++i) (*vectors)(i, j) = cplx(vr[static_cast<size_t>(j) * n + i], 0.0);
      } else if (j + 1 < n) {
        for (int i = 0; i < n; ++i) {
          const double re = vr[static_cast<size_t>(j) * n + i];
          const double im = vr[static_cast<size_t>(j + 1) * n + i];
          (*vectors)(i, j) = cplx(re, im);
          (*vectors)(i, j + 1) = cplx(re, -im);
        }
        ++j;
      }
    }
  }
  return true;
}

bool solve_transpose_full_pivot(const Mat& A, const std::vector<double>& rhs,
                                std::vector<double>& f) {
  const int n = A.rows;
  Mat at(n, n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) at(i, j) = A(j, i);
  std::vector<int> ipiv(n), jpiv(n);
  int info = 0, lda = n;
  scipy_dgetc2_(&n, at.data(), &lda, ipiv.data(), jpiv.data(), &info);
  double maxp = 0.0;
  for (int i = 0; i < n; ++i) maxp = std::max(maxp, std::abs(at(i, i)));
  // Eigen FullPivLU::rank(): pivots strictly above eps * diagsize * maxpivot.
  const double thr = std::numeric_limits<double>::epsilon() * n * maxp;
  if (info != 0 || maxp == 0.0) return false;
  for (int i = 0; i < n; ++i) {
    if (!(std::abs(at(i, i)) > thr)) return false;
  }
  f = rhs;
  double sc = 1.0;
  scipy_dgesc2_(&n, at.data(), &lda, f.data(), ipiv.data(), jpiv.data(), &sc);
  if (sc != 1.0) {
    for (double& v : f) v /= sc;
  }
  return true;
}

Mat householder_q(const Mat& G) {
  const int m = G.rows, k = G.cols;
  Mat a = G;
  std::vector<double> tau(std::max(1, k));
  int info = 0, lda = m, lwork = -1;
  double wq = 0.0;
  scipy_dgeqrf_(&m, &k, a.data(), &lda, tau.data(), &wq, &lwork, &info);
  lwork = std::max(1, static_cast<int>(wq));
  std::vector<double> work(lwork);
  scipy_dgeqrf_(&m, &k, a.data(), &lda, tau.data(), work.data(), &lwork, &info);
  if (info != 0) throw std::runtime_error("householder_q: dgeqrf failed");
  lwork = -1;
  scipy_dorgqr_(&m, &k, &k, a.data(), &lda, tau.data(), &wq, &lwork, &info);
  lwork = std::max(1, static_cast<int>(wq));
  work.assign(lwork, 0.0);
  scipy_dorgqr_(&m, &k, &k, a.data(), &lda, tau.data(), work.data(), &lwork, &info);
  if (info != 0) throw std::runtime_error("householder_q: dorgqr failed");
  return a;
}

Mat matmul(const Mat& A, const Mat& B) {
  Mat C(A.rows, B.cols);
  for (int j = 0; j < B.cols; ++j)
    for (int k = 0; k < A.cols; ++k) {
      const double b = B(k, j);
      for (int i = 0; i < A.rows; ++i) C(i, j) += A(i, k) * b;
    }
  return C;
}

Mat matmul_tn(const Mat& A, const Mat& B) {
  Mat C(A.cols, B.cols);
  for (int j = 0; j < B.cols; ++j)
    for (int i = 0; i < A.cols; ++i) {
      double s = 0.0;
      for (int k = 0; k < A.rows; ++k) s += A(k, i) * B(k, j);
      C(i, j) = s;
    }
  return C;
}

}  // namespace dense
}  // namespace ppa
