#pragma once
// Operators: the reference's operator module (inc/operators.hpp) with
// device-resident vectors.  Names, semantics, counters and exceptions follow
// the reference; the one substitution is the vector type - apply() takes
// device pointers of length dim() instead of Eigen::Ref<VectorXd> (SURVEY
// §8b "Constraint": host vectors would force a 32 MB H2D/D2H per apply).

#include <complex>
#include <functional>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "ppa/cost.hpp"
#include "ppa/device.hpp"
#include "ppa/kernels.hpp"

namespace ppa {

/// Host CSR matrix (inc/operators.hpp:15-33): int32 row_ptr[n+1], int32
/// col_idx strictly increasing per row, fp64 values.
struct CsrMatrix {
  int n = 0;
  std::vector<int> row_ptr;
  std::vector<int> col_idx;
  std::vector<double> values;

  long long nnz() const { return static_cast<long long>(values.size()); }
  double nnzr() const { return n > 0 ? double(nnz()) / double(n) : 0.0; }

  /// Structural invariants; throws std::invalid_argument with the
  /// reference's messages (src/operators.cpp:12-37).
  void validate() const;

  /// Sort by (row, col), sum duplicates in input order, validate
  /// (src/operators.cpp:50-78; the sort is stable here so duplicate sums
  /// are deterministic).
  static CsrMatrix from_triplets(int n, std::vector<std::tuple<int, int, double>> t);

  /// y = A x, uncounted (inc/operators.hpp:27-28); device vectors.  Builds a
  /// device copy of the matrix per call - use CsrOperator for repeated,
  /// counted applies.
  void multiply(const double* x_dev, double* y_dev) const;
};

/// Known eigenvalue list of a test matrix, conjugate-closed
/// (inc/operators.hpp:35-41).
struct SpectrumSpec {
  std::vector<std::complex<double>> eigenvalues;

  int dim() const { return static_cast<int>(eigenvalues.size()); }
  /// True when every eigenvalue has |Im| <= tol (src/operators.cpp:80-85).
  bool real_only(double tol = 0.0) const;
};

enum class OperatorKind { csr, diagonal, shifted, block2, poly, composite, external };

/// A counted action v -> Op v on device vectors (inc/operators.hpp:49-76).
/// Kernels run on the calling thread's current context stream.
class LinearOperator {
 public:
  virtual ~LinearOperator() = default;
  virtual int dim() const = 0;
  virtual OperatorKind kind() const = 0;
  /// y = Op x (device pointers, length dim(), x != y).  Increments rec.mvps
  /// by the base-matrix applications performed.
  virtual void apply(const double* x, double* y, CostRecord& rec) const = 0;
  virtual int mvps_per_apply() const = 0;
  virtual const std::vector<double>* diagonal() const { return nullptr; }
  virtual double nnzr() const = 0;
};

using OperatorPtr = std::shared_ptr<const LinearOperator>;

/// CSR operator whose matrix lives in HBM (uploaded once at construction,
/// validated on the host first; src/operators.cpp:113-130).
/// Device layout of a CSR operator.  `automatic`
/// takes the first that applies of diagonal-coded, packed SELL-32, SELL-32,
/// CSR row blocks; the others cap the choice at that layout (falling back
/// down the same list when the matrix does not fit it).  Every layout gives
/// bit-identical results.
enum class CsrLayout { automatic = 0, csr = 1, sell32 = 2, sell32_packed = 3, dia = 4 };

class CsrOperator final : public LinearOperator {
 public:
  explicit CsrOperator(const CsrMatrix& m, OperatorKind kind = OperatorKind::csr,
                       std::vector<double> diag = {}, CsrLayout layout = CsrLayout::automatic);
  int dim() const override { return n_; }
  OperatorKind kind() const override { return kind_; }
  int mvps_per_apply() const override { return 1; }
  double nnzr() const override { return nnzr_; }
  const std::vector<double>* diagonal() const override {
    return kind_ == OperatorKind::diagonal ? &diag_ : nullptr;
  }
  void apply(const double* x, double* y, CostRecord& rec) const override;

  const kern::CsrDevice& device() const { return dev_; }
  long long nnz() const { return nnz_; }
  bool uses_sell() const { return dev_.sell_val != nullptr; }
  long long sell_entries() const { return dev_.sell_entries; }
  int sell_sigma() const { return dev_.sell_sigma; }
  bool uses_packed() const { return dev_.pk_ptr != nullptr; }
  bool uses_dia() const { return dev_.dia_code != nullptr; }
  /// Matrix-stream bytes one SpMV reads in the layout the kernel uses.
  double stream_bytes() const;
  /// Bytes one SpMV moves under the north-star model:
  /// 12*nnz + 4*(n+1) + 8n (x) + 8n (y).
  double model_bytes() const {
    return 12.0 * double(nnz_) + 4.0 * double(n_ + 1) + 16.0 * double(n_);
  }

 private:
  int n_ = 0;
  long long nnz_ = 0;
  double nnzr_ = 0.0;
  OperatorKind kind_;
  std::vector<double> diag_;
  DBuffer<int> row_ptr_, col_idx_, blk_row_;
  DBuffer<double> values_;
  DBuffer<long long> pk_ptr_;
  kern::DevSell sell_;
  kern::DevDia dia_;
  DBuffer<short> pk_col_;
  DBuffer<unsigned char> pk_code_;
  DBuffer<double> pk_val_, pk_dict_, dia_dict_;
  kern::CsrDevice dev_;

  void upload_packed(const CsrMatrix& m, const std::vector<int>& perm);
  bool upload_dia(cudaStream_t st);
};

OperatorPtr make_csr_operator(const CsrMatrix& matrix,
                              CsrLayout layout = CsrLayout::automatic);
/// Diagonal operator (src/operators.cpp:89-111), stored as a diagonal CSR.
OperatorPtr make_diagonal(std::vector<double> diag_values);
/// 2n-dimensional diag(A, A); one apply costs two applications of A
/// (src/operators.cpp:132-150).
OperatorPtr make_block2(OperatorPtr a);
/// v -> Av - mu v (src/operators.cpp:152-170).
OperatorPtr make_shifted(OperatorPtr a, double mu);

/// A caller-defined device operator: the reference's plugin mechanism (any
/// LinearOperator subclass is accepted by arnoldi_extend, build_gmres_poly
/// and solve; inc/operators.hpp:49-76) for code outside this library, e.g. a
/// matrix-free stencil.  `apply(x, y, stream)` must write y = Op x for device
/// vectors of length dim on `stream` (the calling thread's context stream)
/// and return 0; a nonzero return becomes std::runtime_error.  Each apply
/// charges mvps_per_apply base applications (kind() = external, ours).
using DeviceApplyFn = std::function<int(const double* x, double* y, cudaStream_t stream)>;
OperatorPtr make_callback_operator(int dim, int mvps_per_apply, double nnzr, DeviceApplyFn apply);

/// Strict Matrix Market coordinate reader, real general/symmetric
/// (src/operators.cpp:246-305); symmetric storage is expanded.
CsrMatrix read_matrix_market(const std::string& path);

// ------------------------------------------------------- generators -----
// Deterministic synthetic matrices (BASELINE.json configs; DESIGN.md
// "Generators").  Column order per row is ascending, as the reference's
// generator emits it (src/operators.cpp:215-238).

/// The reference's two-region convection-diffusion matrix
/// (src/operators.cpp:190-244), restated bit-exactly.
CsrMatrix make_convection_diffusion(int grid_n);
/// Constant-coefficient -u_xx - u_yy + beta u_x on a grid_n^2 interior grid,
/// h = 1/(grid_n+1), beta = 2*peclet/h (configs 2 and 5: peclet = 0.5).
CsrMatrix make_convection_diffusion_const(int grid_n, double peclet);
/// 7-point 3D Laplacian (1/h^2 scaling), grid_n^3 unknowns (config 3).
CsrMatrix make_laplacian_3d(int grid_n);
/// Upper bidiagonal a_ii = i (1-based), a_i,i+1 = 1 (config 1).
CsrMatrix make_bidiagonal(int n);
/// Random sparse: row i gets max(1, Poisson(lambda)) off-diagonal entries
/// with uniform columns != i and N(0,1)/8 values, plus a_ii = (i+1)/n*10
/// (config 4).  Duplicates are summed in draw order.
CsrMatrix make_random_poisson(int n, double lambda, unsigned long long seed);

/// BASELINE.json configs 1..5 (matrix only).
CsrMatrix make_config_matrix(int config);

/// FNV-1a over (n, row_ptr, col_idx, values) bytes - the bit-exactness
/// fingerprint compared against the oracle's generator.
unsigned long long csr_fingerprint(const CsrMatrix& m);

}  // namespace ppa
