// Operators and matrix generators (reference: src/operators.cpp).

#include "ppa/operators.hpp"

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>

#include "ppa/rng.hpp"

namespace ppa {

void CsrMatrix::validate() const {
  if (n < 0) throw std::invalid_argument("CsrMatrix: negative dimension");
  if (row_ptr.size() != static_cast<size_t>(n) + 1) {
    throw std::invalid_argument("CsrMatrix: row_ptr length must be n+1");
  }
  if (row_ptr.front() != 0 || row_ptr.back() != nnz()) {
    throw std::invalid_argument("CsrMatrix: row_ptr endpoints invalid");
  }
  if (col_idx.size() != values.size()) {
    throw std::invalid_argument("CsrMatrix: col_idx/values size mismatch");
  }
  for (int i = 0; i < n; ++i) {
    const int b = row_ptr[i], e = row_ptr[i + 1];
    if (e < b) throw std::invalid_argument("CsrMatrix: row_ptr not nondecreasing");
    for (int p = b; p < e; ++p) {
      const int c = col_idx[p];
      if (c < 0 || c >= n) throw std::invalid_argument("CsrMatrix: column index out of range");
      if (p > b && c <= col_idx[p - 1]) {
        throw std::invalid_argument("CsrMatrix: columns not strictly increasing within a row");
      }
    }
  }
}

CsrMatrix CsrMatrix::from_triplets(int n, std::vector<std::tuple<int, int, double>> t) {
  for (const auto& e : t) {
    const int i = std::get<0>(e), j = std::get<1>(e);
    if (i < 0 || i >= n || j < 0 || j >= n) {
      throw std::invalid_argument("from_triplets: index out of range");
    }
  }
  std::stable_sort(t.begin(), t.end(), [](const auto& a, const auto& b) {
    if (std::get<0>(a) != std::get<0>(b)) return std::get<0>(a) < std::get<0>(b);
    return std::get<1>(a) < std::get<1>(b);
  });
  CsrMatrix m;
  m.n = n;
  m.row_ptr.assign(static_cast<size_t>(n) + 1, 0);
  m.col_idx.reserve(t.size());
  m.values.reserve(t.size());
  for (size_t p = 0; p < t.size(); ++p) {
    const int i = std::get<0>(t[p]), j = std::get<1>(t[p]);
    if (p > 0 && std::get<0>(t[p - 1]) == i && std::get<1>(t[p - 1]) == j) {
      m.values.back() += std::get<2>(t[p]);
      continue;
    }
    m.col_idx.push_back(j);
    m.values.push_back(std::get<2>(t[p]));
    ++m.row_ptr[static_cast<size_t>(i) + 1];
  }
  for (int i = 0; i < n; ++i) m.row_ptr[i + 1] += m.row_ptr[i];
  m.validate();
  return m;
}

bool SpectrumSpec::real_only(double tol) const {
  for (const auto& z : eigenvalues) {
    if (std::abs(z.imag()) > tol) return false;
  }
  return true;
}

// ------------------------------------------------------------ operator --

CsrOperator::CsrOperator(const CsrMatrix& m, OperatorKind kind, std::vector<double> diag,
                         CsrLayout layout)
    : kind_(kind), diag_(std::move(diag)) {
  m.validate();
  n_ = m.n;
  nnz_ = m.nnz();
  nnzr_ = m.nnzr();
  std::vector<int> blk;
  kern::build_row_blocks(m.row_ptr.data(), m.n, kern::kSpmvMaxRows, kern::kSpmvMaxNnz, blk);
  const size_t nz = static_cast<size_t>(nnz_);
  const size_t padded = nz + kern::kSpmvPad;
  row_ptr_.resize(static_cast<size_t>(n_) + 1);
  col_idx_.resize(padded);
  values_.resize(padded);
  blk_row_.resize(blk.size());
  PPA_CUDA(cudaMemcpy(row_ptr_.get(), m.row_ptr.data(), (n_ + 1) * sizeof(int),
                      cudaMemcpyHostToDevice));
  PPA_CUDA(cudaMemset(col_idx_.get(), 0, padded * sizeof(int)));
  PPA_CUDA(cudaMemset(values_.get(), 0, padded * sizeof(double)));
  if (nz) {
    PPA_CUDA(cudaMemcpy(col_idx_.get(), m.col_idx.data(), nz * sizeof(int),
                        cudaMemcpyHostToDevice));
    PPA_CUDA(cudaMemcpy(values_.get(), m.values.data(), nz * sizeof(double),
                        cudaMemcpyHostToDevice));
  }
  PPA_CUDA(cudaMemcpy(blk_row_.get(), blk.data(), blk.size() * sizeof(int),
                      cudaMemcpyHostToDevice));
  dev_.n = n_;
  dev_.nnz = nnz_;
  dev_.row_ptr = row_ptr_.get();
  dev_.col_idx = col_idx_.get();
  dev_.values = values_.get();
  dev_.blk_row = blk_row_.get();
  dev_.nblocks = static_cast<int>(blk.size()) - 1;
  int bw = 0;
  for (int i = 0; i < n_; ++i) {
    for (int p = m.row_ptr[i]; p < m.row_ptr[i + 1]; ++p) bw = std::max(bw, std::abs(m.col_idx[p] - i));
  }
  dev_.bandwidth = bw;

  // Layouts are built on the device from the CSR copy (kernels/layout_build.cu):
  // the diagonal-coded form first when allowed (stencils; it needs no SELL
  // copy), else SELL-32 (sigma-sorted when unsorted slices pad too much),
  // then packed SELL-32 over its row order.
  if (layout == CsrLayout::csr || std::getenv("PPA_DISABLE_SELL")) return;
  const cudaStream_t st = current_context().stream();
  const bool dia_ok = layout == CsrLayout::automatic || layout == CsrLayout::dia;
  const bool packed_ok = dia_ok || layout == CsrLayout::sell32_packed;
  if (dia_ok && upload_dia(st)) {
    dev_.nslices = (n_ + 31) / 32;
    return;
  }
  int sigma = 1;
  bool sell = kern::build_sell32_device(row_ptr_.get(), col_idx_.get(), values_.get(), n_, nnz_,
                                        1, sell_, st);
  if (!sell && !std::getenv("PPA_DISABLE_SIGMA")) {
    sigma = kern::kSellSigma;
    sell = kern::build_sell32_device(row_ptr_.get(), col_idx_.get(), values_.get(), n_, nnz_,
                                     sigma, sell_, st);
  }
  if (!sell) return;
  dev_.slice_ptr = sell_.slice_ptr.get();
  dev_.sell_col = sell_.cols.get();
  dev_.sell_val = sell_.vals.get();
  dev_.sell_perm = sell_.perm.size() ? sell_.perm.get() : nullptr;
  dev_.nslices = sell_.nslices;
  dev_.sell_entries = sell_.total;
  dev_.sell_sigma = sigma;
  if (packed_ok) {
    std::vector<int> perm;
    if (dev_.sell_perm) {
      perm.resize(static_cast<size_t>(n_));
      PPA_CUDA(cudaMemcpyAsync(perm.data(), dev_.sell_perm, perm.size() * sizeof(int),
                               cudaMemcpyDeviceToHost, st));
      PPA_CUDA(cudaStreamSynchronize(st));
    }
    upload_packed(m, perm);
  }
}

// Diagonal-coded layout for stencil matrices (kernels/spmv_dia.cu), built on
// the device; PPA_DISABLE_DIA skips it, PPA_DISABLE_DIA_REGULAR keeps every
// row's codes.
bool CsrOperator::upload_dia(cudaStream_t st) {
  if (std::getenv("PPA_DISABLE_DIA")) return false;
  if (!kern::build_dia_device(row_ptr_.get(), col_idx_.get(), values_.get(), n_, nnz_,
                              !std::getenv("PPA_DISABLE_DIA_REGULAR"), dia_, st)) {
    return false;
  }
  dia_dict_.resize(dia_.dict.size());
  PPA_CUDA(cudaMemcpy(dia_dict_.get(), dia_.dict.data(), dia_.dict.size() * sizeof(double),
                      cudaMemcpyHostToDevice));
  dev_.dia_code = dia_.codes.get();
  dev_.dia_dict = dia_dict_.get();
  dev_.dia_ndict = static_cast<int>(dia_.dict.size());
  dev_.dia_ndiag = dia_.ndiag;
  dev_.dia_stride = dia_.stride;
  for (int j = 0; j < dia_.ndiag; ++j) dev_.dia_off[j] = dia_.offsets[j];
  if (dia_.regular) {
    dev_.dia_mask = dia_.mask.get();
    dev_.dia_irr_rows = dia_.irr_rows.get();
    dev_.dia_irr_codes = dia_.irr_codes.get();
    dev_.dia_nirr = dia_.nirr;
    for (int j = 0; j < dia_.ndiag; ++j) dev_.dia_dflt[j] = dia_.defaults[j];
    if (dia_.pres.get()) {
      dev_.dia_pres = dia_.pres.get() + dia_.pres_pad;
      dev_.dia_pres_pad = dia_.pres_pad;
      dev_.grid_nx = dia_.grid[0];
      dev_.grid_ny = dia_.grid[1];
      dev_.grid_nz = dia_.grid[2];
    }
  }
  return true;
}

// Packed SELL-32 over the SELL-32 row order when it shrinks the stream
// (kernels/spmv_packed.cu); PPA_DISABLE_PACKED keeps plain SELL-32.
void CsrOperator::upload_packed(const CsrMatrix& m, const std::vector<int>& perm) {
  if (std::getenv("PPA_DISABLE_PACKED")) return;
  std::vector<long long> pp;
  std::vector<short> pc;
  std::vector<unsigned char> codes;
  std::vector<double> pv, dict;
  if (!kern::build_sell32_packed(m.row_ptr.data(), m.col_idx.data(), m.values.data(), n_, perm,
                                 dev_.sell_entries, pp, pc, codes, pv, dict)) {
    return;
  }
  // +kPackChunk*32 entries of slack so no vector load can run off the end
  const size_t slack = 32 * kern::kPackChunk;
  pk_ptr_.resize(pp.size());
  PPA_CUDA(cudaMemcpy(pk_ptr_.get(), pp.data(), pp.size() * sizeof(long long),
                      cudaMemcpyHostToDevice));
  pk_col_.resize(pc.size() + slack);
  PPA_CUDA(cudaMemcpy(pk_col_.get(), pc.data(), pc.size() * sizeof(short),
                      cudaMemcpyHostToDevice));
  if (!dict.empty()) {
    pk_code_.resize(codes.size() + slack);
    PPA_CUDA(cudaMemcpy(pk_code_.get(), codes.data(), codes.size(), cudaMemcpyHostToDevice));
    pk_dict_.resize(dict.size());
    PPA_CUDA(cudaMemcpy(pk_dict_.get(), dict.data(), dict.size() * sizeof(double),
                        cudaMemcpyHostToDevice));
    dev_.pk_code = pk_code_.get();
    dev_.pk_dict = pk_dict_.get();
    dev_.pk_ndict = static_cast<int>(dict.size());
  } else {
    pk_val_.resize(pv.size() + slack);
    PPA_CUDA(cudaMemcpy(pk_val_.get(), pv.data(), pv.size() * sizeof(double),
                        cudaMemcpyHostToDevice));
    dev_.pk_val = pk_val_.get();
  }
  dev_.pk_col = pk_col_.get();
  dev_.pk_entries = pp.back();
  dev_.pk_ptr = pk_ptr_.get();
}

double CsrOperator::stream_bytes() const {
  if (dev_.dia_mask) {
    return 4.0 * dev_.nslices + double(dev_.dia_nirr) * (4.0 + dev_.dia_stride);
  }
  if (dev_.dia_code) return double(dev_.nslices) * 32.0 * dev_.dia_stride;
  if (dev_.pk_ptr) {
    return double(dev_.pk_entries) * kern::packed_entry_bytes(dev_.pk_ndict) +
           8.0 * double(dev_.nslices + 1);
  }
  if (dev_.sell_val) return 12.0 * double(dev_.sell_entries) + 8.0 * double(dev_.nslices + 1);
  return 12.0 * double(nnz_) + 4.0 * double(n_ + 1);
}

void CsrOperator::apply(const double* x, double* y, CostRecord& rec) const {
  if (x == y) throw std::invalid_argument("CsrOperator::apply: x and y alias");
  ++rec.mvps;
  kern::spmv(dev_, x, y, kern::EpiArgs{}, current_context().stream());
}

void CsrMatrix::multiply(const double* x_dev, double* y_dev) const {
  const CsrOperator op(*this, OperatorKind::csr, {}, CsrLayout::csr);
  CostRecord scratch;  // uncounted
  op.apply(x_dev, y_dev, scratch);
  current_context().sync();
}

OperatorPtr make_csr_operator(const CsrMatrix& matrix, CsrLayout layout) {
  return std::make_shared<CsrOperator>(matrix, OperatorKind::csr, std::vector<double>{}, layout);
}

OperatorPtr make_diagonal(std::vector<double> d) {
  if (d.empty()) throw std::invalid_argument("make_diagonal: empty diagonal");
  CsrMatrix m;
  m.n = static_cast<int>(d.size());
  m.row_ptr.resize(d.size() + 1);
  m.col_idx.resize(d.size());
  m.values = d;
  for (int i = 0; i <= m.n; ++i) m.row_ptr[i] = i;
  for (int i = 0; i < m.n; ++i) m.col_idx[i] = i;
  return std::make_shared<CsrOperator>(m, OperatorKind::diagonal, std::move(d));
}

namespace {

class Block2Operator final : public LinearOperator {
 public:
  explicit Block2Operator(OperatorPtr a) : a_(std::move(a)) {
    if (!a_) throw std::invalid_argument("make_block2: null operator");
  }
  int dim() const override { return 2 * a_->dim(); }
  OperatorKind kind() const override { return OperatorKind::block2; }
  int mvps_per_apply() const override { return 2 * a_->mvps_per_apply(); }
  double nnzr() const override { return a_->nnzr(); }
  void apply(const double* x, double* y, CostRecord& rec) const override {
    const long long n = a_->dim();
    if (const auto* csr = dynamic_cast<const CsrOperator*>(a_.get())) {
      // both halves in one pass over the matrix (multi-RHS SpMV; each column
      // bit-identical to the single SpMV)
      if (x == y) throw std::invalid_argument("Block2Operator::apply: x and y alias");
      rec.mvps += 2;
      kern::spmm(csr->device(), x, n, 2, y, n, current_context().stream());
      return;
    }
    a_->apply(x, y, rec);
    a_->apply(x + n, y + n, rec);
  }

 private:
  OperatorPtr a_;
};

class ShiftedOperator final : public LinearOperator {
 public:
  ShiftedOperator(OperatorPtr a, double mu) : a_(std::move(a)), mu_(mu) {
    if (!a_) throw std::invalid_argument("make_shifted: null operator");
  }
  int dim() const override { return a_->dim(); }
  OperatorKind kind() const override { return OperatorKind::shifted; }
  int mvps_per_apply() const override { return a_->mvps_per_apply(); }
  double nnzr() const override { return a_->nnzr(); }
  void apply(const double* x, double* y, CostRecord& rec) const override {
    a_->apply(x, y, rec);
    if (mu_ != 0.0) {
      kern::axpy(-mu_, x, y, dim(), current_context().stream());
      ++rec.vops;
    }
  }

 private:
  OperatorPtr a_;
  double mu_;
};

class CallbackOperator final : public LinearOperator {
 public:
  CallbackOperator(int n, int mvps, double nnzr, DeviceApplyFn fn)
      : n_(n), mvps_(mvps), nnzr_(nnzr), fn_(std::move(fn)) {
    if (n_ < 1) throw std::invalid_argument("make_callback_operator: dim < 1");
    if (mvps_ < 0) throw std::invalid_argument("make_callback_operator: mvps_per_apply < 0");
    if (!fn_) throw std::invalid_argument("make_callback_operator: null apply");
  }
  int dim() const override { return n_; }
  OperatorKind kind() const override { return OperatorKind::external; }
  int mvps_per_apply() const override { return mvps_; }
  double nnzr() const override { return nnzr_; }
  void apply(const double* x, double* y, CostRecord& rec) const override {
    if (x == nullptr || y == nullptr) throw std::invalid_argument("apply: dimension mismatch");
    const int rc = fn_(x, y, current_context().stream());
    if (rc != 0) {
      throw std::runtime_error("callback operator: apply returned " + std::to_string(rc));
    }
    rec.mvps += mvps_;
  }

 private:
  int n_, mvps_;
  double nnzr_;
  DeviceApplyFn fn_;
};

std::string lower(std::string s) {
  std::transform(s.begin(), s.end(), s.begin(), [](unsigned char c) { return std::tolower(c); });
  return s;
}

}  // namespace

OperatorPtr make_block2(OperatorPtr a) { return std::make_shared<Block2Operator>(std::move(a)); }

OperatorPtr make_shifted(OperatorPtr a, double mu) {
  return std::make_shared<ShiftedOperator>(std::move(a), mu);
}

OperatorPtr make_callback_operator(int dim, int mvps_per_apply, double nnzr, DeviceApplyFn apply) {
  return std::make_shared<CallbackOperator>(dim, mvps_per_apply, nnzr, std::move(apply));
}

CsrMatrix read_matrix_market(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("read_matrix_market: cannot open " + path);
  std::string line;
  if (!std::getline(in, line)) throw std::runtime_error("read_matrix_market: empty file");
  std::istringstream head(line);
  std::string banner, object, format, field, symmetry;
  head >> banner >> object >> format >> field >> symmetry;
  object = lower(object);
  format = lower(format);
  field = lower(field);
  symmetry = lower(symmetry);
  if (banner != "%%MatrixMarket" || object != "matrix" || format != "coordinate") {
    throw std::runtime_error("read_matrix_market: malformed header");
  }
  if (field != "real") {
    throw std::runtime_error("read_matrix_market: unsupported field '" + field + "' (only real)");
  }
  const bool sym = symmetry == "symmetric";
  if (!sym && symmetry != "general") {
    throw std::runtime_error("read_matrix_market: unsupported symmetry '" + symmetry + "'");
  }
  while (std::getline(in, line)) {
    if (!line.empty() && line[0] != '%') break;
  }
  std::istringstream size_line(line);
  long long rows = 0, cols = 0, entries = 0;
  if (!(size_line >> rows >> cols >> entries) || rows <= 0 || cols <= 0) {
    throw std::runtime_error("read_matrix_market: bad size line");
  }
  if (rows != cols) throw std::runtime_error("read_matrix_market: matrix must be square");
  std::vector<std::tuple<int, int, double>> trip;
  trip.reserve(static_cast<size_t>(entries) * (sym ? 2 : 1));
  for (long long e = 0; e < entries; ++e) {
    long long i = 0, j = 0;
    double v = 0.0;
    if (!(in >> i >> j >> v)) throw std::runtime_error("read_matrix_market: truncated entry list");
    if (i < 1 || i > rows || j < 1 || j > cols) {
      throw std::runtime_error("read_matrix_market: index out of range");
    }
    trip.emplace_back(static_cast<int>(i - 1), static_cast<int>(j - 1), v);
    if (sym && i != j) trip.emplace_back(static_cast<int>(j - 1), static_cast<int>(i - 1), v);
  }
  return CsrMatrix::from_triplets(static_cast<int>(rows), std::move(trip));
}

// ---------------------------------------------------------- generators --

CsrMatrix make_convection_diffusion(int grid_n) {
  if (grid_n < 2) throw std::invalid_argument("make_convection_diffusion: grid_n < 2");
  const int n = grid_n * grid_n;
  const double h = 1.0 / (grid_n + 1);
  CsrMatrix m;
  m.n = n;
  m.row_ptr.assign(static_cast<size_t>(n) + 1, 0);
  m.col_idx.reserve(5ull * n);
  m.values.reserve(5ull * n);
  int pos = 0;
  for (int iy = 0; iy < grid_n; ++iy) {
    const double y = (iy + 1) * h;
    const bool lower = y <= 0.5 + 1e-14;
    const double eps = lower ? 1.0 : 100.0;
    const double cc = lower ? 20.0 : 2000.0;
    const double center = 4.0 * eps / (h * h);
    const double east = -eps / (h * h) + cc / (2.0 * h);
    const double west = -eps / (h * h) - cc / (2.0 * h);
    const double ns = -eps / (h * h);
    for (int ix = 0; ix < grid_n; ++ix) {
      const int row = iy * grid_n + ix;
      auto put = [&](int col, double v) {
        m.col_idx.push_back(col);
        m.values.push_back(v);
        ++pos;
      };
      if (iy > 0) put(row - grid_n, ns);
      if (ix > 0) put(row - 1, west);
      put(row, center);
      if (ix + 1 < grid_n) put(row + 1, east);
      if (iy + 1 < grid_n) put(row + grid_n, ns);
      m.row_ptr[static_cast<size_t>(row) + 1] = pos;
    }
  }
  m.validate();
  return m;
}

CsrMatrix make_convection_diffusion_const(int grid_n, double peclet) {
  if (grid_n < 2) throw std::invalid_argument("make_convection_diffusion_const: grid_n < 2");
  const long long nl = static_cast<long long>(grid_n) * grid_n;
  if (nl > 2147483647LL) throw std::invalid_argument("make_convection_diffusion_const: too large");
  const int n = static_cast<int>(nl);
  const double h = 1.0 / (grid_n + 1);
  const double beta = 2.0 * peclet / h;
  const double center = 4.0 / (h * h);
  const double east = -1.0 / (h * h) + beta / (2.0 * h);
  const double west = -1.0 / (h * h) - beta / (2.0 * h);
  const double ns = -1.0 / (h * h);
  CsrMatrix m;
  m.n = n;
  m.row_ptr.assign(static_cast<size_t>(n) + 1, 0);
  const size_t nnz = 5ull * n - 4ull * grid_n;
  m.col_idx.resize(nnz);
  m.values.resize(nnz);
  size_t pos = 0;
  for (int iy = 0; iy < grid_n; ++iy) {
    for (int ix = 0; ix < grid_n; ++ix) {
      const int row = iy * grid_n + ix;
      auto put = [&](int col, double v) {
        m.col_idx[pos] = col;
        m.values[pos] = v;
        ++pos;
      };
      if (iy > 0) put(row - grid_n, ns);
      if (ix > 0) put(row - 1, west);
      put(row, center);
      if (ix + 1 < grid_n) put(row + 1, east);
      if (iy + 1 < grid_n) put(row + grid_n, ns);
      m.row_ptr[static_cast<size_t>(row) + 1] = static_cast<int>(pos);
    }
  }
  m.validate();
  return m;
}

CsrMatrix make_laplacian_3d(int grid_n) {
  if (grid_n < 2) throw std::invalid_argument("make_laplacian_3d: grid_n < 2");
  const long long nl = 1LL * grid_n * grid_n * grid_n;
  if (nl > 2147483647LL / 7) throw std::invalid_argument("make_laplacian_3d: too large");
  const int N = grid_n;
  const int n = static_cast<int>(nl);
  const double h = 1.0 / (grid_n + 1);
  const double center = 6.0 / (h * h);
  const double off = -1.0 / (h * h);
  CsrMatrix m;
  m.n = n;
  m.row_ptr.assign(static_cast<size_t>(n) + 1, 0);
  const size_t nnz = 7ull * n - 6ull * N * N;
  m.col_idx.resize(nnz);
  m.values.resize(nnz);
  size_t pos = 0;
  const int NN = N * N;
  for (int iz = 0; iz < N; ++iz)
    for (int iy = 0; iy < N; ++iy)
      for (int ix = 0; ix < N; ++ix) {
        const int row = (iz * N + iy) * N + ix;
        auto put = [&](int col, double v) {
          m.col_idx[pos] = col;
          m.values[pos] = v;
          ++pos;
        };
        if (iz > 0) put(row - NN, off);
        if (iy > 0) put(row - N, off);
        if (ix > 0) put(row - 1, off);
        put(row, center);
        if (ix + 1 < N) put(row + 1, off);
        if (iy + 1 < N) put(row + N, off);
        if (iz + 1 < N) put(row + NN, off);
        m.row_ptr[static_cast<size_t>(row) + 1] = static_cast<int>(pos);
      }
  m.validate();
  return m;
}

CsrMatrix make_bidiagonal(int n) {
  if (n < 1) throw std::invalid_argument("make_bidiagonal: n < 1");
  CsrMatrix m;
  m.n = n;
  m.row_ptr.resize(static_cast<size_t>(n) + 1);
  m.col_idx.reserve(2ull * n);
  m.values.reserve(2ull * n);
  m.row_ptr[0] = 0;
  for (int i = 0; i < n; ++i) {
    m.col_idx.push_back(i);
    m.values.push_back(static_cast<double>(i + 1));
    if (i + 1 < n) {
      m.col_idx.push_back(i + 1);
      m.values.push_back(1.0);
    }
    m.row_ptr[i + 1] = static_cast<int>(m.col_idx.size());
  }
  m.validate();
  return m;
}

CsrMatrix make_random_poisson(int n, double lambda, unsigned long long seed) {
  if (n < 2) throw std::invalid_argument("make_random_poisson: n < 2");
  const uint64_t mkey = rng::key(seed, rng::kMatrix);
  const double elim = std::exp(-lambda);
  CsrMatrix m;
  m.n = n;
  m.row_ptr.assign(static_cast<size_t>(n) + 1, 0);
  m.col_idx.reserve(static_cast<size_t>(n) * static_cast<size_t>(lambda + 2));
  m.values.reserve(m.col_idx.capacity());
  std::vector<std::pair<int, double>> row;
  for (int i = 0; i < n; ++i) {
    rng::RowStream rs(mkey, static_cast<uint64_t>(i));
    // Knuth's multiplicative Poisson sampler.
    int L = 0;
    double p = 1.0;
    do {
      p *= rs.uniform();
      ++L;
    } while (p > elim);
    L = std::max(1, L - 1);
    row.clear();
    row.emplace_back(i, (static_cast<double>(i) + 1.0) / static_cast<double>(n) * 10.0);
    for (int e = 0; e < L; ++e) {
      int j;
      do {
        j = static_cast<int>(rs.uniform() * n);
        if (j >= n) j = n - 1;
      } while (j == i);
      row.emplace_back(j, rs.normal() / 8.0);
    }
    std::stable_sort(row.begin(), row.end(),
                     [](const auto& a, const auto& b) { return a.first < b.first; });
    int last = -1;
    for (const auto& e : row) {
      if (e.first == last) {
        m.values.back() += e.second;
      } else {
        m.col_idx.push_back(e.first);
        m.values.push_back(e.second);
        last = e.first;
      }
    }
    m.row_ptr[static_cast<size_t>(i) + 1] = static_cast<int>(m.col_idx.size());
  }
  m.validate();
  return m;
}

CsrMatrix make_config_matrix(int config) {
  switch (config) {
    case 1: return make_bidiagonal(5000);
    case 2: return make_convection_diffusion_const(1000, 0.5);
    case 3: return make_laplacian_3d(160);
    case 4: return make_random_poisson(2000000, 16.0, 4);
    case 5: return make_convection_diffusion_const(2048, 0.5);
    default: throw std::invalid_argument("make_config_matrix: config must be 1..5");
  }
}

unsigned long long csr_fingerprint(const CsrMatrix& m) {
  uint64_t h = 0xcbf29ce484222325ull;
  auto eat = [&](const void* p, size_t bytes) {
    const unsigned char* c = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < bytes; ++i) {
      h ^= c[i];
      h *= 0x100000001b3ull;
    }
  };
  eat(&m.n, sizeof(int));
  eat(m.row_ptr.data(), m.row_ptr.size() * sizeof(int));
  eat(m.col_idx.data(), m.col_idx.size() * sizeof(int));
  eat(m.values.data(), m.values.size() * sizeof(double));
  return h;
}

}  // namespace ppa
