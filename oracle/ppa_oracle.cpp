// ===========================================================================
// ORACLE - TEST INFRASTRUCTURE ONLY.
//
// A CPU restatement of the reference library's hot path
// (/root/reference/proj/src/{operators,gmres_poly,arnoldi}.cpp) and of the
// SPEC's solver contract (SPEC.md [MODULE] solver), used by tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
// arm as the CHECKER.  Nothing in the product (paper_1806_08020_b200/)
// links or calls this code.
//
// Why a restatement: the reference cannot be built here - every TU includes
// <Eigen/Core> (inc/operators.hpp:8) and Eigen is neither vendored
// (proj/.gitignore:2) nor installed; solver.cpp does not exist (the solve
// entry points of inc/solver.hpp have no body); CMakeLists.txt:1-6 declares
// no target.  Eigen (version unpinned) is replaced by plain loops for
// vector arithmetic and by LAPACK (scipy's bundled OpenBLAS) for
// EigenSolver / FullPivLU / HouseholderQR.
//
// Pinning: tests/test_oracle_*.py check this oracle against every
// known-answer example SPEC.md gives for the path and against closed-form
// spectra.  The reference ships no test
// vectors, so parity at the Eigen boundary (dense eigensolver ordering,
// dot-product summation order) is unpinned.
//
// Floating point: compiled with -ffp-contract=off so every a*b+c rounds
// twice, as the reference's un-flagged build (CMakeLists.txt:1-6) does.
// Threading (OpenMP) is used only where it cannot change results: the
// row loop of the SpMV and elementwise axpy/scale.  Dots are sequential.
// orc_set_variant(1|2) switches to the roundoff-floor probes (classical
// CGS2 / blocked dots, see g_variant); variant 0, the default, is the
// reference restatement every parity test uses.
// ===========================================================================

#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <numeric>
#include <optional>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

extern "C" {
void scipy_dgeevx_(const char*, const char*, const char*, const char*, const int*, double*,
                   const int*, double*, double*, double*, const int*, double*, const int*, int*,
                   int*, double*, double*, double*, double*, double*, const int*, int*, int*,
                   size_t, size_t, size_t, size_t);
void scipy_dgetc2_(const int*, double*, const int*, int*, int*, int*);
void scipy_dgesc2_(const int*, const double*, const int*, double*, const int*, const int*,
                   double*);
void scipy_dgeqrf_(const int*, const int*, double*, const int*, double*, double*, const int*,
                   int*);
void scipy_dorgqr_(const int*, const int*, const int*, double*, const int*, const double*,
                   double*, const int*, int*);
}

namespace orc {

using cd = std::complex<double>;
using Vec = std::vector<double>;

// ------------------------------------------------------------------ cost --
// inc/cost.hpp:17-23
struct Cost {
  long long mvps = 0, dots = 0, vops = 0;
  double nnzr = 0.0, wall_seconds = 0.0;
};

// Roundoff-floor probe (NOT the reference; test infrastructure for
// tests/golden/roundoff_floor.json).  Variant 0 is the reference: MGS2 with
// sequential dot products (src/arnoldi.cpp:129-140, inc/cost.hpp:51-76).
// Variants 1 and 2 change only the floating-point summation order, which the
// reference leaves to Eigen (unpinned): 1 = classical CGS2 (all coefficients
// of a pass from the same w) with blocked dots, 2 = MGS2 with blocked dots.
// A blocked dot sums 4096-element chunks in order, then the chunk sums in
// order, so it is deterministic for any thread count.  The spread of the
// three variants' results is the oracle's own roundoff floor on a problem.
int g_variant = 0;
constexpr long kDotChunk = 4096;

double blocked_sum(const double* x, const double* y, long n) {
  const long nc = (n + kDotChunk - 1) / kDotChunk;
  std::vector<double> part(static_cast<size_t>(nc));
#pragma omp parallel for schedule(static)
  for (long b = 0; b < nc; ++b) {
    double s = 0.0;
    const long e = std::min(n, (b + 1) * kDotChunk);
    for (long i = b * kDotChunk; i < e; ++i) s += x[i] * y[i];
    part[static_cast<size_t>(b)] = s;
  }
  double s = 0.0;
  for (long b = 0; b < nc; ++b) s += part[static_cast<size_t>(b)];
  return s;
}

// inc/cost.hpp:51-76 - counted length-n kernels.
double dot(const double* x, const double* y, long n, Cost& c) {
  ++c.dots;
  ++c.vops;
  if (g_variant != 0) return blocked_sum(x, y, n);
  double s = 0.0;
  for (long i = 0; i < n; ++i) s += x[i] * y[i];
  return s;
}
double norm(const double* x, long n, Cost& c) {
  ++c.dots;
  ++c.vops;
  if (g_variant != 0) return std::sqrt(blocked_sum(x, x, n));
  double s = 0.0;
  for (long i = 0; i < n; ++i) s += x[i] * x[i];
  return std::sqrt(s);
}
void axpy(double a, const double* x, double* y, long n, Cost& c) {
  ++c.vops;
#pragma omp parallel for schedule(static)
  for (long i = 0; i < n; ++i) y[i] += a * x[i];
}
void scale(double* x, double a, long n, Cost& c) {
  ++c.vops;
#pragma omp parallel for schedule(static)
  for (long i = 0; i < n; ++i) x[i] *= a;
}

// ------------------------------------------------------------------- rng --
// Frozen stream definition; restated
// independently of the product's ppa/rng.hpp.
namespace rng {
inline uint64_t sm(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline uint64_t key(uint64_t seed, uint64_t stream) {
  return sm(seed * 0x9E3779B97F4A7C15ull + stream * 0xD1B54A32D192ED03ull +
            0x8BB84B93962EACC9ull);
}
inline double unif(uint64_t k, uint64_t c) {
  const uint64_t r = sm(k + (c + 1) * 0x9E3779B97F4A7C15ull);
  return (static_cast<double>(r >> 11) + 0.5) * 0x1p-53;
}
inline double gauss(uint64_t k, uint64_t i) {
  const uint64_t pr = i / 2;
  const double a = unif(k, 2 * pr), b = unif(k, 2 * pr + 1);
  const double rad = std::sqrt(-2.0 * std::log(a));
  const double ang = 6.283185307179586 * b;
  return (i % 2 == 0) ? rad * std::cos(ang) : rad * std::sin(ang);
}
Vec gauss_vec(long n, uint64_t seed, uint64_t stream) {
  Vec v(n);
  const uint64_t k = key(seed, stream);
  for (long i = 0; i < n; ++i) v[i] = gauss(k, static_cast<uint64_t>(i));
  return v;
}
enum : uint64_t { NORM = 1, POLY = 2, ARNOLDI = 3, POLY2 = 4, MATRIX = 5 };
}  // namespace rng

// ------------------------------------------------------------------- csr --
struct Csr {
  int n = 0;
  std::vector<int> rp, ci;
  Vec v;
  long long nnz() const { return static_cast<long long>(v.size()); }
  double nnzr() const { return n > 0 ? double(nnz()) / n : 0.0; }

  // src/operators.cpp:12-37
  void validate() const {
    if (n < 0) throw std::invalid_argument("CsrMatrix: negative dimension");
    if (rp.size() != static_cast<size_t>(n) + 1)
      throw std::invalid_argument("CsrMatrix: row_ptr length must be n+1");
    if (rp.front() != 0 || rp.back() != nnz())
      throw std::invalid_argument("CsrMatrix: row_ptr endpoints invalid");
    for (int i = 0; i < n; ++i) {
      if (rp[i + 1] < rp[i]) throw std::invalid_argument("CsrMatrix: row_ptr not nondecreasing");
      for (int p = rp[i]; p < rp[i + 1]; ++p) {
        if (ci[p] < 0 || ci[p] >= n)
          throw std::invalid_argument("CsrMatrix: column index out of range");
        if (p > rp[i] && ci[p] <= ci[p - 1])
          throw std::invalid_argument("CsrMatrix: columns not strictly increasing within a row");
      }
    }
    if (ci.size() != v.size()) throw std::invalid_argument("CsrMatrix: col_idx/values size mismatch");
  }

  // src/operators.cpp:39-48: sequential sum per row (row loop parallel).
  void multiply(const double* x, double* y) const {
#pragma omp parallel for schedule(static, 4096)
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int p = rp[i]; p < rp[i + 1]; ++p) s += v[p] * x[ci[p]];
      y[i] = s;
    }
  }
};

// src/operators.cpp:50-78 (stable sort: duplicate sums in input order).
Csr from_triplets(int n, std::vector<std::tuple<int, int, double>> t) {
  std::stable_sort(t.begin(), t.end(), [](const auto& a, const auto& b) {
    return std::make_pair(std::get<0>(a), std::get<1>(a)) <
           std::make_pair(std::get<0>(b), std::get<1>(b));
  });
  Csr m;
  m.n = n;
  m.rp.assign(n + 1, 0);
  for (size_t p = 0; p < t.size(); ++p) {
    auto [i, j, val] = t[p];
    if (i < 0 || i >= n || j < 0 || j >= n)
      throw std::invalid_argument("from_triplets: index out of range");
    if (!m.ci.empty() && p > 0 && std::get<0>(t[p - 1]) == i && std::get<1>(t[p - 1]) == j) {
      m.v.back() += val;
      continue;
    }
    m.ci.push_back(j);
    m.v.push_back(val);
    ++m.rp[i + 1];
  }
  for (int i = 0; i < n; ++i) m.rp[i + 1] += m.rp[i];
  m.validate();
  return m;
}

// ------------------------------------------------------------ generators --
// src/operators.cpp:190-244 (two-region convection-diffusion).
Csr gen_convdiff_ref(int N) {
  if (N < 2) throw std::invalid_argument("make_convection_diffusion: grid_n < 2");
  Csr m;
  m.n = N * N;
  m.rp.assign(m.n + 1, 0);
  const double h = 1.0 / (N + 1);
  int pos = 0;
  for (int iy = 0; iy < N; ++iy) {
    const double y = (iy + 1) * h;
    const bool lower = y <= 0.5 + 1e-14;
    const double eps = lower ? 1.0 : 100.0;
    const double c = lower ? 20.0 : 2000.0;
    const double center = 4.0 * eps / (h * h);
    const double east = -eps / (h * h) + c / (2.0 * h);
    const double west = -eps / (h * h) - c / (2.0 * h);
    const double ns = -eps / (h * h);
    for (int ix = 0; ix < N; ++ix) {
      if (iy > 0) { m.ci.push_back((iy - 1) * N + ix); m.v.push_back(ns); ++pos; }
      if (ix > 0) { m.ci.push_back(iy * N + ix - 1); m.v.push_back(west); ++pos; }
      m.ci.push_back(iy * N + ix); m.v.push_back(center); ++pos;
      if (ix + 1 < N) { m.ci.push_back(iy * N + ix + 1); m.v.push_back(east); ++pos; }
      if (iy + 1 < N) { m.ci.push_back((iy + 1) * N + ix); m.v.push_back(ns); ++pos; }
      m.rp[iy * N + ix + 1] = pos;
    }
  }
  m.validate();
  return m;
}

// Configs 2/5: constant coefficients, beta = 2 Pe / h.
Csr gen_convdiff_const(int N, double pe) {
  if (N < 2) throw std::invalid_argument("make_convection_diffusion_const: grid_n < 2");
  Csr m;
  m.n = N * N;
  m.rp.assign(static_cast<size_t>(m.n) + 1, 0);
  m.ci.reserve(5ull * m.n);
  m.v.reserve(5ull * m.n);
  const double h = 1.0 / (N + 1);
  const double beta = 2.0 * pe / h;
  const double C = 4.0 / (h * h), E = -1.0 / (h * h) + beta / (2.0 * h),
               W = -1.0 / (h * h) - beta / (2.0 * h), S = -1.0 / (h * h);
  for (int iy = 0; iy < N; ++iy)
    for (int ix = 0; ix < N; ++ix) {
      const int r = iy * N + ix;
      if (iy > 0) { m.ci.push_back(r - N); m.v.push_back(S); }
      if (ix > 0) { m.ci.push_back(r - 1); m.v.push_back(W); }
      m.ci.push_back(r); m.v.push_back(C);
      if (ix + 1 < N) { m.ci.push_back(r + 1); m.v.push_back(E); }
      if (iy + 1 < N) { m.ci.push_back(r + N); m.v.push_back(S); }
      m.rp[r + 1] = static_cast<int>(m.ci.size());
    }
  m.validate();
  return m;
}

// Config 3: 7-point Laplacian, index (iz*N + iy)*N + ix, 1/h^2 scaling.
Csr gen_laplace3d(int N) {
  if (N < 2) throw std::invalid_argument("make_laplacian_3d: grid_n < 2");
  Csr m;
  m.n = N * N * N;
  m.rp.assign(static_cast<size_t>(m.n) + 1, 0);
  m.ci.reserve(7ull * m.n);
  m.v.reserve(7ull * m.n);
  const double h = 1.0 / (N + 1);
  const double C = 6.0 / (h * h), O = -1.0 / (h * h);
  const int P = N * N;
  for (int iz = 0; iz < N; ++iz)
    for (int iy = 0; iy < N; ++iy)
      for (int ix = 0; ix < N; ++ix) {
        const int r = (iz * N + iy) * N + ix;
        if (iz > 0) { m.ci.push_back(r - P); m.v.push_back(O); }
        if (iy > 0) { m.ci.push_back(r - N); m.v.push_back(O); }
        if (ix > 0) { m.ci.push_back(r - 1); m.v.push_back(O); }
        m.ci.push_back(r); m.v.push_back(C);
        if (ix + 1 < N) { m.ci.push_back(r + 1); m.v.push_back(O); }
        if (iy + 1 < N) { m.ci.push_back(r + N); m.v.push_back(O); }
        if (iz + 1 < N) { m.ci.push_back(r + P); m.v.push_back(O); }
        m.rp[r + 1] = static_cast<int>(m.ci.size());
      }
  m.validate();
  return m;
}

// Config 1: upper bidiagonal, a_ii = i (1-based), superdiagonal 1.
Csr gen_bidiag(int n) {
  if (n < 1) throw std::invalid_argument("make_bidiagonal: n < 1");
  Csr m;
  m.n = n;
  m.rp.assign(n + 1, 0);
  for (int i = 0; i < n; ++i) {
    m.ci.push_back(i);
    m.v.push_back(i + 1.0);
    if (i + 1 < n) {
      m.ci.push_back(i + 1);
      m.v.push_back(1.0);
    }
    m.rp[i + 1] = static_cast<int>(m.ci.size());
  }
  m.validate();
  return m;
}

// Config 4: per-row stream; L = max(1, Poisson(lambda)) by Knuth's product
// method; columns uniform != i; values N(0,1)/8; diagonal (i+1)/n*10;
// duplicates summed in draw order (diagonal first).
Csr gen_random_poisson(int n, double lambda, uint64_t seed) {
  if (n < 2) throw std::invalid_argument("make_random_poisson: n < 2");
  const uint64_t mk = rng::key(seed, rng::MATRIX);
  const double lim = std::exp(-lambda);
  Csr m;
  m.n = n;
  m.rp.assign(static_cast<size_t>(n) + 1, 0);
  std::vector<std::pair<int, double>> ent;
  for (int i = 0; i < n; ++i) {
    const uint64_t rk = rng::sm(mk + (static_cast<uint64_t>(i) + 1) * 0xD1B54A32D192ED03ull);
    uint64_t ctr = 0;
    auto U = [&]() { return rng::unif(rk, ctr++); };
    int L = 0;
    double prod = 1.0;
    for (;;) {
      prod *= U();
      ++L;
      if (!(prod > lim)) break;
    }
    L = L - 1 < 1 ? 1 : L - 1;
    ent.assign(1, {i, (i + 1.0) / n * 10.0});
    for (int e = 0; e < L; ++e) {
      int j = i;
      while (j == i) {
        j = static_cast<int>(U() * n);
        if (j >= n) j = n - 1;
      }
      const double a = U(), b = U();
      ent.push_back({j, std::sqrt(-2.0 * std::log(a)) * std::cos(6.283185307179586 * b) / 8.0});
    }
    std::stable_sort(ent.begin(), ent.end(),
                     [](const auto& x, const auto& y) { return x.first < y.first; });
    for (size_t e = 0; e < ent.size(); ++e) {
      if (e > 0 && ent[e].first == ent[e - 1].first) {
        m.v.back() += ent[e].second;
      } else {
        m.ci.push_back(ent[e].first);
        m.v.push_back(ent[e].second);
      }
    }
    m.rp[i + 1] = static_cast<int>(m.ci.size());
  }
  m.validate();
  return m;
}

Csr gen_config(int c) {
  switch (c) {
    case 1: return gen_bidiag(5000);
    case 2: return gen_convdiff_const(1000, 0.5);
    case 3: return gen_laplace3d(160);
    case 4: return gen_random_poisson(2000000, 16.0, 4);
    case 5: return gen_convdiff_const(2048, 0.5);
  }
  throw std::invalid_argument("config must be 1..5");
}

uint64_t fingerprint(const Csr& m) {
  uint64_t h = 14695981039346656037ull;
  auto feed = [&](const void* p, size_t len) {
    const uint8_t* b = static_cast<const uint8_t*>(p);
    for (size_t i = 0; i < len; ++i) h = (h ^ b[i]) * 1099511628211ull;
  };
  feed(&m.n, 4);
  feed(m.rp.data(), m.rp.size() * 4);
  feed(m.ci.data(), m.ci.size() * 4);
  feed(m.v.data(), m.v.size() * 8);
  return h;
}

// ------------------------------------------------------------- operators --
// inc/operators.hpp:49-76
class Op {
 public:
  virtual ~Op() = default;
  virtual int dim() const = 0;
  virtual void apply(const double* x, double* y, Cost& c) const = 0;
  virtual int mvps_per_apply() const = 0;
  virtual const Vec* diagonal() const { return nullptr; }
  virtual double nnzr() const = 0;
};
using OpPtr = std::shared_ptr<const Op>;

// src/operators.cpp:113-130
class CsrOp final : public Op {
 public:
  explicit CsrOp(Csr m, bool diag = false) : m_(std::move(m)), is_diag_(diag) {
    m_.validate();
    if (is_diag_) diag_ = m_.v;
  }
  int dim() const override { return m_.n; }
  int mvps_per_apply() const override { return 1; }
  double nnzr() const override { return m_.nnzr(); }
  const Vec* diagonal() const override { return is_diag_ ? &diag_ : nullptr; }
  void apply(const double* x, double* y, Cost& c) const override {
    ++c.mvps;
    m_.multiply(x, y);
  }
  const Csr& csr() const { return m_; }

 private:
  Csr m_;
  bool is_diag_;
  Vec diag_;
};

// src/operators.cpp:132-150
class Block2Op final : public Op {
 public:
  explicit Block2Op(OpPtr a) : a_(std::move(a)) {}
  int dim() const override { return 2 * a_->dim(); }
  int mvps_per_apply() const override { return 2 * a_->mvps_per_apply(); }
  double nnzr() const override { return a_->nnzr(); }
  void apply(const double* x, double* y, Cost& c) const override {
    const long n = a_->dim();
    a_->apply(x, y, c);
    a_->apply(x + n, y + n, c);
  }

 private:
  OpPtr a_;
};

// src/operators.cpp:152-170
class ShiftedOp final : public Op {
 public:
  ShiftedOp(OpPtr a, double mu) : a_(std::move(a)), mu_(mu) {}
  int dim() const override { return a_->dim(); }
  int mvps_per_apply() const override { return a_->mvps_per_apply(); }
  double nnzr() const override { return a_->nnzr(); }
  void apply(const double* x, double* y, Cost& c) const override {
    a_->apply(x, y, c);
    if (mu_ != 0.0) axpy(-mu_, x, y, dim(), c);
  }

 private:
  OpPtr a_;
  double mu_;
};

// src/operators.cpp:246-305
Csr read_matrix_market(const std::string& path) {
  FILE* f = std::fopen(path.c_str(), "r");
  if (!f) throw std::runtime_error("read_matrix_market: cannot open " + path);
  std::string text;
  char buf[1 << 16];
  size_t got;
  while ((got = std::fread(buf, 1, sizeof(buf), f)) > 0) text.append(buf, got);
  std::fclose(f);
  size_t pos = 0;
  auto next_line = [&](std::string& line) {
    if (pos >= text.size()) return false;
    size_t e = text.find('\n', pos);
    if (e == std::string::npos) e = text.size();
    line = text.substr(pos, e - pos);
    pos = e + 1;
    return true;
  };
  std::string line;
  if (!next_line(line)) throw std::runtime_error("read_matrix_market: empty file");
  char b1[64] = {0}, b2[64] = {0}, b3[64] = {0}, b4[64] = {0}, b5[64] = {0};
  std::sscanf(line.c_str(), "%63s %63s %63s %63s %63s", b1, b2, b3, b4, b5);
  auto low = [](std::string s) {
    for (char& ch : s) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
    return s;
  };
  const std::string obj = low(b2), fmt = low(b3), field = low(b4), sym = low(b5);
  if (std::string(b1) != "%%MatrixMarket" || obj != "matrix" || fmt != "coordinate")
    throw std::runtime_error("read_matrix_market: malformed header");
  if (field != "real")
    throw std::runtime_error("read_matrix_market: unsupported field '" + field + "' (only real)");
  if (sym != "general" && sym != "symmetric")
    throw std::runtime_error("read_matrix_market: unsupported symmetry '" + sym + "'");
  while (next_line(line))
    if (!line.empty() && line[0] != '%') break;
  long long rows = 0, cols = 0, entries = 0;
  if (std::sscanf(line.c_str(), "%lld %lld %lld", &rows, &cols, &entries) != 3 || rows <= 0 ||
      cols <= 0)
    throw std::runtime_error("read_matrix_market: bad size line");
  if (rows != cols) throw std::runtime_error("read_matrix_market: matrix must be square");
  std::vector<std::tuple<int, int, double>> t;
  const char* p = text.c_str() + std::min(pos, text.size());
  for (long long e = 0; e < entries; ++e) {
    long long i, j;
    double v;
    int used = 0;
    if (std::sscanf(p, " %lld %lld %lf%n", &i, &j, &v, &used) != 3)
      throw std::runtime_error("read_matrix_market: truncated entry list");
    p += used;
    if (i < 1 || i > rows || j < 1 || j > cols)
      throw std::runtime_error("read_matrix_market: index out of range");
    t.emplace_back(int(i - 1), int(j - 1), v);
    if (sym == "symmetric" && i != j) t.emplace_back(int(j - 1), int(i - 1), v);
  }
  return from_triplets(static_cast<int>(rows), std::move(t));
}

// ----------------------------------------------------------------- dense --
struct Mat {
  int r = 0, c = 0;
  Vec a;
  Mat() = default;
  Mat(int rows, int cols) : r(rows), c(cols), a(static_cast<size_t>(rows) * cols, 0.0) {}
  double& operator()(int i, int j) { return a[static_cast<size_t>(j) * r + i]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(j) * r + i]; }
};

// Eigen::EigenSolver stand-in: LAPACK dgeevx, no balancing.
bool eigen(const Mat& A, std::vector<cd>& w, std::vector<cd>* V) {
  const int n = A.r;
  Mat a = A;
  Vec wr(n), wi(n), vr(V ? static_cast<size_t>(n) * n : 1), sc(n), rce(n), rcv(n);
  std::vector<int> iw(std::max(1, 2 * n - 2));
  int ilo, ihi, info = 0, one = 1, ldvr = V ? n : 1, lw = -1;
  double ab, wq, vl;
  const char* jv = V ? "V" : "N";
  scipy_dgeevx_("N", "N", jv, "N", &n, a.a.data(), &n, wr.data(), wi.data(), &vl, &one,
                vr.data(), &ldvr, &ilo, &ihi, sc.data(), &ab, rce.data(), rcv.data(), &wq, &lw,
                iw.data(), &info, 1, 1, 1, 1);
  lw = std::max(1, static_cast<int>(wq));
  Vec work(lw);
  scipy_dgeevx_("N", "N", jv, "N", &n, a.a.data(), &n, wr.data(), wi.data(), &vl, &one,
                vr.data(), &ldvr, &ilo, &ihi, sc.data(), &ab, rce.data(), rcv.data(),
                work.data(), &lw, iw.data(), &info, 1, 1, 1, 1);
  if (info) return false;
  w.resize(n);
  for (int i = 0; i < n; ++i) w[i] = cd(wr[i], wi[i]);
  if (V) {
    V->assign(static_cast<size_t>(n) * n, cd());
    for (int j = 0; j < n; ++j) {
      if (wi[j] == 0.0) {
        for (int i = 0; i < n; ++i) (*V)[static_cast<size_t>(j) * n + i] = vr[static_cast<size_t>(j) * n + i];
      } else {
        for (int i = 0; i < n; ++i) {
          const double re = vr[static_cast<size_t>(j) * n + i], im = vr[static_cast<size_t>(j + 1) * n + i];
          (*V)[static_cast<size_t>(j) * n + i] = cd(re, im);
          (*V)[static_cast<size_t>(j + 1) * n + i] = cd(re, -im);
        }
        ++j;
      }
    }
  }
  return true;
}

// Eigen::FullPivLU<MatrixXd>(M).isInvertible() + solve, via dgetc2/dgesc2.
bool fullpiv_solve(const Mat& M, Vec& rhs) {
  const int n = M.r;
  Mat a = M;
  std::vector<int> ip(n), jp(n);
  int info = 0;
  scipy_dgetc2_(&n, a.a.data(), &n, ip.data(), jp.data(), &info);
  double mx = 0.0;
  for (int i = 0; i < n; ++i) mx = std::max(mx, std::abs(a(i, i)));
  if (info || mx == 0.0) return false;
  const double thr = std::numeric_limits<double>::epsilon() * n * mx;
  for (int i = 0; i < n; ++i)
    if (!(std::abs(a(i, i)) > thr)) return false;
  double scl = 1.0;
  scipy_dgesc2_(&n, a.a.data(), &n, rhs.data(), ip.data(), jp.data(), &scl);
  if (scl != 1.0)
    for (double& x : rhs) x /= scl;
  return true;
}

// Eigen::HouseholderQR(G).householderQ() * Identity(m, k)
Mat thin_q(const Mat& G) {
  const int m = G.r, k = G.c;
  Mat a = G;
  Vec tau(std::max(1, k));
  int info = 0, lw = -1;
  double wq;
  scipy_dgeqrf_(&m, &k, a.a.data(), &m, tau.data(), &wq, &lw, &info);
  lw = std::max(1, static_cast<int>(wq));
  Vec w(lw);
  scipy_dgeqrf_(&m, &k, a.a.data(), &m, tau.data(), w.data(), &lw, &info);
  lw = -1;
  scipy_dorgqr_(&m, &k, &k, a.a.data(), &m, tau.data(), &wq, &lw, &info);
  lw = std::max(1, static_cast<int>(wq));
  w.assign(lw, 0.0);
  scipy_dorgqr_(&m, &k, &k, a.a.data(), &m, tau.data(), w.data(), &lw, &info);
  if (info) throw std::runtime_error("thin_q: LAPACK failure");
  return a;
}

// --------------------------------------------------------------- arnoldi --
// inc/arnoldi.hpp:18-26: V n x (m+1), H (m+1) x m.
struct State {
  int n = 0;
  Vec V;  // column-major, ld = n
  Mat H;
  int max_dim = 0, cur_dim = 0, restart_k = 0, cycle_count = 0;
  bool breakdown = false;
  double* col(int j) { return V.data() + static_cast<size_t>(j) * n; }
  const double* col(int j) const { return V.data() + static_cast<size_t>(j) * n; }
};

constexpr double kBreakdownTol = 1e-14;  // src/arnoldi.cpp:15
constexpr double kPairTol = 1e-10;       // src/arnoldi.cpp:16

bool a_is_complex(const cd& z) { return std::abs(z.imag()) > kPairTol * std::max(1.0, std::abs(z)); }
bool a_is_pair(const cd& a, const cd& b) {
  return std::abs(a - std::conj(b)) <= kPairTol * std::max(1.0, std::abs(a));
}

enum Ordering { SMALLEST = 0, LARGEST = 1, TARGET_ONE = 2 };

double okey(const cd& z, int ord) {
  if (ord == SMALLEST) return std::abs(z);
  if (ord == LARGEST) return -std::abs(z);
  return std::abs(1.0 - z);
}

struct Ritz {
  std::vector<cd> values;
  std::vector<cd> vec;  // d x count, column-major
  int d = 0;
  Vec residuals;
  int ordering = SMALLEST;
  int count() const { return static_cast<int>(values.size()); }
  cd& g(int i, int j) { return vec[static_cast<size_t>(j) * d + i]; }
  const cd& g(int i, int j) const { return vec[static_cast<size_t>(j) * d + i]; }
};

// src/arnoldi.cpp:40-95
void sort_pairs(Ritz& s) {
  const int d = s.count();
  std::vector<int> idx(d);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
    return okey(s.values[a], s.ordering) < okey(s.values[b], s.ordering);
  });
  std::vector<int> arr;
  std::vector<bool> used(d, false);
  for (int r = 0; r < d; ++r) {
    const int i = idx[r];
    if (used[i]) continue;
    used[i] = true;
    if (!a_is_complex(s.values[i])) { arr.push_back(i); continue; }
    int mate = -1;
    for (int q = 0; q < d; ++q) {
      const int j = idx[q];
      if (!used[j] && a_is_pair(s.values[i], s.values[j])) { mate = j; break; }
    }
    if (mate < 0) { arr.push_back(i); continue; }
    used[mate] = true;
    if (s.values[i].imag() >= 0.0) { arr.push_back(i); arr.push_back(mate); }
    else { arr.push_back(mate); arr.push_back(i); }
  }
  Ritz t = s;
  for (int r = 0; r < d; ++r) {
    t.values[r] = s.values[arr[r]];
    t.residuals[r] = s.residuals[arr[r]];
    for (int i = 0; i < s.d; ++i) t.g(i, r) = s.g(i, arr[r]);
  }
  s = std::move(t);
}

// src/arnoldi.cpp:99-113
State arnoldi_init(const Vec& v0, int m, Cost& c) {
  if (m < 1) throw std::invalid_argument("arnoldi_init: m < 1");
  if (static_cast<long>(v0.size()) < m + 1) throw std::invalid_argument("arnoldi_init: m+1 exceeds dimension");
  State st;
  st.n = static_cast<int>(v0.size());
  st.max_dim = m;
  st.V.assign(static_cast<size_t>(st.n) * (m + 1), 0.0);
  st.H = Mat(m + 1, m);
  const double nb = norm(v0.data(), st.n, c);
  if (nb == 0.0) throw std::invalid_argument("arnoldi_init: zero start");
  std::copy(v0.begin(), v0.end(), st.col(0));
  scale(st.col(0), 1.0 / nb, st.n, c);
  return st;
}

// src/arnoldi.cpp:115-152: MGS + one MGS reorthogonalisation pass.
void arnoldi_extend(State& st, const Op& op, int to_dim, Cost& c) {
  if (to_dim > st.max_dim) throw std::invalid_argument("arnoldi_extend: to_dim > max_dim");
  if (to_dim <= st.cur_dim) throw std::invalid_argument("arnoldi_extend: to_dim <= cur_dim");
  if (op.dim() != st.n) throw std::invalid_argument("arnoldi_extend: dimension mismatch");
  const long n = st.n;
  Vec w(n);
  for (int j = st.cur_dim; j < to_dim; ++j) {
    op.apply(st.col(j), w.data(), c);
    if (g_variant == 1) {
      // roundoff-floor variant 1: classical Gram-Schmidt, two passes
      std::vector<double> h(static_cast<size_t>(j) + 1);
      for (int pass = 0; pass < 2; ++pass) {
        for (int i = 0; i <= j; ++i) h[i] = dot(st.col(i), w.data(), n, c);
        for (int i = 0; i <= j; ++i) {
          st.H(i, j) = pass == 0 ? h[i] : st.H(i, j) + h[i];
          axpy(-h[i], st.col(i), w.data(), n, c);
        }
      }
    } else {
      for (int i = 0; i <= j; ++i) {
        const double h = dot(st.col(i), w.data(), n, c);
        st.H(i, j) = h;
        axpy(-h, st.col(i), w.data(), n, c);
      }
      for (int i = 0; i <= j; ++i) {
        const double h = dot(st.col(i), w.data(), n, c);
        st.H(i, j) += h;
        axpy(-h, st.col(i), w.data(), n, c);
      }
    }
    const double hsub = norm(w.data(), n, c);
    st.H(j + 1, j) = hsub;
    st.cur_dim = j + 1;
    double cn = 0.0;
    for (int i = 0; i <= j + 1; ++i) cn += st.H(i, j) * st.H(i, j);
    if (hsub <= kBreakdownTol * std::sqrt(cn)) {
      st.H(j + 1, j) = 0.0;
      st.breakdown = true;
      return;
    }
    double* dst = st.col(j + 1);
    for (long i = 0; i < n; ++i) dst[i] = w[i] / hsub;
    ++c.vops;
  }
}

Mat lead(const State& st, int d) {
  Mat M(d, d);
  for (int j = 0; j < d; ++j)
    for (int i = 0; i < d; ++i) M(i, j) = st.H(i, j);
  return M;
}

// src/arnoldi.cpp:154-176
Ritz ritz_pairs(const State& st, int ord) {
  const int d = st.cur_dim;
  if (d < 1) throw std::invalid_argument("ritz_pairs: empty state");
  Ritz s;
  s.ordering = ord;
  s.d = d;
  if (!eigen(lead(st, d), s.values, &s.vec)) throw std::runtime_error("ritz_pairs: Hessenberg eigensolver failed");
  s.residuals.resize(d);
  const double hsub = st.H(d, d - 1);
  for (int i = 0; i < d; ++i) {
    double nn = 0.0;
    for (int r = 0; r < d; ++r) nn += std::norm(s.g(r, i));
    nn = std::sqrt(nn);
    for (int r = 0; r < d; ++r) s.g(r, i) /= nn;
    s.residuals[i] = std::abs(hsub) * std::abs(s.g(d - 1, i));
  }
  sort_pairs(s);
  return s;
}

// src/arnoldi.cpp:178-206
std::vector<cd> harmonic_ritz_values(const State& st) {
  const int d = st.cur_dim;
  if (d < 1) throw std::invalid_argument("harmonic_ritz_values: empty state");
  Mat M = lead(st, d);
  const double hsub = st.H(d, d - 1);
  if (hsub != 0.0) {
    Mat T(d, d);
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) T(i, j) = M(j, i);
    Vec f(d, 0.0);
    f[d - 1] = 1.0;
    if (!fullpiv_solve(T, f))
      throw std::runtime_error(
          "harmonic_ritz_values: singular projection (GMRES stagnation); try a different starting vector");
    for (int i = 0; i < d; ++i) M(i, d - 1) += (hsub * hsub) * f[i];
  }
  std::vector<cd> w;
  if (!eigen(M, w, nullptr)) throw std::runtime_error("harmonic_ritz_values: eigensolver failed");
  return w;
}

// src/arnoldi.cpp:208-246: harmonic selection for restarting.  The
// eigenpairs of H_d + h^2 f e_d^T (f = H_d^{-T} e_d), unit vectors, and the
// exact subspace residual ||[H_d g - theta g ; h g_d]||.
Ritz harmonic_restart_selection(const State& st, int ord) {
  const int d = st.cur_dim;
  if (d < 1) throw std::invalid_argument("harmonic_restart_selection: empty");
  const Mat Hd = lead(st, d);
  Mat M = Hd;
  const double hsub = st.H(d, d - 1);
  if (hsub != 0.0) {
    Mat T(d, d);
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) T(i, j) = Hd(j, i);
    Vec f(d, 0.0);
    f[d - 1] = 1.0;
    if (!fullpiv_solve(T, f))
      throw std::runtime_error(
          "harmonic_restart_selection: singular projection; try a different starting vector");
    for (int i = 0; i < d; ++i) M(i, d - 1) += (hsub * hsub) * f[i];
  }
  Ritz s;
  s.ordering = ord;
  s.d = d;
  if (!eigen(M, s.values, &s.vec))
    throw std::runtime_error("harmonic_restart_selection: eigensolver failed");
  s.residuals.resize(d);
  for (int i = 0; i < d; ++i) {
    double nn = 0.0;
    for (int r = 0; r < d; ++r) nn += std::norm(s.g(r, i));
    nn = std::sqrt(nn);
    for (int r = 0; r < d; ++r) s.g(r, i) /= nn;
    double top2 = 0.0;
    for (int r = 0; r < d; ++r) {
      cd acc = 0.0;
      for (int q = 0; q < d; ++q) acc += Hd(r, q) * s.g(q, i);
      top2 += std::norm(acc - s.values[i] * s.g(r, i));
    }
    const cd last = hsub * s.g(d - 1, i);
    s.residuals[i] = std::sqrt(top2 + std::norm(last));
  }
  sort_pairs(s);
  return s;
}

// The solve's restart selection (SolveConfig::variant, inc/solver.hpp:31).
Ritz select_pairs(const State& st, int ord, int variant) {
  return variant == 1 ? harmonic_restart_selection(st, ord) : ritz_pairs(st, ord);
}

// src/arnoldi.cpp:252-265: unit Ritz vector (re, im parts).
void ritz_vector(const State& st, const Ritz& s, int j, Vec& yr, Vec& yi, bool& cplx, Cost& c) {
  const int d = s.d;
  if (j < 0 || j >= s.count()) throw std::invalid_argument("ritz_vector: index out of range");
  const long n = st.n;
  double im2 = 0.0;
  for (int r = 0; r < d; ++r) im2 += s.g(r, j).imag() * s.g(r, j).imag();
  cplx = std::sqrt(im2) > 0.0;
  yr.assign(n, 0.0);
  yi.assign(n, 0.0);
  for (int r = 0; r < d; ++r) {
    const double gr = s.g(r, j).real(), gi = s.g(r, j).imag();
    const double* v = st.col(r);
    for (long i = 0; i < n; ++i) {
      yr[i] += v[i] * gr;
      yi[i] += v[i] * gi;
    }
  }
  c.vops += (cplx ? 2 : 1) * d;
  double nn = 0.0;
  for (long i = 0; i < n; ++i) nn += yr[i] * yr[i] + yi[i] * yi[i];
  nn = std::sqrt(nn);
  for (long i = 0; i < n; ++i) {
    yr[i] /= nn;
    yi[i] /= nn;
  }
  c.dots += cplx ? 2 : 1;
  c.vops += cplx ? 4 : 2;
}

// src/arnoldi.cpp:267-334
int thick_restart(State& st, const Ritz& keep, int k, Cost& c) {
  const int m = st.cur_dim;
  if (m != st.max_dim) throw std::invalid_argument("thick_restart: cycle not at full dimension");
  if (k <= 0 || k >= m) throw std::invalid_argument("thick_restart: bad k");
  if (keep.count() < k) throw std::invalid_argument("thick_restart: selection smaller than k");
  if (st.H(m, m - 1) == 0.0) throw std::runtime_error("thick_restart: no residual vector (breakdown)");
  Mat G(m, k);
  int col = 0, j = 0;
  while (col < k && j < keep.count()) {
    if (!a_is_complex(keep.values[j])) {
      for (int r = 0; r < m; ++r) G(r, col) = keep.g(r, j).real();
      ++col;
      ++j;
    } else {
      if (col + 2 > k) break;
      for (int r = 0; r < m; ++r) {
        G(r, col) = keep.g(r, j).real();
        G(r, col + 1) = keep.g(r, j).imag();
      }
      col += 2;
      j += 2;
    }
  }
  const int kk = col;
  if (kk == 0) throw std::invalid_argument("thick_restart: k too small");
  Mat Gk(m, kk);
  for (int cc = 0; cc < kk; ++cc)
    for (int r = 0; r < m; ++r) Gk(r, cc) = G(r, cc);
  const Mat Q = thin_q(Gk);
  // Hk = Q^T Hm Q ; hrow = h_{m+1,m} Q(m-1,:)
  Mat HQ(m, kk), Hk(kk, kk);
  for (int cc = 0; cc < kk; ++cc)
    for (int q = 0; q < m; ++q)
      for (int r = 0; r < m; ++r) HQ(r, cc) += st.H(r, q) * Q(q, cc);
  for (int cc = 0; cc < kk; ++cc)
    for (int r = 0; r < kk; ++r) {
      double s = 0.0;
      for (int q = 0; q < m; ++q) s += Q(q, r) * HQ(q, cc);
      Hk(r, cc) = s;
    }
  Vec hrow(kk);
  for (int cc = 0; cc < kk; ++cc) hrow[cc] = st.H(m, m - 1) * Q(m - 1, cc);
  // V(:,0:kk) = V(:,0:m) Q
  const long n = st.n;
  Vec NV(static_cast<size_t>(n) * kk, 0.0);
#pragma omp parallel for schedule(static)
  for (long i = 0; i < n; ++i)
    for (int cc = 0; cc < kk; ++cc) {
      double s = 0.0;
      for (int q = 0; q < m; ++q) s += st.V[static_cast<size_t>(q) * n + i] * Q(q, cc);
      NV[static_cast<size_t>(cc) * n + i] = s;
    }
  std::copy(NV.begin(), NV.end(), st.V.begin());
  c.vops += static_cast<long long>(m) * kk;
  std::copy(st.col(m), st.col(m) + n, st.col(kk));
  Vec corr(kk, 0.0);
  for (int i = 0; i < kk; ++i) {
    const double h = dot(st.col(i), st.col(kk), n, c);
    corr[i] = h;
    axpy(-h, st.col(i), st.col(kk), n, c);
  }
  const double rn = norm(st.col(kk), n, c);
  scale(st.col(kk), 1.0 / rn, n, c);
  for (int cc = 0; cc < kk; ++cc)
    for (int r = 0; r < kk; ++r) Hk(r, cc) += corr[r] * hrow[cc];
  std::fill(st.H.a.begin(), st.H.a.end(), 0.0);
  for (int cc = 0; cc < kk; ++cc) {
    for (int r = 0; r < kk; ++r) st.H(r, cc) = Hk(r, cc);
    st.H(kk, cc) = rn * hrow[cc];
  }
  st.cur_dim = kk;
  st.restart_k = kk;
  ++st.cycle_count;
  return kk;
}

// Harmonic thick restart (our decision for RestartVariant::harmonic,
// DESIGN.md section 5; SPEC.md:178 asks the restart to keep the Krylov
// property): keep span{[G; 0], p} with p = [-h f; 1], H_m^T f = e_m, the
// direction every harmonic residual Hbar g - theta [g; 0] lies along.
int harmonic_thick_restart(State& st, const Ritz& keep, int k, Cost& c) {
  const int m = st.cur_dim;
  if (m != st.max_dim) throw std::invalid_argument("thick_restart: cycle not at full dimension");
  if (k <= 0 || k >= m) throw std::invalid_argument("thick_restart: bad k");
  if (keep.count() < k) throw std::invalid_argument("thick_restart: selection smaller than k");
  const double hm = st.H(m, m - 1);
  if (hm == 0.0) throw std::runtime_error("thick_restart: no residual vector (breakdown)");
  Mat G(m, k);
  int col = 0, j = 0;
  while (col < k && j < keep.count()) {
    if (!a_is_complex(keep.values[j])) {
      for (int r = 0; r < m; ++r) G(r, col) = keep.g(r, j).real();
      ++col;
      ++j;
    } else {
      if (col + 2 > k) break;
      for (int r = 0; r < m; ++r) {
        G(r, col) = keep.g(r, j).real();
        G(r, col + 1) = keep.g(r, j).imag();
      }
      col += 2;
      j += 2;
    }
  }
  const int kk = col;
  if (kk == 0) throw std::invalid_argument("thick_restart: k too small");
  Mat T(m, m);
  for (int r = 0; r < m; ++r)
    for (int q = 0; q < m; ++q) T(r, q) = st.H(q, r);
  Vec f(m, 0.0);
  f[m - 1] = 1.0;
  if (!fullpiv_solve(T, f))
    throw std::runtime_error("harmonic_restart_selection: singular projection; try a different starting vector");
  Mat P(m + 1, kk + 1);
  for (int cc = 0; cc < kk; ++cc)
    for (int r = 0; r < m; ++r) P(r, cc) = G(r, cc);
  for (int r = 0; r < m; ++r) P(r, kk) = -hm * f[r];
  P(m, kk) = 1.0;
  const Mat Qh = thin_q(P);
  // Hn = Qh^T Hbar Qh(0:m, 0:kk), (kk+1) x kk
  Mat HQ(m + 1, kk), Hn(kk + 1, kk);
  for (int cc = 0; cc < kk; ++cc)
    for (int q = 0; q < m; ++q)
      for (int r = 0; r <= m; ++r) HQ(r, cc) += st.H(r, q) * Qh(q, cc);
  for (int cc = 0; cc < kk; ++cc)
    for (int r = 0; r <= kk; ++r) {
      double s = 0.0;
      for (int q = 0; q <= m; ++q) s += Qh(q, r) * HQ(q, cc);
      Hn(r, cc) = s;
    }
  // V(:,0:kk+1) = V(:,0:m+1) Qh
  const long n = st.n;
  Vec NV(static_cast<size_t>(n) * (kk + 1), 0.0);
#pragma omp parallel for schedule(static)
  for (long i = 0; i < n; ++i)
    for (int cc = 0; cc <= kk; ++cc) {
      double s = 0.0;
      for (int q = 0; q <= m; ++q) s += st.V[static_cast<size_t>(q) * n + i] * Qh(q, cc);
      NV[static_cast<size_t>(cc) * n + i] = s;
    }
  std::copy(NV.begin(), NV.end(), st.V.begin());
  c.vops += static_cast<long long>(m + 1) * (kk + 1);
  Vec corr(kk, 0.0);
  for (int i = 0; i < kk; ++i) {
    const double h = dot(st.col(i), st.col(kk), n, c);
    corr[i] = h;
    axpy(-h, st.col(i), st.col(kk), n, c);
  }
  const double rn = norm(st.col(kk), n, c);
  scale(st.col(kk), 1.0 / rn, n, c);
  std::fill(st.H.a.begin(), st.H.a.end(), 0.0);
  for (int cc = 0; cc < kk; ++cc) {
    for (int r = 0; r < kk; ++r) st.H(r, cc) = Hn(r, cc) + corr[r] * Hn(kk, cc);
    st.H(kk, cc) = rn * Hn(kk, cc);
  }
  st.cur_dim = kk;
  st.restart_k = kk;
  ++st.cycle_count;
  return kk;
}

// ------------------------------------------------------------ gmres_poly --
constexpr double kImagTol = 1e-13;  // src/gmres_poly.cpp:13
constexpr double kLogFloor = -690.0;

bool p_is_complex(const cd& z) { return std::abs(z.imag()) > kImagTol * std::abs(z); }

struct Poly {
  std::vector<cd> roots;
  std::vector<int> mult;
  int base_degree = 0;
  bool truncated = false;
  int eff() const { return static_cast<int>(roots.size()); }
};

std::vector<cd> distinct(const Poly& p) {  // src/gmres_poly.cpp:20-26
  std::vector<cd> out;
  for (const cd& r : p.roots)
    if (std::find(out.begin(), out.end(), r) == out.end()) out.push_back(r);
  return out;
}
void refresh(Poly& p) {  // src/gmres_poly.cpp:28-34
  p.mult.assign(p.roots.size(), 0);
  for (size_t i = 0; i < p.roots.size(); ++i)
    p.mult[i] = static_cast<int>(std::count(p.roots.begin(), p.roots.end(), p.roots[i]));
}

// src/gmres_poly.cpp:38-93
std::vector<cd> leja_order(const std::vector<cd>& roots) {
  const int d = static_cast<int>(roots.size());
  if (d == 0) throw std::invalid_argument("leja_order: empty root list");
  for (const cd& r : roots)
    if (r == cd(0.0, 0.0)) throw std::invalid_argument("leja_order: zero root");
  std::vector<cd> out;
  std::vector<bool> used(d, false);
  auto take_conj = [&](int i) {
    for (int k = 0; k < d; ++k) {
      if (!used[k] && k != i && std::abs(roots[k] - std::conj(roots[i])) <= 1e-10 * std::abs(roots[i])) {
        used[k] = true;
        out.push_back(roots[k]);
        return;
      }
    }
  };
  int first = 0;
  for (int i = 1; i < d; ++i)
    if (std::abs(roots[i]) > std::abs(roots[first])) first = i;
  used[first] = true;
  out.push_back(roots[first]);
  if (p_is_complex(roots[first])) take_conj(first);
  while (static_cast<int>(out.size()) < d) {
    int best = -1;
    double bs = -std::numeric_limits<double>::infinity();
    for (int i = 0; i < d; ++i) {
      if (used[i]) continue;
      double sc = 0.0;
      for (const cd& c : out) {
        const double dist = std::abs(roots[i] - c);
        sc += dist > 0.0 ? std::log(dist) : kLogFloor;
      }
      if (sc > bs) { bs = sc; best = i; }
    }
    used[best] = true;
    out.push_back(roots[best]);
    if (p_is_complex(roots[best])) take_conj(best);
  }
  return out;
}

// src/gmres_poly.cpp:95-115
Poly build_gmres_poly(const Op& a, const Vec& b, int degree, Cost& c) {
  if (degree < 1) throw std::invalid_argument("build_gmres_poly: degree < 1");
  if (static_cast<int>(b.size()) != a.dim()) throw std::invalid_argument("build_gmres_poly: dimension mismatch");
  double bn = 0.0;
  for (double x : b) bn += x * x;
  if (std::sqrt(bn) == 0.0) throw std::invalid_argument("build_gmres_poly: zero starting vector");
  const int d = std::min(degree, a.dim());
  State st = arnoldi_init(b, d, c);
  arnoldi_extend(st, a, d, c);
  Poly p;
  p.roots = leja_order(harmonic_ritz_values(st));
  p.base_degree = p.eff();
  p.truncated = p.base_degree < degree;
  refresh(p);
  return p;
}

// src/gmres_poly.cpp:228-264
Poly build_two_vector_poly(const OpPtr& a, const Vec& b1, const Vec& b2, int degree, Cost& c) {
  const long n = a->dim();
  if (static_cast<long>(b1.size()) != n || static_cast<long>(b2.size()) != n)
    throw std::invalid_argument("build_two_vector_poly: dimension mismatch");
  const double n1 = norm(b1.data(), n, c), n2 = norm(b2.data(), n, c);
  if (n1 == 0.0 || n2 == 0.0) throw std::invalid_argument("build_two_vector_poly: zero starting vector");
  Vec bhat(2 * n);
  for (long i = 0; i < n; ++i) {
    bhat[i] = b1[i] / (n1 * std::sqrt(2.0));
    bhat[n + i] = b2[i] / (n2 * std::sqrt(2.0));
  }
  c.vops += 2;
  const Block2Op block(a);
  return build_gmres_poly(block, bhat, degree, c);
}

// src/gmres_poly.cpp:266-283
Vec damped_start(const Op& a, const Vec& b, double alpha, int power, Cost& c) {
  if (power != 1 && power != 2) throw std::invalid_argument("damped_start: power must be 1 or 2");
  if (alpha < 0.0) throw std::invalid_argument("damped_start: alpha < 0");
  const long n = a.dim();
  Vec w(n);
  a.apply(b.data(), w.data(), c);
  if (power == 2) {
    Vec w2(n);
    a.apply(w.data(), w2.data(), c);
    w.swap(w2);
  } else if (alpha != 0.0) {
    axpy(alpha, b.data(), w.data(), n, c);
  }
  const double nw = norm(w.data(), n, c);
  if (nw == 0.0) throw std::runtime_error("damped_start: damped vector vanished");
  scale(w.data(), 1.0 / nw, n, c);
  return w;
}

// src/gmres_poly.cpp:117-147
void apply_poly(const Poly& p, const Op& a, const double* v, double* out, Cost& c) {
  const long n = a.dim();
  std::copy(v, v + n, out);
  Vec t1(n), t2(n);
  size_t i = 0;
  while (i < p.roots.size()) {
    const cd th = p.roots[i];
    if (!p_is_complex(th)) {
      a.apply(out, t1.data(), c);
      axpy(-1.0 / th.real(), t1.data(), out, n, c);
      i += 1;
    } else {
      if (i + 1 >= p.roots.size() || std::abs(p.roots[i + 1] - std::conj(th)) > 1e-10 * std::abs(th))
        throw std::logic_error("apply_poly: complex root without adjacent conjugate");
      const double inv = 1.0 / std::norm(th);
      const double tr = 2.0 * th.real() * inv;
      a.apply(out, t1.data(), c);
      a.apply(t1.data(), t2.data(), c);
      axpy(-tr, t1.data(), out, n, c);
      axpy(inv, t2.data(), out, n, c);
      i += 2;
    }
  }
}

cd eval_poly(const Poly& p, cd z) {  // src/gmres_poly.cpp:149-153
  cd val(1.0, 0.0);
  for (const cd& th : p.roots) val *= (1.0 - z / th);
  return val;
}

struct Pof {
  Vec lg;
  std::vector<int> copies;
  double maxlg = 0.0;
  int total = 0;
};

Pof compute_pof(const Poly& p) {  // src/gmres_poly.cpp:155-179
  const auto base = distinct(p);
  const int d = static_cast<int>(base.size());
  if (d < 2) throw std::invalid_argument("compute_pof: needs at least two roots");
  Pof r;
  r.lg.resize(d);
  r.copies.resize(d);
  r.maxlg = -std::numeric_limits<double>::infinity();
  for (int j = 0; j < d; ++j) {
    double lg = 0.0;
    for (int i = 0; i < d; ++i) {
      if (i == j) continue;
      const double f = std::abs(1.0 - base[j] / base[i]);
      lg += f > 0.0 ? std::log10(f) : kLogFloor;
    }
    r.lg[j] = lg;
    r.copies[j] = lg > 4.0 ? static_cast<int>(std::ceil((lg - 4.0) / 14.0)) : 0;
    r.total += r.copies[j];
    r.maxlg = std::max(r.maxlg, lg);
  }
  return r;
}

Poly add_stability_roots(const Poly& p, int maxc) {  // src/gmres_poly.cpp:181-226
  const Pof rep = compute_pof(p);
  const auto base = distinct(p);
  Poly out = p;
  std::vector<bool> handled(base.size(), false);
  for (size_t j = 0; j < base.size(); ++j) {
    if (handled[j]) continue;
    handled[j] = true;
    const int c = std::min(rep.copies[j], maxc);
    if (c <= 0) continue;
    const cd th = base[j];
    std::vector<cd> grp{th};
    if (p_is_complex(th)) {
      for (size_t k = 0; k < base.size(); ++k) {
        if (!handled[k] && std::abs(base[k] - std::conj(th)) <= 1e-10 * std::abs(th)) {
          handled[k] = true;
          grp.push_back(base[k]);
          break;
        }
      }
    }
    const long long L = static_cast<long long>(out.roots.size());
    const long long jpos = std::find(out.roots.begin(), out.roots.end(), th) - out.roots.begin();
    std::vector<long long> pos;
    for (int r = 1; r < c; ++r)
      pos.push_back(jpos + static_cast<long long>(std::llround(double(r) * double(L - jpos) / double(c))));
    std::sort(pos.rbegin(), pos.rend());
    out.roots.insert(out.roots.end(), grp.begin(), grp.end());
    for (long long q : pos) out.roots.insert(out.roots.begin() + q, grp.begin(), grp.end());
  }
  refresh(out);
  return out;
}

// src/gmres_poly.cpp:287-318
class PolyOp final : public Op {
 public:
  PolyOp(OpPtr a, Poly p, bool comp) : a_(std::move(a)), p_(std::move(p)), comp_(comp) {}
  int dim() const override { return a_->dim(); }
  int mvps_per_apply() const override { return p_.eff() * a_->mvps_per_apply(); }
  double nnzr() const override { return a_->nnzr(); }
  void apply(const double* x, double* y, Cost& c) const override {
    const long n = dim();
    Vec w(n);
    apply_poly(p_, *a_, x, w.data(), c);
    if (comp_) {
      std::copy(x, x + n, y);
      axpy(-1.0, w.data(), y, n, c);
    } else {
      std::copy(w.begin(), w.end(), y);
    }
  }

 private:
  OpPtr a_;
  Poly p_;
  bool comp_;
};

// ---------------------------------------------------------------- solver --
// SPEC.md [MODULE] solver with the frozen decisions of DESIGN.md (the same
// choices the product implements; restated here independently).
struct Config {
  int m = 50, k = 20, nev = 15, degree = 0;
  double rtol_mult = 1e-8, rtol_abs = 0.0;
  int stability = 0, d1 = 0, d2 = 0, use_double = 0, max_cycles = 100;
  uint64_t seed = 1;
  int allow_nev_above_k = 0;
  int damping = 0;  // 0 off, 1 auto heuristic, 2 forced
  double damping_alpha = 0.0;
  int damping_power = 1;
  int mid_stride = 0;  // > 0: check_mid_cycle with this stride
  int variant = 0;  // RestartVariant: 0 ritz, 1 harmonic (inc/solver.hpp:17)
  int stag_window = 0;  // > 0: stagnation_stop over this many cycles
  double stag_rtol = 0.01;
};

// inc/solver.hpp:96-99: |mu_1| <= ... <= |mu_nev| and
// strictly below every remaining magnitude.
bool check_ideal_order(const std::vector<cd>& mu, int nev) {
  if (nev < 1 || nev > static_cast<int>(mu.size()))
    throw std::invalid_argument("check_ideal_order: need 1 <= nev <= size");
  for (int j = 1; j < nev; ++j)
    if (std::abs(mu[j]) < std::abs(mu[j - 1])) return false;
  for (size_t j = nev; j < mu.size(); ++j)
    if (!(std::abs(mu[nev - 1]) < std::abs(mu[j]))) return false;
  return true;
}

struct Result {
  std::vector<cd> mu;
  Vec res;
  std::vector<int> conv;
  int converged = 0, cycles = 0, composite = 0, discarded = 0;
  double rtol = 0.0, max_err = 0.0, norm_est = 0.0;
  Cost cost;
  Poly poly, inner;
  Vec cycle_max;
};

double norm_estimate(const Op& a, uint64_t seed, Cost& c) {
  if (const Vec* d = a.diagonal()) {
    double mx = 0.0;
    for (double x : *d) mx = std::max(mx, std::abs(x));
    return mx;
  }
  const long n = a.dim();
  Vec x = rng::gauss_vec(n, seed, rng::NORM), y(n);
  const double nx = norm(x.data(), n, c);
  if (nx == 0.0) return 0.0;
  scale(x.data(), 1.0 / nx, n, c);
  double est = 0.0;
  for (int it = 0; it < 5; ++it) {
    a.apply(x.data(), y.data(), c);
    est = norm(y.data(), n, c);
    if (est == 0.0) break;
    if (it + 1 < 5) {
      x = y;
      scale(x.data(), 1.0 / est, n, c);
    }
  }
  return est;
}

void check_and_record(const State& st, const Ritz& s, int nev, const Op& A, Result& R, bool& all,
                      double& mx, Cost& c) {
  const int nchk = std::min(nev, s.count());
  const long n = st.n;
  R.mu.assign(nchk, cd());
  R.res.assign(nchk, 0.0);
  Vec yr, yi, ar(n), ai(n);
  for (int j = 0; j < nchk;) {
    const bool pair = a_is_complex(s.values[j]) && j + 1 < s.count();
    bool cx;
    ritz_vector(st, s, j, yr, yi, cx, c);
    if (!pair) {
      A.apply(yr.data(), ar.data(), c);
      const double mu = dot(yr.data(), ar.data(), n, c);
      Vec r(ar);
      axpy(-mu, yr.data(), r.data(), n, c);
      const double rn = norm(r.data(), n, c);
      R.mu[j] = mu;
      R.res[j] = rn;
      j += 1;
    } else {
      A.apply(yr.data(), ar.data(), c);
      A.apply(yi.data(), ai.data(), c);
      const double a1 = dot(yr.data(), ar.data(), n, c), a2 = dot(yi.data(), ai.data(), n, c);
      const double a3 = dot(yr.data(), ai.data(), n, c), a4 = dot(yi.data(), ar.data(), n, c);
      const cd mu(a1 + a2, a3 - a4);
      double s2 = 0.0;
      for (long i = 0; i < n; ++i) {
        const double rr = ar[i] - (mu.real() * yr[i] - mu.imag() * yi[i]);
        const double ri = ai[i] - (mu.real() * yi[i] + mu.imag() * yr[i]);
        s2 += rr * rr + ri * ri;
      }
      c.vops += 4;
      c.dots += 2;
      c.vops += 2;
      R.mu[j] = mu;
      R.res[j] = std::sqrt(s2);
      if (j + 1 < nchk) {
        R.mu[j + 1] = std::conj(mu);
        R.res[j + 1] = R.res[j];
      }
      j += 2;
    }
  }
  all = nchk == nev;
  mx = 0.0;
  for (double r : R.res) {
    mx = std::max(mx, r);
    all = all && r <= R.rtol;
  }
  R.conv.assign(nchk, 0);
  for (int i = 0; i < nchk; ++i) R.conv[i] = R.res[i] <= R.rtol;
}

void validate(const Config& g) {
  if (g.m < 2) throw std::invalid_argument("SolveConfig: m must be >= 2");
  if (g.k <= 0 || g.k >= g.m) throw std::invalid_argument("SolveConfig: need 0 < k < m");
  if (g.nev <= 0) throw std::invalid_argument("SolveConfig: need nev > 0");
  if (!g.allow_nev_above_k && g.nev > g.k) throw std::invalid_argument("SolveConfig: need nev <= k");
  if (g.nev >= g.m) throw std::invalid_argument("SolveConfig: need nev < m");
  if (g.degree < 0) throw std::invalid_argument("SolveConfig: degree < 0");
  if (g.max_cycles < 1) throw std::invalid_argument("SolveConfig: max_cycles < 1");
}

Result solve(const OpPtr& A, const Config& g) {
  validate(g);
  const auto t0 = std::chrono::steady_clock::now();
  Result R;
  Cost c;
  c.nnzr = A->nnzr();
  const long n = A->dim();
  if (n < g.m + 1) throw std::invalid_argument("solve: dimension must be >= m+1");
  R.norm_est = norm_estimate(*A, g.seed, c);
  R.rtol = g.rtol_abs > 0 ? g.rtol_abs : g.rtol_mult * R.norm_est;
  OpPtr op = A;
  int ord = SMALLEST;
  State probe_state;
  Ritz probe_set;
  std::vector<cd> probe_mu;
  Vec probe_res;
  bool has_probe = false;
  if (g.use_double) {
    if (g.d1 < 1 || g.d2 < 1) throw std::invalid_argument("solve_double: d1, d2 must be >= 1");
    Poly p1 = build_gmres_poly(*A, rng::gauss_vec(n, g.seed, rng::POLY), g.d1, c);
    OpPtr tau = std::make_shared<PolyOp>(A, p1, true);
    Poly p2 = build_gmres_poly(*tau, rng::gauss_vec(n, g.seed, rng::POLY2), g.d2, c);
    if (g.stability && distinct(p2).size() >= 2 && p2.roots.size() >= 2) p2 = add_stability_roots(p2, 1 << 20);
    R.composite = p1.eff() * p2.eff();
    op = std::make_shared<PolyOp>(tau, p2, false);
    R.inner = p1;
    R.poly = p2;
    ord = TARGET_ONE;
  } else if (g.degree > 0) {
    const Vec b = rng::gauss_vec(n, g.seed, rng::POLY);
    auto stab = [&](Poly p) { return (g.stability && p.roots.size() >= 2) ? add_stability_roots(p, 1 << 20) : p; };
    Poly p;
    if (g.damping == 1) {
      // PAPER.md 6.3 / SPEC.md:169-177: probe one Arnoldi(m,k) cycle; on an
      // ideal-order failure rebuild from Ab, then halve d until a probe passes
      // or d = 1.  A passing probe becomes cycle 1.
      Vec ab;
      int d = g.degree;
      bool damped = false;
      for (;;) {
        p = stab(build_gmres_poly(*A, damped ? ab : b, d, c));
        OpPtr pop = std::make_shared<PolyOp>(A, p, false);
        State ps = arnoldi_init(rng::gauss_vec(n, g.seed, rng::ARNOLDI), g.m, c);
        arnoldi_extend(ps, *pop, g.m, c);
        Ritz pset = select_pairs(ps, TARGET_ONE, g.variant);
        Result tmp;
        tmp.rtol = R.rtol;
        bool all_k;
        double mx_k;
        check_and_record(ps, pset, g.k, *A, tmp, all_k, mx_k, c);
        const bool pass = static_cast<int>(tmp.mu.size()) >= g.nev && check_ideal_order(tmp.mu, g.nev);
        if (pass) {
          probe_state = std::move(ps);
          probe_set = std::move(pset);
          probe_mu = tmp.mu;
          probe_res = tmp.res;
          has_probe = true;
          break;
        }
        ++R.discarded;
        if (d <= 1) break;
        if (!damped) {
          ab = damped_start(*A, b, 0.0, 1, c);
          damped = true;
        } else {
          d /= 2;
        }
      }
    } else if (g.damping == 2) {
      p = stab(build_gmres_poly(*A, damped_start(*A, b, g.damping_alpha, g.damping_power, c), g.degree, c));
    } else {
      p = stab(build_gmres_poly(*A, b, g.degree, c));
    }
    R.composite = p.eff();
    op = std::make_shared<PolyOp>(A, p, false);
    R.poly = p;
    ord = TARGET_ONE;
  }
  State st = has_probe ? std::move(probe_state)
                       : arnoldi_init(rng::gauss_vec(n, g.seed, rng::ARNOLDI), g.m, c);
  R.max_err = std::numeric_limits<double>::infinity();
  std::vector<double> best;
  for (int cyc = 1; cyc <= g.max_cycles; ++cyc) {
    Ritz s;
    bool all;
    double mx;
    if (cyc == 1 && has_probe) {
      s = std::move(probe_set);
      const int keep = std::min<int>(g.nev, static_cast<int>(probe_mu.size()));
      R.mu.assign(probe_mu.begin(), probe_mu.begin() + keep);
      R.res.assign(probe_res.begin(), probe_res.begin() + keep);
      all = keep == g.nev;
      mx = 0.0;
      for (double r : R.res) {
        mx = std::max(mx, r);
        all = all && r <= R.rtol;
      }
      R.conv.assign(keep, 0);
      for (int i = 0; i < keep; ++i) R.conv[i] = R.res[i] <= R.rtol;
    } else if (g.mid_stride > 0) {
      // SPEC.md:421 mid-cycle checks: test the partial factorisation every
      // mid_stride steps once it holds nev columns; the full check at m
      all = false;
      for (;;) {
        const int to = std::min(g.m, st.cur_dim + g.mid_stride);
        arnoldi_extend(st, *op, to, c);
        if (st.breakdown || st.cur_dim >= g.m) break;
        if (st.cur_dim < g.nev) continue;
        s = select_pairs(st, ord, g.variant);
        check_and_record(st, s, g.nev, *A, R, all, mx, c);
        if (all) break;
      }
      if (!all) {
        s = select_pairs(st, ord, g.variant);
        check_and_record(st, s, g.nev, *A, R, all, mx, c);
      }
    } else {
      arnoldi_extend(st, *op, g.m, c);
      s = select_pairs(st, ord, g.variant);
      check_and_record(st, s, g.nev, *A, R, all, mx, c);
    }
    R.cycles = cyc;
    R.cycle_max.push_back(mx);
    R.max_err = std::min(R.max_err, mx);
    best.push_back(R.max_err);
    // SPEC.md:621 stagnation: best max-residual improved by < stag_rtol over
    // the last stag_window cycles
    const int w = g.stag_window;
    const bool stalled = w > 0 && cyc > w && best[cyc - 1] > (1.0 - g.stag_rtol) * best[cyc - 1 - w];
    if ((w > 0 ? stalled : all) || cyc == g.max_cycles || st.breakdown || st.cur_dim < g.m) {
      R.converged = all;
      break;
    }
    if (g.variant == 1) {
      harmonic_thick_restart(st, s, g.k, c);
    } else {
      thick_restart(st, s, g.k, c);
    }
  }
  c.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  R.cost = c;
  return R;
}

}  // namespace orc

// ===================================================================== C API
// (ctypes; tests/ and bench.py only)

struct orc_csr {
  orc::Csr m;
};
struct orc_op {
  orc::OpPtr p;
};

namespace {
thread_local std::string g_err;
template <typename F>
int wrap(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}
orc::Poly mkpoly(const double* re, const double* im, int n) {
  orc::Poly p;
  for (int i = 0; i < n; ++i) p.roots.emplace_back(re[i], im[i]);
  p.base_degree = n;
  orc::refresh(p);
  return p;
}
void addc(double* out5, const orc::Cost& c) {
  if (!out5) return;
  out5[0] += static_cast<double>(c.mvps);
  out5[1] += static_cast<double>(c.dots);
  out5[2] += static_cast<double>(c.vops);
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
void orc_set_threads(int t) { omp_set_num_threads(t < 1 ? 1 : t); }
void orc_set_variant(int v) { orc::g_variant = (v >= 0 && v <= 2) ? v : 0; }
int orc_get_variant(void) { return orc::g_variant; }
int orc_max_threads() { return omp_get_max_threads(); }

int orc_gen_config(int c, orc_csr** out) {
  return wrap([&] { *out = new orc_csr{orc::gen_config(c)}; });
}
int orc_gen_convdiff_ref(int N, orc_csr** out) {
  return wrap([&] { *out = new orc_csr{orc::gen_convdiff_ref(N)}; });
}
int orc_gen_convdiff_const(int N, double pe, orc_csr** out) {
  return wrap([&] { *out = new orc_csr{orc::gen_convdiff_const(N, pe)}; });
}
int orc_gen_laplace3d(int N, orc_csr** out) {
  return wrap([&] { *out = new orc_csr{orc::gen_laplace3d(N)}; });
}
int orc_gen_bidiag(int n, orc_csr** out) {
  return wrap([&] { *out = new orc_csr{orc::gen_bidiag(n)}; });
}
int orc_gen_random_poisson(int n, double lam, unsigned long long seed, orc_csr** out) {
  return wrap([&] { *out = new orc_csr{orc::gen_random_poisson(n, lam, seed)}; });
}
int orc_csr_create(int n, long long nnz, const int* rp, const int* ci, const double* v, orc_csr** out) {
  return wrap([&] {
    orc::Csr m;
    m.n = n;
    m.rp.assign(rp, rp + n + 1);
    m.ci.assign(ci, ci + nnz);
    m.v.assign(v, v + nnz);
    m.validate();
    *out = new orc_csr{std::move(m)};
  });
}
int orc_csr_from_triplets(int n, long long cnt, const int* r, const int* c, const double* v, orc_csr** out) {
  return wrap([&] {
    std::vector<std::tuple<int, int, double>> t;
    for (long long i = 0; i < cnt; ++i) t.emplace_back(r[i], c[i], v[i]);
    *out = new orc_csr{orc::from_triplets(n, std::move(t))};
  });
}
int orc_csr_info(const orc_csr* m, int* n, long long* nnz, unsigned long long* fp) {
  return wrap([&] {
    if (n) *n = m->m.n;
    if (nnz) *nnz = m->m.nnz();
    if (fp) *fp = orc::fingerprint(m->m);
  });
}
int orc_csr_arrays(const orc_csr* m, const int** rp, const int** ci, const double** v) {
  return wrap([&] {
    *rp = m->m.rp.data();
    *ci = m->m.ci.data();
    *v = m->m.v.data();
  });
}
void orc_csr_free(orc_csr* m) { delete m; }

int orc_normal_vector(long long n, unsigned long long seed, unsigned long long stream, double* out) {
  return wrap([&] {
    const uint64_t k = orc::rng::key(seed, stream);
    for (long long i = 0; i < n; ++i) out[i] = orc::rng::gauss(k, static_cast<uint64_t>(i));
  });
}

int orc_csr_operator(const orc_csr* m, orc_op** out) {
  return wrap([&] { *out = new orc_op{std::make_shared<orc::CsrOp>(m->m)}; });
}
int orc_diag_operator(int n, const double* d, orc_op** out) {
  return wrap([&] {
    orc::Csr m;
    m.n = n;
    for (int i = 0; i <= n; ++i) m.rp.push_back(i);
    for (int i = 0; i < n; ++i) m.ci.push_back(i);
    m.v.assign(d, d + n);
    *out = new orc_op{std::make_shared<orc::CsrOp>(m, true)};
  });
}
int orc_poly_operator(const orc_op* a, const double* re, const double* im, int n, int comp, orc_op** out) {
  return wrap([&] { *out = new orc_op{std::make_shared<orc::PolyOp>(a->p, mkpoly(re, im, n), comp != 0)}; });
}
void orc_op_free(orc_op* o) { delete o; }
int orc_op_apply(const orc_op* o, const double* x, double* y, double* cost) {
  return wrap([&] {
    orc::Cost c;
    o->p->apply(x, y, c);
    addc(cost, c);
  });
}
int orc_spmv(const orc_op* o, const double* x, double* y) {
  return wrap([&] {
    orc::Cost c;
    o->p->apply(x, y, c);
  });
}
int orc_apply_poly(const double* re, const double* im, int n, const orc_op* a, const double* v, double* out,
                   double* cost) {
  return wrap([&] {
    orc::Cost c;
    orc::apply_poly(mkpoly(re, im, n), *a->p, v, out, c);
    addc(cost, c);
  });
}
int orc_build_gmres_poly(const orc_op* a, const double* b, int degree, double* re, double* im, int* nr,
                         int* trunc, double* cost) {
  return wrap([&] {
    orc::Cost c;
    orc::Vec bv(b, b + a->p->dim());
    const orc::Poly p = orc::build_gmres_poly(*a->p, bv, degree, c);
    for (int i = 0; i < p.eff(); ++i) {
      re[i] = p.roots[i].real();
      im[i] = p.roots[i].imag();
    }
    *nr = p.eff();
    *trunc = p.truncated;
    addc(cost, c);
  });
}
int orc_leja_order(const double* re, const double* im, int n, double* ore, double* oim) {
  return wrap([&] {
    std::vector<orc::cd> r;
    for (int i = 0; i < n; ++i) r.emplace_back(re[i], im[i]);
    const auto o = orc::leja_order(r);
    for (size_t i = 0; i < o.size(); ++i) {
      ore[i] = o[i].real();
      oim[i] = o[i].imag();
    }
  });
}
int orc_compute_pof(const double* re, const double* im, int n, double* lg, int* copies, int* nd,
                    double* maxlg, int* total) {
  return wrap([&] {
    const orc::Pof r = orc::compute_pof(mkpoly(re, im, n));
    for (size_t i = 0; i < r.lg.size(); ++i) {
      lg[i] = r.lg[i];
      copies[i] = r.copies[i];
    }
    *nd = static_cast<int>(r.lg.size());
    *maxlg = r.maxlg;
    *total = r.total;
  });
}
int orc_add_stability_roots(const double* re, const double* im, int n, int maxc, int cap, double* ore,
                            double* oim, int* on) {
  return wrap([&] {
    const orc::Poly p = orc::add_stability_roots(mkpoly(re, im, n), maxc);
    if (p.eff() > cap) throw std::invalid_argument("capacity");
    for (int i = 0; i < p.eff(); ++i) {
      ore[i] = p.roots[i].real();
      oim[i] = p.roots[i].imag();
    }
    *on = p.eff();
  });
}
int orc_eval_poly(const double* re, const double* im, int n, double zr, double zi, double* ore, double* oim) {
  return wrap([&] {
    const orc::cd v = orc::eval_poly(mkpoly(re, im, n), orc::cd(zr, zi));
    *ore = v.real();
    *oim = v.imag();
  });
}

// Arnoldi on an operator: init + extend + (ritz values, H) in one call.
int orc_arnoldi(const orc_op* a, const double* v0, int m, int to_dim, double* H, int* cur_dim, int* breakdown,
                double* V, double* cost) {
  return wrap([&] {
    orc::Cost c;
    orc::Vec v(v0, v0 + a->p->dim());
    orc::State st = orc::arnoldi_init(v, m, c);
    orc::arnoldi_extend(st, *a->p, to_dim, c);
    std::copy(st.H.a.begin(), st.H.a.end(), H);
    *cur_dim = st.cur_dim;
    *breakdown = st.breakdown;
    if (V) std::copy(st.V.begin(), st.V.end(), V);
    addc(cost, c);
  });
}
int orc_harmonic_from_H(const double* H, int m, int d, double* re, double* im) {
  return wrap([&] {
    orc::State st;
    st.max_dim = m;
    st.cur_dim = d;
    st.H = orc::Mat(m + 1, m);
    std::copy(H, H + static_cast<size_t>(m + 1) * m, st.H.a.begin());
    const auto w = orc::harmonic_ritz_values(st);
    for (size_t i = 0; i < w.size(); ++i) {
      re[i] = w[i].real();
      im[i] = w[i].imag();
    }
  });
}
int orc_ritz_from_H(const double* H, int m, int d, int ord, double* re, double* im, double* res) {
  return wrap([&] {
    orc::State st;
    st.max_dim = m;
    st.cur_dim = d;
    st.H = orc::Mat(m + 1, m);
    std::copy(H, H + static_cast<size_t>(m + 1) * m, st.H.a.begin());
    const orc::Ritz s = orc::ritz_pairs(st, ord);
    for (int i = 0; i < s.count(); ++i) {
      re[i] = s.values[i].real();
      im[i] = s.values[i].imag();
      res[i] = s.residuals[i];
    }
  });
}

struct orc_solve_out {
  int cap_nev, cap_roots, cap_cycles;
  double* eig_re;
  double* eig_im;
  double* residuals;
  int* conv;
  double* poly_re;
  double* poly_im;
  double* inner_re;
  double* inner_im;
  double* cycle_max;
  int n_eig, n_poly, n_inner, n_cycles;
  int converged, cycles, composite, discarded;
  double rtol, max_err, norm_est;
  long long mvps, dots, vops;
  double wall;
};

int orc_solve(const orc_op* a, int m, int k, int nev, int degree, double rtol_mult, double rtol_abs,
              int stability, int use_double, int d1, int d2, int max_cycles, unsigned long long seed,
              int allow_nev_above_k, int damping, double damping_alpha, int damping_power,
              int mid_stride, int stag_window, double stag_rtol, int variant,
              orc_solve_out* out) {
  return wrap([&] {
    orc::Config g;
    g.variant = variant;
    g.mid_stride = mid_stride;
    g.stag_window = stag_window;
    if (stag_rtol > 0) g.stag_rtol = stag_rtol;
    g.damping = damping;
    g.damping_alpha = damping_alpha;
    g.damping_power = damping_power > 0 ? damping_power : 1;
    g.m = m;
    g.k = k;
    g.nev = nev;
    g.degree = degree;
    g.rtol_mult = rtol_mult;
    g.rtol_abs = rtol_abs;
    g.stability = stability;
    g.use_double = use_double;
    g.d1 = d1;
    g.d2 = d2;
    g.max_cycles = max_cycles;
    g.seed = seed;
    g.allow_nev_above_k = allow_nev_above_k;
    const orc::Result R = orc::solve(a->p, g);
    out->n_eig = static_cast<int>(R.mu.size());
    for (int i = 0; i < out->n_eig && i < out->cap_nev; ++i) {
      out->eig_re[i] = R.mu[i].real();
      out->eig_im[i] = R.mu[i].imag();
      out->residuals[i] = R.res[i];
      out->conv[i] = R.conv[i];
    }
    out->n_poly = R.poly.eff();
    for (int i = 0; i < out->n_poly && i < out->cap_roots; ++i) {
      out->poly_re[i] = R.poly.roots[i].real();
      out->poly_im[i] = R.poly.roots[i].imag();
    }
    out->n_inner = R.inner.eff();
    for (int i = 0; i < out->n_inner && i < out->cap_roots; ++i) {
      out->inner_re[i] = R.inner.roots[i].real();
      out->inner_im[i] = R.inner.roots[i].imag();
    }
    out->n_cycles = static_cast<int>(R.cycle_max.size());
    for (int i = 0; i < out->n_cycles && i < out->cap_cycles; ++i) out->cycle_max[i] = R.cycle_max[i];
    out->converged = R.converged;
    out->cycles = R.cycles;
    out->composite = R.composite;
    out->discarded = R.discarded;
    out->rtol = R.rtol;
    out->max_err = R.max_err;
    out->norm_est = R.norm_est;
    out->mvps = R.cost.mvps;
    out->dots = R.cost.dots;
    out->vops = R.cost.vops;
    out->wall = R.cost.wall_seconds;
  });
}

int orc_block2_operator(const orc_op* a, orc_op** out) {
  return wrap([&] { *out = new orc_op{std::make_shared<orc::Block2Op>(a->p)}; });
}
int orc_shifted_operator(const orc_op* a, double mu, orc_op** out) {
  return wrap([&] { *out = new orc_op{std::make_shared<orc::ShiftedOp>(a->p, mu)}; });
}
int orc_build_two_vector_poly(const orc_op* a, const double* b1, const double* b2, int degree, double* re,
                              double* im, int* nr, double* cost) {
  return wrap([&] {
    orc::Cost c;
    const long n = a->p->dim();
    const orc::Poly p = orc::build_two_vector_poly(a->p, orc::Vec(b1, b1 + n), orc::Vec(b2, b2 + n), degree, c);
    for (int i = 0; i < p.eff(); ++i) {
      re[i] = p.roots[i].real();
      im[i] = p.roots[i].imag();
    }
    *nr = p.eff();
    addc(cost, c);
  });
}
int orc_damped_start(const orc_op* a, const double* b, double alpha, int power, double* out, double* cost) {
  return wrap([&] {
    orc::Cost c;
    const long n = a->p->dim();
    const orc::Vec w = orc::damped_start(*a->p, orc::Vec(b, b + n), alpha, power, c);
    std::copy(w.begin(), w.end(), out);
    addc(cost, c);
  });
}
int orc_check_ideal_order(const double* re, const double* im, int count, int nev, int* holds) {
  return wrap([&] {
    std::vector<orc::cd> mu;
    for (int i = 0; i < count; ++i) mu.emplace_back(re[i], im[i]);
    *holds = orc::check_ideal_order(mu, nev) ? 1 : 0;
  });
}
int orc_read_matrix_market(const char* path, orc_csr** out) {
  return wrap([&] { *out = new orc_csr{orc::read_matrix_market(path)}; });
}

// cpu_baseline / reference arm: time `reps` applications of the first
// `nfactors` factors of pi(A) (real roots: SpMV + axpy each), seconds.
double orc_time_poly_factors(const orc_op* a, const double* re, const double* im, int nroots, int nfactors,
                             int reps) {
  orc::Poly p;
  for (int i = 0; i < nroots && static_cast<int>(p.roots.size()) < nfactors; ++i) p.roots.emplace_back(re[i], im[i]);
  // keep conjugate pairs whole
  if (!p.roots.empty() && orc::p_is_complex(p.roots.back()) && static_cast<int>(p.roots.size()) < nroots) {
    const size_t L = p.roots.size();
    if (L >= 2 && std::abs(p.roots[L - 2] - std::conj(p.roots[L - 1])) > 1e-10 * std::abs(p.roots[L - 1]))
      p.roots.emplace_back(re[L], im[L]);
  }
  const long n = a->p->dim();
  orc::Vec v = orc::rng::gauss_vec(n, 1, orc::rng::POLY), out(n);
  orc::Cost c;
  const auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < reps; ++r) orc::apply_poly(p, *a->p, v.data(), out.data(), c);
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Seconds per orthogonalisation step of arnoldi_extend at basis size c (the
// MGS + MGS reorthogonalisation loops, the norm and the scaled store of
// src/arnoldi.cpp:129-150, without the operator application), mean of reps.
// The timing does not depend on the values: the basis is c scaled Gaussian
// columns.  For bench.py's CPU arm only.
double orc_time_mgs2_step(long n, int c, int reps) {
  orc::Vec V(static_cast<size_t>(n) * (c + 1));
  for (int j = 0; j < c; ++j) {
    const orc::Vec g = orc::rng::gauss_vec(n, 100 + j, orc::rng::ARNOLDI);
    const double s = 1.0 / std::sqrt(static_cast<double>(n));
    for (long i = 0; i < n; ++i) V[static_cast<size_t>(j) * n + i] = g[i] * s;
  }
  const orc::Vec w0 = orc::rng::gauss_vec(n, 7, orc::rng::ARNOLDI);
  orc::Vec w(n);
  std::vector<double> h(static_cast<size_t>(c) + 1);
  orc::Cost cost;
  double total = 0.0;
  for (int r = 0; r < reps; ++r) {
    w = w0;
    const auto t0 = std::chrono::steady_clock::now();
    for (int pass = 0; pass < 2; ++pass) {
      for (int i = 0; i < c; ++i) {
        const double hi = orc::dot(V.data() + static_cast<size_t>(i) * n, w.data(), n, cost);
        h[i] = pass == 0 ? hi : h[i] + hi;
        orc::axpy(-hi, V.data() + static_cast<size_t>(i) * n, w.data(), n, cost);
      }
    }
    const double hsub = orc::norm(w.data(), n, cost);
    double* dst = V.data() + static_cast<size_t>(c) * n;
    for (long i = 0; i < n; ++i) dst[i] = w[i] / hsub;
    total += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  return total / std::max(1, reps);
}

}  // extern "C"
