#pragma once
// Thick-restarted Arnoldi (reference inc/arnoldi.hpp) with the basis V in
// HBM and the projection H on the host.

#include <complex>
#include <vector>

#include "ppa/cost.hpp"
#include "ppa/dense.hpp"
#include "ppa/device.hpp"
#include "ppa/operators.hpp"

namespace ppa {

/// Op V_j = V_{j+1} H_{j+1,j} (inc/arnoldi.hpp:18-26).  V is n x (m+1),
/// column-major on the device with ld = n rounded up to 32 doubles; H is
/// (m+1) x m column-major on the host.
/// Orthogonalisation of arnoldi_extend: classic CGS2 (three sweeps per
/// step, the default) or delayed CGS2 (two sweeps per step; arnoldi.cpp).
enum class Orthogonalization { cgs2 = 0, dcgs2 = 1 };

struct ArnoldiState {
  PoolBuffer V;  // (max_dim + 1) columns of ld doubles
  Orthogonalization ortho = Orthogonalization::cgs2;
  long long ld = 0;
  int n = 0;
  std::vector<double> H;
  int max_dim = 0;
  int cur_dim = 0;
  int restart_k = 0;
  int cycle_count = 0;
  bool breakdown = false;

  double& h(int i, int j) { return H[static_cast<size_t>(j) * (max_dim + 1) + i]; }
  double h(int i, int j) const { return H[static_cast<size_t>(j) * (max_dim + 1) + i]; }
  double* col(int j) { return V.get() + static_cast<long long>(j) * ld; }
  const double* col(int j) const { return V.get() + static_cast<long long>(j) * ld; }
};

/// v0: device vector of length n (src/arnoldi.cpp:99-113).
ArnoldiState arnoldi_init(const double* v0, int n, int m, CostRecord& rec);

/// CGS2 extension to to_dim (src/arnoldi.cpp:115-152; counters charged as
/// the reference's MGS2: dots += 2c+1, vops += 4c+2 per step).
void arnoldi_extend(ArnoldiState& state, const LinearOperator& op, int to_dim, CostRecord& rec);

enum class RitzOrdering { smallest_magnitude, largest_magnitude, target_one };

/// inc/arnoldi.hpp:46-54; vectors_h is cur_dim x count (column-major).
struct RitzSet {
  std::vector<std::complex<double>> values;
  dense::CMat vectors_h;
  std::vector<double> residuals;
  RitzOrdering ordering = RitzOrdering::smallest_magnitude;
  bool harmonic = false;
  int count() const { return static_cast<int>(values.size()); }
};

RitzSet ritz_pairs(const ArnoldiState& state, RitzOrdering ordering);
std::vector<std::complex<double>> harmonic_ritz_values(const ArnoldiState& state);
RitzSet harmonic_restart_selection(const ArnoldiState& state, RitzOrdering ordering);

/// Unit-norm Ritz vector j as device (re, im) vectors (src/arnoldi.cpp:252-265).
struct DeviceComplexVector {
  DBuffer<double> re, im;
  bool complex = false;
};
DeviceComplexVector ritz_vector(const ArnoldiState& state, const RitzSet& set, int j,
                                CostRecord& rec);

/// src/arnoldi.cpp:267-334; V(:,0:kk) = V(:,0:m) Q runs in place on the device.
int thick_restart(ArnoldiState& state, const RitzSet& keep, int k, CostRecord& rec);
/// Thick restart for harmonic keep-sets (the solve's harmonic variant): keeps
/// span{harmonic vectors, harmonic residual direction} so the compressed
/// factorisation stays an Arnoldi relation (arnoldi.cpp).
int harmonic_thick_restart(ArnoldiState& state, const RitzSet& keep, int k, CostRecord& rec);

/// Ritz-value classification used by sort_pairs / thick_restart
/// (src/arnoldi.cpp:18-25).
bool ritz_is_complex(const std::complex<double>& z);

}  // namespace ppa
