#pragma once
// Work counters of one solve, with the paper's composite cost metric
// cost = nnzr * mvps + vops (section 4).
//
// Conventions are the reference's (inc/cost.hpp:10-16): `mvps` counts
// base-matrix applications, `dots` counts length-n inner products with norms
// included, `vops` counts every length-n vector operation, dots included.
// Device kernels fuse several of those operations into one launch; the host
// code still charges each fused operation separately, so the numbers stay
// comparable with the CPU oracle.

#include <stdexcept>

namespace ppa {

struct CostRecord {
  long long mvps = 0;
  long long dots = 0;
  long long vops = 0;
  double nnzr = 0.0;  // nonzeros per row of the base matrix; 0 = not set
  double wall_seconds = 0.0;
};

/// Paper metric; nnzr must have been set.
inline double cost_estimate(const CostRecord& c) {
  if (!(c.nnzr > 0.0)) throw std::invalid_argument("cost_estimate: nnzr is unset");
  return c.nnzr * static_cast<double>(c.mvps) + static_cast<double>(c.vops);
}

/// Sum of two records that describe the same matrix (nnzr must agree when
/// both are set).
inline CostRecord merge(const CostRecord& x, const CostRecord& y) {
  const bool both = x.nnzr > 0.0 && y.nnzr > 0.0;
  if (both && x.nnzr != y.nnzr) throw std::invalid_argument("merge: mismatched nnzr");
  CostRecord s;
  s.mvps = x.mvps + y.mvps;
  s.dots = x.dots + y.dots;
  s.vops = x.vops + y.vops;
  s.nnzr = x.nnzr > 0.0 ? x.nnzr : y.nnzr;
  s.wall_seconds = x.wall_seconds + y.wall_seconds;
  return s;
}

}  // namespace ppa
