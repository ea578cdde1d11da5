#pragma once
// Operation counters.  Field-for-field the reference's CostRecord
// (inc/cost.hpp:17-23) with the same counting conventions
// (inc/cost.hpp:10-16): mvps = base-matrix applications, dots = length-n
// inner products (norms included), vops = every length-n vector operation
// (dots included).  The device kernels fuse several reference operations
// into one launch; the host side charges the reference's increments for
// each fused operation so the counters stay comparable.

#include <stdexcept>

namespace ppa {

struct CostRecord {
  long long mvps = 0;
  long long dots = 0;
  long long vops = 0;
  double nnzr = 0.0;  // average nonzeros per row; 0 means unset
  double wall_seconds = 0.0;
};

/// cost = nnzr * mvps + vops (inc/cost.hpp:26-32).
inline double cost_estimate(const CostRecord& rec) {
  if (rec.nnzr <= 0.0) {
    throw std::invalid_argument("cost_estimate: nnzr is unset");
  }
  return rec.nnzr * static_cast<double>(rec.mvps) +
         static_cast<double>(rec.vops);
}

/// Componentwise sum (inc/cost.hpp:35-46).
inline CostRecord merge(const CostRecord& a, const CostRecord& b) {
  if (a.nnzr > 0.0 && b.nnzr > 0.0 && a.nnzr != b.nnzr) {
    throw std::invalid_argument("merge: mismatched nnzr");
  }
  CostRecord out;
  out.mvps = a.mvps + b.mvps;
  out.dots = a.dots + b.dots;
  out.vops = a.vops + b.vops;
  out.nnzr = a.nnzr > 0.0 ? a.nnzr : b.nnzr;
  out.wall_seconds = a.wall_seconds + b.wall_seconds;
  return out;
}

}  // namespace ppa
