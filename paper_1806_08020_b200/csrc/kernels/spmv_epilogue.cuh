#pragma once
// Polynomial-factor epilogue shared by the SpMV kernels (kernels.hpp "Fused
// epilogues"): the reference's operation order of src/gmres_poly.cpp:129-143
// and the complement of src/gmres_poly.cpp:306-308, without FMA contraction.
//
// Nested double polynomials (solve_double: phi(psi(A)) with psi = tau =
// I - pi_1) also fold the OUTER factor into the last inner launch, in the
// order of the reference's generic loop (src/gmres_poly.cpp:129-143 over the
// tau operator): with u = base - z the tau output of this launch,
//   outer real : y = oo + oc0 * u                  (out += c0 * t1)
//   outer pair : y = (oo + oc1 * base) + oc0 * u    (out += c1 * t1; out += c0 * t2)
// where base is tau's input (t1 for a pair) and oo the outer running product.

#include "ppa/kernels.hpp"

namespace ppa {
namespace kern {

struct EpiDev {
  double c0, c1;
  const double* o;
  const double* base;
  int outer;  // 0 none, 1 outer real factor, 2 outer pair (requires base)
  double oc0, oc1;
  const double* oo;
};

inline EpiDev epi_dev(const EpiArgs& a) {
  return EpiDev{a.c0, a.c1, a.o, a.base, a.outer, a.oc0, a.oc1, a.oo};
}

// xr = x[r], already in a register (the gather kernels hold the centre).
template <int MODE, bool COMPL>
__device__ __forceinline__ double epilogue_x(int r, double s, double xr, const EpiDev& e) {
  double z;
  if (MODE == 0) {
    z = s;
  } else if (MODE == 1) {
    z = __dadd_rn(xr, __dmul_rn(e.c0, s));
  } else {
    z = __dadd_rn(__dadd_rn(e.o[r], __dmul_rn(e.c1, xr)), __dmul_rn(e.c0, s));
  }
  if (COMPL) {
    const double b = e.base[r];
    z = __dsub_rn(b, z);
    if (e.outer == 1) {
      z = __dadd_rn(e.oo[r], __dmul_rn(e.oc0, z));
    } else if (e.outer == 2) {
      z = __dadd_rn(__dadd_rn(e.oo[r], __dmul_rn(e.oc1, b)), __dmul_rn(e.oc0, z));
    }
  }
  return z;
}

template <int MODE, bool COMPL>
__device__ __forceinline__ double epilogue(int r, double s, const double* __restrict__ x,
                                           const EpiDev& e) {
  return epilogue_x<MODE, COMPL>(r, s, MODE == 0 ? 0.0 : __ldg(x + r), e);
}

}  // namespace kern
}  // namespace ppa
