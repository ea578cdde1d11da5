#pragma once
// Polynomial-factor epilogue shared by the SpMV kernels (kernels.hpp "Fused
// epilogues"): the reference's operation order of src/gmres_poly.cpp:129-143
// and the complement of src/gmres_poly.cpp:306-308, without FMA contraction.

namespace ppa {
namespace kern {

template <int MODE, bool COMPL>
__device__ __forceinline__ double epilogue(int r, double s, const double* __restrict__ x,
                                           double c0, double c1, const double* o,
                                           const double* base) {
  double z;
  if (MODE == 0) {
    z = s;
  } else if (MODE == 1) {
    z = __dadd_rn(__ldg(x + r), __dmul_rn(c0, s));
  } else {
    z = __dadd_rn(__dadd_rn(o[r], __dmul_rn(c1, __ldg(x + r))), __dmul_rn(c0, s));
  }
  if (COMPL) z = __dsub_rn(base[r], z);
  return z;
}

}  // namespace kern
}  // namespace ppa
