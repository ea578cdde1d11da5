#pragma once
// Layout of ReduceWorkspace::scalars (device doubles) shared by the kernels.

namespace ppa {
namespace kern {

constexpr int kScalH1 = 0;      // CGS2 pass-1 coefficients
constexpr int kScalH2 = 256;    // CGS2 pass-2 coefficients
constexpr int kScalHsub = 512;  // hsub, ||w|| after pass 1
constexpr int kScalCount = 1024;
constexpr int kMaxCols = 128;   // widest basis block the tall-skinny kernels take

void check_cols(int c, const char* who);

}  // namespace kern
}  // namespace ppa
