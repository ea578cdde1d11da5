// Box-grid two-factor pass: the 5-point kernels with 4 cells per thread
// (every block size, root kind, complement, single-factor and slab form).
#include "spmv_grid2_kernel.cuh"

PPA_G2_DEFINE(5, 4)
