#pragma once
// Programmatic dependent launch (sm_90+) for the dependent kernel chains of
// pi(A)v: a kernel launched with launch_pdl() may be scheduled while the
// previous kernel on the stream is still draining; it runs its independent
// prologue (matrix-structure loads) and then waits in pdl_wait() until the
// previous grid has completed and its writes are visible.  Every kernel
// launched through launch_pdl() must call pdl_wait() before it reads data a
// previous kernel wrote or writes data a previous kernel reads.
// PPA_DISABLE_PDL=1 launches normally (the wait is then a no-op).

#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

#include "ppa/device.hpp"

namespace ppa {
namespace kern {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

inline bool pdl_enabled() {
  static const bool on = std::getenv("PPA_DISABLE_PDL") == nullptr;
  return on;
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  PPA_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

}  // namespace kern
}  // namespace ppa
