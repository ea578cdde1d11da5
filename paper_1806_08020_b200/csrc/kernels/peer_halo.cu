// Halo exchange of the row-sharded pi(A)v over peer memory (NVLink /
// NVSwitch), without NCCL: every rank maps its neighbours' vector buffers
// and epoch flags with CUDA IPC (dist.py PeerHalo) and, before each SpMV,
// pulls the halo entries it needs straight from the owners' HBM.
//
// Protocol (per exchange e of a buffer role X):
//   owner : after the kernel that wrote X, publish(flag, e) - a system-scope
//           fence then a release store of e into its own flag;
//   reader: k_halo_pull waits (acquire load, system scope) until every
//           owner's flag >= e, then gathers x_ext[off_p + i] = X_p[idx_p[i]].
// A buffer is rewritten only after the rank's next pull, which waits for
// every reader's next publish, which that reader issues after its pull of
// this exchange: no reader can still be reading it.
// Before a rank writes a role buffer at the start of a new product it fences
// (publish + wait only): the last exchange of the previous product may still
// be read by peers whose publish came before their pull.
// The wait is bounded: a flag that does not arrive within ~10 s sets an
// error word and the kernel returns instead of hanging the GPU.

#include <algorithm>
#include <cstdint>

#include "ppa/kernels.hpp"

namespace ppa {
namespace kern {
namespace {

__device__ __forceinline__ long long ld_acquire_sys(const long long* p) {
  long long v;
  asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(long long* p, long long v) {
  asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void k_publish(long long* flag, long long epoch) {
  if (threadIdx.x == 0) {
    // every write of this stream's earlier kernels is complete (stream
    // order); make it visible system-wide before the flag
    asm volatile("fence.sc.sys;" ::: "memory");
    st_release_sys(flag, epoch);
  }
}

// grid.y = peer; each CTA waits on its peer's flag, then copies a strided
// share of that peer's halo entries
__global__ void k_halo_pull(const PeerHaloDesc* __restrict__ peers, double* __restrict__ x_ext,
                            long long epoch, int* __restrict__ error) {
  const PeerHaloDesc d = peers[blockIdx.y];
  __shared__ int ok;
  if (threadIdx.x == 0) {
    long long spins = 0;
    int good = 1;
    long long seen;
    while ((seen = ld_acquire_sys(d.flag)) < epoch) {
      __nanosleep(256);
      if (++spins > (1LL << 25)) {  // ~10 s
        atomicExch(error, 1);
        atomicExch(error + 1, static_cast<int>(seen));  // the last epoch seen
        good = 0;
        break;
      }
    }
    ok = good;
  }
  __syncthreads();
  if (!ok || x_ext == nullptr) return;  // x_ext == nullptr: a fence (wait only)
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < d.count;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    x_ext[d.dst_offset + i] = d.src[d.src_index[i]];
  }
}

}  // namespace

void publish(long long* flag, long long epoch, cudaStream_t st) {
  k_publish<<<1, 32, 0, st>>>(flag, epoch);
  PPA_CUDA(cudaGetLastError());
}

void halo_pull(const PeerHaloDesc* peers_dev, int npeers, long long max_count, double* x_ext,
               long long epoch, int* error, cudaStream_t st) {
  if (npeers <= 0) return;
  const int blocks = static_cast<int>(std::min<long long>(64, (max_count + 255) / 256));
  k_halo_pull<<<dim3(blocks > 0 ? blocks : 1, npeers), 256, 0, st>>>(peers_dev, x_ext, epoch,
                                                                     error);
  PPA_CUDA(cudaGetLastError());
}

}  // namespace kern
}  // namespace ppa
