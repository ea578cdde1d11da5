// Random-gather throughput of the B200: the LSU path (one 8-byte load per
// lane, every lane a different 32-byte sector) against the Blackwell TMA
// gather (cp.async.bulk.tensor.2d ... tile::gather4: four 16-byte rows of a
// 2-D view of x per instruction, into shared memory).  Config 4's SpMV makes
// 34 M such gathers over a 16 MB x.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather4_rate gather4_rate.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// LSU gathers: each thread sums x[idx[i]] over its share of idx
__global__ void k_lsu(const double* __restrict__ x, const int* __restrict__ idx, long long m,
                      double* out) {
  double s = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x)
    s += __ldg(x + idx[i]);
  if (s == 1234.5) out[0] = s;
}

// TMA gather4: warp 0 lane 0 issues gathers of 4 x 16-byte rows into a ring of
// stages; the other warps consume (sum) and release.  Row r of the 2-D view
// holds x[2r], x[2r+1]; element c comes from row c/2.
constexpr int STAGES = 8;
constexpr int G4_PER_STAGE = 32;  // 128 rows = 2 KB per stage
__global__ void k_tma(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx,
                      long long m, double* out) {
  __shared__ __align__(128) double buf[STAGES][G4_PER_STAGE * 16];  // 128-byte aligned destinations
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int ncons = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(ncons));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long per_stage = G4_PER_STAGE * 4;
  const long long nst = m / per_stage;
  double s = 0;
  if (warp == 0) {
    // lane g issues gather g of the stage (G4_PER_STAGE == 32)
    // indices prefetched PF stages ahead (a global load is ~1 us; without the
    // prefetch the producer issues one stage per index round trip)
    constexpr int PF = 6;
    int4 q[PF];
#pragma unroll
    for (int j = 0; j < PF; ++j) {
      const long long kk = blockIdx.x + (long long)j * gridDim.x;
      q[j] = kk < nst ? reinterpret_cast<const int4*>(idx + kk * per_stage)[lane] : make_int4(0, 0, 0, 0);
    }
    for (long long k = blockIdx.x, it = 0; k < nst; k += gridDim.x, ++it) {
      const int st = it % STAGES;
      const int4 rr = q[0];
#pragma unroll
      for (int j = 0; j < PF - 1; ++j) q[j] = q[j + 1];
      {
        const long long kk = k + (long long)PF * gridDim.x;
        q[PF - 1] = kk < nst ? reinterpret_cast<const int4*>(idx + kk * per_stage)[lane] : make_int4(0, 0, 0, 0);
      }
      if (lane == 0) {
        if (it >= STAGES) {
          const uint32_t ph = ((it / STAGES) - 1) & 1;
          asm volatile(
              "{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" ::"r"(
                  su32(&empty[st])),
              "r"(ph)
              : "memory");
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[st])),
                     "r"(G4_PER_STAGE * 4 * 16)
                     : "memory");
      }
      __syncwarp();
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(&buf[st][lane * 16])),
          "l"(&tm), "r"(0), "r"(rr.x >> 1), "r"(rr.y >> 1), "r"(rr.z >> 1), "r"(rr.w >> 1),
          "r"(su32(&full[st]))
          : "memory");
    }
  } else {
    for (long long k = blockIdx.x, it = 0; k < nst; k += gridDim.x, ++it) {
      const int st = it % STAGES;
      const uint32_t ph = (it / STAGES) & 1;
      asm volatile(
          "{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" ::"r"(
              su32(&full[st])),
          "r"(ph)
          : "memory");
      // consumer warp w sums its slice of the stage
      for (int j = (warp - 1) * 32 + lane; j < G4_PER_STAGE * 8; j += ncons * 32) s += buf[st][(j >> 3) * 16 + (j & 7)];
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[st])) : "memory");
    }
  }
  if (s == 1234.5) out[0] = s;
}

// correctness of the 2-D view: gather4 of rows r0..r3 lands x[2r], x[2r+1]
__global__ void k_tma_check(const __grid_constant__ CUtensorMap tm, int r0, int r1, int r2, int r3,
                            double* out) {
  __shared__ __align__(128) double b[8];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 64;" ::"r"(su32(&bar)) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(b)),
        "l"(&tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(&bar))
        : "memory");
    asm volatile(
        "{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" ::"r"(
            su32(&bar))
        : "memory");
    for (int i = 0; i < 8; ++i) out[i] = b[i];
  }
}

int main(int argc, char** argv) {
  const unsigned bh = argc > 1 ? atoi(argv[1]) : 1;
  const long long n = 2000000, m = 34 * 1000000LL;  // config 4: 2 M columns, 34 M gathers
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::vector<double> hx(n);
  for (long long i = 0; i < n; ++i) hx[i] = (double)i;
  std::vector<int> hi(m);
  uint64_t z = 12345;
  for (long long i = 0; i < m; ++i) {
    z = z * 6364136223846793005ull + 1442695040888963407ull;
    hi[i] = (int)((z >> 33) % n);
  }
  double *x, *out;
  int* idx;
  CK(cudaMalloc(&x, n * 8));
  CK(cudaMalloc(&out, 64));
  CK(cudaMalloc(&idx, m * 4));
  CK(cudaMemcpy(x, hx.data(), n * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(idx, hi.data(), m * 4, cudaMemcpyHostToDevice));

  CUtensorMap tm;
  cuuint64_t gdim[2] = {2, (cuuint64_t)(n / 2)};
  cuuint64_t gstride[1] = {16};
  cuuint32_t box[2] = {2, bh};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, gdim, gstride, box,
                                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("tensor map (box 2x%u): %d\n", bh, (int)r);
  k_tma_check<<<1, 32>>>(tm, 5, 999, 7, 123456, out);
  CK(cudaDeviceSynchronize());
  double ho[8];
  CK(cudaMemcpy(ho, out, 64, cudaMemcpyDeviceToHost));
  printf("gather4 rows 5,999,7,123456 -> %g %g | %g %g | %g %g | %g %g\n", ho[0], ho[1], ho[2],
         ho[3], ho[4], ho[5], ho[6], ho[7]);

  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k_lsu<<<sms * 8, 256>>>(x, idx, m, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
  }
  printf("LSU gathers: %.1f us for %lld (%.2f per clk per SM at 1.965 GHz)\n", ms * 1e3, m,
         m / (ms * 1e-3) / sms / 1.965e9);
  for (int cpb : {1, 2, 4}) {
    for (int warps : {2, 4, 8}) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k_tma<<<sms * cpb, 32 * warps>>>(tm, idx, m, out);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
      }
      CK(cudaGetLastError());
      printf("TMA gather4 (%d CTA/SM, %d warps): %.1f us (%.2f per clk per SM)\n", cpb, warps,
             ms * 1e3, m / (ms * 1e-3) / sms / 1.965e9);
    }
  }
  return 0;
}
