// Execution context: stream, reduction workspace, stream-ordered scratch.

#include <cstdint>
#include <memory>

#include "ppa/device.hpp"
#include "ppa/kernels.hpp"

namespace ppa {

Context::Context(cudaStream_t s) : stream_(s) {
  int dev = 0;
  PPA_CUDA(cudaGetDevice(&dev));
  PPA_CUDA(cudaDeviceGetAttribute(&sm_count_, cudaDevAttrMultiProcessorCount, dev));
  // Keep freed scratch in the pool: apply() allocates temporaries per call
  // like the reference (src/gmres_poly.cpp:124, 304) and must stay cheap.
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  kern::ensure_workspace(ws_, 148 * 16, 8);
  results_.resize(64);
}

Context::~Context() {
  if (pinned_) cudaFreeHost(pinned_);
  if (pinned_aux_) cudaFreeHost(pinned_aux_);
}

void Context::sync() const { PPA_CUDA(cudaStreamSynchronize(stream_)); }

double* Context::scratch(size_t count) {
  void* p = nullptr;
  PPA_CUDA(cudaMallocAsync(&p, count * sizeof(double), stream_));
  return static_cast<double*>(p);
}

void Context::release_scratch(double* p) {
  if (p) cudaFreeAsync(p, stream_);
}

double* Context::pinned(size_t count) {
  if (count > pinned_count_) {
    if (pinned_) {
      PPA_CUDA(cudaStreamSynchronize(stream_));
      cudaFreeHost(pinned_);
      pinned_ = nullptr;
    }
    const size_t c = count < 4096 ? 4096 : count;
    PPA_CUDA(cudaMallocHost(&pinned_, c * sizeof(double)));
    pinned_count_ = c;
  }
  return pinned_;
}

double* Context::pinned_aux(size_t count) {
  if (count > pinned_aux_count_) {
    if (pinned_aux_) {
      PPA_CUDA(cudaStreamSynchronize(stream_));
      cudaFreeHost(pinned_aux_);
      pinned_aux_ = nullptr;
    }
    const size_t c = count < 4096 ? 4096 : count;
    PPA_CUDA(cudaMallocHost(&pinned_aux_, c * sizeof(double)));
    pinned_aux_count_ = c;
  }
  return pinned_aux_;
}

double* Context::results() { return results_.get(); }

double Context::nrm2_sync(const double* x, long long n) {
  kern::nrm2(x, n, results_.get(), ws_, sm_count_, stream_);
  double* h = pinned(1);
  PPA_CUDA(cudaMemcpyAsync(h, results_.get(), sizeof(double), cudaMemcpyDeviceToHost, stream_));
  sync();
  return h[0];
}

double Context::dot_sync(const double* x, const double* y, long long n) {
  kern::dot(x, y, n, results_.get(), ws_, sm_count_, stream_);
  double* h = pinned(1);
  PPA_CUDA(cudaMemcpyAsync(h, results_.get(), sizeof(double), cudaMemcpyDeviceToHost, stream_));
  sync();
  return h[0];
}

namespace {
thread_local std::unique_ptr<Context> t_ctx;
}

Context& current_context() {
  if (!t_ctx) t_ctx = std::make_unique<Context>(nullptr);
  return *t_ctx;
}

void set_current_stream(cudaStream_t s) { current_context().set_stream(s); }

}  // namespace ppa
