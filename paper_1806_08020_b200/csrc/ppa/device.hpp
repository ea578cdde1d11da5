#pragma once
// Device plumbing: owning buffers, the execution context (stream + the
// deterministic-reduction workspace) and CUDA error mapping.
//
// The reference has no device; its vectors are Eigen::VectorXd.  Here every
// length-n vector lives in HBM and the host only sees small (m-sized) data.

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>

namespace ppa {

class CudaError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
  }
}
#define PPA_CUDA(call) ::ppa::cuda_check((call), #call)

/// Owning device allocation (256-byte aligned by cudaMalloc).
template <typename T>
class DBuffer {
 public:
  DBuffer() = default;
  explicit DBuffer(size_t count) { resize(count); }
  ~DBuffer() { release(); }
  DBuffer(const DBuffer&) = delete;
  DBuffer& operator=(const DBuffer&) = delete;
  DBuffer(DBuffer&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
  DBuffer& operator=(DBuffer&& o) noexcept {
    if (this != &o) { release(); p_ = o.p_; n_ = o.n_; o.p_ = nullptr; o.n_ = 0; }
    return *this;
  }
  void resize(size_t count) {
    if (count == n_) return;
    release();
    if (count) PPA_CUDA(cudaMalloc(&p_, count * sizeof(T)));
    n_ = count;
  }
  void release() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

/// Workspace for the two-stage deterministic reductions: each reduction
/// kernel writes one partial row per block and the last block to finish
/// (ticket counter) sums the rows in block order.
struct ReduceWorkspace {
  DBuffer<double> partials;       // [max_blocks * max_width]
  DBuffer<unsigned int> tickets;  // one counter per concurrent reduction
  DBuffer<double> scalars;        // small device-resident results
  int max_blocks = 0;
  int max_width = 0;
};

/// Execution context: the stream every kernel of one solver run is
/// launched on plus its reduction workspace.  One solve is single-threaded
/// (SPEC.md concurrency model), so a context is owned by one thread.
class Context {
 public:
  explicit Context(cudaStream_t s = nullptr);
  ~Context();
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  cudaStream_t stream() const { return stream_; }
  /// Switching streams first drains the old one: the reduction workspace
  /// is shared by everything launched through this context.
  void set_stream(cudaStream_t s) {
    if (s != stream_) {
      PPA_CUDA(cudaStreamSynchronize(stream_));
      stream_ = s;
    }
  }
  /// Replace the stream without draining the old one: only for recording a
  /// launch sequence into a CUDA graph on a capture stream (nothing runs).
  cudaStream_t swap_stream(cudaStream_t s) {
    const cudaStream_t old = stream_;
    stream_ = s;
    return old;
  }
  ReduceWorkspace& ws() { return ws_; }
  int sm_count() const { return sm_count_; }
  void sync() const;

  /// Scratch length-n vectors from the stream-ordered pool.
  double* scratch(size_t count);
  void release_scratch(double* p);

  /// Pinned host staging for small device->host reads.
  double* pinned(size_t count);
  /// A second pinned area, owned by arnoldi_extend's in-flight Hessenberg
  /// columns, so an operator that uses pinned() inside apply() cannot
  /// clobber them.
  double* pinned_aux(size_t count);

  /// Small synchronous helpers (device reduction + read-back).
  double nrm2_sync(const double* x, long long n);
  double dot_sync(const double* x, const double* y, long long n);
  /// Device scratch for up to 64 reduction results (separate from ws()).
  double* results();

 private:
  cudaStream_t stream_ = nullptr;
  ReduceWorkspace ws_;
  int sm_count_ = 148;
  double* pinned_ = nullptr;
  size_t pinned_count_ = 0;
  double* pinned_aux_ = nullptr;
  size_t pinned_aux_count_ = 0;
  DBuffer<double> results_;

 public:
};

/// The calling thread's current context (created on first use, default
/// stream).  Mirrors torch's "current stream" idea so the reference-style
/// signatures (apply(x, y, rec)) need no extra argument.
Context& current_context();
void set_current_stream(cudaStream_t s);

/// RAII scratch vector from the current context's stream-ordered pool.
class Scratch {
 public:
  explicit Scratch(size_t count) : ctx_(&current_context()) { p_ = ctx_->scratch(count); }
  ~Scratch() { if (p_) ctx_->release_scratch(p_); }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  double* get() const { return p_; }

 private:
  Context* ctx_;
  double* p_ = nullptr;
};

/// Device array from the context's stream-ordered pool (release threshold
/// unlimited), so large per-solve buffers - the Krylov basis V, 1.3 GB at
/// config 3 - are recycled between solves instead of cudaMalloc'd each time.
/// Movable; freed on the stream of the context that allocated it.
class PoolBuffer {
 public:
  PoolBuffer() = default;
  ~PoolBuffer() { release(); }
  PoolBuffer(const PoolBuffer&) = delete;
  PoolBuffer& operator=(const PoolBuffer&) = delete;
  PoolBuffer(PoolBuffer&& o) noexcept : ctx_(o.ctx_), p_(o.p_), n_(o.n_) {
    o.p_ = nullptr;
    o.n_ = 0;
  }
  PoolBuffer& operator=(PoolBuffer&& o) noexcept {
    if (this != &o) {
      release();
      ctx_ = o.ctx_;
      p_ = o.p_;
      n_ = o.n_;
      o.p_ = nullptr;
      o.n_ = 0;
    }
    return *this;
  }
  void resize(size_t count) {
    if (count == n_) return;
    release();
    ctx_ = &current_context();
    if (count) p_ = ctx_->scratch(count);
    n_ = count;
  }
  void release() {
    if (p_ && ctx_) ctx_->release_scratch(p_);
    p_ = nullptr;
    n_ = 0;
  }
  double* get() const { return p_; }
  size_t size() const { return n_; }

 private:
  Context* ctx_ = nullptr;
  double* p_ = nullptr;
  size_t n_ = 0;
};

}  // namespace ppa
