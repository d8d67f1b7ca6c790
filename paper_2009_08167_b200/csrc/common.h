// Shared internals of libriga_b200.so (host + device).
#pragma once

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/riga_b200.h"

namespace riga {

// thread-local last error message (riga_last_error)
void set_error(const std::string& msg);
const char* last_error();

#define RIGA_CHECK_ARG(cond, msg)          \
  do {                                     \
    if (!(cond)) {                         \
      ::riga::set_error(msg);              \
      return RIGA_BAD_ARG;                 \
    }                                      \
  } while (0)

#define RIGA_CUDA(call)                                                                  \
  do {                                                                                   \
    cudaError_t _e = (call);                                                             \
    if (_e != cudaSuccess) {                                                             \
      ::riga::set_error(std::string("CUDA error ") + cudaGetErrorString(_e) + " at " +   \
                        __FILE__ + ":" + std::to_string(__LINE__));                      \
      return _e == cudaErrorMemoryAllocation ? RIGA_OOM : RIGA_CUDA_ERROR;               \
    }                                                                                    \
  } while (0)

#define RIGA_TRY(call)              \
  do {                              \
    int _s = (call);                \
    if (_s != RIGA_OK) return _s;   \
  } while (0)

// Device buffer with RAII release.  Stream-ordered allocation
// (cudaMallocAsync / cudaFreeAsync on the owner's stream): no device-wide
// synchronisation, so concurrent slices on other streams keep running.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  int alloc(size_t count, cudaStream_t stream) {
    release();
    s = stream;
    if (count == 0) return RIGA_OK;
    cudaError_t e = cudaMallocAsync(&p, count * sizeof(T), stream);
    if (e != cudaSuccess) {
      p = nullptr;
      set_error(std::string("cudaMallocAsync of ") + std::to_string(count * sizeof(T)) +
                " bytes failed: " + cudaGetErrorString(e));
      return e == cudaErrorMemoryAllocation ? RIGA_OOM : RIGA_CUDA_ERROR;
    }
    n = count;
    return RIGA_OK;
  }
  // grow-only: keeps the buffer when it already holds `count` elements of this stream
  int reserve(size_t count, cudaStream_t stream) {
    if (p && n >= count && s == stream) return RIGA_OK;
    return alloc(count, stream);
  }
  int upload(const T* host, size_t count, cudaStream_t st) {
    int rc = alloc(count, st);
    if (rc) return rc;
    if (count) RIGA_CUDA(cudaMemcpyAsync(p, host, count * sizeof(T), cudaMemcpyHostToDevice, st));
    return RIGA_OK;
  }
  void swap(DevBuf& o) {
    std::swap(p, o.p);
    std::swap(n, o.n);
    std::swap(s, o.s);
  }
};

}  // namespace riga

struct riga_ctx {
  std::atomic<int> refs{1};  // riga_ctx_destroy + every object created on it
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  double* scratch_host = nullptr;  // pinned scratch for small D2H reads
  double* scratch_dev = nullptr;   // small device scratch (reductions)
  size_t scratch_dev_n = 0;
  // side streams of the factorization (factor.cu, created on first use): [0] panel chain (high
  // priority), [1] solve-side companions (low priority); events for the hand-offs
  cudaStream_t aux[2] = {nullptr, nullptr};
  cudaEvent_t aux_ev[4] = {nullptr, nullptr, nullptr, nullptr};
};

// Device guard: sets the current device for the scope.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

namespace riga {
// Objects keep their context (and so the stream their buffers are freed on)
// alive: declared as the FIRST member of an object, it is destroyed last,
// after every DevBuf of the object has been released on the stream.
void ctx_release(riga_ctx* c);
struct CtxRef {
  riga_ctx* c = nullptr;
  CtxRef() = default;
  CtxRef(const CtxRef&) = delete;
  CtxRef& operator=(const CtxRef&) = delete;
  void set(riga_ctx* x) {
    if (x == c) return;
    if (x) x->refs.fetch_add(1);
    ctx_release(c);
    c = x;
  }
  ~CtxRef() { ctx_release(c); }
};
// Wait for a stream with a blocking-sync event: the host thread sleeps
// instead of spinning (16 slice threads spinning in cudaStreamSynchronize
// would take every core and starve the threads that launch work).
cudaError_t stream_sync(cudaStream_t s);
// Process-wide cache of pinned host blocks: cudaMallocHost / cudaFreeHost
// synchronise the device, so blocks are recycled instead of freed.
void* pinned_get(size_t bytes);
void pinned_put(void* p);
}  // namespace riga
