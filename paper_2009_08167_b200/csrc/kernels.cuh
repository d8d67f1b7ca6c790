// Device helpers shared by the kernels of libriga_b200.so.
#pragma once

#include <cub/cub.cuh>

#include "common.h"

namespace riga {

constexpr int kDotScratch = 1024;  // doubles of device scratch per reduction

// ---- programmatic dependent launch (PDL) -----------------------------------
// The Lanczos step is a chain of ~60 dependent small kernels replayed as a
// CUDA graph; launched with programmatic stream serialization, kernel N+1's
// CTAs are scheduled while kernel N drains, and wait in pdl_start() until N
// has completed and its writes are visible.  pdl_start() is the first
// statement of every step kernel (no global access before it, so no
// read-after-write or write-after-read hazard with the predecessor); the
// trigger after the wait lets the successor launch one kernel ahead only.
// Outside a PDL launch both instructions are no-ops.
__device__ __forceinline__ void pdl_start() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

extern bool g_pdl;  // RIGA_PDL=1 enables

template <typename... KArgs, typename... Args>
inline cudaError_t launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                          Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

__host__ __device__ __forceinline__ int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum, result broadcast to every thread.  red: >= 32 doubles.
__device__ __forceinline__ double block_sum(double v, double* red) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = (threadIdx.x < nw) ? red[threadIdx.x] : 0.0;
  if (w == 0) t = warp_sum(t);
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  double r = red[0];
  __syncthreads();
  return r;
}

__device__ __forceinline__ double block_max(double v, double* red) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = (threadIdx.x < nw) ? red[threadIdx.x] : 0.0;
  if (w == 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
  }
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  double r = red[0];
  __syncthreads();
  return r;
}

inline int inclusive_scan_i64(cudaStream_t s, int64_t* data, int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, bytes, data, data, (int)n, s);
  void* tmp = nullptr;
  RIGA_CUDA(cudaMallocAsync(&tmp, bytes, s));
  cub::DeviceScan::InclusiveSum(tmp, bytes, data, data, (int)n, s);
  RIGA_CUDA(cudaFreeAsync(tmp, s));
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

}  // namespace riga
