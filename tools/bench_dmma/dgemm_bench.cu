// Standalone throughput of the FP64 DMMA tile used by the frontal updates:
// C(n x n, lower) -= A D A^T, A n x k column-major.  nvcc -I ../../paper_2009_08167_b200/csrc
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "dmma.cuh"

using namespace riga;

__global__ void __launch_bounds__(256, 1) syrk_tiles128(const double* A, int64_t lda, const double* D, int64_t k,
                                                        double* C, int64_t n) {
  extern __shared__ double sm[];
  const int64_t nt = (n + 127) / 128;
  const int64_t ti = blockIdx.x / nt, tj = blockIdx.x % nt;
  if (ti < tj) return;
  dmma_tile128(A, lda, A, lda, D, 0, k, ti * 128, tj * 128, n, n, C, n, 0, sm);
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 4096, k = argc > 2 ? atoll(argv[2]) : 2048;
  double *A, *C, *D;
  cudaMalloc(&A, n * k * 8);
  cudaMalloc(&C, n * n * 8);
  cudaMalloc(&D, k * 8);
  cudaMemset(A, 0, n * k * 8);
  cudaMemset(C, 0, n * n * 8);
  cudaMemset(D, 0, k * 8);
  cudaFuncSetAttribute(syrk_tiles128, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kT128Smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaFuncSetAttribute(syrk_tiles128, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kT128Smem);
  const int64_t nt2 = (n + 127) / 128;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    syrk_tiles128<<<(unsigned)(nt2 * nt2), 256, kT128Smem>>>(A, n, D, k, C, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = (double)n * (n + 128) * k;
    if (rep) printf("syrk tile128 n=%lld k=%lld: %.3f ms  %.2f TFLOP/s\n", (long long)n, (long long)k, ms,
                    flops / ms / 1e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
