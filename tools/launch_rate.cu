// Device-wide kernel launch throughput: S streams each replaying a CUDA graph
// of K dependent tiny kernels (grid G x 256 threads, a few loads each).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__global__ void tiny(double* p, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = p[i] * 1.0000001 + 1.0;
}

int main(int argc, char** argv) {
  int S = argc > 1 ? atoi(argv[1]) : 16, K = argc > 2 ? atoi(argv[2]) : 400, G = argc > 3 ? atoi(argv[3]) : 64;
  int reps = 20;
  std::vector<cudaStream_t> st(S);
  std::vector<cudaGraphExec_t> ge(S);
  std::vector<double*> buf(S);
  for (int s = 0; s < S; ++s) {
    cudaStreamCreateWithFlags(&st[s], cudaStreamNonBlocking);
    cudaMalloc(&buf[s], G * 256 * sizeof(double));
    cudaMemset(buf[s], 0, G * 256 * sizeof(double));
    cudaGraph_t g;
    cudaStreamBeginCapture(st[s], cudaStreamCaptureModeThreadLocal);
    for (int k = 0; k < K; ++k) tiny<<<G, 256, 0, st[s]>>>(buf[s], G * 256);
    cudaStreamEndCapture(st[s], &g);
    cudaGraphInstantiate(&ge[s], g, 0);
    cudaGraphDestroy(g);
  }
  cudaDeviceSynchronize();
  for (int w = 0; w < 2; ++w) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, 0);
    for (int s = 0; s < S; ++s) cudaStreamWaitEvent(st[s], e0, 0);
    for (int r = 0; r < reps; ++r)
      for (int s = 0; s < S; ++s) cudaGraphLaunch(ge[s], st[s]);
    for (int s = 0; s < S; ++s) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, st[s]);
      cudaStreamWaitEvent(0, e, 0);
    }
    cudaEventRecord(e1, 0);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (w) printf("streams=%d kernels/graph=%d grid=%d: %.1f k kernels/s (%.2f us per kernel per stream)\n", S, K, G,
                  (double)S * K * reps / ms, ms * 1e3 / (K * reps));
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
