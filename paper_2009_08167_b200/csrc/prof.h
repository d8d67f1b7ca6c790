// Launch counting and per-category device timing (CUDA events on the
// launching stream) used by bench.py for the roofline numbers.
#pragma once

#include <atomic>
#include <cstdint>

#include <cuda_runtime.h>

namespace riga {

enum ProfCat {
  kProfFactor = 0,  // numeric LDL^T (work = factor_flops)
  kProfSolve = 1,   // supernodal fwd/bwd solve (bytes = 16 fill + 32 n)
  kProfSpmv = 2,    // CSR SpMV (bytes = 12 nnz + 4 (n+1) + 16 n)
  kProfCgs = 3,     // one CGS pass (bytes = 2 rows n 8)
  kProfVec = 4,     // dots / residual / normalise
  kProfLift = 5,    // lift / restart skinny GEMMs
  kProfTrail = 6,   // frontal Schur-complement updates (k_trail128; work = their flops)
  kProfCount = 7
};

extern std::atomic<long long> g_launches;
// launches issued by this thread (graph capture is thread-local, so the
// kernels a capture recorded are this counter's difference across it)
extern thread_local long long t_launches;
inline void count_launch(int n = 1) {
  g_launches.fetch_add(n, std::memory_order_relaxed);
  t_launches += n;
}

bool prof_on();  // per-category timing enabled (riga_prof_enable)

struct ProfScope {
  int cat;
  cudaStream_t s;
  double work;
  cudaEvent_t e0 = nullptr;
  ProfScope(int cat, cudaStream_t s, double work);
  ~ProfScope();
};

}  // namespace riga
