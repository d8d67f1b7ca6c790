// FP64 tensor-core tiles: the frontal Schur-complement updates (dmma_tile128),
// the chain-inverse doubling GEMMs and the Lanczos lift / locking GEMMs.
//
// sm_100a has no tcgen05 kind for f64, so FP64 MMA is the warp-level
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  The 64x64 tiles use 4 warps of
// 32x32 (32 fp64 accumulators per thread) with operands staged in shared
// memory k-major at a 72-double pitch (conflict-free fragment loads).
#pragma once

#include <cstdint>

namespace riga {

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

}  // namespace riga

namespace riga {

// C(i, j) = alpha * sum_{t in [k0, k1)} A(i, t) B(t, j) for the 64x64 tile at
// (i0, j0), i < mend, j < nend; A(i, t) = A[t * lda + i] (column-major),
// B(t, j) = B[j * ldb + t] (column-major, t contiguous); C(i, j) =
// C[j * ldc + i] is overwritten.  blockDim.x == 128, 4 warps x 32x32.
__device__ __forceinline__ void dmma_gemm_tile(const double* __restrict__ A, int64_t lda,
                                               const double* __restrict__ B, int64_t ldb, int64_t k0,
                                               int64_t k1, int64_t i0, int64_t j0, int64_t mend, int64_t nend,
                                               double* __restrict__ C, int64_t ldc, double alpha) {
  __shared__ double As[2][16][72];
  __shared__ double Bs[2][16][72];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  double ra[8], rb[8];
  auto load = [&](int64_t kt) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = tid + 128 * u;
      {  // A: 16 k x 64 rows, rows contiguous
        const int t = idx >> 6, i = idx & 63;
        const int64_t kk = kt + t;
        ra[u] = (kk < k1 && i0 + i < mend) ? A[kk * lda + i0 + i] : 0.0;
      }
      {  // B: 64 cols x 16 k, k contiguous
        const int t = idx & 15, j = idx >> 4;
        const int64_t kk = kt + t;
        rb[u] = (kk < k1 && j0 + j < nend) ? B[(j0 + j) * ldb + kk] : 0.0;
      }
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = tid + 128 * u;
      As[buf][idx >> 6][idx & 63] = ra[u];
      Bs[buf][idx & 15][idx >> 4] = rb[u];
    }
  };
  int buf = 0;
  if (k0 < k1) {
    load(k0);
    store(0);
  }
  __syncthreads();
  for (int64_t kt = k0; kt < k1; kt += 16) {
    const bool more = kt + 16 < k1;
    if (more) load(kt + 16);
#pragma unroll
    for (int k4 = 0; k4 < 4; ++k4) {
      const int kr = k4 * 4 + (lane & 3);
      double av[4], bv[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) av[m] = As[buf][kr][wm * 32 + m * 8 + (lane >> 2)];
#pragma unroll
      for (int q = 0; q < 4; ++q) bv[q] = Bs[buf][kr][wn * 32 + q * 8 + (lane >> 2)];
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int q = 0; q < 4; ++q) dmma_8x8x4(acc[m][q][0], acc[m][q][1], av[m], bv[q]);
    }
    if (more) {
      store(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
  const int r = lane >> 2, cc = (lane & 3) * 2;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int64_t i = i0 + wm * 32 + m * 8 + r;
    if (i >= mend) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t j = j0 + wn * 32 + q * 8 + cc;
      if (j < nend) C[j * ldc + i] = alpha * acc[m][q][0];
      if (j + 1 < nend) C[(j + 1) * ldc + i] = alpha * acc[m][q][1];
    }
  }
}

}  // namespace riga

namespace riga {

// ---------------------------------------------------------------------------
// 128 x 128 FP64 DMMA tile with a cp.async pipeline (large frontal updates).
//
//   C(i - coff, j - coff) -= sum_{t in [k0, k1)} A[t lda + i] d[t] B[t ldb + j]
//   for i in [i0, i0 + 128), i < mend, and j in [j0, j0 + 128), j < nend.
//
// 256 threads = 8 warps as 2 (rows) x 4 (cols), each warp 64 x 32 = 8 x 4
// DMMA.8x8x4 tiles (64 fp64 accumulators per thread).  k runs in steps of kT128K
// through kT128Stages shared-memory stages filled by 8-byte cp.async (rows
// of a front are not 16-byte aligned in general) with zero fill outside the
// ranges.  The pivots d (or 1 for nullptr) and the sign are folded into the A
// stage in shared memory one stage ahead of its use, by the thread that copied
// the element (cp.async.wait_group covers a thread's own copies, so no extra
// barrier): the k loop is fragment loads and DMMAs only.  (With the scaling
// in the k loop -- one DMUL per A fragment on the pipe the DMMAs use, in the
// LDS -> DMUL -> DMMA chain of a single reused fragment register -- ncu showed
// the DMMA pipe 67 % active on K = 512 frontal updates.)  Pitch 132 doubles
// (== 4 mod 16): the 16 lanes of a half warp (4 k rows x 4 columns) hit 16
// distinct bank pairs.
// ---------------------------------------------------------------------------
constexpr int kT128 = 128;
#ifndef RIGA_T128K
#define RIGA_T128K 16
#endif
constexpr int kT128K = RIGA_T128K;  // k rows per stage (16 or 32)
constexpr int kT128KG = kT128K / 16;  // k rows of a stage per loader thread
constexpr int kT128P = 132;
constexpr int kT128Stages = kT128K == 16 ? 4 : 3;
constexpr int kT128StageDoubles = 2 * kT128K * kT128P;
constexpr size_t kT128Smem = (size_t)kT128Stages * kT128StageDoubles * sizeof(double) + 2 * kT128Stages * sizeof(uint64_t);

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async8n(double* smem, const double* gmem, int nbytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(nbytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// mbarrier helpers of the tile's stage ring (CTA scope; arrive = release, wait = acquire)
__device__ __forceinline__ void t128_bar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void t128_bar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void t128_bar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned ok = 0;
  while (!ok) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  }
}

// EPI 0: C(i - coff, j - coff) -= A d B^T; EPI 2: the same with the columns j >= jsplit going to C2
// (ld ldc2, rows and columns offset by jsplit) and only i >= j touched (a front's pivot columns and its
// update block in one trailing update; c2_overwrite: C2 = -A d B^T, nothing read from it).  The C tile
// is loaded into the accumulators before the K loop (its 64 loads per thread in flight together,
// overlapping the pipeline prologue) and the MMAs subtract (negated A stage), so the epilogue is
// stores only.
template <int EPI = 0>
__device__ __forceinline__ void dmma_tile128(const double* __restrict__ A, int64_t lda,
                                             const double* __restrict__ B, int64_t ldb,
                                             const double* __restrict__ d, int64_t k0, int64_t k1,
                                             int64_t i0, int64_t j0, int64_t mend, int64_t nend,
                                             double* C, int64_t ldc, int64_t coff,
                                             double* __restrict__ smem, double* C2 = nullptr, int64_t ldc2 = 0,
                                             int64_t jsplit = 0, bool c2_overwrite = false) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  const int r = lane >> 2, cc = (lane & 3) * 2;
  auto cptr = [&](int64_t i, int64_t j) -> double* {
    if (i >= mend || j >= nend) return nullptr;
    if (EPI == 2) {
      if (j > i) return nullptr;
      return j < jsplit ? C + j * ldc + i : C2 + (j - jsplit) * ldc2 + (i - jsplit);
    }
    return C + (j - coff) * ldc + (i - coff);
  };
  double acc[8][4][2];
#pragma unroll
  for (int m = 0; m < 8; ++m)
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t jc = j0 + wn * 32 + q * 8 + cc + e;
        const double* p = cptr(i0 + wm * 64 + m * 8 + r, jc);
        // c2_overwrite: the C2 part holds nothing yet (a front's update block at its first update)
        acc[m][q][e] = p && !(EPI == 2 && c2_overwrite && jc >= jsplit) ? *p : 0.0;
      }
  const int nk = (int)((k1 - k0 + kT128K - 1) / kT128K);
  // thread -> k row kr, columns c8 + 16 u (u < 8) of a stage: one pivot per thread and stage, the
  // 8 copies of an operand at constant offsets from one pointer
  const int kr = tid >> 4, c8 = tid & 15;
  unsigned ma = 0, mb = 0;  // column predicates
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    ma |= (i0 + c8 + 16 * u < mend ? 1u : 0u) << u;
    mb |= (j0 + c8 + 16 * u < nend ? 1u : 0u) << u;
  }
  const bool full = ma == 0xffu && mb == 0xffu;
  const double* Ab = A + (k0 + kr) * lda + i0 + c8;
  const double* Bb = B + (k0 + kr) * ldb + j0 + c8;
  double* const S0 = smem + kr * kT128P + c8;  // this thread's first A element of stage 0
  auto load = [&](int it) {
#pragma unroll
    for (int g = 0; g < kT128KG; ++g) {
      double* As = S0 + (it % kT128Stages) * kT128StageDoubles + 16 * g * kT128P;
      double* Bs = As + kT128K * kT128P;
      const double* pa = Ab + ((int64_t)it * kT128K + 16 * g) * lda;
      const double* pb = Bb + ((int64_t)it * kT128K + 16 * g) * ldb;
      const bool kin = k0 + (int64_t)it * kT128K + 16 * g + kr < k1;
      if (full && kin) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          cp_async8n(As + 16 * u, pa + 16 * u, 8);
          cp_async8n(Bs + 16 * u, pb + 16 * u, 8);
        }
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const bool ina = kin && (ma >> u & 1u), inb = kin && (mb >> u & 1u);
          cp_async8n(As + 16 * u, ina ? pa + 16 * u : A, ina ? 8 : 0);
          cp_async8n(Bs + 16 * u, inb ? pb + 16 * u : B, inb ? 8 : 0);
        }
      }
    }
  };
  // d of this thread's k rows in stage `it` (zero-filled rows: any finite value); the values are only
  // consumed by the next iteration's scale(), so the loads' latency hides behind a stage of MMAs
  auto pivot = [&](int it, int g) -> double {
    const int64_t kk = k0 + (int64_t)it * kT128K + 16 * g + kr;
    return d ? (it < nk && kk < k1 ? d[kk] : 0.0) : 1.0;
  };
  // fold -d into this thread's own A elements of stage `it` (its copies have landed)
  auto scale = [&](int it, const double (&dk)[kT128KG]) {
#pragma unroll
    for (int g = 0; g < kT128KG; ++g) {
      double* As = S0 + (it % kT128Stages) * kT128StageDoubles + 16 * g * kT128P;
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = As[16 * u];
#pragma unroll
      for (int u = 0; u < 8; ++u) As[16 * u] = v[u] * -dk[g];
    }
  };
  // Stage ring without a CTA-wide barrier per stage: full[b] counts the 256 threads that have copied and
  // scaled their part of the stage in buffer b, empty[b] the 256 that have finished reading it.  A thread
  // publishes stage it + 1 before it computes stage it, so by the time any warp wants stage it + 1 the
  // others published it a whole stage ago; the refill of a buffer waits for empty only after the next
  // stage's MMAs have been issued.  (A __syncthreads per stage drained the DMMA pipe at every stage.)
  uint64_t* bfull = reinterpret_cast<uint64_t*>(smem + (size_t)kT128Stages * kT128StageDoubles);
  uint64_t* bempty = bfull + kT128Stages;
  if (tid == 0) {
#pragma unroll
    for (int b = 0; b < kT128Stages; ++b) {
      t128_bar_init(bfull + b, 256);
      t128_bar_init(bempty + b, 256);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < kT128Stages - 1; ++s) {
    if (s < nk) load(s);
    cp_async_commit();
  }
  double dpend[kT128KG];  // pivots of the stage scaled next (loaded one iteration ahead of their use)
  {
    double d0[kT128KG];
#pragma unroll
    for (int g = 0; g < kT128KG; ++g) {
      d0[g] = pivot(0, g);
      dpend[g] = pivot(1, g);
    }
    cp_async_wait<kT128Stages - 2>();
    if (nk > 0) {
      scale(0, d0);
      t128_bar_arrive(bfull + 0);
    }
  }
  const double* Af = smem + (lane & 3) * kT128P + wm * 64 + (lane >> 2);
  const double* Bf = smem + kT128K * kT128P + (lane & 3) * kT128P + wn * 32 + (lane >> 2);
  for (int it = 0; it < nk; ++it) {
    const int buf = it % kT128Stages;
    cp_async_wait<kT128Stages - 3>();  // this thread's copies of stage it + 1 have landed
    if (it + 1 < nk) {
      scale(it + 1, dpend);
      t128_bar_arrive(bfull + (it + 1) % kT128Stages);
    }
#pragma unroll
    for (int g = 0; g < kT128KG; ++g) dpend[g] = pivot(it + 2, g);
    t128_bar_wait(bfull + buf, (unsigned)(it / kT128Stages) & 1u);
    const double* As = Af + buf * kT128StageDoubles;
    const double* Bs = Bf + buf * kT128StageDoubles;
    double av[2][8], bv[2][4];
#pragma unroll
    for (int m = 0; m < 8; ++m) av[0][m] = As[m * 8];
#pragma unroll
    for (int q = 0; q < 4; ++q) bv[0][q] = Bs[q * 8];
#pragma unroll
    for (int k4 = 0; k4 < kT128K / 4; ++k4) {
      const int cur = k4 & 1, nxt = cur ^ 1;
      if (k4 < kT128K / 4 - 1) {
#pragma unroll
        for (int m = 0; m < 8; ++m) av[nxt][m] = As[(k4 + 1) * 4 * kT128P + m * 8];
#pragma unroll
        for (int q = 0; q < 4; ++q) bv[nxt][q] = Bs[(k4 + 1) * 4 * kT128P + q * 8];
      }
#pragma unroll
      for (int m = 0; m < 8; ++m)
#pragma unroll
        for (int q = 0; q < 4; ++q) dmma_8x8x4(acc[m][q][0], acc[m][q][1], av[cur][m], bv[cur][q]);
      if (k4 == 0) {
        // refill: stage it + Stages - 1 goes into the buffer stage it - 1 used; every thread has read it once
        // empty completes (its MMAs of stage it - 1 were issued a stage ago, so this rarely waits)
        const int nx = it + kT128Stages - 1;
        if (nx < nk) {
          if (it >= 1) t128_bar_wait(bempty + nx % kT128Stages, (unsigned)((it - 1) / kT128Stages) & 1u);
          load(nx);
        }
        cp_async_commit();
      }
    }
    t128_bar_arrive(bempty + buf);
  }
  cp_async_wait<0>();
#pragma unroll
  for (int m = 0; m < 8; ++m)
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double* p = cptr(i0 + wm * 64 + m * 8 + r, j0 + wn * 32 + q * 8 + cc + e);
        if (p) *p = acc[m][q][e];
      }
}

}  // namespace riga

namespace riga {

// General-stride 64 x 64 FP64 DMMA tile (4 warps x 32 x 32):
//   acc(i, j) = sum_{t in [k0, k1)} A(i, t) B(j, t)
//   A(i, t) = A[i as_i + t as_t],  B(j, t) = B[j bs_j + t bs_t]
//   C(i, j) = C[i cs_i + j cs_j]  <- alpha acc  (sub: C -= acc)
// Operand loads are coalesced along whichever of i / t has unit stride.
__device__ __forceinline__ void dmma_tile_gen(const double* __restrict__ A, int64_t as_i, int64_t as_t,
                                              const double* __restrict__ B, int64_t bs_j, int64_t bs_t, int64_t k0,
                                              int64_t k1, int64_t i0, int64_t j0, int64_t mend, int64_t nend,
                                              double* __restrict__ C, int64_t cs_i, int64_t cs_j, double alpha,
                                              bool sub) {
  __shared__ double As[2][16][72];
  __shared__ double Bs[2][16][72];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const bool a_icont = as_i == 1, b_jcont = bs_j == 1;
  double ra[8], rb[8];
  auto load = [&](int64_t kt) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = tid + 128 * u;
      {
        const int t = a_icont ? idx >> 6 : idx & 15, i = a_icont ? idx & 63 : idx >> 4;
        const int64_t kk = kt + t;
        ra[u] = (kk < k1 && i0 + i < mend) ? A[(i0 + i) * as_i + kk * as_t] : 0.0;
      }
      {
        const int t = b_jcont ? idx >> 6 : idx & 15, j = b_jcont ? idx & 63 : idx >> 4;
        const int64_t kk = kt + t;
        rb[u] = (kk < k1 && j0 + j < nend) ? B[(j0 + j) * bs_j + kk * bs_t] : 0.0;
      }
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = tid + 128 * u;
      if (a_icont) As[buf][idx >> 6][idx & 63] = ra[u];
      else As[buf][idx & 15][idx >> 4] = ra[u];
      if (b_jcont) Bs[buf][idx >> 6][idx & 63] = rb[u];
      else Bs[buf][idx & 15][idx >> 4] = rb[u];
    }
  };
  int buf = 0;
  if (k0 < k1) {
    load(k0);
    store(0);
  }
  __syncthreads();
  for (int64_t kt = k0; kt < k1; kt += 16) {
    const bool more = kt + 16 < k1;
    if (more) load(kt + 16);
#pragma unroll
    for (int k4 = 0; k4 < 4; ++k4) {
      const int kr = k4 * 4 + (lane & 3);
      double av[4], bv[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) av[m] = As[buf][kr][wm * 32 + m * 8 + (lane >> 2)];
#pragma unroll
      for (int q = 0; q < 4; ++q) bv[q] = Bs[buf][kr][wn * 32 + q * 8 + (lane >> 2)];
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int q = 0; q < 4; ++q) dmma_8x8x4(acc[m][q][0], acc[m][q][1], av[m], bv[q]);
    }
    if (more) {
      store(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
  const int r = lane >> 2, cc = (lane & 3) * 2;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int64_t i = i0 + wm * 32 + m * 8 + r;
    if (i >= mend) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t j = j0 + wn * 32 + q * 8 + cc;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (j + e < nend) {
          double* p = C + i * cs_i + (j + e) * cs_j;
          *p = sub ? *p - acc[m][q][e] : alpha * acc[m][q][e];
        }
      }
    }
  }
}

}  // namespace riga
