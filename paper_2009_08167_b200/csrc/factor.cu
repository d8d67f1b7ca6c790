// Multifrontal supernodal LDL^T of K - sigma M and the supernodal solves.
//
//  riga_factor       <- factor_ldl + _ldl_numeric  ref sparsela.py:212-262, :118-159
//  riga_factor_solve <- solve_fb + _ldl_solve      ref sparsela.py:265-277, :162-175
//
// Schedule (per factorization, all on one stream, level by level bottom-up):
//   k_tol            zero_tol = rel * max|K - sigma M| (device reduction)
//   k_asm_large      original entries -> panels of the large fronts
//   per level:
//     k_extend_add   child update blocks -> large parent fronts (rounds of
//                    distinct parents, so no atomics and a fixed order)
//     k_small_front  one CTA per front with f <= kSmallFront: the whole front
//                    (originals + children) in shared memory, dense LDL^T of
//                    the pivot block, Schur complement written back
//     large fronts   right-looking blocked LDL^T in HBM: per 128-column block
//                    k_diag128 (diagonal block in shared memory), k_trsm128
//                    (rows below, blocked substitution), narrow k_trail128
//                    inside the nb2-column outer block and one wide
//                    k_trail128 per outer block over the remaining pivot
//                    columns AND the update block (K = nb2, 128 x 128 tiles
//                    of mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4)
// Inertia = count of negative pivots (integer atomics, order independent).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <utility>

#include "dmma.cuh"
#include "internal.h"
#include "kernels.cuh"
#include "prof.h"

namespace riga {


// ---------------------------------------------------------------------------
__global__ void k_tol(int64_t nnz, const double* __restrict__ K, const double* __restrict__ M,
                      double sigma, double rel, double* __restrict__ partial,
                      unsigned* __restrict__ ticket, double* __restrict__ tol,
                      int64_t* __restrict__ stat, int64_t n) {
  __shared__ double red[32];
  __shared__ bool last;
  double m = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz;
       q += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(__dsub_rn(K[q], __dmul_rn(sigma, M[q]))));
  m = block_max(m, red);
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = m;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    double t = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x)
      t = fmax(t, ((volatile double*)partial)[i]);
    t = block_max(t, red);
    if (threadIdx.x == 0) {
      tol[0] = t;
      tol[1] = rel * t;
      stat[0] = 0;
      stat[1] = n;
      *ticket = 0u;
    }
  }
}

__global__ void k_asm_large(SymDev S, const int32_t* __restrict__ nodes,
                            const double* __restrict__ K, const double* __restrict__ M,
                            double sigma, double* __restrict__ panel) {
  int s = nodes[blockIdx.x];
  double* P = panel + S.panel_off[s];
  for (int64_t e = S.asm_ptr[s] + threadIdx.x; e < S.asm_ptr[s + 1]; e += blockDim.x) {
    int32_t q = S.asm_slot[e];
    P[S.asm_local[e]] = __dsub_rn(K[q], __dmul_rn(sigma, M[q]));
  }
}

// child update block (lower triangle, ld nu_c) scatter-added into the parent:
// part 0 = the columns that land in the parent's pivot columns (before the
// parent is factored), part 1 = the columns that land in the parent's update
// block (after the parent's own Schur complement has been written there)
constexpr int kEaRows = 1024;  // rows of a child column handled by one CTA (grid z = row chunks)
__global__ void __launch_bounds__(256) k_extend_add(SymDev S, const int32_t* __restrict__ items, int part,
                                                    double* __restrict__ panel, double* __restrict__ cb) {
  const int c = items[blockIdx.y];
  const int p = S.sparent[c];
  const int64_t nuc = S.front[c] - S.ncol[c];
  const int64_t b0 = (int64_t)blockIdx.x * 32;
  const int64_t z0 = (int64_t)blockIdx.z * kEaRows, z1 = min(z0 + kEaRows, nuc);
  if (b0 >= nuc || z1 <= b0) return;  // past the child's columns, or a chunk above the diagonal
  const int64_t fp = S.front[p], npp = S.ncol[p], nup = fp - npp;
  const double* src = cb + S.cb_off[c];
  const int32_t* __restrict__ rp = S.relpos + S.upd_off[c];
  double* P = panel + S.panel_off[p];
  double* C = cb + S.cb_off[p];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t b = b0 + w; b < min(b0 + 32, nuc); b += nw) {
    const int64_t rb = rp[b];
    if ((rb < npp) != (part == 0)) continue;
    // destination column: entry (ra, rb) of the parent front
    double* dst = rb < npp ? P + rb * fp : C + (rb - npp) * nup - npp;
    const double* sc = src + b * nuc;
    int64_t a = max(b, z0) + lane;
    for (; a + 224 < z1; a += 256) {  // eight independent read-modify-writes in flight per lane (16: no gain)
      int32_t r[8];
      double v[8], d[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) r[u] = rp[a + 32 * u];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = sc[a + 32 * u];
#pragma unroll
      for (int u = 0; u < 8; ++u) d[u] = dst[r[u]];
#pragma unroll
      for (int u = 0; u < 8; ++u) dst[r[u]] = d[u] + v[u];
    }
    for (; a + 96 < z1; a += 128) {
      const int32_t r0 = rp[a], r1 = rp[a + 32], r2 = rp[a + 64], r3 = rp[a + 96];
      const double v0 = sc[a], v1 = sc[a + 32], v2 = sc[a + 64], v3 = sc[a + 96];
      const double d0 = dst[r0], d1 = dst[r1], d2 = dst[r2], d3 = dst[r3];
      dst[r0] = d0 + v0;
      dst[r1] = d1 + v1;
      dst[r2] = d2 + v2;
      dst[r3] = d3 + v3;
    }
    for (; a < z1; a += 32) dst[rp[a]] += sc[a];
  }
}

// ---------------------------------------------------------------------------
// Small fronts: whole front in shared memory (column-major, odd ld).
// ---------------------------------------------------------------------------
#ifndef RIGA_SF_PANEL
#define RIGA_SF_PANEL 8
#endif
constexpr int kSfPanel = RIGA_SF_PANEL;  // pivots per panel of k_small_front
__global__ void __launch_bounds__(512) k_small_front(SymDev S, const int32_t* __restrict__ nodes,
                                                     const double* __restrict__ K,
                                                     const double* __restrict__ M, double sigma,
                                                     const double* __restrict__ tol,
                                                     double* __restrict__ panel,
                                                     double* __restrict__ cb,
                                                     double* __restrict__ D,
                                                     int64_t* __restrict__ stat) {
  extern __shared__ double F[];
  const int s = nodes[blockIdx.x];
  const int f = (int)S.front[s], np = (int)S.ncol[s], nu = f - np;
  const int ld = f | 1;
  const int64_t col0 = S.col0[s];
  double* lb0 = F + f * ld;  // 2 x kSfPanel x f: the scaled pivot columns of two panels
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
  for (int i = tid; i < f * ld; i += blockDim.x) F[i] = 0.0;
  __syncthreads();
  for (int64_t e = S.asm_ptr[s] + tid; e < S.asm_ptr[s + 1]; e += blockDim.x) {
    int loc = S.asm_local[e];
    int col = loc / f, row = loc - col * f;
    int32_t q = S.asm_slot[e];
    F[col * ld + row] = __dsub_rn(K[q], __dmul_rn(sigma, M[q]));
  }
  __syncthreads();
  for (int64_t t = S.child_ptr[s]; t < S.child_ptr[s + 1]; ++t) {
    int c = S.child_list[t];
    int nuc = (int)(S.front[c] - S.ncol[c]);
    const double* src = cb + S.cb_off[c];
    const int32_t* rp = S.relpos + S.upd_off[c];
    for (int b = w; b < nuc; b += nw) {
      int rb = rp[b];
      for (int a = b + lane; a < nuc; a += 32) F[rb * ld + rp[a]] += src[b * nuc + a];
    }
    __syncthreads();
  }
  const double tv = tol[1];
  int neg = 0;
  int64_t bad = INT64_MAX;
  // Right-looking LDL^T in panels of kSfPanel pivots: inside a panel each pivot updates only the panel's
  // remaining columns; the columns to its right then take the panel's kSfPanel rank-1 updates in one pass
  // (one load and one store of an entry per panel instead of per pivot, the same fused multiply-adds in the
  // same order: the factor is bitwise that of the pivot-by-pivot loop).  Two panel buffers of scaled columns,
  // so a panel's write-back overlaps the next panel's first pivot.
  for (int k0 = 0, pb = 0; k0 < np; k0 += kSfPanel, pb ^= 1) {
    const int pw = min(kSfPanel, np - k0);
    double* lbp = lb0 + pb * kSfPanel * f;
    for (int q = 0; q < pw; ++q) {
      const int k = k0 + q;
      double* lb = lbp + q * f;
      const double d = F[k * ld + k];
      if (tid == 0) {
        D[col0 + k] = d;
        if (d < 0.0) neg++;
        if (fabs(d) < tv && bad == INT64_MAX) bad = col0 + k;
      }
      for (int i = k + 1 + tid; i < f; i += blockDim.x) lb[i] = F[k * ld + i] / d;
      __syncthreads();
      const int j = k + 1 + w;  // the panel's remaining columns (at most kSfPanel - 1 warps busy)
      if (j < k0 + pw) {
        const double cj = F[k * ld + j];
        double* Fj = F + j * ld;
        for (int i = j + lane; i < f; i += 32) Fj[i] -= lb[i] * cj;
      }
      if (q + 1 < pw) __syncthreads();
    }
    for (int j = k0 + pw + w; j < f; j += nw) {
      double c[kSfPanel];
#pragma unroll
      for (int q = 0; q < kSfPanel; ++q) c[q] = q < pw ? F[(k0 + q) * ld + j] : 0.0;
      double* Fj = F + j * ld;
      if (pw == kSfPanel) {
        for (int i = j + lane; i < f; i += 32) {
          double x = Fj[i];
#pragma unroll
          for (int q = 0; q < kSfPanel; ++q) x -= lbp[q * f + i] * c[q];
          Fj[i] = x;
        }
      } else {
        for (int i = j + lane; i < f; i += 32) {
          double x = Fj[i];
          for (int q = 0; q < pw; ++q) x -= lbp[q * f + i] * c[q];
          Fj[i] = x;
        }
      }
    }
    __syncthreads();
    for (int q = 0; q < pw; ++q)
      for (int i = k0 + q + 1 + tid; i < f; i += blockDim.x) F[(k0 + q) * ld + i] = lbp[q * f + i];
  }
  __syncthreads();
  if (tid == 0) {
    if (neg) atomicAdd((unsigned long long*)&stat[0], (unsigned long long)neg);
    if (bad != INT64_MAX) atomicMin((long long*)&stat[1], (long long)bad);
  }
  double* P = panel + S.panel_off[s];
  for (int c = w; c < np; c += nw)
    for (int r = lane; r < f; r += 32) P[(int64_t)c * f + r] = F[c * ld + r];
  if (nu > 0) {
    double* C = cb + S.cb_off[s];
    for (int b = w; b < nu; b += nw)
      for (int a = b + lane; a < nu; a += 32) C[(int64_t)b * nu + a] = F[(np + b) * ld + np + a];
  }
}

// ---------------------------------------------------------------------------
// Large fronts: blocked right-looking LDL^T with 128-column blocks, three
// launches per block (all large fronts of a level batched in grid y):
//   k_diag128   one CTA per front: the nb x nb diagonal block (nb <= 128) in
//               shared memory in 32-column steps -- warp 0 factors the 32 x 32
//               sub-block in registers, the rows below it inside the block
//               are solved by substitution (thread per row), the rest of the
//               block takes the rank-32 update on DMMA; writes L11 (d on the
//               diagonal), D and the inertia / zero-pivot counters
//   k_trsm128   L21 = A21 L11^{-T} D^{-1} for every row below the block by
//               blocked substitution: warp per 32 rows, per 32-column step the
//               update from the earlier steps on DMMA, then substitution
//   k_trail128  trailing columns -= L21 D L21^T (128 x 128 DMMA tiles)
// No triangular factor is ever inverted explicitly: explicit inverses (128 x
// 128 or even 32 x 32 diagonal blocks) measured 1.6-1.9e-10 solve backward
// error on cfg4 IGA against 4e-12 for substitution.
// ---------------------------------------------------------------------------
constexpr int kDB = 128;
constexpr int kDBP = kDB + 1;
constexpr size_t kDiag128Smem = ((size_t)kDB * kDBP + 2 * kDB) * sizeof(double);

// acc(i, j) += sum_{t < kcount} fa(i, t) fb(t, j) for a 32 x 32 warp tile (kcount % 4 == 0)
template <class FA, class FB>
__device__ __forceinline__ void warp_mma32(double (&acc)[4][4][2], FA fa, FB fb, int kcount) {
  const int lane = threadIdx.x & 31;
  for (int k4 = 0; k4 < kcount; k4 += 4) {
    const int kr = k4 + (lane & 3);
    double av[4], bv[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) av[m] = fa(m * 8 + (lane >> 2), kr);
#pragma unroll
    for (int q = 0; q < 4; ++q) bv[q] = fb(kr, q * 8 + (lane >> 2));
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int q = 0; q < 4; ++q) dmma_8x8x4(acc[m][q][0], acc[m][q][1], av[m], bv[q]);
  }
}

__device__ __forceinline__ void zero_acc(double (&acc)[4][4][2]) {
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[m][q][0] = acc[m][q][1] = 0.0;
}

// accumulator element e of (m, q): row m * 8 + lane / 4, column q * 8 + 2 (lane % 4) + e
#define RIGA_ACC_FOR(body)                                                     \
  _Pragma("unroll") for (int m = 0; m < 4; ++m)                                \
    _Pragma("unroll") for (int q = 0; q < 4; ++q)                              \
      _Pragma("unroll") for (int e = 0; e < 2; ++e) {                          \
        const int ai = m * 8 + (lane >> 2), aj = q * 8 + (lane & 3) * 2 + e; \
        body                                                                   \
      }

// Warp: unblocked LDL^T of the 32 x 32 lower block at A[c * ld + r] (r >= c) in
// registers (lane = row); L (strict lower) and d (diagonal) are written back.
// The pivot steps are template instances (compile-time indices), so the
// register array never falls back to local memory.
template <int K>
__device__ __forceinline__ void ldl32_step(double (&a)[32], int lane, double& dl) {
  const double dk = __shfl_sync(0xffffffffu, a[K], K);
  const double lk = a[K] * (1.0 / dk);
  // every lane updates its whole row: the entries right of the diagonal (lane < j) hold garbage that no
  // later step reads and the write-back skips, so the update needs no per-element predicate
#pragma unroll
  for (int j = K + 1; j < 32; ++j) {
    const double ajk = __shfl_sync(0xffffffffu, a[K], j);  // A(j, K), not yet scaled
    a[j] = fma(-lk, ajk, a[j]);
  }
  if (lane == K) dl = dk;
  if (lane > K) a[K] = lk;
}

// One row of a 32-column block solve by substitution: w[c] <- (w[c] - sum_{t<c} w[t] d(t) L(c, t)) / d(c),
// i.e. row L(r, kb:kb+32) = A(r, kb:kb+32) L_bb^{-T} D_b^{-1} with compile-time column indices.
template <int C, class FL>
__device__ __forceinline__ void sub32_col(double (&w)[32], FL L) {
  // w[t < C] hold u_t = L(r, t) d_t; u_C = A(r, C) - sum_{t<C} u_t L(C, t) in four independent chains
  double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int t = 0; t < C; ++t) s[t & 3] = fma(w[t], L(C, t), s[t & 3]);
  w[C] -= (s[0] + s[1]) + (s[2] + s[3]);
}

// One row of a 32-column block solve by substitution, L(r, kb:kb+32) = A(r, kb:kb+32) L_bb^{-T} D_b^{-1}
// (compile-time column indices): on return w[c] = L(r, c); rd(c) = 1 / d_c.
template <class FL, class FR, int... C>
__device__ __forceinline__ void sub32_all(double (&w)[32], FL L, FR rd, std::integer_sequence<int, C...>) {
  (sub32_col<C>(w, L), ...);
#pragma unroll
  for (int c = 0; c < 32; ++c) w[c] *= rd(c);
}

template <int... K>
__device__ __forceinline__ void ldl32_all(double (&a)[32], int lane, double& dl, std::integer_sequence<int, K...>) {
  (ldl32_step<K>(a, lane, dl), ...);
}

__device__ __forceinline__ void warp_ldl32(double* A, int ld, double& d_out) {
  const int lane = threadIdx.x & 31;
  double dl = 0.0;
  double a[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) a[j] = j <= lane ? A[j * ld + lane] : 0.0;
  ldl32_all(a, lane, dl, std::make_integer_sequence<int, 32>{});
#pragma unroll
  for (int j = 0; j < 32; ++j)
    if (j <= lane) A[j * ld + lane] = j == lane ? dl : a[j];
  d_out = dl;
}

__global__ void __launch_bounds__(256) k_diag128(SymDev S, const int32_t* __restrict__ nodes, int kbo,
                                                 const double* __restrict__ tol, double* __restrict__ panel,
                                                 double* __restrict__ D, int64_t* __restrict__ stat) {
  extern __shared__ double sm[];
  double* A = sm;               // A[c * kDBP + r], lower triangle
  double* dd = A + kDB * kDBP;  // pivots
  double* rdd = dd + kDB;       // their reciprocals
  const int s = nodes[blockIdx.x];
  const int64_t f = S.front[s], np = S.ncol[s];
  if (kbo >= np) return;
  const int nb = (int)imin(kDB, np - kbo);
  const int nbp = (nb + 31) & ~31;
  const int64_t col0 = S.col0[s];
  double* P = panel + S.panel_off[s] + (int64_t)kbo * f + kbo;  // (r, c) of the block at P[c f + r]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // stage the block with cp.async (every load in flight at once; padding rows/columns: zero fill,
  // identity pivots written after the wait); warp per column, lanes along the rows
  for (int c = warp; c < nbp; c += 8)
    for (int r = (c & ~31) + lane; r < nbp; r += 32) {
      const bool in = r >= c && r < nb && c < nb;
      if (r >= c) cp_async8(A + c * kDBP + r, in ? P + (int64_t)c * f + r : P, in);
    }
  cp_async_commit();
  cp_async_wait<0>();
  for (int c = nb + tid; c < nbp; c += blockDim.x) A[c * kDBP + c] = 1.0;
  __syncthreads();
  for (int kb = 0; kb < nbp; kb += 32) {
    if (warp == 0) {
      double dl;
      warp_ldl32(A + kb * kDBP + kb, kDBP, dl);
      dd[kb + lane] = dl;
      rdd[kb + lane] = 1.0 / dl;
    }
    __syncthreads();
    // rows below the sub-block inside the block: substitution, thread per row
    const int nr = nbp - kb - 32;
    if (tid < nr) {
      const int r = kb + 32 + tid;
      double w[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) w[c] = A[(kb + c) * kDBP + r];
      sub32_all(w, [&](int c, int t) { return A[(kb + t) * kDBP + kb + c]; }, [&](int c) { return rdd[kb + c]; },
                std::make_integer_sequence<int, 32>{});
#pragma unroll
      for (int c = 0; c < 32; ++c) A[(kb + c) * kDBP + r] = w[c];
    }
    __syncthreads();
    // the rest of the block -= L D L^T (rank 32): 32 x 32 lower tiles on DMMA, one per warp
    const int n3 = nr / 32;
    for (int t = warp; t < n3 * (n3 + 1) / 2; t += 8) {
      int ti = 0;
      while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
      const int tj = t - ti * (ti + 1) / 2;
      const int i0 = kb + 32 + 32 * ti, j0 = kb + 32 + 32 * tj;
      double acc[4][4][2];
      zero_acc(acc);
      warp_mma32(acc, [&](int i, int k) { return A[(kb + k) * kDBP + i0 + i] * dd[kb + k]; },
                 [&](int k, int j) { return A[(kb + k) * kDBP + j0 + j]; }, 32);
      RIGA_ACC_FOR(if (i0 + ai >= j0 + aj) A[(j0 + aj) * kDBP + i0 + ai] -= acc[m][q][e];)
    }
    __syncthreads();
  }
  if (tid == 0) {  // pivots: D, inertia, first zero pivot
    int neg = 0;
    int64_t bad = INT64_MAX;
    const double tv = tol[1];
    for (int k = 0; k < nb; ++k) {
      const double d = dd[k];
      D[col0 + kbo + k] = d;
      if (d < 0.0) neg++;
      if (fabs(d) < tv && bad == INT64_MAX) bad = col0 + kbo + k;
    }
    if (neg) atomicAdd((unsigned long long*)&stat[0], (unsigned long long)neg);
    if (bad != INT64_MAX) atomicMin((long long*)&stat[1], (long long)bad);
  }
  for (int c = warp; c < nb; c += 8)  // L11, d on the diagonal
    for (int r = (c & ~31) + lane; r < nb; r += 32)
      if (r >= c) P[(int64_t)c * f + r] = A[c * kDBP + r];
}

// L21 = A21 L11^{-T} D^{-1} for the rows below the block, by blocked substitution: a CTA of four warps takes
// 128 rows, one warp per 32 rows.  Per 32-column step b the CTA stages the L11 row strip L(b rows, 0 : b + 32)
// once for its four warps; a warp stages its 32 x 32 slice A_b, subtracts sum_{t<b} W_t D_t L_bt^T on DMMA
// (the earlier slices W_t are read back from the panel, where the warp stored them as final L21 columns --
// ld.global.cg, one fragment ahead of its use), then W_b = T L_bb^{-T} D_b^{-1} row by row (lane = row) and
// stores it.  Only the strip and one 32 x 32 tile per warp live in shared memory (74 KB per CTA: twelve
// warps per SM; the previous one-warp CTAs kept their whole 32 x 128 row block there, three warps per SM).
constexpr int kTrsmP = 36;  // pitch == 4 mod 16: conflict-free DMMA fragment loads
constexpr int kTrsmWarps = 4;
constexpr size_t kTrsmSmem = ((size_t)kDB * kTrsmP + kTrsmWarps * 32 * kTrsmP + 2 * kDB) * sizeof(double);

__device__ __forceinline__ void cp_async8_cg(double* smem, const double* gmem, bool pred) {
  // 8-byte cp.async has only the .ca form; the slices a warp re-reads after storing them go through
  // ld.global.cg instead (below), so a stale L1 line is never consulted
  cp_async8(smem, gmem, pred);
}

__global__ void __launch_bounds__(32 * kTrsmWarps, 3) k_trsm128(SymDev S, const int32_t* __restrict__ nodes, int kbo,
                                                             double* __restrict__ panel,
                                                             const double* __restrict__ D) {
  extern __shared__ double sm[];
  const int s = nodes[blockIdx.y];
  const int64_t f = S.front[s], np = S.ncol[s];
  if (kbo >= np) return;
  const int nb = (int)imin(kDB, np - kbo);
  const int nbp = (nb + 31) & ~31;
  const int64_t R0 = kbo + nb + (int64_t)blockIdx.x * (32 * kTrsmWarps);
  if (R0 >= f) return;  // CTA-uniform
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = R0 + 32 * warp;
  const bool active = r0 < f;
  const int nr = active ? (int)imin(32, f - r0) : 0;
  const int64_t col0 = S.col0[s];
  double* Ls = sm;                                   // strip: L(kb + j, t) at Ls[t * kTrsmP + j]
  double* Wt = Ls + kDB * kTrsmP + warp * 32 * kTrsmP;  // this warp's slice: (row, kb + c) at Wt[c * kTrsmP + row]
  double* ds = sm + kDB * kTrsmP + kTrsmWarps * 32 * kTrsmP;  // pivots
  double* rds = ds + kDB;                            // their reciprocals
  const double* Lb = panel + S.panel_off[s] + (int64_t)kbo * f + kbo;  // L11(r, c) at Lb[c f + r]
  double* Pr = panel + S.panel_off[s] + (int64_t)kbo * f + r0;         // A21(row, c) at Pr[c f + row]
  for (int c = threadIdx.x; c < nbp; c += blockDim.x) {
    const double d = c < nb ? D[col0 + kbo + c] : 1.0;
    ds[c] = d;
    rds[c] = 1.0 / d;
  }
  for (int kb = 0; kb < nbp; kb += 32) {
    const bool rowin = kb + lane < nb;
    for (int t = warp; t < kb + 32; t += kTrsmWarps) {
      const bool in = rowin && t < nb;
      cp_async8(Ls + t * kTrsmP + lane, in ? Lb + (int64_t)t * f + kb + lane : Lb, in);
    }
#pragma unroll 8
    for (int c = 0; c < 32; ++c) {
      const bool in = kb + c < nb && lane < nr;
      cp_async8_cg(Wt + c * kTrsmP + lane, in ? Pr + (int64_t)(kb + c) * f + lane : Lb, in);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();  // strip (and ds / rds on the first pass) visible to the four warps
    if (active) {
      if (kb > 0) {  // T = A_b - sum_{t < b} W_t D_t L_bt^T, the W_t read back from the panel
        double acc[4][4][2];
        zero_acc(acc);
        const int kq = lane & 3, ir = lane >> 2;
        auto load_a = [&](double (&av)[4], int k4) {
          const int kr = k4 + kq;
          const double dk = ds[kr];
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            const int i = m * 8 + ir;
            av[m] = i < nr ? __ldcg(Pr + (int64_t)kr * f + i) * dk : 0.0;
          }
        };
        double an[4];
        load_a(an, 0);
        for (int k4 = 0; k4 < kb; k4 += 4) {
          double av[4], bv[4];
#pragma unroll
          for (int m = 0; m < 4; ++m) av[m] = an[m];
          if (k4 + 4 < kb) load_a(an, k4 + 4);
#pragma unroll
          for (int q = 0; q < 4; ++q) bv[q] = Ls[(k4 + kq) * kTrsmP + q * 8 + ir];
#pragma unroll
          for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int q = 0; q < 4; ++q) dmma_8x8x4(acc[m][q][0], acc[m][q][1], av[m], bv[q]);
        }
        RIGA_ACC_FOR(Wt[aj * kTrsmP + ai] -= acc[m][q][e];)
        __syncwarp();
      }
      double w[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) w[c] = Wt[c * kTrsmP + lane];
      sub32_all(w, [&](int c, int t) { return Ls[(kb + t) * kTrsmP + c]; }, [&](int c) { return rds[kb + c]; },
                std::make_integer_sequence<int, 32>{});
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (kb + c < nb && lane < nr) Pr[(int64_t)(kb + c) * f + lane] = w[c];
      __syncwarp();  // the stores are ordered before the next step's fragment loads of this warp
    }
    __syncthreads();  // every warp is done with the strip before it is restaged
  }
}

// Trailing update of a front over its pivot columns [k0, min(k1, n_p)), lower triangle, rows to f.
//   narrow (wide = 0): the columns [c0, min(c1, n_p)) -- the rest of the current outer block;
//   wide   (wide = 1): every column right of min(c0, n_p) -- the remaining pivot columns and the update
//                      block (columns >= n_p live in the front's update block, so the update block takes
//                      its Schur complement slice by slice with the pivot columns instead of one long-K
//                      pass at the end).
// tri != 0: blockIdx.x enumerates the lower tiles of a triangle of ntj x ntj tiles.
// first != 0: the update block holds nothing yet and is written, not accumulated (the children's
// contributions are extend-added into it afterwards), so it is never zeroed or read here.
__global__ void __launch_bounds__(256, 1) k_trail128(SymDev S, const int32_t* __restrict__ nodes, int64_t k0,
                                                     int64_t k1, int64_t c0, int64_t c1, int wide, int ntj,
                                                     int tri, int first, double* __restrict__ panel,
                                                     double* __restrict__ cb, const double* __restrict__ D) {
  extern __shared__ double sm[];
  const int s = nodes[blockIdx.y];
  const int64_t f = S.front[s], np = S.ncol[s];
  const int64_t kend = imin(k1, np);
  if (k0 >= kend) return;
  const int64_t cs = imin(c0, np), ce = wide ? f : imin(c1, np);
  if (cs >= ce) return;
  int64_t ti, tj;
  if (tri) {
    const int64_t t = blockIdx.x;
    ti = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
    while (ti * (ti + 1) / 2 > t) --ti;
    tj = t - ti * (ti + 1) / 2;
  } else {
    ti = blockIdx.x / ntj;
    tj = blockIdx.x % ntj;
  }
  const int64_t i0 = cs + ti * kT128, j0 = cs + tj * kT128;
  if (i0 >= f || j0 >= ce || i0 + kT128 - 1 < j0) return;
  double* L = panel + S.panel_off[s];
  dmma_tile128<2>(L, f, L, f, D + S.col0[s], k0, kend, i0, j0, f, ce, L, f, 0, sm, cb + S.cb_off[s], f - np, np,
                  first != 0);
}

// ---------------------------------------------------------------------------
// host drivers
// ---------------------------------------------------------------------------
static int build_plan(riga_symbolic* sym) {
  const SymbolicHost& h = sym->h;
  sym->plan.assign(h.nlevels, LevelPlan());
  sym->ea_items_host.clear();
  std::vector<int32_t> large;
  static const int bounds[] = {32, 64, 96, 128, kSmallFront};
  for (int64_t l = 0; l < h.nlevels; ++l) {
    LevelPlan& P = sym->plan[l];
    P.begin = h.level_ptr[l];
    int64_t end = h.level_ptr[l + 1];
    P.nsmall = h.level_nsmall[l];
    P.nlarge = end - P.begin - P.nsmall;
    int64_t i = P.begin;
    for (int b : bounds) {
      int64_t j = i;
      while (j < P.begin + P.nsmall && h.front[h.level_nodes[j]] <= b) ++j;
      if (j > i) {
        P.cls_begin.push_back(i);
        P.cls_f.push_back(b);
      }
      i = j;
    }
    P.cls_begin.push_back(P.begin + P.nsmall);
    for (int64_t q = P.begin; q < end; ++q) {
      int32_t s = h.level_nodes[q];
      P.max_f = std::max<int64_t>(P.max_f, h.front[s]);
      P.max_np = std::max<int64_t>(P.max_np, h.ncol[s]);
      if (q >= P.begin + P.nsmall) {
        P.max_np_large = std::max<int64_t>(P.max_np_large, h.ncol[s]);
        P.max_f_large = std::max<int64_t>(P.max_f_large, h.front[s]);
        P.max_nu_large = std::max<int64_t>(P.max_nu_large, h.front[s] - h.ncol[s]);
        large.push_back(s);
      }
    }
    // extend-add rounds into the large parents of this level
    int64_t maxch = 0;
    for (int64_t q = P.begin + P.nsmall; q < end; ++q) {
      int32_t s = h.level_nodes[q];
      maxch = std::max<int64_t>(maxch, h.child_ptr[s + 1] - h.child_ptr[s]);
    }
    for (int64_t r = 0; r < maxch; ++r) {
      P.ea_round_begin.push_back((int64_t)sym->ea_items_host.size());
      int64_t mx = 0;
      for (int64_t q = P.begin + P.nsmall; q < end; ++q) {
        int32_t s = h.level_nodes[q];
        if (h.child_ptr[s] + r < h.child_ptr[s + 1]) {
          int32_t c = h.child_list[h.child_ptr[s] + r];
          sym->ea_items_host.push_back(c);
          mx = std::max<int64_t>(mx, h.front[c] - h.ncol[c]);
        }
      }
      P.ea_round_maxnu.push_back(mx);
    }
    P.ea_round_begin.push_back((int64_t)sym->ea_items_host.size());
  }
  sym->n_large = (int64_t)large.size();
  sym->large_host = large;
  return RIGA_OK;
}

template <typename T>
static int up(DevBuf<T>& d, const std::vector<T>& v, cudaStream_t s) {
  return d.upload(v.data(), v.size(), s);
}

// ---- scatter map of the original entries, built on the device -----------------------------------------
// (what symbolic.cpp 5d builds on the host for a host-only analysis: for every supernode the lower-triangle
// entries of its pivot columns as (CSR slot, position in the panel), columns in elimination order, a column's
// entries in CSR order.)  One warp per elimination column: count, exclusive scan, fill.
__global__ void k_asm_count(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colidx,
                            const int32_t* __restrict__ order, const int32_t* __restrict__ io,
                            int64_t* __restrict__ cnt) {
  const int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  const int64_t o = order[j];
  int c = 0;
  for (int64_t q = rowptr[o] + lane; q < rowptr[o + 1]; q += 32) c += io[colidx[q]] >= j;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
  if (lane == 0) cnt[j] = c;
}

__global__ void k_asm_fill(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colidx,
                           const int32_t* __restrict__ order, const int32_t* __restrict__ io,
                           const int32_t* __restrict__ sn_of, const int64_t* __restrict__ col0,
                           const int64_t* __restrict__ ncol, const int64_t* __restrict__ front,
                           const int64_t* __restrict__ rows_off, const int32_t* __restrict__ rows,
                           const int64_t* __restrict__ colptr, int32_t* __restrict__ slot,
                           int32_t* __restrict__ local, int* __restrict__ bad) {
  const int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  const int64_t o = order[j];
  const int s = sn_of[j];
  const int64_t c0 = col0[s], np = ncol[s], f = front[s];
  const int32_t* upd = rows + rows_off[s] + np;  // the front's update rows, ascending
  const int64_t nu = f - np;
  int64_t w = colptr[j];
  for (int64_t q0 = rowptr[o]; q0 < rowptr[o + 1]; q0 += 32) {
    const int64_t q = q0 + lane;
    int64_t i = -1;
    if (q < rowptr[o + 1]) i = io[colidx[q]];
    const bool take = i >= j;
    const unsigned m = __ballot_sync(0xffffffffu, take);
    if (take) {
      int64_t r;
      if (i < c0 + np) {
        r = i - c0;
      } else {
        int64_t a = 0, b = nu;  // lower bound of i in upd
        while (a < b) {
          const int64_t h = (a + b) >> 1;
          if (upd[h] < i) a = h + 1;
          else b = h;
        }
        if (a >= nu || upd[a] != i) *bad = 1;
        r = np + a;
      }
      const int64_t e = w + __popc(m & ((1u << lane) - 1));
      slot[e] = (int32_t)q;
      local[e] = (int32_t)((j - c0) * f + r);
    }
    w += __popc(m);
  }
}

__global__ void k_asm_ptr(int64_t ns, int64_t n, const int64_t* __restrict__ col0, const int64_t* __restrict__ colptr,
                          int64_t* __restrict__ asm_ptr) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s < ns) asm_ptr[s] = colptr[col0[s]];
  if (s == ns) asm_ptr[ns] = colptr[n];
}

// needs d_order, d_col0, d_ncol, d_front, d_rows_off, d_rows on the device
static int build_asm_map_device(riga_symbolic* sym) {
  cudaStream_t st = sym->ctx->stream;
  SymbolicHost& h = sym->h;
  const int64_t n = h.n, ns = h.nsuper;
  RIGA_CHECK_ARG(sym->sys && sym->sys->n == n, "device scatter map needs the device pattern");
  std::vector<int32_t> sn_of(n);
  for (int64_t s = 0; s < ns; ++s)
    for (int64_t j = h.col0[s]; j < h.col0[s] + h.ncol[s]; ++j) sn_of[j] = (int32_t)s;
  DevBuf<int32_t> d_sn, d_io;
  DevBuf<int64_t> colptr;
  DevBuf<int> bad;
  RIGA_TRY(up(d_sn, sn_of, st));
  RIGA_TRY(up(d_io, h.iorder, st));
  RIGA_TRY(colptr.alloc(n + 1, st));
  RIGA_TRY(bad.alloc(1, st));
  RIGA_CUDA(cudaMemsetAsync(colptr.p, 0, sizeof(int64_t), st));
  RIGA_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
  const unsigned gw = (unsigned)((n * 32 + 255) / 256);
  k_asm_count<<<gw, 256, 0, st>>>(n, sym->sys->rowptr.p, sym->sys->colidx.p, sym->d_order.p, d_io.p, colptr.p + 1);
  RIGA_TRY(inclusive_scan_i64(st, colptr.p + 1, n));
  int64_t total = 0;
  RIGA_CUDA(cudaMemcpyAsync(&total, colptr.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  RIGA_CUDA(stream_sync(st));
  RIGA_CHECK_ARG(total > 0 && total < (int64_t)1 << 31, "scatter map size out of range");
  RIGA_TRY(sym->d_asm_ptr.alloc(ns + 1, st));
  RIGA_TRY(sym->d_asm_slot.alloc(total, st));
  RIGA_TRY(sym->d_asm_local.alloc(total, st));
  k_asm_fill<<<gw, 256, 0, st>>>(n, sym->sys->rowptr.p, sym->sys->colidx.p, sym->d_order.p, d_io.p, d_sn.p,
                                sym->d_col0.p, sym->d_ncol.p, sym->d_front.p, sym->d_rows_off.p, sym->d_rows.p,
                                colptr.p, sym->d_asm_slot.p, sym->d_asm_local.p, bad.p);
  k_asm_ptr<<<(unsigned)((ns + 1 + 255) / 256), 256, 0, st>>>(ns, n, sym->d_col0.p, colptr.p, sym->d_asm_ptr.p);
  RIGA_CUDA(cudaGetLastError());
  int hb = 0;
  RIGA_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  RIGA_CUDA(stream_sync(st));
  if (hb) {
    set_error("symbolic analysis: original entry outside its front");
    return RIGA_BAD_ARG;
  }
  h.nnz_lower = total;
  return RIGA_OK;
}

static int upload_symbolic(riga_symbolic* sym) {
  cudaStream_t s = sym->ctx->stream;
  SymbolicHost& h = sym->h;
  RIGA_TRY(up(sym->d_col0, h.col0, s));
  RIGA_TRY(up(sym->d_ncol, h.ncol, s));
  RIGA_TRY(up(sym->d_front, h.front, s));
  RIGA_TRY(up(sym->d_rows_off, h.rows_off, s));
  RIGA_TRY(up(sym->d_panel_off, h.panel_off, s));
  RIGA_TRY(up(sym->d_cb_off, h.cb_off, s));
  RIGA_TRY(up(sym->d_upd_off, h.upd_off, s));
  RIGA_TRY(up(sym->d_child_ptr, h.child_ptr, s));
  RIGA_TRY(up(sym->d_sparent, h.sparent, s));
  RIGA_TRY(up(sym->d_rows, h.rows, s));
  RIGA_TRY(up(sym->d_relpos, h.relpos, s));
  RIGA_TRY(up(sym->d_child_list, h.child_list, s));
  RIGA_TRY(up(sym->d_level_nodes, h.level_nodes, s));
  std::vector<int32_t> ord32(h.order.begin(), h.order.end());
  RIGA_TRY(up(sym->d_order, ord32, s));
  if (h.asm_ptr.empty()) {  // device analysis: the scatter map is built here
    RIGA_TRY(build_asm_map_device(sym));
  } else {
    RIGA_TRY(up(sym->d_asm_ptr, h.asm_ptr, s));
    std::vector<int32_t> slot32(h.asm_slot.begin(), h.asm_slot.end());
    RIGA_TRY(up(sym->d_asm_slot, slot32, s));
    RIGA_TRY(up(sym->d_asm_local, h.asm_local, s));
  }
  RIGA_TRY(up(sym->d_ea_items, sym->ea_items_host, s));
  RIGA_TRY(up(sym->d_large_nodes, sym->large_host, s));
  RIGA_TRY(upload_solve_plan(sym, s));
  RIGA_CUDA(stream_sync(s));
  sym->on_device = true;
  return RIGA_OK;
}

static int g_lookahead = 1;  // RIGA_FACTOR_LOOKAHEAD=0: everything on the factor stream
static int64_t g_nb2 = 512;  // outer block of the trailing updates (multiple of 128; RIGA_FACTOR_NB2)

static int set_smem_attrs() {
  static bool done = false;
  if (done) return RIGA_OK;
  {
    const char* e = getenv("RIGA_FACTOR_NB2");
    if (e && atoll(e) >= 128) g_nb2 = atoll(e) / 128 * 128;
    const char* la = getenv("RIGA_FACTOR_LOOKAHEAD");
    if (la && *la) g_lookahead = atoi(la);
  }
  RIGA_CUDA(cudaFuncSetAttribute(k_trsm128, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTrsmSmem));
  RIGA_CUDA(cudaFuncSetAttribute(k_trail128, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kT128Smem));
  RIGA_CUDA(cudaFuncSetAttribute(k_diag128, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDiag128Smem));
  int dev = 0, maxsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa;
  RIGA_CUDA(cudaFuncGetAttributes(&fa, k_small_front));
  RIGA_CUDA(cudaFuncSetAttribute(k_small_front, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 maxsm - (int)fa.sharedSizeBytes));
  done = true;
  return RIGA_OK;
}

// Side streams and events of a context (created on first use): aux[0] runs the
// panel chain of the large fronts one outer block ahead of the trailing
// updates (high priority), aux[1] builds the solve-side companions (G blocks)
// of the lower levels while the upper levels are still being factored.
static int ctx_aux(riga_ctx* ctx) {
  if (ctx->aux[0]) return RIGA_OK;
  int lo = 0, hi = 0;
  RIGA_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  RIGA_CUDA(cudaStreamCreateWithPriority(&ctx->aux[0], cudaStreamNonBlocking, hi));
  RIGA_CUDA(cudaStreamCreateWithPriority(&ctx->aux[1], cudaStreamNonBlocking, lo));
  for (auto& e : ctx->aux_ev) RIGA_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return RIGA_OK;
}


static int numeric(riga_factor* F, cudaStream_t st, const double* Kv, const double* Mv,
                   double sigma, double rel) {
  riga_symbolic* sym = F->sym;
  const SymbolicHost& h = sym->h;
  SymDev S = sym->dev();
  RIGA_TRY(set_smem_attrs());
  ProfScope prof(kProfFactor, st, (double)h.factor_flops);
  double* scratch = nullptr;
  RIGA_CUDA(cudaMallocAsync(&scratch, 1024 * sizeof(double), st));
  RIGA_CUDA(cudaMemsetAsync(scratch, 0, 1024 * sizeof(double), st));
  int nb = (int)std::min<int64_t>(592, (sym->sys->nnz + 255) / 256);
  k_tol<<<std::max(nb, 1), 256, 0, st>>>(sym->sys->nnz, Kv, Mv, sigma, rel, scratch,
                                          reinterpret_cast<unsigned*>(scratch + 1000), F->tol.p,
                                          F->stat.p, h.n); count_launch();
  RIGA_CUDA(cudaGetLastError());
  double* cbuf = nullptr;
  if (h.cb_total) RIGA_CUDA(cudaMallocAsync(&cbuf, h.cb_total * sizeof(double), st));
  if (h.panel_large) RIGA_CUDA(cudaMemsetAsync(F->panel.p, 0, h.panel_large * 8, st));
  if (sym->n_large) {
    k_asm_large<<<(unsigned)sym->n_large, 256, 0, st>>>(S, sym->d_large_nodes.p, Kv, Mv, sigma,
                                                        F->panel.p); count_launch();
    RIGA_CUDA(cudaGetLastError());
  }
  // does any level have more than one outer block?  then the panel chain runs ahead on aux[0]
  bool ahead = false;
  for (int64_t l = 0; l < h.nlevels; ++l) ahead = ahead || (sym->plan[l].nlarge && sym->plan[l].max_np_large > g_nb2);
  // with the per-kernel timing scopes on, everything stays on one stream so a scope times its kernel alone
  ahead = ahead && g_lookahead && !prof_on();
  riga_ctx* ctx = F->ctx;
  if (ahead) RIGA_TRY(ctx_aux(ctx));
  // G blocks of the small supernodes: on the low-priority side stream as soon as their last level is
  // factored, beside the upper levels (whose panel chains leave SMs idle); joined at the end
  // (forked no earlier than six levels from the top: lower down every SM is busy with frontal updates and
  // the G kernels would only take time from them -- measured: forked at level 9 of 19 they doubled level 10)
  const int64_t g_last = small_g_top_level(sym);
  const int64_t g_top = g_last < 0 ? -1 : std::max<int64_t>(g_last, h.nlevels - 6);
  const SolvePlanHost& SP = sym->sp;
  if (g_top >= 0 && !F->gsmall.p) RIGA_TRY(F->gsmall.alloc(SP.g_total, st));
  bool g_forked = false;
  // RIGA_FACTOR_TRACE=1: per-level device time (events on the factor stream), printed after the factorization
  static const bool trace = getenv("RIGA_FACTOR_TRACE") != nullptr;
  std::vector<cudaEvent_t> tev;
  auto mark = [&]() {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    tev.push_back(e);
  };
  mark();
  cudaStream_t sp = ahead ? ctx->aux[0] : st;
  cudaEvent_t evH = ahead ? ctx->aux_ev[0] : nullptr, evP = ahead ? ctx->aux_ev[1] : nullptr;
  for (int64_t l = 0; l < h.nlevels; ++l) {
    const LevelPlan& P = sym->plan[l];
    auto extend_add = [&](int part) -> int {
      for (size_t r = 0; r + 1 < P.ea_round_begin.size(); ++r) {
        int64_t cnt = P.ea_round_begin[r + 1] - P.ea_round_begin[r];
        if (!cnt) continue;
        dim3 g((unsigned)((P.ea_round_maxnu[r] + 31) / 32), (unsigned)cnt,
               (unsigned)((P.ea_round_maxnu[r] + kEaRows - 1) / kEaRows));
        if (g.x == 0) continue;
        k_extend_add<<<g, 256, 0, st>>>(S, sym->d_ea_items.p + P.ea_round_begin[r], part, F->panel.p, cbuf);
        count_launch();
        RIGA_CUDA(cudaGetLastError());
      }
      return RIGA_OK;
    };
    RIGA_TRY(extend_add(0));  // children -> pivot columns of the large fronts
    for (size_t c = 0; c + 1 < P.cls_begin.size(); ++c) {
      int64_t cnt = P.cls_begin[c + 1] - P.cls_begin[c];
      if (!cnt) continue;
      int fm = P.cls_f[c];
      size_t smem = (size_t)fm * (fm | 1) * 8 + 2 * kSfPanel * (size_t)fm * 8;
      // a class whose fronts take an SM's shared memory alone (> 113 KB) runs 16 warps per front instead of 8
      // (cfg3: 17 concurrent factorizations 41.5 -> 35.1 ms; 32 warps: no further gain)
      const unsigned nthr = fm >= 113 ? 512 : 256;
      k_small_front<<<(unsigned)cnt, nthr, smem, st>>>(S, sym->d_level_nodes.p + P.cls_begin[c], Kv,
                                                       Mv, sigma, F->tol.p, F->panel.p, cbuf,
                                                       F->D.p, F->stat.p); count_launch();
      RIGA_CUDA(cudaGetLastError());
    }
    if (P.nlarge) {
    const int32_t* ln = sym->d_level_nodes.p + P.begin + P.nsmall;
    const unsigned nl = (unsigned)P.nlarge;
    // trailing update of pivot columns [k0, k1): narrow = the pivot columns [c0, c1); wide = every
    // column right of c0, update block included (first: the update block is written, not accumulated)
    auto trail = [&](cudaStream_t ts, int64_t k0, int64_t k1, int64_t c0, int64_t c1, bool wide, bool first) -> int {
      // rows [c0', f) with c0' = min(c0, n_p) per front: tile counts bounded over the level's fronts
      const int64_t rows = wide ? std::max(P.max_f_large - c0, P.max_nu_large) : P.max_f_large - c0;
      const int64_t nti = (rows + kT128 - 1) / kT128;
      if (nti <= 0) return RIGA_OK;
      const int64_t ntj = wide ? nti : (std::min(c1, P.max_np_large) - c0 + kT128 - 1) / kT128;
      if (ntj <= 0) return RIGA_OK;
      const int64_t ntiles = wide ? nti * (nti + 1) / 2 : nti * ntj;
      double work = 0.0;  // algorithmic flops: 2 K per updated lower entry, over the level's fronts
      for (int64_t q = P.begin + P.nsmall; q < P.begin + P.nsmall + P.nlarge; ++q) {
          const int64_t sn = h.level_nodes[q], f = h.front[sn], np = h.ncol[sn];
          const int64_t kend = std::min(k1, np), cs = std::min(c0, np), ce = wide ? f : std::min(c1, np);
          if (k0 >= kend || cs >= ce) continue;
        work += 2.0 * (double)(kend - k0) * ((double)(ce - cs) * f - 0.5 * (double)(ce - 1 + cs) * (ce - cs));
      }
      ProfScope prof_t(kProfTrail, ts, work);
      k_trail128<<<dim3((unsigned)ntiles, nl), 256, kT128Smem, ts>>>(S, ln, k0, k1, c0, c1, wide ? 1 : 0, (int)ntj,
                                                                     wide ? 1 : 0, first ? 1 : 0, F->panel.p, cbuf,
                                                                     F->D.p);
      count_launch();
      RIGA_CUDA(cudaGetLastError());
      return RIGA_OK;
    };
    // panel chain of the outer block [kbo, kbo + nb2): per 128 columns the diagonal block, the rows
    // below it, and the block's remaining columns (narrow, K = 128)
    auto panel_block = [&](cudaStream_t ts, int64_t kbo) -> int {
      const int64_t kend = std::min<int64_t>(kbo + g_nb2, P.max_np_large);
      for (int64_t kb = kbo; kb < kend; kb += kDB) {
        k_diag128<<<nl, 256, kDiag128Smem, ts>>>(S, ln, (int)kb, F->tol.p, F->panel.p, F->D.p, F->stat.p);
        const unsigned nti = (unsigned)((P.max_f_large - kb + 32 * kTrsmWarps - 1) / (32 * kTrsmWarps));
        k_trsm128<<<dim3(nti, nl), 32 * kTrsmWarps, kTrsmSmem, ts>>>(S, ln, (int)kb, F->panel.p, F->D.p);
        count_launch(2);
        RIGA_CUDA(cudaGetLastError());
        if (kb + kDB < kend) RIGA_TRY(trail(ts, kb, kb + kDB, kb + kDB, kbo + g_nb2, false, false));
      }
      return RIGA_OK;
    };
    const bool la = ahead && P.max_np_large > g_nb2;
    if (!la) {
      for (int64_t kbo = 0; kbo < P.max_np_large; kbo += g_nb2) {
        RIGA_TRY(panel_block(st, kbo));
        // everything right of the block -- pivot columns and update block -- in one K = nb2 slice
        RIGA_TRY(trail(st, kbo, kbo + g_nb2, kbo + g_nb2, 0, true, kbo == 0));
      }
    } else {
      // look-ahead: the next outer block's pivot columns take the K = nb2 slice first (head), then its
      // panel chain runs on the high-priority side stream while the factor stream updates the rest
      RIGA_CUDA(cudaEventRecord(evH, st));
      RIGA_CUDA(cudaStreamWaitEvent(sp, evH, 0));
      RIGA_TRY(panel_block(sp, 0));
      RIGA_CUDA(cudaEventRecord(evP, sp));
      for (int64_t kbo = 0; kbo < P.max_np_large; kbo += g_nb2) {
        RIGA_CUDA(cudaStreamWaitEvent(st, evP, 0));
        const bool more = kbo + g_nb2 < P.max_np_large;
        if (more) {
          RIGA_TRY(trail(st, kbo, kbo + g_nb2, kbo + g_nb2, kbo + 2 * g_nb2, false, false));
          RIGA_CUDA(cudaEventRecord(evH, st));
          RIGA_CUDA(cudaStreamWaitEvent(sp, evH, 0));
          RIGA_TRY(panel_block(sp, kbo + g_nb2));
          RIGA_CUDA(cudaEventRecord(evP, sp));
        }
        RIGA_TRY(trail(st, kbo, kbo + g_nb2, kbo + (more ? 2 : 1) * g_nb2, 0, true, kbo == 0));
      }
    }
    RIGA_TRY(extend_add(1));  // children -> update blocks, on top of the fronts' own Schur complements
    }
    mark();
    if (ahead && l == g_top && l + 1 < h.nlevels) {
      RIGA_CUDA(cudaEventRecord(ctx->aux_ev[2], st));
      RIGA_CUDA(cudaStreamWaitEvent(ctx->aux[1], ctx->aux_ev[2], 0));
      RIGA_TRY(build_small_g(F, ctx->aux[1]));
      RIGA_CUDA(cudaEventRecord(ctx->aux_ev[3], ctx->aux[1]));
      g_forked = true;
    }
  }
  if (trace) {
    cudaStreamSynchronize(st);
    for (size_t l = 0; l + 1 < tev.size(); ++l) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tev[l], tev[l + 1]);
      const LevelPlan& P = sym->plan[l];
      fprintf(stderr, "[riga] level %2zu: %4lld large fronts, max np %5lld, max f %5lld: %7.3f ms\n", l,
              (long long)P.nlarge, (long long)P.max_np_large, (long long)P.max_f_large, ms);
    }
    for (auto e : tev) cudaEventDestroy(e);
  }
  if (g_forked)
    RIGA_CUDA(cudaStreamWaitEvent(st, ctx->aux_ev[3], 0));
  else if (g_top >= 0)
    RIGA_TRY(build_small_g(F, st));
  if (cbuf) RIGA_CUDA(cudaFreeAsync(cbuf, st));
  RIGA_CUDA(cudaFreeAsync(scratch, st));
  return build_chain_inverse(F, st);
}

// Chain supernodes whose inverse probe (build_chain_inverse) exceeds the
// tolerance get a local refinement step in every solve: per-supernode device
// flags, per-level host flags (levels without one launch nothing extra).
int flag_inverse_refinement(riga_factor* F, cudaStream_t st) {
  riga_symbolic* sym = F->sym;
  const SolvePlanHost& L = sym->sp;
  const SymbolicHost& h = sym->h;
  F->fix_level.assign(h.nlevels, 0);
  F->n_fix = 0;
  if (!L.inv_fix || !L.chain_inv || L.ifwd.empty() || !F->inv_err.p) return RIGA_OK;
  static const double tol = [] {
    const char* e = getenv("RIGA_INV_FIX_TOL");
    return e && *e ? atof(e) : 1e-11;
  }();
  std::vector<unsigned long long> eb(h.nsuper);
  RIGA_CUDA(cudaMemcpyAsync(eb.data(), F->inv_err.p, h.nsuper * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  RIGA_CUDA(stream_sync(st));
  std::vector<int> flag(h.nsuper, 0);
  double emax = 0.0;
  int nchain = 0;
  for (int64_t l = 0; l < h.nlevels; ++l)
    for (int64_t t = L.ifwd_ptr[l]; t < L.ifwd_ptr[l + 1]; ++t) {
      const int sn = L.ifwd[t].x;
      if (L.ifwd[t].y == 0) ++nchain;
      const double e = __longlong_as_double_host((long long)eb[sn]);
      emax = std::max(emax, e);
      if (e > tol || e != e) {
        if (!flag[sn]) ++F->n_fix;
        flag[sn] = 1;
        F->fix_level[l] = 1;
      }
    }
  if (getenv("RIGA_INV_FIX_DEBUG"))
    fprintf(stderr, "[riga] inverse probe: %d of %d chain supernodes above %.1e (max %.3e)\n", F->n_fix, nchain, tol,
            emax);
  RIGA_TRY(F->fix_flag.upload(flag.data(), flag.size(), st));
  return RIGA_OK;
}

}  // namespace riga

using namespace riga;

extern "C" {

static int finish_symbolic(riga_symbolic* sym) {
  RIGA_TRY(build_plan(sym));
  return build_solve_plan(sym);
}

int riga_symbolic_analyze(int64_t n, const int64_t* rowptr, const int32_t* colidx,
                          const int64_t* perm, riga_symbolic** out) {
  RIGA_CHECK_ARG(out && rowptr && colidx && perm && n > 0, "null arg");
  auto sym = std::make_unique<riga_symbolic>();
  std::string err;
  if (analyze(n, rowptr, colidx, perm, sym->h, err)) {
    set_error("symbolic analysis: " + err);
    return RIGA_BAD_ARG;
  }
  RIGA_TRY(finish_symbolic(sym.get()));
  *out = sym.release();
  return RIGA_OK;
}

int riga_symbolic_create(riga_system* sys, const int64_t* perm, riga_symbolic** out) {
  RIGA_CHECK_ARG(sys && perm && out, "null arg");
  DeviceGuard g(sys->ctx->device);
  std::vector<int64_t> rp(sys->n + 1);
  std::vector<int32_t> ci(sys->nnz);
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  RIGA_TRY(riga_system_download(sys, rp.data(), ci.data(), nullptr, nullptr));
  auto sym = std::make_unique<riga_symbolic>();
  sym->ctx = sys->ctx;
  sym->ctxref.set(sys->ctx);
  sym->sys = sys;
  std::string err;
  const auto t1 = clk::now();
  if (analyze(sys->n, rp.data(), ci.data(), perm, sym->h, err, /*with_asm_map=*/false)) {
    set_error("symbolic analysis: " + err);
    return RIGA_BAD_ARG;
  }
  const auto t2 = clk::now();
  RIGA_TRY(finish_symbolic(sym.get()));
  const auto t3 = clk::now();
  RIGA_TRY(upload_symbolic(sym.get()));
  if (std::getenv("RIGA_SYM_TIME")) {
    auto ms = [](clk::time_point a, clk::time_point b) {
      return std::chrono::duration<double, std::milli>(b - a).count();
    };
    std::fprintf(stderr, "symbolic_create: download %.1f analyze %.1f plans %.1f upload %.1f ms\n", ms(t0, t1),
                 ms(t1, t2), ms(t2, t3), ms(t3, clk::now()));
  }
  *out = sym.release();
  return RIGA_OK;
}

int riga_symbolic_stats(riga_symbolic* sym, int64_t* st) {
  RIGA_CHECK_ARG(sym && st, "null arg");
  const SymbolicHost& h = sym->h;
  int64_t nsmall = 0;
  for (int64_t s = 0; s < h.nsuper; ++s) nsmall += h.front[s] <= kSmallFront;
  int64_t v[16] = {h.fill_nnz,    h.factor_flops, h.nsuper,         h.max_front,
                   h.nlevels,     h.panel_total,  h.cb_total,       h.max_ncol,
                   h.fundamental, h.stored_L,     nsmall,           h.nsuper - nsmall,
                   h.nnz_lower,   h.tree_height,  h.relaxed_flops,  0};
  std::memcpy(st, v, sizeof(v));
  return RIGA_OK;
}

int riga_symbolic_order(riga_symbolic* sym, int64_t* order) {
  RIGA_CHECK_ARG(sym && order, "null arg");
  std::memcpy(order, sym->h.order.data(), sym->h.n * sizeof(int64_t));
  return RIGA_OK;
}

int riga_symbolic_asm_map(riga_symbolic* sym, int64_t* count, int64_t* asm_ptr, int32_t* slot, int32_t* local) {
  RIGA_CHECK_ARG(sym && count, "null arg");
  const SymbolicHost& h = sym->h;
  *count = h.nnz_lower;
  if (!asm_ptr && !slot && !local) return RIGA_OK;
  RIGA_CHECK_ARG(asm_ptr && slot && local, "null arg");
  if (!h.asm_ptr.empty()) {  // host analysis
    std::copy(h.asm_ptr.begin(), h.asm_ptr.end(), asm_ptr);
    for (size_t e = 0; e < h.asm_slot.size(); ++e) slot[e] = (int32_t)h.asm_slot[e];
    std::copy(h.asm_local.begin(), h.asm_local.end(), local);
    return RIGA_OK;
  }
  RIGA_CHECK_ARG(sym->on_device, "no scatter map");
  DeviceGuard g(sym->ctx->device);
  cudaStream_t st = sym->ctx->stream;
  RIGA_CUDA(cudaMemcpyAsync(asm_ptr, sym->d_asm_ptr.p, (h.nsuper + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  RIGA_CUDA(cudaMemcpyAsync(slot, sym->d_asm_slot.p, h.nnz_lower * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  RIGA_CUDA(cudaMemcpyAsync(local, sym->d_asm_local.p, h.nnz_lower * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  RIGA_CUDA(stream_sync(st));
  return RIGA_OK;
}

int riga_symbolic_colcounts(riga_symbolic* sym, int64_t* counts) {
  RIGA_CHECK_ARG(sym && counts, "null arg");
  const SymbolicHost& h = sym->h;
  for (int64_t k = 0; k < h.n; ++k) counts[h.post[k]] = h.colcount[k];
  return RIGA_OK;
}

int riga_symbolic_supernodes(riga_symbolic* sym, int64_t* col0, int64_t* ncol, int64_t* front,
                             int64_t* parent, int64_t* level) {
  RIGA_CHECK_ARG(sym, "null arg");
  const SymbolicHost& h = sym->h;
  for (int64_t s = 0; s < h.nsuper; ++s) {
    if (col0) col0[s] = h.col0[s];
    if (ncol) ncol[s] = h.ncol[s];
    if (front) front[s] = h.front[s];
    if (parent) parent[s] = h.sparent[s];
    if (level) level[s] = h.level[s];
  }
  return RIGA_OK;
}

int riga_symbolic_destroy(riga_symbolic* sym) {
  if (!sym) return RIGA_OK;
  if (sym->ctx) {
    DeviceGuard g(sym->ctx->device);
    stream_sync(sym->ctx->stream);
    delete sym;
  } else {
    delete sym;
  }
  return RIGA_OK;
}

int riga_factor_create(riga_ctx* ctx, riga_symbolic* sym, double sigma, double rel_zero_tol,
                riga_factor** out, int64_t* n_negative, int64_t* bad_pivot) {
  RIGA_CHECK_ARG(sym && out, "null arg");
  RIGA_CHECK_ARG(sym->on_device && sym->sys, "symbolic handle has no device system");
  if (!ctx) ctx = sym->ctx;
  DeviceGuard g(ctx->device);
  cudaStream_t st = ctx->stream;
  const SymbolicHost& h = sym->h;
  auto F = std::make_unique<riga_factor>();
  F->ctx = ctx;
  F->ctxref.set(ctx);
  F->sym = sym;
  F->sigma = sigma;
  RIGA_TRY(F->panel.alloc(std::max<int64_t>(h.panel_total, 1), st));
  RIGA_TRY(F->D.alloc(h.n, st));
  RIGA_TRY(F->xperm.alloc(h.n, st));
  RIGA_TRY(F->upd.alloc(std::max<int64_t>(sym->sp.upd_doubles, 1), st));
  RIGA_TRY(F->stat.alloc(2, st));
  RIGA_TRY(F->tol.alloc(2, st));
  RIGA_TRY(F->cvec.alloc(h.n, st));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  int rc = numeric(F.get(), st, sym->sys->K.p, sym->sys->M.p, sigma, rel_zero_tol);
  cudaEventRecord(e1, st);
  if (rc) {
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return rc;
  }
  int64_t stat[2];
  double tol[2];
  RIGA_CUDA(cudaMemcpyAsync(stat, F->stat.p, sizeof(stat), cudaMemcpyDeviceToHost, st));
  RIGA_CUDA(cudaMemcpyAsync(tol, F->tol.p, sizeof(tol), cudaMemcpyDeviceToHost, st));
  RIGA_CUDA(stream_sync(st));
  cudaEventElapsedTime(&F->factor_ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  RIGA_TRY(flag_inverse_refinement(F.get(), st));
  if (n_negative) *n_negative = stat[0];
  if (bad_pivot) *bad_pivot = stat[1] < h.n ? stat[1] : -1;
  if (tol[0] == 0.0) {
    set_error("matrix is identically zero");
    if (bad_pivot) *bad_pivot = -1;
    return RIGA_ZERO_PIVOT;
  }
  if (stat[1] < h.n) {
    char buf[160];
    snprintf(buf, sizeof(buf), "pivot %lld below %.3e (shift at an eigenvalue?)",
             (long long)stat[1], tol[1]);
    set_error(buf);
    *out = F.release();
    return RIGA_ZERO_PIVOT;
  }
  *out = F.release();
  return RIGA_OK;
}

int riga_factor_solve(riga_factor* f, const double* b, double* x) {
  RIGA_CHECK_ARG(f && b && x, "null arg");
  DeviceGuard g(f->ctx->device);
  return factor_solve(f, f->ctx->stream, b, x, false, true);
}

int riga_factor_time_ms(riga_factor* f, float* ms) {
  RIGA_CHECK_ARG(f && ms, "null arg");
  *ms = f->factor_ms;
  return RIGA_OK;
}

int riga_factor_D(riga_factor* f, double* D) {
  RIGA_CHECK_ARG(f && D, "null arg");
  DeviceGuard g(f->ctx->device);
  RIGA_CUDA(cudaMemcpyAsync(D, f->D.p, f->sym->h.n * 8, cudaMemcpyDeviceToHost, f->ctx->stream));
  RIGA_CUDA(stream_sync(f->ctx->stream));
  return RIGA_OK;
}

int riga_factor_export(riga_factor* f, int64_t* Lp, int32_t* Li, double* Lx) {
  RIGA_CHECK_ARG(f && Lp && Li && Lx, "null arg");
  DeviceGuard g(f->ctx->device);
  const SymbolicHost& h = f->sym->h;
  std::vector<double> panel(h.panel_total);
  RIGA_CUDA(cudaMemcpyAsync(panel.data(), f->panel.p, h.panel_total * 8, cudaMemcpyDeviceToHost,
                            f->ctx->stream));
  RIGA_CUDA(stream_sync(f->ctx->stream));
  int64_t q = 0;
  Lp[0] = 0;
  for (int64_t s = 0; s < h.nsuper; ++s) {
    int64_t fr = h.front[s], np = h.ncol[s];
    const int32_t* rows = &h.rows[h.rows_off[s]];
    const double* P = &panel[h.panel_off[s]];
    for (int64_t c = 0; c < np; ++c) {
      for (int64_t r = c + 1; r < fr; ++r) {
        Li[q] = rows[r];
        Lx[q] = P[c * fr + r];
        ++q;
      }
      Lp[h.col0[s] + c + 1] = q;
    }
  }
  return RIGA_OK;
}

int riga_factor_destroy(riga_factor* f) {
  if (!f) return RIGA_OK;
  DeviceGuard g(f->ctx->device);
  stream_sync(f->ctx->stream);
  delete f;
  return RIGA_OK;
}

}  // extern "C"
