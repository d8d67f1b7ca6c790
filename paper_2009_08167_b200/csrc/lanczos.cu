// Device Lanczos state: shift-invert steps, CGS2 full reorthogonalisation,
// lift / thick-restart skinny GEMMs, locking.
//
//  riga_lanczos_extend  <- LanczosState.step / lanczos_extend  ref eigensolver.py:235-295
//  CGS2 (k_gemv_t + k_gemv_n, two passes) <- _orthogonalize   ref eigensolver.py:204-212
//  riga_lanczos_lift    <- LanczosState.lift                   ref eigensolver.py:270-274
//  riga_lanczos_restart <- thick_restart                       ref eigensolver.py:326-357
//
// Layout: V and MV are (max_dim+1) rows of ld >= n doubles (row-major, each
// basis vector contiguous); the pending normalised direction r (and M r)
// always sits in row k.  Locked vectors L, LM: rows of ld doubles.
//
// The recurrence state (k, coupling window, locked count, stop flag) lives
// in device memory (LzDev), so one Lanczos step -- permuted gather, the
// supernodal solve, alpha/|w| dots, residual, CGS2 against basis + locked
// set, M-SpMV, beta, normalisation -- is a fixed kernel sequence that is
// captured once as a CUDA graph and replayed; the host syncs once per
// extend.  A breakdown sets the stop flag and the remaining replays are
// no-ops.  Reductions are two-phase with a fixed order (bitwise
// reproducible).
#include <algorithm>
#include <cmath>
#include <cstring>

#include "dmma.cuh"
#include "internal.h"
#include "kernels.cuh"
#include "prof.h"

namespace riga {

constexpr int kChunk = 512;  // columns per CTA in the tall-skinny GEMV

// LzDev (device recurrence state): internal.h

// rows used by a CGS pass: basis rows [0, k + add) and/or the locked set
struct RowSel {
  const double* V;
  const double* L;
  int64_t ld;
  int add;        // basis rows = k + add (k from the device state)
  int use_basis;  // 0: locked set only
};

__device__ __forceinline__ void rows_of(const RowSel& A, const LzDev* st, int64_t& na, int64_t& nb) {
  na = A.use_basis ? (int64_t)st->k + A.add : 0;
  nb = st->nlocked;
}

// ---- tall-skinny GEMVs of the Gram-Schmidt passes --------------------------
// dots:   partial[chunk * Rmax + i] = sum_{c in chunk} row_i[c] x[c], then
//         coef[i] = sum_chunk partial (fixed order, by the CTA finishing the
//         row group's last chunk)
// update: upart[g][c] = sum_{i in group g} row_i[c] coef[i]  (grid columns x
//         kUpdGroups), then y[c] -= sum_g upart[g][c]  (fixed order, by the
//         last group of the column strip)
constexpr int kDotCols = 1024;
#ifndef RIGA_DOT_COLS
#define RIGA_DOT_COLS 2048  // columns of a delayed-CGS2 dots tile (>= kDotCols: partial buffers; 2048 > 1024 by 6 %)
#endif
constexpr int kDotColsD = RIGA_DOT_COLS;
constexpr int kUpdGroups = 8;
constexpr int kUpdCols = 512;   // columns per update CTA (2 per thread)
#ifndef RIGA_UPD_UNROLL
#define RIGA_UPD_UNROLL 8
#endif
constexpr int kUpdUnroll = RIGA_UPD_UNROLL;  // row loads in flight per thread

__device__ __forceinline__ const double* sel_row(const RowSel& A, int64_t na, int64_t i) {
  return i < na ? A.V + i * A.ld : A.L + (i - na) * A.ld;
}

// dots: warp tiles (row i, column chunk of kDotCols) handed out over a
// fixed persistent grid (the step graph is captured once; R is read from the
// device state), chunk-major so the warps of a CTA share their x chunk in
// L1.  A lane issues its 16 double2 row loads and 16 x loads at once.  The
// warp finishing the last chunk of a row (per-row ticket) reduces that row's
// partials in fixed order into coef: no block barriers, no reduce launch.
constexpr int kDotGrid = 2 * 148;
// CTAs of the delayed-CGS2 dots sweep (grid-stride over the row tiles):
// RIGA_DOT_CTAS overrides 2 x 148 (two 125-register CTAs fill an SM's registers)
static int dcgs_dot_grid() {
  static const int g = [] {
    const char* e = getenv("RIGA_DOT_CTAS");
    const int v = e ? atoi(e) : 0;
    return v > 0 ? v : kDotGrid;
  }();
  return g;
}
__global__ void __launch_bounds__(256, 2) k_cgs_dots(RowSel A, const LzDev* st, int64_t n, int64_t Rmax,
                                                     const double* __restrict__ x, double* __restrict__ partial,
                                                     double* __restrict__ coef, unsigned* __restrict__ tickets) {
  pdl_start();
  if (st->stop) return;
  int64_t na, nb;
  rows_of(A, st, na, nb);
  const int64_t R = na + nb;
  const int lane = threadIdx.x & 31;
  const int nchunk = (int)((n + kDotCols - 1) / kDotCols);
  const int64_t ntiles = (int64_t)nchunk * R;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < ntiles; t += nwarps) {
    const int chunk = (int)(t / R);
    const int64_t i = t - (int64_t)chunk * R;
    const int64_t c0 = (int64_t)chunk * kDotCols;
    const double* row = sel_row(A, na, i) + c0;
    double acc = 0.0;
    if (c0 + kDotCols <= n) {
      double2 v[16], xv[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        v[u] = __ldcs(reinterpret_cast<const double2*>(row) + 32 * u + lane);
        xv[u] = __ldg(reinterpret_cast<const double2*>(x + c0) + 32 * u + lane);
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        acc = fma(v[u].x, xv[u].x, acc);
        acc = fma(v[u].y, xv[u].y, acc);
      }
    } else {
      for (int64_t c = 2 * lane; c0 + c < n; c += 64) {
        acc = fma(row[c], x[c0 + c], acc);
        if (c0 + c + 1 < n) acc = fma(row[c + 1], x[c0 + c + 1], acc);
      }
    }
    acc = warp_sum(acc);
    unsigned done = 0;
    if (lane == 0) {
      partial[(int64_t)chunk * Rmax + i] = acc;
      __threadfence();
      done = atomicAdd(&tickets[i], 1u);
    }
    done = __shfl_sync(0xffffffffu, done, 0);
    if (done == (unsigned)nchunk - 1) {
      __threadfence();
      double v = 0.0;
      for (int b = lane; b < nchunk; b += 32) v += __ldcg(partial + (int64_t)b * Rmax + i);
      v = warp_sum(v);
      if (lane == 0) {
        coef[i] = v;
        tickets[i] = 0;
      }
    }
  }
}

// y[c] -= sum_i row_i[c] coef[i]: CTA (column strip, row group g) writes
// upart[g]; the last group of a strip to finish sums the kUpdGroups parts
// in order and updates y (no separate final launch)
__global__ void __launch_bounds__(256) k_cgs_upd(RowSel A, const LzDev* st, int64_t n, int64_t ldu,
                                                 const double* __restrict__ coef, double* __restrict__ upart,
                                                 double* __restrict__ y, unsigned* __restrict__ tickets) {
  pdl_start();
  if (st->stop) return;
  __shared__ double cs[1024];
  __shared__ bool last;
  int64_t na, nb;
  rows_of(A, st, na, nb);
  const int64_t R = na + nb;
  const int64_t per = (R + kUpdGroups - 1) / kUpdGroups;
  const int64_t i0 = (int64_t)blockIdx.y * per, i1 = imin(R, i0 + per);
  const int cnt = (int)(i1 > i0 ? i1 - i0 : 0);
  for (int t = threadIdx.x; t < cnt && t < 1024; t += blockDim.x) cs[t] = coef[i0 + t];
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * kUpdCols + 2 * threadIdx.x;
  const bool valid = c < n;
  const bool pair = c + 1 < n;
  double2 acc = make_double2(0.0, 0.0);
  if (valid) {
    if (pair) {
      // kUpdUnroll rows per round trip, the last round predicated (no serial tail)
      for (int t = 0; t < cnt; t += kUpdUnroll) {
        double2 v[kUpdUnroll];
#pragma unroll
        for (int u = 0; u < kUpdUnroll; ++u)
          v[u] = t + u < cnt ? __ldcs(reinterpret_cast<const double2*>(sel_row(A, na, i0 + t + u) + c))
                             : make_double2(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < kUpdUnroll; ++u) {
          if (t + u < cnt) {
            const double cf = t + u < 1024 ? cs[t + u] : coef[i0 + t + u];
            acc.x = fma(v[u].x, cf, acc.x);
            acc.y = fma(v[u].y, cf, acc.y);
          }
        }
      }
    } else {
      for (int t = 0; t < cnt; ++t) {
        const double cf = t < 1024 ? cs[t] : coef[i0 + t];
        acc.x = fma(sel_row(A, na, i0 + t)[c], cf, acc.x);
      }
    }
    double* dst = upart + (int64_t)blockIdx.y * ldu + c;
    dst[0] = acc.x;
    if (pair) dst[1] = acc.y;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&tickets[blockIdx.x], 1u) == gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (valid) {
    double sx = 0.0, sy = 0.0;
#pragma unroll
    for (int g = 0; g < kUpdGroups; ++g) {
      sx += __ldcg(upart + (int64_t)g * ldu + c);
      if (pair) sy += __ldcg(upart + (int64_t)g * ldu + c + 1);
    }
    y[c] -= sx;
    if (pair) y[c + 1] -= sy;
  }
  if (threadIdx.x == 0) tickets[blockIdx.x] = 0;
}

__device__ __forceinline__ bool broke_down(const LzDev* st, double& beta, double& wn);

// ---- delayed CGS2 (one sweep of dots + one sweep of updates per step) -----
// The step's two Gram-Schmidt passes are the reference's (_orthogonalize,
// eigensolver.py:204-212, two passes against basis + locked), reorganised
// so that the second pass of the new direction r_k runs one step later,
// inside the first pass of the next product w~ = H r~_k (delayed CGS2):
//   dots:   s = U M r~,  z = U M w~       one read of MV/LM rows for both
//   update: r~ -= U^T s, w~ -= U^T z      one read of V/L rows for both
// with U = basis rows [0, k) + locked rows.  The recurrence coefficients
// are corrected for the delay exactly (see k_dcgs_scalars), so the host
// sees the same alpha, beta, |w| as with the undelayed passes up to
// rounding.  Row k (the pending direction) is part of the row sweep with
// a zero coefficient: its dots give r~.M r~ (z side: r~.M w~), and the
// extra tile row R (x2 itself) gives |w~|^2.

// dots of x1 = V[k] (pending row) and x2 against rows [0, k] + locked and,
// as tile row R, x2.x2: coef[i] (x1 side), coef[Rmax + i] (x2 side)
#ifndef RIGA_DOT_W
#define RIGA_DOT_W 8  // double2 row loads per lane per round of the delayed-CGS2 dots
#endif
#ifndef RIGA_DOT_MINB
#define RIGA_DOT_MINB 2
#endif
__device__ __forceinline__ void k_dcgs_dots_body(RowSel A, const LzDev* st, int64_t n, int64_t Rmax,
                                                      const double* __restrict__ Vbase,
                                                      const double* __restrict__ x2, double* __restrict__ partial,
                                                      double* __restrict__ coef, unsigned* __restrict__ tickets) {
  pdl_start();
  if (st->stop) return;
  int64_t na, nb;
  rows_of(A, st, na, nb);
  const int64_t R = na + nb, RT = R + 1;
  const double* x1 = Vbase + (int64_t)st->k * A.ld;
  const int lane = threadIdx.x & 31;
  const int nchunk = (int)((n + kDotColsD - 1) / kDotColsD);
  const int64_t P2 = (int64_t)nchunk * Rmax;
  const int64_t ntiles = (int64_t)nchunk * RT;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < ntiles; t += nwarps) {
    const int chunk = (int)(t / RT);
    const int64_t i = t - (int64_t)chunk * RT;
    const int64_t c0 = (int64_t)chunk * kDotColsD;
    const double* row = (i < R ? sel_row(A, na, i) : x2) + c0;
    double a1 = 0.0, a2 = 0.0;
    if (c0 + kDotColsD <= n) {
#pragma unroll
      for (int h = 0; h < kDotColsD / 64 / RIGA_DOT_W; ++h) {
        double2 v[RIGA_DOT_W], p[RIGA_DOT_W], q[RIGA_DOT_W];
#pragma unroll
        for (int u = 0; u < RIGA_DOT_W; ++u) {
          const int o = 32 * (RIGA_DOT_W * h + u) + lane;
          v[u] = i < R ? __ldcs(reinterpret_cast<const double2*>(row) + o)
                       : __ldg(reinterpret_cast<const double2*>(row) + o);
          p[u] = __ldg(reinterpret_cast<const double2*>(x1 + c0) + o);
          q[u] = __ldg(reinterpret_cast<const double2*>(x2 + c0) + o);
        }
#pragma unroll
        for (int u = 0; u < RIGA_DOT_W; ++u) {
          a1 = fma(v[u].x, p[u].x, a1);
          a1 = fma(v[u].y, p[u].y, a1);
          a2 = fma(v[u].x, q[u].x, a2);
          a2 = fma(v[u].y, q[u].y, a2);
        }
      }
    } else {
      for (int64_t c = 2 * lane; c0 + c < n; c += 64) {
        a1 = fma(row[c], x1[c0 + c], a1);
        a2 = fma(row[c], x2[c0 + c], a2);
        if (c0 + c + 1 < n) {
          a1 = fma(row[c + 1], x1[c0 + c + 1], a1);
          a2 = fma(row[c + 1], x2[c0 + c + 1], a2);
        }
      }
    }
    a1 = warp_sum(a1);
    a2 = warp_sum(a2);
    unsigned done = 0;
    if (lane == 0) {
      partial[(int64_t)chunk * Rmax + i] = a1;
      partial[P2 + (int64_t)chunk * Rmax + i] = a2;
      __threadfence();
      done = atomicAdd(&tickets[i], 1u);
    }
    done = __shfl_sync(0xffffffffu, done, 0);
    if (done == (unsigned)nchunk - 1) {
      __threadfence();
      double s1 = 0.0, s2 = 0.0;
      for (int b = lane; b < nchunk; b += 32) {
        s1 += __ldcg(partial + (int64_t)b * Rmax + i);
        s2 += __ldcg(partial + P2 + (int64_t)b * Rmax + i);
      }
      s1 = warp_sum(s1);
      s2 = warp_sum(s2);
      if (lane == 0) {
        coef[i] = s1;
        coef[Rmax + i] = s2;
        tickets[i] = 0;
      }
    }
  }
}

__global__ void __launch_bounds__(256, RIGA_DOT_MINB) k_dcgs_dots(RowSel A, const LzDev* st, int64_t n, int64_t Rmax,
                                                      const double* __restrict__ Vbase,
                                                      const double* __restrict__ x2, double* __restrict__ partial,
                                                      double* __restrict__ coef, unsigned* __restrict__ tickets) {
  k_dcgs_dots_body(A, st, n, Rmax, Vbase, x2, partial, coef, tickets);
}

// Scalars of the delayed pass (one CTA).  With r~ = eta v + U^T s (v the
// finished direction, U M-orthonormal) and w~ = H r~:
//   eta^2 = r~.M r~ - |s|^2
//   alpha = v.M H v = (r~.M w~ - s.z) / eta^2 - (s.b) / eta,  b = U M H v
// where b is the coupling column (beta_{k-1} e_{k-1} inside a run, the
// arrowhead couplings after a restart, 0 on locked rows); the previous
// step's beta becomes beta~ eta.  The coefficient of v in the first pass of
// w~ / eta is (r~.M w~ - s.z) / eta^2.
// scal: [0] alpha, [1] |w|^2, [5] eta, [6] coefficient of v
__device__ __forceinline__ void k_dcgs_scalars_body(LzDev* st, int64_t Rmax, double* __restrict__ coef,
                                                      double* __restrict__ cpl, double* __restrict__ ob) {
  pdl_start();
  if (st->stop) return;
  __shared__ double red[32];
  const int k = st->k, clo = st->clo;
  const int64_t R = (int64_t)k + 1 + st->nlocked;
  const double vmv = coef[k], a0 = coef[Rmax + k], ww = coef[Rmax + R];
  double ss = 0.0, sz = 0.0;
  for (int64_t i = threadIdx.x; i < R; i += blockDim.x) {
    if (i == k) continue;
    const double s = coef[i];
    ss = fma(s, s, ss);
    sz = fma(s, coef[Rmax + i], sz);
  }
  ss = block_sum(ss, red);
  sz = block_sum(sz, red);
  const double eta = sqrt(fmax(vmv - ss, 1e-300));
  double sb = 0.0;
  for (int i = clo + threadIdx.x; i < k; i += blockDim.x) {
    double b = cpl[i];
    if (i == k - 1 && st->steps > 0) b *= eta;  // previous step's beta, finished now
    sb = fma(coef[i], b, sb);
  }
  sb = block_sum(sb, red);
  if (threadIdx.x == 0) {
    if (st->steps > 0 && k >= 1) {
      cpl[k - 1] *= eta;
      ob[st->steps - 1] *= eta;
    }
    const double e2 = eta * eta;
    st->scal[0] = (a0 - sz) / e2 - sb / eta;
    st->scal[1] = ww / e2;
    st->scal[5] = eta;
    st->scal[6] = (a0 - sz) / e2;
    coef[k] = 0.0;  // row k takes no part in its own update
    coef[Rmax + k] = 0.0;
  }
}

__global__ void __launch_bounds__(256) k_dcgs_scalars(LzDev* st, int64_t Rmax, double* __restrict__ coef,
                                                      double* __restrict__ cpl, double* __restrict__ ob) {
  k_dcgs_scalars_body(st, Rmax, coef, cpl, ob);
}

// r~ -= U^T s, w~ -= U^T z over the rows of A (row k with zero
// coefficients); the last row group of a column strip finishes:
//   vt = (r~ - U^T s) / eta          (the finished direction v_k)
//   r  = (w~ - U^T z) / eta - c_v vt (first pass of the new residual)
__device__ __forceinline__ void k_dcgs_upd_body(RowSel A, const LzDev* st, int64_t n, int64_t ldu,
                                                  int64_t Rmax, const double* __restrict__ coef,
                                                  double* __restrict__ upart, const double* __restrict__ w,
                                                  double* __restrict__ vt, double* __restrict__ r,
                                                  unsigned* __restrict__ tickets, const double* __restrict__ cpl) {
  pdl_start();
  if (st->stop) return;
  __shared__ double cs[2][1024];
  __shared__ double red[32];
  __shared__ bool last;
  int64_t na, nb;
  rows_of(A, st, na, nb);
  const int64_t R = na + nb;
  const int k = st->k;
  // scalars of the delayed pass (see k_dcgs_scalars), computed by every CTA
  // in the same order; CTA (0, 0) publishes alpha, |w|^2, eta, c_v; the
  // previous beta's correction by eta is applied by k_step_finish
  double ss = 0.0, sz = 0.0;
  for (int64_t i = threadIdx.x; i < R; i += blockDim.x) {
    if (i == k) continue;
    const double sv = coef[i];
    ss = fma(sv, sv, ss);
    sz = fma(sv, coef[Rmax + i], sz);
  }
  ss = block_sum(ss, red);
  sz = block_sum(sz, red);
  const double vmv = coef[k], a0 = coef[Rmax + k];
  const double eta = sqrt(fmax(vmv - ss, 1e-300));
  const double cv = (a0 - sz) / (eta * eta);
  if (blockIdx.x == 0 && blockIdx.y == 0) {
    double sb = 0.0;
    for (int i = st->clo + threadIdx.x; i < k; i += blockDim.x) {
      double bb = cpl[i];
      if (i == k - 1 && st->steps > 0) bb *= eta;  // previous step's beta, finished now
      sb = fma(coef[i], bb, sb);
    }
    sb = block_sum(sb, red);
    if (threadIdx.x == 0) {
      LzDev* sw = const_cast<LzDev*>(st);
      sw->scal[0] = cv - sb / eta;
      sw->scal[1] = coef[Rmax + R] / (eta * eta);
      sw->scal[5] = eta;
      sw->scal[6] = cv;
    }
  }
  const int64_t per = (R + kUpdGroups - 1) / kUpdGroups;
  const int64_t i0 = (int64_t)blockIdx.y * per, i1 = imin(R, i0 + per);
  const int cnt = (int)(i1 > i0 ? i1 - i0 : 0);
  for (int t = threadIdx.x; t < cnt && t < 1024; t += blockDim.x) {
    const bool self = i0 + t == k;  // row k takes no part in its own update
    cs[0][t] = self ? 0.0 : coef[i0 + t];
    cs[1][t] = self ? 0.0 : coef[Rmax + i0 + t];
  }
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * kUpdCols + 2 * threadIdx.x;
  const bool valid = c < n;
  const bool pair = c + 1 < n;
  double2 as = make_double2(0.0, 0.0), az = make_double2(0.0, 0.0);
  if (valid) {
    if (pair) {
      for (int t = 0; t < cnt; t += kUpdUnroll) {
        double2 v[kUpdUnroll];
#pragma unroll
        for (int u = 0; u < kUpdUnroll; ++u)
          v[u] = t + u < cnt ? __ldcs(reinterpret_cast<const double2*>(sel_row(A, na, i0 + t + u) + c))
                             : make_double2(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < kUpdUnroll; ++u) {
          if (t + u < cnt) {
            const double f = t + u < 1024 ? cs[0][t + u] : coef[i0 + t + u];
            const double g = t + u < 1024 ? cs[1][t + u] : coef[Rmax + i0 + t + u];
            as.x = fma(v[u].x, f, as.x);
            as.y = fma(v[u].y, f, as.y);
            az.x = fma(v[u].x, g, az.x);
            az.y = fma(v[u].y, g, az.y);
          }
        }
      }
    } else {
      for (int t = 0; t < cnt; ++t) {
        const double x = sel_row(A, na, i0 + t)[c];
        as.x = fma(x, t < 1024 ? cs[0][t] : coef[i0 + t], as.x);
        az.x = fma(x, t < 1024 ? cs[1][t] : coef[Rmax + i0 + t], az.x);
      }
    }
    double* dst = upart + (int64_t)blockIdx.y * ldu + c;
    double* dsz = upart + (int64_t)(kUpdGroups + blockIdx.y) * ldu + c;
    dst[0] = as.x;
    dsz[0] = az.x;
    if (pair) {
      dst[1] = as.y;
      dsz[1] = az.y;
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&tickets[blockIdx.x], 1u) == gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (valid) {
    const double* vk = A.V + (int64_t)k * A.ld;
    for (int e = 0; e < (pair ? 2 : 1); ++e) {
      double ps = 0.0, pz = 0.0;
#pragma unroll
      for (int g = 0; g < kUpdGroups; ++g) {
        ps += __ldcg(upart + (int64_t)g * ldu + c + e);
        pz += __ldcg(upart + (int64_t)(kUpdGroups + g) * ldu + c + e);
      }
      const double v = (vk[c + e] - ps) / eta;
      vt[c + e] = v;
      r[c + e] = (w[c + e] - pz) / eta - cv * v;
    }
  }
  if (threadIdx.x == 0) tickets[blockIdx.x] = 0;
}

__global__ void __launch_bounds__(256) k_dcgs_upd(RowSel A, const LzDev* st, int64_t n, int64_t ldu,
                                                  int64_t Rmax, const double* __restrict__ coef,
                                                  double* __restrict__ upart, const double* __restrict__ w,
                                                  double* __restrict__ vt, double* __restrict__ r,
                                                  unsigned* __restrict__ tickets, const double* __restrict__ cpl) {
  k_dcgs_upd_body(A, st, n, ldu, Rmax, coef, upart, w, vt, r, tickets, cpl);
}

// row k <- (vt, M vt); row k+1 <- (r, M r) / beta~ unless the step broke down
__device__ __forceinline__ void k_dcgs_store_body(const LzDev* st, int64_t n, int64_t ld, const double* __restrict__ vt,
                             const double* __restrict__ mvt, const double* __restrict__ r,
                             const double* __restrict__ Mr, double* __restrict__ V, double* __restrict__ MV) {
  pdl_start();
  if (st->stop) return;
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int64_t o = (int64_t)st->k * ld + c;
  V[o] = vt[c];
  MV[o] = mvt[c];
  double beta, wn;
  if (broke_down(st, beta, wn)) return;
  V[o + ld] = r[c] / beta;
  MV[o + ld] = Mr[c] / beta;
}

__global__ void k_dcgs_store(const LzDev* st, int64_t n, int64_t ld, const double* __restrict__ vt,
                             const double* __restrict__ mvt, const double* __restrict__ r,
                             const double* __restrict__ Mr, double* __restrict__ V, double* __restrict__ MV) {
  k_dcgs_store_body(st, n, ld, vt, mvt, r, Mr, V, MV);
}

// finish of a run: row k /= sqrt(s) (its delayed second pass is done), the
// last beta of the run *= sqrt(s)
__global__ void k_dcgs_finish_row(const LzDev* st, int64_t n, int64_t ld, const double* __restrict__ s,
                                  double* __restrict__ V, double* __restrict__ MV, double* __restrict__ ob,
                                  int last) {
  const double nrm = sqrt(fmax(s[0], 0.0));
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c == 0 && last >= 0) ob[last] *= nrm;
  if (c >= n) return;
  const int64_t o = (int64_t)st->k * ld + c;
  V[o] /= nrm;
  MV[o] /= nrm;
}

// out[0] = <a, b>, out[1] = <c, d>; `a` offset by k rows when koff_a != 0
__device__ __forceinline__ void k_dot2_body(const LzDev* st, int64_t n, int64_t ld, const double* __restrict__ a, int koff_a,
                       const double* __restrict__ b, const double* __restrict__ c,
                       const double* __restrict__ d, double* __restrict__ partial,
                       unsigned* __restrict__ ticket, double* __restrict__ out) {
  pdl_start();
  if (st->stop) return;
  __shared__ double red[32];
  __shared__ bool last;
  const double* aa = a + (koff_a ? (int64_t)st->k * ld : 0);
  double s0 = 0.0, s1 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    s0 = fma(aa[i], b[i], s0);
    s1 = fma(c[i], d[i], s1);
  }
  s0 = block_sum(s0, red);
  s1 = block_sum(s1, red);
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = s0;
    partial[2 * blockIdx.x + 1] = s1;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    double t0 = 0.0, t1 = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
      t0 += ((volatile double*)partial)[2 * i];
      t1 += ((volatile double*)partial)[2 * i + 1];
    }
    t0 = block_sum(t0, red);
    t1 = block_sum(t1, red);
    if (threadIdx.x == 0) {
      out[0] = t0;
      out[1] = t1;
      *ticket = 0u;
    }
  }
}

__global__ void k_dot2(const LzDev* st, int64_t n, int64_t ld, const double* __restrict__ a, int koff_a,
                       const double* __restrict__ b, const double* __restrict__ c,
                       const double* __restrict__ d, double* __restrict__ partial,
                       unsigned* __restrict__ ticket, double* __restrict__ out) {
  k_dot2_body(st, n, ld, a, koff_a, b, c, d, partial, ticket, out);
}

// bp[j] = MV[k][order[j]]: the solve's right-hand side in elimination order
__device__ __forceinline__ void k_perm_row_body(const LzDev* st, int64_t n, int64_t ld, const double* __restrict__ MV,
                           const int32_t* __restrict__ order, double* __restrict__ bp) {
  pdl_start();
  if (st->stop) return;
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < n) bp[j] = MV[(int64_t)st->k * ld + order[j]];
}

__global__ void k_perm_row(const LzDev* st, int64_t n, int64_t ld, const double* __restrict__ MV,
                           const int32_t* __restrict__ order, double* __restrict__ bp) {
  k_perm_row_body(st, n, ld, MV, order, bp);
}

// r = w - alpha V[k] - sum_{i in [clo, k)} cpl[i] V[i]
__global__ void k_residual(const LzDev* st, int64_t n, int64_t ld, const double* __restrict__ w,
                           const double* __restrict__ V, const double* __restrict__ cpl,
                           double* __restrict__ r) {
  pdl_start();
  if (st->stop) return;
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int k = st->k, clo = st->clo;
  const double alpha = st->scal[0];
  double x = w[c] - alpha * V[(int64_t)k * ld + c];
  if (clo < k) {
    double acc = 0.0;
    for (int i = clo; i < k; ++i) acc = fma(V[(int64_t)i * ld + c], cpl[i], acc);
    x -= acc;
  }
  r[c] = x;
}

__device__ __forceinline__ bool broke_down(const LzDev* st, double& beta, double& wn) {
  beta = sqrt(fmax(st->scal[2], 0.0));
  wn = sqrt(fmax(st->scal[1], 0.0));
  return beta <= fmax(st->btol, 1e-13 * wn);
}

// V[k+1] = r / beta, MV[k+1] = Mr / beta (unless the step broke down)
__global__ void k_normalize_next(const LzDev* st, int64_t n, int64_t ld, const double* __restrict__ r,
                                 const double* __restrict__ Mr, double* __restrict__ V,
                                 double* __restrict__ MV) {
  pdl_start();
  if (st->stop) return;
  double beta, wn;
  if (broke_down(st, beta, wn)) return;
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int64_t o = (int64_t)(st->k + 1) * ld + c;
  V[o] = r[c] / beta;
  MV[o] = Mr[c] / beta;
}

// bookkeeping of a finished step (one thread)
__device__ __forceinline__ void k_step_finish_body(LzDev* st, double* __restrict__ cpl, double* __restrict__ oa,
                              double* __restrict__ ob, double* __restrict__ ow, int delayed) {
  pdl_start();
  if (st->stop) return;
  double beta, wn;
  const bool broke = broke_down(st, beta, wn);
  const int k = st->k, i = st->steps;
  if (delayed && i > 0 && k >= 1) {  // the previous step's beta, finished by this step's pass: beta~ eta
    cpl[k - 1] *= st->scal[5];
    ob[i - 1] *= st->scal[5];
  }
  oa[i] = st->scal[0];
  ob[i] = beta;
  ow[i] = wn;
  st->steps = i + 1;
  st->k = k + 1;
  if (broke) {
    st->stop = 1;
    return;
  }
  cpl[k] = beta;
  st->clo = k;
  if (k + 1 >= st->limit) st->stop = 2;
}

__global__ void k_step_finish(LzDev* st, double* __restrict__ cpl, double* __restrict__ oa,
                              double* __restrict__ ob, double* __restrict__ ow, int delayed) {
  k_step_finish_body(st, cpl, oa, ob, ow, delayed);
}

// row k of V / MV = a, b scaled by 1 / sqrt(s[0])
__global__ void k_normalize_k(const LzDev* st, int64_t n, int64_t ld, const double* __restrict__ s,
                              const double* __restrict__ a, double* __restrict__ V,
                              const double* __restrict__ b, double* __restrict__ MV) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  const double nrm = sqrt(fmax(s[0], 0.0));
  const int64_t o = (int64_t)st->k * ld + c;
  V[o] = a[c] / nrm;
  MV[o] = b[c] / nrm;
}

// X[q][c] = sum_i W[i + q*k] * V[i][c]  for q < qn (W column-major k x qn)
template <int NQ>
__global__ void __launch_bounds__(256) k_lift(int64_t n, const double* __restrict__ V, int64_t ld,
                                              int k, const double* __restrict__ W, int q0, int qn,
                                              double* __restrict__ X, int64_t ldx) {
  extern __shared__ double ws[];  // NQ x k
  for (int q = 0; q < NQ; ++q)
    for (int i = threadIdx.x; i < k; i += blockDim.x)
      ws[q * k + i] = (q0 + q < qn) ? W[(int64_t)(q0 + q) * k + i] : 0.0;
  __syncthreads();
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  for (int i = 0; i < k; ++i) {
    const double v = __ldg(V + (int64_t)i * ld + c);
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = fma(ws[q * k + i], v, acc[q]);
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q)
    if (q0 + q < qn) X[(int64_t)(q0 + q) * ldx + c] = acc[q];
}

// X = V[:k]^T W on FP64 tensor cores: C(col, q) = sum_t V[t][col] W[t + q k],
// one 64 x 64 (column x Ritz vector) tile per CTA (dmma.cuh)
__global__ void __launch_bounds__(128) k_lift_dmma(const double* __restrict__ V, int64_t ld, int64_t n, int k,
                                                   const double* __restrict__ W, int c, double* __restrict__ X) {
  dmma_gemm_tile(V, ld, W, k, 0, k, (int64_t)blockIdx.x * 64, (int64_t)blockIdx.y * 64, n, c, X, ld, 1.0);
}

// batched locking on FP64 tensor cores (dmma_tile_gen):
//   k_mdots_dmma  partial[z][i][q] = sum_{t in K-chunk z} A_i[t] X_q[t]  (split-K over n)
//   k_mupd_dmma   Y_q[col] -= sum_i C[i][q] B_i[col]
constexpr int kMKChunk = 512;
static const bool g_lift_dmma = [] {  // RIGA_LIFT_DMMA=0: the CUDA-core lift / locking kernels
  const char* e = getenv("RIGA_LIFT_DMMA");
  return !(e && e[0] == '0');
}();

__global__ void __launch_bounds__(128) k_mdots_dmma(const double* __restrict__ A, int64_t lda, int R,
                                                    const double* __restrict__ X, int64_t ldx, int c, int64_t n,
                                                    double* __restrict__ partial) {
  const int64_t k0 = (int64_t)blockIdx.z * kMKChunk, k1 = imin(n, k0 + kMKChunk);
  dmma_tile_gen(A, lda, 1, X, ldx, 1, k0, k1, (int64_t)blockIdx.x * 64, (int64_t)blockIdx.y * 64, R, c,
                partial + (int64_t)blockIdx.z * R * c, c, 1, 1.0, false);
}
__global__ void __launch_bounds__(128) k_mupd_dmma(const double* __restrict__ B, int64_t ldb, int R,
                                                   const double* __restrict__ C, int c, double* __restrict__ Y,
                                                   int64_t ldy, int64_t n) {
  dmma_tile_gen(B, 1, ldb, C, 1, c, 0, R, (int64_t)blockIdx.x * 64, (int64_t)blockIdx.y * 64, n, c, Y, 1, ldy,
                1.0, true);
}
// mode 1 of k_mupd (strictly upper: earlier batch members only) as a mask on C
__global__ void k_mask_upper(double* __restrict__ C, int c) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < c * c && t / c >= t % c) C[t] = 0.0;  // C[i][q], keep i < q
}

// --- batched locking (ref _sweep :483-523), one converged pair at a time ---
// LzDev scal slots: [5] x.Mx before, [6] after projection; pad[0] = projected?
__global__ void k_pair_begin(LzDev* st) {
  st->pad[0] = st->nlocked > 0 ? 1 : 0;  // the reference projects only if something is locked
  st->pad[1] = 0;                        // rejected?
}

// x, mx /= sqrt(s) (first normalisation; s <= 0 rejects the pair)
__global__ void k_pair_scale(LzDev* st, int64_t n, double* __restrict__ x, double* __restrict__ mx,
                             int slot, int only_if_projected) {
  if (st->pad[1]) return;
  if (only_if_projected && !st->pad[0]) return;
  const double s = st->scal[slot];
  const double nrm = sqrt(fmax(s, 0.0));
  if (!only_if_projected && nrm <= 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) st->pad[1] = 1;
    return;
  }
  if (only_if_projected && nrm < 0.3) {  // a copy of something known
    if (blockIdx.x == 0 && threadIdx.x == 0) st->pad[1] = 1;
    return;
  }
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  x[c] = x[c] / nrm;
  mx[c] = mx[c] / nrm;
}

// append an accepted pair to the locked set (row nlocked) and record the flag
__global__ void k_pair_append(const LzDev* st, int64_t n, int64_t ld, const double* __restrict__ x,
                              const double* __restrict__ mx, double* __restrict__ L,
                              double* __restrict__ LM) {
  if (st->pad[1]) return;
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int64_t o = (int64_t)st->nlocked * ld + c;
  L[o] = x[c];
  LM[o] = mx[c];
}

__global__ void k_pair_end(LzDev* st, int* __restrict__ flags, int q) {
  flags[q] = st->pad[1] ? 0 : 1;
  if (!st->pad[1]) st->nlocked += 1;
}

// --- batched locking: multi-vector Gram-Schmidt against a row set -----------
// mdots: partial[chunk][i][q] = sum_{c in chunk} A_i[c] X_q[c]
//        grid (column chunks of kMChunk, row groups of 32, q groups of 8)
// mred:  C[i][q] = sum_chunk partial[chunk][i][q]
// mupd:  Y_q[c] -= sum_i C[i][q] B_i[c]   (B read once per q group of 8)
constexpr int kMChunk = 4096;

__global__ void __launch_bounds__(256) k_mdots(const double* __restrict__ A, int64_t lda, int R,
                                               const double* __restrict__ X, int64_t ldx, int c,
                                               int64_t n, double* __restrict__ partial) {
  extern __shared__ double xt[];  // 8 x 1024
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int q0 = blockIdx.z * 8, nq = min(8, c - q0);
  const int i = blockIdx.y * 32 + w * 4;
  double acc[4][8];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[a][q] = 0.0;
  const int64_t cbeg = (int64_t)blockIdx.x * kMChunk, cend = imin(n, cbeg + kMChunk);
  for (int64_t s0 = cbeg; s0 < cend; s0 += 1024) {
    const int sn = (int)imin(1024, cend - s0);
    __syncthreads();
    for (int q = 0; q < 8; ++q)
      for (int t = threadIdx.x; t < 1024; t += blockDim.x)
        xt[q * 1024 + t] = (q < nq && t < sn) ? X[(int64_t)(q0 + q) * ldx + s0 + t] : 0.0;
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      if (i + a >= R) break;
      const double* row = A + (int64_t)(i + a) * lda + s0;
      for (int t = lane; t < sn; t += 32) {
        const double v = row[t];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[a][q] = fma(v, xt[q * 1024 + t], acc[a][q]);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    if (i + a >= R) break;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double v = warp_sum(acc[a][q]);
      if (lane == 0 && q < nq) partial[((int64_t)blockIdx.x * R + i + a) * c + q0 + q] = v;
    }
  }
}

__global__ void k_mred(int nchunk, int R, int c, const double* __restrict__ partial,
                       double* __restrict__ C) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)R * c) return;
  double s = 0.0;
  for (int b = 0; b < nchunk; ++b) s += partial[(int64_t)b * R * c + t];
  C[t] = s;
}

// mode 0: coefficients C[i][q] for all i < R;  mode 1: strictly-upper only
// (i < q: the intra-batch projection onto earlier members)
__global__ void __launch_bounds__(256) k_mupd(const double* __restrict__ B, int64_t ldb, int R,
                                              const double* __restrict__ C, int c, int mode,
                                              double* __restrict__ Y, int64_t ldy, int64_t n) {
  __shared__ double cs[8][512];
  const int q0 = blockIdx.y * 8, nq = min(8, c - q0);
  const int64_t col = (int64_t)blockIdx.x * 256 + threadIdx.x;
  double acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = 0.0;
  for (int i0 = 0; i0 < R; i0 += 512) {
    const int ni = min(512, R - i0);
    __syncthreads();
    for (int t = threadIdx.x; t < 8 * 512; t += blockDim.x) {
      const int q = t / 512, ii = t % 512;
      double v = 0.0;
      if (q < nq && ii < ni) {
        v = C[(int64_t)(i0 + ii) * c + q0 + q];
        if (mode == 1 && i0 + ii >= q0 + q) v = 0.0;
      }
      cs[q][ii] = v;
    }
    __syncthreads();
    if (col < n) {
      for (int ii = 0; ii < ni; ++ii) {
        const double v = B[(int64_t)(i0 + ii) * ldb + col];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = fma(v, cs[q][ii], acc[q]);
      }
    }
  }
  if (col < n)
    for (int q = 0; q < nq; ++q) Y[(int64_t)(q0 + q) * ldy + col] -= acc[q];
}

// nrm2[q] = X_q . MX_q (one CTA per row, fixed order)
__global__ void k_rowdots(const double* __restrict__ X, const double* __restrict__ MX, int64_t ld,
                          int64_t n, double* __restrict__ out) {
  __shared__ double red[32];
  const double* x = X + (int64_t)blockIdx.x * ld;
  const double* mx = MX + (int64_t)blockIdx.x * ld;
  double s = 0.0;
  for (int64_t c = threadIdx.x; c < n; c += blockDim.x) s = fma(x[c], mx[c], s);
  s = block_sum(s, red);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// rows q with flag[q] != 0: X_q, MX_q /= sqrt(nrm2[q])
__global__ void k_rowscale(double* __restrict__ X, double* __restrict__ MX, int64_t ld, int64_t n,
                           const double* __restrict__ nrm2, const int* __restrict__ flag) {
  const int q = blockIdx.y;
  if (flag && !flag[q]) return;
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  const double nrm = sqrt(fmax(nrm2[q], 0.0));
  X[(int64_t)q * ld + c] /= nrm;
  MX[(int64_t)q * ld + c] /= nrm;
}

}  // namespace riga

using namespace riga;

struct riga_lanczos {
  riga::CtxRef ctxref;
  riga_ctx* ctx = nullptr;
  riga_system* sys = nullptr;
  riga_factor* op = nullptr;
  int64_t n = 0, ld = 0, max_dim = 0, k = 0;
  int64_t nlocked = 0, cap = 0;
  DevBuf<double> V, MV, L, LM, w, r, Mr, bp, coef, partial, upart, cpl, Wd, outs, dscratch;
  DevBuf<double> vt, mvt;            // finished direction of the delayed pass and its M product
  DevBuf<double> lk_part, lk_C, lk_G, lk_nrm, lk_Xt, lk_MXt;  // scratch of riga_lanczos_lock_block (grow-only)
  bool delayed = true;               // delayed CGS2 step (RIGA_CGS=classic: two passes per step)
  DevBuf<unsigned> tk_dots, tk_upd;  // last-block tickets of the Gram-Schmidt kernels (self-resetting)
  DevBuf<double> kt1, kt2;           // scratch of the Kronecker mass product
  bool kron_ok = false;
  DevBuf<LzDev> st;
  LzDev* hst = nullptr;    // pinned mirror
  double* hbuf = nullptr;  // pinned readback
  int nblk = 0;
  // captured step graph (valid for one operator and one locked-buffer layout)
  cudaGraphExec_t gexec = nullptr;
  bool gvalid = false;  // false: gexec holds a stale operator (update before replay)
  riga_factor* gop = nullptr;
  const double* gL = nullptr;
  int64_t gR = 0;
  long long gnodes = 0;  // kernel launches per replay
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;  // around the last extend's replays
  bool ev_valid = false;
  cudaStream_t cur = nullptr;   // stream the step helpers launch on
  cudaStream_t capst = nullptr; // private stream for graph capture (never legacy)
  ~riga_lanczos() {
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (gexec) cudaGraphExecDestroy(gexec);
    if (capst) cudaStreamDestroy(capst);
    if (hbuf) riga::pinned_put(hbuf);
    if (hst) riga::pinned_put(hst);
  }
};

namespace {

void drop_graph(riga_lanczos* lz) {
  if (lz->gexec) cudaGraphExecDestroy(lz->gexec);
  lz->gexec = nullptr;
}

int grow_locked(riga_lanczos* lz, int64_t need) {
  if (need <= lz->cap) return RIGA_OK;
  int64_t cap = std::max<int64_t>(std::max<int64_t>(16, lz->max_dim), lz->cap);
  while (cap < need) cap *= 2;
  cudaStream_t s = lz->ctx->stream;
  DevBuf<double> nL, nLM;
  RIGA_TRY(nL.alloc(cap * lz->ld, s));
  RIGA_TRY(nLM.alloc(cap * lz->ld, s));
  if (lz->nlocked) {
    RIGA_CUDA(cudaMemcpyAsync(nL.p, lz->L.p, lz->nlocked * lz->ld * 8, cudaMemcpyDeviceToDevice, s));
    RIGA_CUDA(cudaMemcpyAsync(nLM.p, lz->LM.p, lz->nlocked * lz->ld * 8, cudaMemcpyDeviceToDevice, s));
  }
  lz->L.swap(nL);
  lz->LM.swap(nLM);
  lz->cap = cap;
  const int64_t R = lz->max_dim + 1 + cap;
  RIGA_TRY(lz->coef.alloc(2 * R, s));
  RIGA_TRY(lz->partial.alloc(2 * (int64_t)((lz->n + kDotCols - 1) / kDotCols) * R, s));
  RIGA_TRY(lz->tk_dots.alloc(R, s));
  RIGA_CUDA(cudaMemsetAsync(lz->tk_dots.p, 0, R * sizeof(unsigned), s));
  lz->gvalid = false;
  return RIGA_OK;
}

// push the host mirror of the recurrence state to the device
int push_state(riga_lanczos* lz, int64_t clo, int64_t limit, double btol, cudaStream_t on = nullptr) {
  LzDev& h = *lz->hst;
  std::memset(&h, 0, sizeof(LzDev));
  h.k = (int)lz->k;
  h.clo = (int)clo;
  h.nlocked = (int)lz->nlocked;
  h.limit = (int)limit;
  h.btol = btol;
  RIGA_CUDA(cudaMemcpyAsync(lz->st.p, &h, sizeof(LzDev), cudaMemcpyHostToDevice, on ? on : lz->ctx->stream));
  return RIGA_OK;
}

int pull_state(riga_lanczos* lz) {
  RIGA_CUDA(cudaMemcpyAsync(lz->hst, lz->st.p, sizeof(LzDev), cudaMemcpyDeviceToHost, lz->ctx->stream));
  RIGA_CUDA(stream_sync(lz->ctx->stream));
  return RIGA_OK;
}

RowSel sel_basis(riga_lanczos* lz, bool mv, int add) {
  return RowSel{mv ? lz->MV.p : lz->V.p, mv ? lz->LM.p : lz->L.p, lz->ld, add, 1};
}
RowSel sel_locked(riga_lanczos* lz, bool mv) {
  return RowSel{nullptr, mv ? lz->LM.p : lz->L.p, lz->ld, 0, 0};
}

// `passes` x: r -= U^T (D r) over the selected rows; r2 -= U2^T (D r) if given
int cgs_passes(riga_lanczos* lz, RowSel dots, RowSel upd, RowSel upd2, double* r, double* r2,
               int passes, int64_t rows_hint) {
  cudaStream_t s = lz->cur;
  const int64_t Rmax = lz->max_dim + 1 + lz->cap;
  const dim3 gu((unsigned)((lz->n + kUpdCols - 1) / kUpdCols), kUpdGroups);
  for (int p = 0; p < passes; ++p) {
    ProfScope prof(kProfCgs, s, 2.0 * (double)rows_hint * lz->n * 8.0);
    RIGA_CUDA(launch(k_cgs_dots, kDotGrid, 256, 0, s, dots, lz->st.p, lz->n, Rmax, r, lz->partial.p, lz->coef.p,
                                        lz->tk_dots.p));
    RIGA_CUDA(launch(k_cgs_upd, gu, 256, 0, s, upd, lz->st.p, lz->n, lz->ld, lz->coef.p, lz->upart.p, r, lz->tk_upd.p));
    count_launch(2);
    if (r2) {
      RIGA_CUDA(launch(k_cgs_upd, gu, 256, 0, s, upd2, lz->st.p, lz->n, lz->ld, lz->coef.p, lz->upart.p, r2, lz->tk_upd.p));
      count_launch();
    }
  }
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

int mass_apply(riga_lanczos* lz, const double* x, double* y) {
  cudaStream_t s = lz->cur;
  if (lz->sys && lz->sys->kdim && lz->kron_ok) return kron_mass_apply(lz->sys, s, x, y, lz->kt1.p, lz->kt2.p);
  if (lz->sys) return system_spmv(lz->sys, s, 1, 0.0, x, y);
  RIGA_CUDA(cudaMemcpyAsync(y, x, lz->n * 8, cudaMemcpyDeviceToDevice, s));
  return RIGA_OK;
}

int dot2(riga_lanczos* lz, const double* a, int koff_a, const double* b, const double* c,
         const double* d, int slot) {
  cudaStream_t s = lz->cur;
  ProfScope prof(kProfVec, s, 32.0 * lz->n);
  const int blocks = (int)std::min<int64_t>(296, (lz->n + 255) / 256);
  RIGA_CUDA(launch(k_dot2, blocks, 256, 0, s, lz->st.p, lz->n, lz->ld, a, koff_a, b, c, d, lz->dscratch.p,
                                reinterpret_cast<unsigned*>(lz->dscratch.p + 2 * 296),
                                lz->st.p->scal + slot));
  count_launch();
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

// the second half of a step, once w = H v is in lz->w (ref step :244-267)
int step_tail(riga_lanczos* lz) {
  cudaStream_t s = lz->cur;
  const unsigned g1 = (unsigned)((lz->n + 255) / 256);
  RIGA_TRY(dot2(lz, lz->MV.p, 1, lz->w.p, lz->w.p, lz->w.p, 0));  // alpha, |w|^2
  RIGA_CUDA(launch(k_residual, g1, 256, 0, s, lz->st.p, lz->n, lz->ld, lz->w.p, lz->V.p, lz->cpl.p, lz->r.p));
  count_launch();
  RIGA_TRY(cgs_passes(lz, sel_basis(lz, true, 1), sel_basis(lz, false, 1), RowSel{}, lz->r.p, nullptr, 2,
                      lz->k + 1 + lz->nlocked));
  RIGA_TRY(mass_apply(lz, lz->r.p, lz->Mr.p));
  RIGA_TRY(dot2(lz, lz->r.p, 0, lz->Mr.p, lz->r.p, lz->Mr.p, 2));  // beta^2
  RIGA_CUDA(launch(k_normalize_next, g1, 256, 0, s, lz->st.p, lz->n, lz->ld, lz->r.p, lz->Mr.p, lz->V.p, lz->MV.p));
  count_launch();
  RIGA_CUDA(launch(k_step_finish, 1, 1, 0, s, lz->st.p, lz->cpl.p, lz->outs.p, lz->outs.p + (lz->max_dim + 1),
                                lz->outs.p + 2 * (lz->max_dim + 1), 0));
  count_launch();
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

// one full step with the device operator
int step_full(riga_lanczos* lz) {
  cudaStream_t s = lz->cur;
  const unsigned g1 = (unsigned)((lz->n + 255) / 256);
  RIGA_CUDA(launch(k_perm_row, g1, 256, 0, s, lz->st.p, lz->n, lz->ld, lz->MV.p, lz->op->sym->d_order.p, lz->bp.p));
  count_launch();
  RIGA_TRY(factor_solve(lz->op, s, lz->bp.p, lz->w.p, true));
  if (!lz->delayed) return step_tail(lz);
  // delayed CGS2: one dots sweep + one update sweep (see k_dcgs_dots)
  const int64_t Rmax = lz->max_dim + 1 + lz->cap;
  double* ob = lz->outs.p + (lz->max_dim + 1);
  {
    ProfScope prof(kProfCgs, s, 2.0 * (double)(lz->k + 1 + lz->nlocked) * lz->n * 8.0);
    RIGA_CUDA(launch(k_dcgs_dots, dcgs_dot_grid(), 256, 0, s, sel_basis(lz, true, 1), lz->st.p, lz->n, Rmax, lz->V.p, lz->w.p,
                                         lz->partial.p, lz->coef.p, lz->tk_dots.p));
    const dim3 gu((unsigned)((lz->n + kUpdCols - 1) / kUpdCols), kUpdGroups);
    RIGA_CUDA(launch(k_dcgs_upd, gu, 256, 0, s, sel_basis(lz, false, 1), lz->st.p, lz->n, lz->ld, Rmax, lz->coef.p,
                     lz->upart.p, lz->w.p, lz->vt.p, lz->r.p, lz->tk_upd.p, lz->cpl.p));
    count_launch(2);
  }
  RIGA_TRY(mass_apply(lz, lz->vt.p, lz->mvt.p));
  RIGA_TRY(mass_apply(lz, lz->r.p, lz->Mr.p));
  RIGA_TRY(dot2(lz, lz->r.p, 0, lz->Mr.p, lz->r.p, lz->Mr.p, 2));  // beta~^2
  RIGA_CUDA(launch(k_dcgs_store, g1, 256, 0, s, lz->st.p, lz->n, lz->ld, lz->vt.p, lz->mvt.p, lz->r.p, lz->Mr.p, lz->V.p,
                                  lz->MV.p));
  RIGA_CUDA(launch(k_step_finish, 1, 1, 0, s, lz->st.p, lz->cpl.p, lz->outs.p, ob, lz->outs.p + 2 * (lz->max_dim + 1), 1));
  count_launch(2);
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

// end of a delayed run: the pending row k gets its second pass against rows
// [0, k) + locked and is renormalised; the run's last beta *= that norm
int finish_pending(riga_lanczos* lz, int last, cudaStream_t on = nullptr) {
  cudaStream_t s = on ? on : lz->ctx->stream;
  RIGA_TRY(push_state(lz, lz->k, lz->k, 0.0, s));
  double* x = lz->V.p + lz->k * lz->ld;
  double* mx = lz->MV.p + lz->k * lz->ld;
  RIGA_TRY(cgs_passes(lz, sel_basis(lz, true, 0), sel_basis(lz, false, 0), RowSel{}, x, nullptr, 1,
                      lz->k + lz->nlocked));
  RIGA_TRY(mass_apply(lz, x, mx));
  RIGA_TRY(dot2(lz, x, 0, mx, x, mx, 6));
  k_dcgs_finish_row<<<(unsigned)((lz->n + 255) / 256), 256, 0, s>>>(lz->st.p, lz->n, lz->ld, lz->st.p->scal + 6,
                                                                     lz->V.p, lz->MV.p,
                                                                     lz->outs.p + (lz->max_dim + 1), last);
  count_launch();
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

int ensure_graph(riga_lanczos* lz) {
  const int64_t Rmax = lz->max_dim + 1 + lz->cap;
  if (lz->gexec && lz->gvalid && lz->gop == lz->op && lz->gL == lz->L.p && lz->gR == Rmax) return RIGA_OK;
  cudaStream_t s = lz->ctx->stream;
  // kernel attributes must be set outside the capture
  RIGA_TRY(prepare_solve());
  RIGA_CUDA(stream_sync(s));
  cudaGraph_t g = nullptr;
  if (!lz->capst) RIGA_CUDA(cudaStreamCreateWithFlags(&lz->capst, cudaStreamNonBlocking));
  const long long n0 = t_launches;
  RIGA_CUDA(cudaStreamBeginCapture(lz->capst, cudaStreamCaptureModeThreadLocal));
  lz->cur = lz->capst;
  const int rc = step_full(lz);
  lz->cur = lz->ctx->stream;
  cudaError_t e = cudaStreamEndCapture(lz->capst, &g);
  lz->gnodes = t_launches - n0;
  g_launches.fetch_sub(lz->gnodes);  // captured, not launched
  if (rc) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  RIGA_CUDA(e);
  // same kernel sequence, new parameters (operator / buffers): update the
  // executable graph in place (cheaper than instantiating a new one)
  bool updated = false;
  if (lz->gexec) {
    cudaGraphExecUpdateResultInfo info;
    updated = cudaGraphExecUpdate(lz->gexec, g, &info) == cudaSuccess;
    if (!updated) {
      cudaGetLastError();
      drop_graph(lz);
    }
  }
  if (!updated) e = cudaGraphInstantiate(&lz->gexec, g, 0);
  cudaGraphDestroy(g);
  RIGA_CUDA(e);
  lz->gvalid = true;
  lz->gop = lz->op;
  lz->gL = lz->L.p;
  lz->gR = Rmax;
  return RIGA_OK;
}

}  // namespace

extern "C" {

int riga_lanczos_create(riga_ctx* ctx, riga_system* mass, int64_t n, int64_t max_dim,
                        riga_lanczos** out) {
  RIGA_CHECK_ARG(out && max_dim >= 1 && n >= 1, "bad arg");
  RIGA_CHECK_ARG(!mass || mass->n == n, "mass dimension mismatch");
  if (!ctx && mass) ctx = mass->ctx;
  RIGA_CHECK_ARG(ctx, "null ctx");
  DeviceGuard g(ctx->device);
  auto lz = std::make_unique<riga_lanczos>();
  lz->ctx = ctx;
  lz->ctxref.set(ctx);
  lz->cur = ctx->stream;
  lz->sys = mass;
  lz->n = n;
  lz->ld = (n + 3) / 4 * 4;
  lz->max_dim = std::min<int64_t>(max_dim, n);
  lz->nblk = (int)((lz->n + kChunk - 1) / kChunk);
  const int64_t rows = lz->max_dim + 1;
  cudaStream_t cs = ctx->stream;
  RIGA_TRY(lz->V.alloc(rows * lz->ld, cs));
  RIGA_TRY(lz->MV.alloc(rows * lz->ld, cs));
  RIGA_CUDA(cudaMemsetAsync(lz->V.p, 0, rows * lz->ld * 8, cs));
  RIGA_CUDA(cudaMemsetAsync(lz->MV.p, 0, rows * lz->ld * 8, cs));
  RIGA_TRY(lz->w.alloc(lz->ld, cs));
  RIGA_TRY(lz->r.alloc(lz->ld, cs));
  RIGA_TRY(lz->Mr.alloc(lz->ld, cs));
  RIGA_TRY(lz->bp.alloc(lz->ld, cs));
  RIGA_TRY(lz->upart.alloc(2 * kUpdGroups * lz->ld, cs));
  RIGA_TRY(lz->vt.alloc(lz->ld, cs));
  RIGA_TRY(lz->mvt.alloc(lz->ld, cs));
  {
    const char* e = getenv("RIGA_CGS");
    lz->delayed = !(e && std::strcmp(e, "classic") == 0);
  }
  RIGA_TRY(lz->tk_upd.alloc((lz->n + kUpdCols - 1) / kUpdCols, cs));
  RIGA_CUDA(cudaMemsetAsync(lz->tk_upd.p, 0, ((lz->n + kUpdCols - 1) / kUpdCols) * sizeof(unsigned), cs));
  RIGA_TRY(lz->cpl.alloc(rows, cs));
  RIGA_TRY(lz->outs.alloc(3 * rows, cs));
  RIGA_TRY(lz->dscratch.alloc(2 * 296 + 8, cs));
  RIGA_CUDA(cudaMemsetAsync(lz->dscratch.p, 0, (2 * 296 + 8) * 8, cs));
  RIGA_TRY(lz->st.alloc(1, cs));
  if (mass && mass->kdim && !getenv("RIGA_CSR_MASS")) {
    RIGA_TRY(lz->kt1.alloc(n, cs));
    RIGA_TRY(lz->kt2.alloc(n, cs));
    lz->kron_ok = true;
  }
  RIGA_CUDA(cudaMemsetAsync(lz->st.p, 0, sizeof(LzDev), cs));
  RIGA_TRY(grow_locked(lz.get(), 16));
  lz->hst = static_cast<LzDev*>(pinned_get(sizeof(LzDev)));
  lz->hbuf = static_cast<double*>(pinned_get(std::max<int64_t>(64, 3 * rows + 8) * 8));
  if (!lz->hst || !lz->hbuf) {
    set_error("pinned host allocation failed");
    return RIGA_OOM;
  }
  RIGA_CUDA(stream_sync(cs));
  *out = lz.release();
  return RIGA_OK;
}

int riga_lanczos_destroy(riga_lanczos* lz) {
  if (!lz) return RIGA_OK;
  DeviceGuard g(lz->ctx->device);
  stream_sync(lz->ctx->stream);
  delete lz;
  return RIGA_OK;
}

int riga_lanczos_reset(riga_lanczos* lz, riga_system* mass) {
  RIGA_CHECK_ARG(lz, "null arg");
  RIGA_CHECK_ARG(!mass || mass->n == lz->n, "mass dimension mismatch");
  DeviceGuard g(lz->ctx->device);
  lz->sys = mass;
  if (mass && mass->kdim && !getenv("RIGA_CSR_MASS")) {
    if (!lz->kt1.p) {
      RIGA_TRY(lz->kt1.alloc(lz->n, lz->ctx->stream));
      RIGA_TRY(lz->kt2.alloc(lz->n, lz->ctx->stream));
    }
    lz->kron_ok = true;
  } else {
    lz->kron_ok = false;
  }
  lz->k = 0;
  lz->nlocked = 0;
  lz->ev_valid = false;
  // the captured step graph holds the previous operator's device pointers;
  // a new factor may reuse the old one's host address (riga_factor*), so the
  // pointer comparison in ensure_graph cannot be trusted across states
  lz->gvalid = false;  // re-captured (and updated in place) before the next extend
  lz->op = nullptr;
  return push_state(lz, 0, 0, 0.0);
}

int riga_lanczos_set_operator(riga_lanczos* lz, riga_factor* f) {
  RIGA_CHECK_ARG(lz && f, "null arg");
  RIGA_CHECK_ARG(f->sym->h.n == lz->n, "operator dimension mismatch");
  if (lz->op != f) lz->gvalid = false;
  lz->op = f;
  return RIGA_OK;
}

int riga_lanczos_k(riga_lanczos* lz, int64_t* k) {
  RIGA_CHECK_ARG(lz && k, "null arg");
  *k = lz->k;
  return RIGA_OK;
}

int riga_lanczos_locked_count(riga_lanczos* lz, int64_t* c) {
  RIGA_CHECK_ARG(lz && c, "null arg");
  *c = lz->nlocked;
  return RIGA_OK;
}

int riga_lanczos_set_start(riga_lanczos* lz, const double* r_host) {
  RIGA_CHECK_ARG(lz && r_host, "null arg");
  DeviceGuard g(lz->ctx->device);
  cudaStream_t s = lz->ctx->stream;
  RIGA_TRY(push_state(lz, lz->k, lz->k, 0.0));
  RIGA_CUDA(cudaMemcpyAsync(lz->r.p, r_host, lz->n * 8, cudaMemcpyHostToDevice, s));
  RIGA_TRY(mass_apply(lz, lz->r.p, lz->Mr.p));
  RIGA_TRY(dot2(lz, lz->r.p, 0, lz->Mr.p, lz->r.p, lz->Mr.p, 0));
  RIGA_TRY(pull_state(lz));
  if (!(std::sqrt(std::max(lz->hst->scal[0], 0.0)) > 0.0)) {
    set_error("start vector has zero mass norm");
    return RIGA_BAD_ARG;
  }
  k_normalize_k<<<(unsigned)((lz->n + 255) / 256), 256, 0, s>>>(lz->st.p, lz->n, lz->ld, lz->st.p->scal,
                                                                  lz->r.p, lz->V.p, lz->Mr.p, lz->MV.p);
  count_launch();
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

int riga_lanczos_fresh(riga_lanczos* lz, const double* r_host, int* accepted) {
  RIGA_CHECK_ARG(lz && r_host && accepted, "null arg");
  DeviceGuard g(lz->ctx->device);
  cudaStream_t s = lz->ctx->stream;
  RIGA_TRY(push_state(lz, lz->k, lz->k, 0.0));
  RIGA_CUDA(cudaMemcpyAsync(lz->r.p, r_host, lz->n * 8, cudaMemcpyHostToDevice, s));
  RIGA_TRY(mass_apply(lz, lz->r.p, lz->Mr.p));
  RIGA_TRY(dot2(lz, lz->r.p, 0, lz->Mr.p, lz->r.p, lz->Mr.p, 4));  // ref norm^2 -> scal[4]
  RIGA_TRY(cgs_passes(lz, sel_basis(lz, true, 0), sel_basis(lz, false, 0), RowSel{}, lz->r.p, nullptr, 2,
                      lz->k + lz->nlocked));
  RIGA_TRY(mass_apply(lz, lz->r.p, lz->Mr.p));
  RIGA_TRY(dot2(lz, lz->r.p, 0, lz->Mr.p, lz->r.p, lz->Mr.p, 0));
  RIGA_TRY(pull_state(lz));
  const double ref = std::sqrt(std::max(lz->hst->scal[4], 0.0));
  const double nrm = std::sqrt(std::max(lz->hst->scal[0], 0.0));
  *accepted = nrm > 1e-8 * std::max(ref, 1e-300);
  if (*accepted) {
    k_normalize_k<<<(unsigned)((lz->n + 255) / 256), 256, 0, s>>>(lz->st.p, lz->n, lz->ld, lz->st.p->scal,
                                                                    lz->r.p, lz->V.p, lz->Mr.p, lz->MV.p);
    count_launch();
    RIGA_CUDA(cudaGetLastError());
  }
  return RIGA_OK;
}

int riga_lanczos_lock(riga_lanczos* lz, const double* x, const double* mx) {
  RIGA_CHECK_ARG(lz && x && mx, "null arg");
  DeviceGuard g(lz->ctx->device);
  RIGA_TRY(grow_locked(lz, lz->nlocked + 1));
  cudaStream_t s = lz->ctx->stream;
  RIGA_CUDA(cudaMemcpyAsync(lz->L.p + lz->nlocked * lz->ld, x, lz->n * 8, cudaMemcpyDeviceToDevice, s));
  RIGA_CUDA(cudaMemcpyAsync(lz->LM.p + lz->nlocked * lz->ld, mx, lz->n * 8, cudaMemcpyDeviceToDevice, s));
  lz->nlocked++;
  return RIGA_OK;
}

int riga_lanczos_extend(riga_lanczos* lz, int64_t limit, const double* coupling_host,
                        double breakdown_tol, double* alpha, double* beta, double* wnorm,
                        int64_t* steps) {
  RIGA_CHECK_ARG(lz && alpha && beta && wnorm && steps, "null arg");
  RIGA_CHECK_ARG(lz->op, "no operator set");
  DeviceGuard g(lz->ctx->device);
  cudaStream_t s = lz->ctx->stream;
  limit = std::min(limit, lz->max_dim);
  *steps = 0;
  if (lz->k >= limit) return RIGA_OK;
  int64_t clo = lz->k;
  if (coupling_host && lz->k > 0) {
    RIGA_CUDA(cudaMemcpyAsync(lz->cpl.p, coupling_host, lz->k * 8, cudaMemcpyHostToDevice, s));
    clo = 0;
  }
  RIGA_TRY(ensure_graph(lz));
  RIGA_TRY(push_state(lz, clo, limit, breakdown_tol));
  if (!lz->ev0) {
    RIGA_CUDA(cudaEventCreate(&lz->ev0));
    RIGA_CUDA(cudaEventCreate(&lz->ev1));
  }
  RIGA_CUDA(cudaEventRecord(lz->ev0, s));
  for (int64_t i = lz->k; i < limit; ++i) RIGA_CUDA(cudaGraphLaunch(lz->gexec, s));
  RIGA_CUDA(cudaEventRecord(lz->ev1, s));
  lz->ev_valid = true;
  count_launch((int)((limit - lz->k) * lz->gnodes));
  const int64_t rows = lz->max_dim + 1;
  if (lz->delayed) {
    RIGA_TRY(pull_state(lz));
    const int ns0 = lz->hst->steps, stop0 = lz->hst->stop, k0 = lz->hst->k;
    if (stop0 != 1 && ns0 > 0) {
      lz->k = k0;
      RIGA_TRY(finish_pending(lz, ns0 - 1));
    }
    RIGA_CUDA(cudaMemcpyAsync(lz->hbuf, lz->outs.p, 3 * rows * 8, cudaMemcpyDeviceToHost, s));
    RIGA_CUDA(stream_sync(s));
    lz->hst->steps = ns0;
    lz->hst->stop = stop0;
    lz->hst->k = k0;
  } else {
    RIGA_CUDA(cudaMemcpyAsync(lz->hbuf, lz->outs.p, 3 * rows * 8, cudaMemcpyDeviceToHost, s));
    RIGA_TRY(pull_state(lz));
  }
  const int ns = lz->hst->steps;
  for (int i = 0; i < ns; ++i) {
    alpha[i] = lz->hbuf[i];
    beta[i] = lz->hbuf[rows + i];
    wnorm[i] = lz->hbuf[2 * rows + i];
  }
  *steps = ns;
  lz->k = lz->hst->k;
  return lz->hst->stop == 1 ? RIGA_BREAKDOWN : RIGA_OK;
}

int riga_lanczos_last_extend_ms(riga_lanczos* lz, float* ms) {
  RIGA_CHECK_ARG(lz && ms, "null arg");
  *ms = 0.0f;
  if (!lz->ev_valid) return RIGA_OK;
  DeviceGuard g(lz->ctx->device);
  RIGA_CUDA(cudaEventSynchronize(lz->ev1));
  RIGA_CUDA(cudaEventElapsedTime(ms, lz->ev0, lz->ev1));
  return RIGA_OK;
}

int riga_lanczos_step_given(riga_lanczos* lz, const double* w_dev, const double* coupling_host,
                            double breakdown_tol, double* alpha, double* beta, double* wnorm) {
  RIGA_CHECK_ARG(lz && w_dev && alpha && beta && wnorm, "null arg");
  RIGA_CHECK_ARG(lz->k < lz->max_dim, "basis is full");
  DeviceGuard g(lz->ctx->device);
  cudaStream_t s = lz->ctx->stream;
  int64_t clo = lz->k;
  if (coupling_host && lz->k > 0) {
    RIGA_CUDA(cudaMemcpyAsync(lz->cpl.p, coupling_host, lz->k * 8, cudaMemcpyHostToDevice, s));
    clo = 0;
  }
  RIGA_TRY(push_state(lz, clo, lz->k + 1, breakdown_tol));
  RIGA_CUDA(cudaMemcpyAsync(lz->w.p, w_dev, lz->n * 8, cudaMemcpyDeviceToDevice, s));
  RIGA_TRY(step_tail(lz));
  const int64_t rows = lz->max_dim + 1;
  RIGA_CUDA(cudaMemcpyAsync(lz->hbuf, lz->outs.p, 3 * rows * 8, cudaMemcpyDeviceToHost, s));
  RIGA_TRY(pull_state(lz));
  *alpha = lz->hbuf[0];
  *beta = lz->hbuf[rows];
  *wnorm = lz->hbuf[2 * rows];
  lz->k = lz->hst->k;
  return lz->hst->stop == 1 ? RIGA_BREAKDOWN : RIGA_OK;
}

}  // extern "C"


namespace {

// C (R x c) = A (R rows) . X^T (c rows)
int mdots(riga_lanczos* lz, const double* A, int R, const double* X, int c, double* C, DevBuf<double>& part) {
  cudaStream_t s = lz->ctx->stream;
  if (R == 0 || c == 0) return RIGA_OK;
  if (g_lift_dmma) {
    const int nz = (int)((lz->n + kMKChunk - 1) / kMKChunk);
    RIGA_TRY(part.reserve((int64_t)nz * R * c, s));
    const dim3 g((unsigned)((R + 63) / 64), (unsigned)((c + 63) / 64), (unsigned)nz);
    k_mdots_dmma<<<g, 128, 0, s>>>(A, lz->ld, R, X, lz->ld, c, lz->n, part.p);
    k_mred<<<(unsigned)(((int64_t)R * c + 255) / 256), 256, 0, s>>>(nz, R, c, part.p, C);
    count_launch(2);
    RIGA_CUDA(cudaGetLastError());
    return RIGA_OK;
  }
  const int nchunk = (int)((lz->n + kMChunk - 1) / kMChunk);
  RIGA_TRY(part.reserve((int64_t)nchunk * R * c, s));
  const dim3 g(nchunk, (unsigned)((R + 31) / 32), (unsigned)((c + 7) / 8));
  k_mdots<<<g, 256, 8 * 1024 * 8, s>>>(A, lz->ld, R, X, lz->ld, c, lz->n, part.p);
  k_mred<<<(unsigned)(((int64_t)R * c + 255) / 256), 256, 0, s>>>(nchunk, R, c, part.p, C);
  count_launch(2);
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

// Y_q -= sum_i C[i][q] B_i
int mupd(riga_lanczos* lz, const double* B, int R, const double* C, int c, int mode, double* Y) {
  if (R == 0 || c == 0) return RIGA_OK;
  if (g_lift_dmma && mode == 0) {
    const dim3 g((unsigned)((lz->n + 63) / 64), (unsigned)((c + 63) / 64));
    k_mupd_dmma<<<g, 128, 0, lz->ctx->stream>>>(B, lz->ld, R, C, c, Y, lz->ld, lz->n);
    count_launch();
    RIGA_CUDA(cudaGetLastError());
    return RIGA_OK;
  }
  const dim3 g((unsigned)((lz->n + 255) / 256), (unsigned)((c + 7) / 8));
  k_mupd<<<g, 256, 0, lz->ctx->stream>>>(B, lz->ld, R, C, c, mode, Y, lz->ld, lz->n);
  count_launch();
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

}  // namespace

extern "C" {

int riga_lanczos_lock_block(riga_lanczos* lz, double* X, double* MX, int64_t c, int64_t ldx,
                            double* nrm2_host) {
  RIGA_CHECK_ARG(lz && X && MX && nrm2_host && c >= 0, "null arg");
  RIGA_CHECK_ARG(ldx == lz->ld, "rows must use the basis leading dimension");
  if (c == 0) return RIGA_OK;
  DeviceGuard g(lz->ctx->device);
  cudaStream_t s = lz->ctx->stream;
  static int attr = 0;
  if (!attr) {
    RIGA_CUDA(cudaFuncSetAttribute(k_mdots, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 1024 * 8));
    attr = 1;
  }
  const int nl = (int)lz->nlocked, cc = (int)c;
  // scratch kept on the state (grow-only): no stream-ordered allocations inside a slice's lock phase
  DevBuf<double>&part = lz->lk_part, &C = lz->lk_C, &G = lz->lk_G, &nrm = lz->lk_nrm, &Xt = lz->lk_Xt, &MXt = lz->lk_MXt;
  RIGA_TRY(C.reserve(std::max<int64_t>((int64_t)nl * cc, 1), s));
  RIGA_TRY(G.reserve((int64_t)cc * cc, s));
  RIGA_TRY(nrm.reserve(cc, s));
  RIGA_TRY(Xt.reserve(c * lz->ld, s));
  RIGA_TRY(MXt.reserve(c * lz->ld, s));
  const dim3 gs((unsigned)((lz->n + 255) / 256), (unsigned)cc);
  // M-normalise the lifted vectors (ref: x /= sqrt(x.Mx))
  k_rowdots<<<cc, 256, 0, s>>>(X, MX, lz->ld, lz->n, nrm.p);
  k_rowscale<<<gs, 256, 0, s>>>(X, MX, lz->ld, lz->n, nrm.p, nullptr);
  count_launch(2);
  for (int p = 0; p < 2; ++p) {
    if (nl > 0) {  // against the locked set: C = LM X^T, X -= L^T C, MX -= LM^T C
      RIGA_TRY(mdots(lz, lz->LM.p, nl, X, cc, C.p, part));
      RIGA_TRY(mupd(lz, lz->L.p, nl, C.p, cc, 0, X));
      RIGA_TRY(mupd(lz, lz->LM.p, nl, C.p, cc, 0, MX));
    }
    if (cc > 1) {  // against the earlier members of the batch
      RIGA_TRY(mdots(lz, MX, cc, X, cc, G.p, part));
      if (g_lift_dmma) {  // mode 1 (earlier batch members only) as a mask, then plain updates
        k_mask_upper<<<(unsigned)((cc * cc + 255) / 256), 256, 0, s>>>(G.p, cc);
        count_launch();
      }
      RIGA_CUDA(cudaMemcpyAsync(Xt.p, X, c * lz->ld * 8, cudaMemcpyDeviceToDevice, s));
      RIGA_CUDA(cudaMemcpyAsync(MXt.p, MX, c * lz->ld * 8, cudaMemcpyDeviceToDevice, s));
      RIGA_TRY(mupd(lz, Xt.p, cc, G.p, cc, g_lift_dmma ? 0 : 1, X));
      RIGA_TRY(mupd(lz, MXt.p, cc, G.p, cc, g_lift_dmma ? 0 : 1, MX));
    }
  }
  k_rowdots<<<cc, 256, 0, s>>>(X, MX, lz->ld, lz->n, nrm.p);
  count_launch();
  RIGA_CUDA(cudaMemcpyAsync(nrm2_host, nrm.p, c * 8, cudaMemcpyDeviceToHost, s));
  RIGA_CUDA(stream_sync(s));
  return RIGA_OK;
}

int riga_lanczos_append_rows(riga_lanczos* lz, double* X, double* MX, int64_t c, int64_t ldx,
                             const double* nrm2_host, const int* scale_host) {
  RIGA_CHECK_ARG(lz && X && MX && c >= 0 && ldx == lz->ld, "bad arg");
  if (c == 0) return RIGA_OK;
  DeviceGuard g(lz->ctx->device);
  cudaStream_t s = lz->ctx->stream;
  RIGA_TRY(grow_locked(lz, lz->nlocked + c));
  DevBuf<double> nrm;
  DevBuf<int> flag;
  RIGA_TRY(nrm.upload(nrm2_host, c, s));
  RIGA_TRY(flag.upload(scale_host, c, s));
  const dim3 gs((unsigned)((lz->n + 255) / 256), (unsigned)c);
  k_rowscale<<<gs, 256, 0, s>>>(X, MX, lz->ld, lz->n, nrm.p, flag.p);
  count_launch();
  RIGA_CUDA(cudaMemcpyAsync(lz->L.p + lz->nlocked * lz->ld, X, c * lz->ld * 8, cudaMemcpyDeviceToDevice, s));
  RIGA_CUDA(cudaMemcpyAsync(lz->LM.p + lz->nlocked * lz->ld, MX, c * lz->ld * 8, cudaMemcpyDeviceToDevice, s));
  lz->nlocked += c;
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

}  // extern "C"

static int lift_rows(riga_lanczos* lz, const double* Vb, int64_t k, const double* Wd, int64_t c,
                     double* X) {
  cudaStream_t s = lz->ctx->stream;
  ProfScope prof(kProfLift, s, 8.0 * (double)k * lz->n * ((c + 7) / 8));
  if (g_lift_dmma && c >= 16) {  // (a 64-wide tile wastes most of its MMAs on fewer vectors)
    const dim3 g((unsigned)((lz->n + 63) / 64), (unsigned)((c + 63) / 64));
    k_lift_dmma<<<g, 128, 0, s>>>(Vb, lz->ld, lz->n, (int)k, Wd, (int)c, X);
    count_launch();
  } else {
    const unsigned g1 = (unsigned)((lz->n + 255) / 256);
    for (int64_t q0 = 0; q0 < c; q0 += 8) {
      k_lift<8><<<g1, 256, k * 8 * 8, s>>>(lz->n, Vb, lz->ld, (int)k, Wd, (int)q0, (int)c, X, lz->ld);
      count_launch();
    }
  }
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

extern "C" {

int riga_lanczos_lift(riga_lanczos* lz, const double* W_host, int64_t c, double* X, double* MX) {
  RIGA_CHECK_ARG(lz && W_host && X && MX && c >= 0, "null arg");
  if (c == 0) return RIGA_OK;
  DeviceGuard g(lz->ctx->device);
  cudaStream_t s = lz->ctx->stream;
  const int64_t k = lz->k;
  RIGA_TRY(lz->Wd.alloc(std::max<int64_t>(k * c, 1), s));
  RIGA_CUDA(cudaMemcpyAsync(lz->Wd.p, W_host, k * c * 8, cudaMemcpyHostToDevice, s));
  RIGA_TRY(lift_rows(lz, lz->V.p, k, lz->Wd.p, c, X));
  RIGA_TRY(lift_rows(lz, lz->MV.p, k, lz->Wd.p, c, MX));
  return RIGA_OK;
}

int riga_lanczos_restart(riga_lanczos* lz, const double* W_host, int64_t c) {
  RIGA_CHECK_ARG(lz && c >= 0 && c < lz->max_dim, "bad arg");
  DeviceGuard g(lz->ctx->device);
  cudaStream_t s = lz->ctx->stream;
  const int64_t k = lz->k, ld = lz->ld;
  if (c > 0) {
    RIGA_CHECK_ARG(W_host, "null weights");
    DevBuf<double> nv, nmv;
    RIGA_TRY(nv.alloc(c * ld, s));
    RIGA_TRY(nmv.alloc(c * ld, s));
    RIGA_TRY(lz->Wd.alloc(k * c, s));
    RIGA_CUDA(cudaMemcpyAsync(lz->Wd.p, W_host, k * c * 8, cudaMemcpyHostToDevice, s));
    RIGA_TRY(lift_rows(lz, lz->V.p, k, lz->Wd.p, c, nv.p));
    RIGA_TRY(lift_rows(lz, lz->MV.p, k, lz->Wd.p, c, nmv.p));
    RIGA_CUDA(cudaMemcpyAsync(lz->V.p, nv.p, c * ld * 8, cudaMemcpyDeviceToDevice, s));
    RIGA_CUDA(cudaMemcpyAsync(lz->MV.p, nmv.p, c * ld * 8, cudaMemcpyDeviceToDevice, s));
  }
  // keep the pending direction: row k -> row c
  if (c != k) {
    RIGA_CUDA(cudaMemcpyAsync(lz->V.p + c * ld, lz->V.p + k * ld, ld * 8, cudaMemcpyDeviceToDevice, s));
    RIGA_CUDA(cudaMemcpyAsync(lz->MV.p + c * ld, lz->MV.p + k * ld, ld * 8, cudaMemcpyDeviceToDevice, s));
  }
  lz->k = c;
  return RIGA_OK;
}

int riga_lanczos_lock_batch(riga_lanczos* lz, double* X, double* MX, int64_t c, int64_t ldx,
                            int* accepted) {
  RIGA_CHECK_ARG(lz && X && MX && accepted && c >= 0, "null arg");
  if (c == 0) return RIGA_OK;
  DeviceGuard g(lz->ctx->device);
  cudaStream_t s = lz->ctx->stream;
  RIGA_TRY(grow_locked(lz, lz->nlocked + c));
  DevBuf<int> flags;
  RIGA_TRY(flags.alloc(c, s));
  RIGA_TRY(push_state(lz, lz->k, lz->k, 0.0));
  const unsigned g1 = (unsigned)((lz->n + 255) / 256);
  for (int64_t q = 0; q < c; ++q) {
    double* x = X + q * ldx;
    double* mx = MX + q * ldx;
    k_pair_begin<<<1, 1, 0, s>>>(lz->st.p);
    RIGA_TRY(dot2(lz, x, 0, mx, x, mx, 5));
    k_pair_scale<<<g1, 256, 0, s>>>(lz->st.p, lz->n, x, mx, 5, 0);
    // two passes against the locked set (empty set: the kernels do nothing)
    RIGA_TRY(cgs_passes(lz, sel_locked(lz, true), sel_locked(lz, false), sel_locked(lz, true), x, mx, 2,
                        lz->nlocked + q));
    RIGA_TRY(dot2(lz, x, 0, mx, x, mx, 6));
    k_pair_scale<<<g1, 256, 0, s>>>(lz->st.p, lz->n, x, mx, 6, 1);
    k_pair_append<<<g1, 256, 0, s>>>(lz->st.p, lz->n, lz->ld, x, mx, lz->L.p, lz->LM.p);
    k_pair_end<<<1, 1, 0, s>>>(lz->st.p, flags.p, (int)q);
    count_launch(6);
  }
  RIGA_CUDA(cudaGetLastError());
  RIGA_CUDA(cudaMemcpyAsync(accepted, flags.p, c * sizeof(int), cudaMemcpyDeviceToHost, s));
  RIGA_TRY(pull_state(lz));
  lz->nlocked = lz->hst->nlocked;
  return RIGA_OK;
}

int riga_lanczos_cgs_probe(riga_lanczos* lz, double* x, int passes, int64_t* rows) {
  RIGA_CHECK_ARG(lz && x && passes >= 0, "null arg");
  DeviceGuard g(lz->ctx->device);
  RIGA_TRY(push_state(lz, lz->k, lz->k, 0.0));
  if (rows) *rows = lz->k + lz->nlocked;
  return cgs_passes(lz, sel_basis(lz, true, 0), sel_basis(lz, false, 0), RowSel{}, x, nullptr, passes,
                    lz->k + lz->nlocked);
}

int riga_lanczos_dcgs_probe(riga_lanczos* lz, const double* w, int64_t* rows) {
  RIGA_CHECK_ARG(lz && w && lz->k < lz->max_dim, "bad arg");
  DeviceGuard g(lz->ctx->device);
  cudaStream_t s = lz->ctx->stream;
  RIGA_TRY(push_state(lz, lz->k, lz->k, 0.0));  // steps = 0: no beta correction
  const int64_t Rmax = lz->max_dim + 1 + lz->cap;
  if (rows) *rows = lz->k + 1 + lz->nlocked;
  // events around the two sweeps alone (riga_lanczos_last_extend_ms reads them): the state upload above is
  // not part of the step's sweeps
  if (!lz->ev0) {
    RIGA_CUDA(cudaEventCreate(&lz->ev0));
    RIGA_CUDA(cudaEventCreate(&lz->ev1));
  }
  RIGA_CUDA(cudaEventRecord(lz->ev0, s));
  RIGA_CUDA(launch(k_dcgs_dots, dcgs_dot_grid(), 256, 0, s, sel_basis(lz, true, 1), lz->st.p, lz->n, Rmax, lz->V.p, w,
                   lz->partial.p, lz->coef.p, lz->tk_dots.p));
  const dim3 gu((unsigned)((lz->n + kUpdCols - 1) / kUpdCols), kUpdGroups);
  RIGA_CUDA(launch(k_dcgs_upd, gu, 256, 0, s, sel_basis(lz, false, 1), lz->st.p, lz->n, lz->ld, Rmax, lz->coef.p,
                   lz->upart.p, w, lz->vt.p, lz->r.p, lz->tk_upd.p, lz->cpl.p));
  RIGA_CUDA(cudaEventRecord(lz->ev1, s));
  lz->ev_valid = true;
  count_launch(2);
  return RIGA_OK;
}

int riga_lanczos_project_locked(riga_lanczos* lz, double* x, double* mx, int passes) {
  RIGA_CHECK_ARG(lz && x && mx, "null arg");
  if (!lz->nlocked) return RIGA_OK;
  DeviceGuard g(lz->ctx->device);
  RIGA_TRY(push_state(lz, lz->k, lz->k, 0.0));
  return cgs_passes(lz, sel_locked(lz, true), sel_locked(lz, false), sel_locked(lz, true), x, mx, passes,
                    lz->nlocked);
}

int riga_lanczos_gram(riga_lanczos* lz, double* G) {
  RIGA_CHECK_ARG(lz && G, "null arg");
  DeviceGuard g(lz->ctx->device);
  cudaStream_t s = lz->ctx->stream;
  const int64_t k = lz->k;
  if (!k) return RIGA_OK;
  // G[i][j] = V[i] . MV[j]: row V[i] against MV[:k] (locked rows excluded)
  const int64_t saved = lz->nlocked;
  lz->nlocked = 0;
  RIGA_TRY(push_state(lz, k, k, 0.0));
  lz->nlocked = saved;
  const RowSel dots = sel_basis(lz, true, 0);
  const int64_t Rmax = lz->max_dim + 1 + lz->cap;
  for (int64_t i = 0; i < k; ++i) {
    k_cgs_dots<<<kDotGrid, 256, 0, s>>>(dots, lz->st.p, lz->n, Rmax, lz->V.p + i * lz->ld, lz->partial.p,
                                        lz->coef.p, lz->tk_dots.p);
    count_launch();
    RIGA_CUDA(cudaMemcpyAsync(G + i * k, lz->coef.p, k * 8, cudaMemcpyDeviceToHost, s));
  }
  RIGA_CUDA(stream_sync(s));
  return RIGA_OK;
}

int riga_lanczos_bytes(riga_lanczos* lz, int64_t* bytes) {
  RIGA_CHECK_ARG(lz && bytes, "null arg");
  const DevBuf<double>* bufs[] = {&lz->V, &lz->MV, &lz->L, &lz->LM, &lz->w, &lz->r, &lz->Mr, &lz->bp, &lz->coef,
                                  &lz->partial, &lz->upart, &lz->cpl, &lz->Wd, &lz->outs, &lz->dscratch, &lz->vt,
                                  &lz->mvt, &lz->kt1, &lz->kt2, &lz->lk_part, &lz->lk_C, &lz->lk_G, &lz->lk_nrm,
                                  &lz->lk_Xt, &lz->lk_MXt};
  int64_t b = 0;
  for (const DevBuf<double>* d : bufs) b += (int64_t)d->n * 8;
  *bytes = b;
  return RIGA_OK;
}

int riga_lanczos_basis(riga_lanczos* lz, double** V, double** MV, int64_t* ld) {
  RIGA_CHECK_ARG(lz, "null arg");
  if (V) *V = lz->V.p;
  if (MV) *MV = lz->MV.p;
  if (ld) *ld = lz->ld;
  return RIGA_OK;
}

}  // extern "C"
