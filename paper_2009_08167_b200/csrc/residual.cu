// Eigenpair residual norms on the device (the north-star residual gate) and
// the batched multi-RHS solve used to refine pairs that fail it.
//
//  riga_residuals        <- the residual loop of solve_spectrum
//                           ref eigensolver.py:784-792 (K x, M x per pair),
//                           evaluated for every returned pair as
//                           ||K x - lam M x|| / (|lam| ||M x||)  (north_star)
//                           and ||K x - lam M x|| / ||K x||      (reference)
//  riga_spmv_many        <- mass_matvec over the rows of a block (ref sparsela.py:280-290)
//  riga_factor_solve_many <- solve_fb over the columns of a block
//                           ref sparsela.py:265-277 (SURVEY §8b solve(fact, x, nrhs))
//
// One pass over the shared CSR pattern of K and M serves NV vectors: each
// 16-lane row group loads (col, K, M) once per element and applies them to
// the NV vectors, accumulating K x and M x; lane 0 of the row folds
// r = Kx - lam Mx into three per-vector sums (|r|^2, |Mx|^2, |Kx|^2).  Row
// groups stride over the rows with a fixed grid, partial sums are reduced
// per CTA and then across CTAs in a fixed order: the result is
// bitwise-reproducible run to run (no floating-point atomics).
#include "internal.h"
#include "kernels.cuh"
#include "prof.h"

namespace riga {

constexpr int kResLanes = 16;
constexpr int kResThreads = 256;
constexpr int kResRows = kResThreads / kResLanes;  // row groups per CTA
constexpr int kResNV = 8;                          // vectors per pass

template <int NV>
__global__ void __launch_bounds__(kResThreads) k_resid(int64_t n, const int64_t* __restrict__ rp,
                                                       const int32_t* __restrict__ ci,
                                                       const double* __restrict__ K,
                                                       const double* __restrict__ M,
                                                       const double* __restrict__ X, int64_t ldx, int nv,
                                                       const double* __restrict__ lam,
                                                       double* __restrict__ partial) {
  const int sub = threadIdx.x % kResLanes;
  const int grp = threadIdx.x / kResLanes;
  double lv[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) lv[v] = v < nv ? lam[v] : 0.0;
  double acc[NV][3];
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v][0] = acc[v][1] = acc[v][2] = 0.0;
  // the row-group loop bound is CTA-uniform (base), so every lane reaches the width-16 shuffles
  for (int64_t base = (int64_t)blockIdx.x * kResRows; base < n; base += (int64_t)gridDim.x * kResRows) {
    const int64_t row = base + grp;
    const bool valid = row < n;
    double kx[NV], mx[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) kx[v] = mx[v] = 0.0;
    const int64_t e = valid ? rp[row + 1] : 0;
    for (int64_t q = (valid ? rp[row] : 0) + sub; q < e; q += kResLanes) {
      const double kv = __ldg(K + q), mv = __ldg(M + q);
      const int64_t c = __ldg(ci + q);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        if (v < nv) {
          const double x = __ldg(X + v * ldx + c);
          kx[v] = fma(kv, x, kx[v]);
          mx[v] = fma(mv, x, mx[v]);
        }
      }
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
#pragma unroll
      for (int o = kResLanes / 2; o > 0; o >>= 1) {
        kx[v] += __shfl_down_sync(0xffffffffu, kx[v], o, kResLanes);
        mx[v] += __shfl_down_sync(0xffffffffu, mx[v], o, kResLanes);
      }
    }
    if (sub == 0 && valid) {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const double r = kx[v] - lv[v] * mx[v];
        acc[v][0] = fma(r, r, acc[v][0]);
        acc[v][1] = fma(mx[v], mx[v], acc[v][1]);
        acc[v][2] = fma(kx[v], kx[v], acc[v][2]);
      }
    }
  }
  // CTA reduction in row-group order
  __shared__ double red[kResRows][NV * 3];
  if (sub == 0) {
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int j = 0; j < 3; ++j) red[grp][v * 3 + j] = acc[v][j];
  }
  __syncthreads();
  if (threadIdx.x < NV * 3) {
    double s = 0.0;
    for (int g = 0; g < kResRows; ++g) s += red[g][threadIdx.x];
    partial[(int64_t)blockIdx.x * NV * 3 + threadIdx.x] = s;
  }
}

// out[v*3 + j] = sum over CTAs (fixed order) of partial[b][v][j]
__global__ void k_resid_final(int nblocks, int nv, const double* __restrict__ partial, double* __restrict__ out) {
  const int t = threadIdx.x;
  if (t >= nv * 3) return;
  double s = 0.0;
  for (int b = 0; b < nblocks; ++b) s += partial[(int64_t)b * kResNV * 3 + t];
  out[t] = s;
}

int residual_norms(riga_system* sys, cudaStream_t s, const double* X, int64_t ldx, int64_t nvec,
                   const double* lam_host, double* out_host) {
  const int64_t n = sys->n;
  int dev = 0;
  RIGA_CUDA(cudaGetDevice(&dev));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t groups = (n + kResRows - 1) / kResRows;
  const int nblocks = (int)std::min<int64_t>(groups, (int64_t)sms * 8);
  DevBuf<double> lam, part, out;
  RIGA_TRY(lam.upload(lam_host, nvec, s));
  RIGA_TRY(part.alloc((size_t)nblocks * kResNV * 3, s));
  RIGA_TRY(out.alloc((size_t)nvec * 3, s));
  for (int64_t v0 = 0; v0 < nvec; v0 += kResNV) {
    const int nv = (int)std::min<int64_t>(kResNV, nvec - v0);
    k_resid<kResNV><<<nblocks, kResThreads, 0, s>>>(n, sys->rowptr.p, sys->colidx.p, sys->K.p, sys->M.p,
                                                     X + v0 * ldx, ldx, nv, lam.p + v0, part.p);
    count_launch();
    k_resid_final<<<1, 32, 0, s>>>(nblocks, nv, part.p, out.p + v0 * 3);
    count_launch();
  }
  RIGA_CUDA(cudaGetLastError());
  RIGA_CUDA(cudaMemcpyAsync(out_host, out.p, nvec * 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
  RIGA_CUDA(stream_sync(s));
  return RIGA_OK;
}

}  // namespace riga

using namespace riga;

extern "C" {

int riga_residuals(riga_ctx* ctx, riga_system* sys, const double* X_dev, int64_t ldx, int64_t nvec,
                   const double* lam_host, double* out_host) {
  RIGA_CHECK_ARG(sys && (X_dev || nvec == 0) && (lam_host || nvec == 0) && (out_host || nvec == 0), "null arg");
  RIGA_CHECK_ARG(nvec >= 0 && (nvec == 0 || ldx >= sys->n), "bad block shape");
  if (nvec == 0) return RIGA_OK;
  riga_ctx* c = ctx ? ctx : sys->ctx;
  DeviceGuard g(c->device);
  return residual_norms(sys, c->stream, X_dev, ldx, nvec, lam_host, out_host);
}

int riga_spmv_many(riga_ctx* ctx, riga_system* sys, int which, double sigma, const double* X_dev, int64_t ldx,
                   int64_t nvec, double* Y_dev, int64_t ldy) {
  RIGA_CHECK_ARG(sys && ((X_dev && Y_dev) || nvec == 0), "null arg");
  RIGA_CHECK_ARG(nvec >= 0 && (nvec == 0 || (ldx >= sys->n && ldy >= sys->n)), "bad block shape");
  riga_ctx* c = ctx ? ctx : sys->ctx;
  DeviceGuard g(c->device);
  for (int64_t j = 0; j < nvec; ++j) RIGA_TRY(system_spmv(sys, c->stream, which, sigma, X_dev + j * ldx, Y_dev + j * ldy));
  return RIGA_OK;
}

int riga_factor_solve_many(riga_ctx* ctx, riga_factor* f, const double* B_dev, int64_t ldb, int64_t nrhs,
                           double* X_dev, int64_t ldx) {
  RIGA_CHECK_ARG(f && ((B_dev && X_dev) || nrhs == 0), "null arg");
  const int64_t n = f->sym->h.n;
  RIGA_CHECK_ARG(nrhs >= 0 && (nrhs == 0 || (ldb >= n && ldx >= n)), "bad block shape");
  if (nrhs == 0) return RIGA_OK;
  riga_ctx* c = ctx ? ctx : f->ctx;
  DeviceGuard g(c->device);
  cudaStream_t s = c->stream;
  if (s != f->ctx->stream) {
    // the factor's own stream finished building it (and its last solve)
    cudaEvent_t ev;
    RIGA_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    RIGA_CUDA(cudaEventRecord(ev, f->ctx->stream));
    RIGA_CUDA(cudaStreamWaitEvent(s, ev, 0));
    cudaEventDestroy(ev);
  }
  for (int64_t j = 0; j < nrhs; ++j) RIGA_TRY(factor_solve(f, s, B_dev + j * ldb, X_dev + j * ldx, false, true));
  if (s != f->ctx->stream) {
    // later work on the factor's stream sees these solves' workspace use done
    cudaEvent_t ev;
    RIGA_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    RIGA_CUDA(cudaEventRecord(ev, s));
    RIGA_CUDA(cudaStreamWaitEvent(f->ctx->stream, ev, 0));
    cudaEventDestroy(ev);
  }
  return RIGA_OK;
}

}  // extern "C"
