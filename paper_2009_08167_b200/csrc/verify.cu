// Tensor-product evaluation kernels of the eigen-error study (verify.py).
//
//  riga_tp_contract   <- ErrorEvaluator._contract        ref verify.py:218-225
//                        (u_h or one partial derivative on the tensor Gauss
//                        grid: one banded contraction per direction)
//  riga_tp_reduce     <- ErrorEvaluator.integrate applied to (u_h - u)^2 and
//                        u_h u                            ref verify.py:227-255
//                        with the exact mode u = prod_t sqrt(2) sin(k_t pi x_t)
//                        (ref :105-133) formed on the fly
//  riga_row_dots      <- the c^T M c normalisations       ref verify.py:296-300
//
// A collocation matrix has p + 1 non-zeros per quadrature point, so a
// direction's contraction is a banded gather (HBM-bound: read the tensor
// once, write it once), not a dense GEMM.  Layouts are (outer, axis, inner)
// row-major; batch members are the leading part of `outer`.  All reductions
// run in a fixed order (no floating-point atomics): results are bitwise
// reproducible.
#include "internal.h"
#include "kernels.cuh"
#include "prof.h"

namespace riga {

constexpr double kPi = 3.141592653589793238462643383279502884;

// out[o, q, i] = s[o / opb] * sum_j vals[q p1 + j] * in[o, first[q] + j - off, i]; indices outside
// [0, n_in) read as zero (the Dirichlet layers of the embedded coefficient tensor)
__global__ void __launch_bounds__(256) k_tp_axis(const double* __restrict__ in, double* __restrict__ out,
                                                 int64_t outer, int64_t n_in, int64_t n_out, int64_t inner,
                                                 int p1, int off, const int32_t* __restrict__ first,
                                                 const double* __restrict__ vals,
                                                 const double* __restrict__ bscale, int64_t opb) {
  const int64_t total = outer * n_out * inner;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % inner, oq = t / inner;
    const int64_t q = oq % n_out, o = oq / n_out;
    const double* src = in + o * n_in * inner + i;
    const double* v = vals + q * p1;
    const int64_t j0 = (int64_t)first[q] - off;
    double acc = 0.0;
    for (int j = 0; j < p1; ++j) {
      const int64_t r = j0 + j;
      if (r >= 0 && r < n_in) acc = fma(v[j], src[r * inner], acc);
    }
    out[t] = bscale ? acc * bscale[o / opb] : acc;
  }
}

// F[(b, q)] = sqrt(2) sin(k_b pi x_q), or sqrt(2) k_b pi cos(k_b pi x_q) for the derivative direction
__global__ void k_tp_factors(const double* __restrict__ x, int64_t nq, const int32_t* __restrict__ kidx,
                             int kstride, int64_t nbatch, int deriv, double* __restrict__ F) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nbatch * nq) return;
  const int64_t b = t / nq, q = t % nq;
  const double k = (double)kidx[b * kstride];
  const double arg = k * kPi * x[q];
  F[t] = deriv ? sqrt(2.0) * k * kPi * cos(arg) : sqrt(2.0) * sin(arg);
}

// R[b, row] = sum_x w_x f(g G[b, row, x], E), E = rowf[b, row] * Fx[b, x]; mode 0: f = (g G - E)^2,
// mode 1: f = G E, mode 2: f = G (plain quadrature).  One warp per (b, row), lanes stride x, fixed-order shuffle reduction.
// rowf[b, row] = prod over the slower directions of their factors (rows = q_z * nq_y + q_y).
__global__ void __launch_bounds__(256) k_tp_rowreduce(const double* __restrict__ G, int64_t nbatch, int64_t rows,
                                                      int64_t nx, int64_t ny, const double* __restrict__ Fx,
                                                      const double* __restrict__ Fy,
                                                      const double* __restrict__ Fz, int64_t nz,
                                                      const double* __restrict__ wx,
                                                      const double* __restrict__ gsign, int mode,
                                                      double* __restrict__ R) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (w >= nbatch * rows) return;
  const int64_t b = w / rows, row = w % rows;
  double rf = 1.0;
  if (Fy) rf *= Fy[b * ny + row % ny];
  if (Fz) rf *= Fz[b * nz + row / ny];
  const double g = gsign ? gsign[b] : 1.0;
  const double* Gr = G + w * nx;
  const double* fx = Fx + b * nx;
  double acc = 0.0;
  for (int64_t x = lane; x < nx; x += 32) {
    const double e = rf * fx[x], u = g * Gr[x];
    const double d = mode == 0 ? (u - e) * (u - e) : mode == 1 ? Gr[x] * e : Gr[x];
    acc = fma(wx[x], d, acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) R[w] = acc;
}

// out[o] = sum_j w[j] R[o, j]: one warp per o
__global__ void __launch_bounds__(256) k_tp_wsum(const double* __restrict__ R, int64_t outer, int64_t n,
                                                 const double* __restrict__ w, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t o = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (o >= outer) return;
  double acc = 0.0;
  for (int64_t j = lane; j < n; j += 32) acc = fma(w[j], R[o * n + j], acc);
  acc = warp_sum(acc);
  if (lane == 0) out[o] = acc;
}

// out[v] = X[v, :] . Y[v, :]: one CTA per row, fixed-order block reduction
__global__ void __launch_bounds__(256) k_row_dots(const double* __restrict__ X, int64_t ldx,
                                                  const double* __restrict__ Y, int64_t ldy, int64_t n,
                                                  double* __restrict__ out) {
  __shared__ double red[32];
  const double* x = X + blockIdx.x * ldx;
  const double* y = Y + blockIdx.x * ldy;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc = fma(x[i], y[i], acc);
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

}  // namespace riga

using namespace riga;

extern "C" {

int riga_tp_contract(riga_ctx* ctx, const double* in_dev, double* out_dev, int64_t outer, int64_t n_in,
                     int64_t n_out, int64_t inner, int p1, int off, const int32_t* first_dev,
                     const double* vals_dev, const double* bscale_dev, int64_t outer_per_batch) {
  RIGA_CHECK_ARG(ctx && in_dev && out_dev && first_dev && vals_dev, "null arg");
  RIGA_CHECK_ARG(outer > 0 && n_in > 0 && n_out > 0 && inner > 0 && p1 > 0, "bad shape");
  RIGA_CHECK_ARG(!bscale_dev || outer_per_batch > 0, "bad batch stride");
  DeviceGuard g(ctx->device);
  const int64_t total = outer * n_out * inner;
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
  k_tp_axis<<<grid, 256, 0, ctx->stream>>>(in_dev, out_dev, outer, n_in, n_out, inner, p1, off, first_dev, vals_dev,
                                           bscale_dev, outer_per_batch);
  count_launch();
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

int riga_tp_reduce(riga_ctx* ctx, const double* G_dev, int64_t nbatch, int dim, const int64_t* nq_host,
                   const double* const* x_dev, const double* const* w_dev, const int32_t* kidx_dev, int deriv,
                   int mode, const double* gsign_dev, double* out_dev) {
  RIGA_CHECK_ARG(ctx && G_dev && nq_host && x_dev && w_dev && kidx_dev && out_dev, "null arg");
  RIGA_CHECK_ARG(dim >= 1 && dim <= 3 && nbatch > 0 && mode >= 0 && mode <= 2, "bad arg");
  DeviceGuard g(ctx->device);
  cudaStream_t st = ctx->stream;
  const int64_t nx = nq_host[0], ny = dim > 1 ? nq_host[1] : 1, nz = dim > 2 ? nq_host[2] : 1;
  const int64_t rows = ny * nz;
  DevBuf<double> F, R, R2;
  RIGA_TRY(F.alloc(nbatch * (nx + ny + nz), st));
  RIGA_TRY(R.alloc(nbatch * rows, st));
  double* Fx = F.p;
  double* Fy = dim > 1 ? Fx + nbatch * nx : nullptr;
  double* Fz = dim > 2 ? Fy + nbatch * ny : nullptr;
  double* Ft[3] = {Fx, Fy, Fz};
  for (int t = 0; t < dim; ++t) {
    const int64_t n = nbatch * nq_host[t];
    k_tp_factors<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x_dev[t], nq_host[t], kidx_dev + t, dim, nbatch,
                                                               deriv == t ? 1 : 0, Ft[t]);
    count_launch();
  }
  const int64_t warps = nbatch * rows;
  k_tp_rowreduce<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(G_dev, nbatch, rows, nx, ny, Fx, Fy, Fz, nz, w_dev[0],
                                                               gsign_dev, mode, R.p);
  count_launch();
  const double* cur = R.p;
  if (dim > 1) {  // y, then z
    RIGA_TRY(R2.alloc(nbatch * nz, st));
    k_tp_wsum<<<(unsigned)((nbatch * nz + 7) / 8), 256, 0, st>>>(cur, nbatch * nz, ny, w_dev[1],
                                                                 dim > 2 ? R2.p : out_dev);
    count_launch();
    cur = R2.p;
    if (dim > 2) {
      k_tp_wsum<<<(unsigned)((nbatch + 7) / 8), 256, 0, st>>>(cur, nbatch, nz, w_dev[2], out_dev);
      count_launch();
    }
  } else {
    RIGA_CUDA(cudaMemcpyAsync(out_dev, cur, nbatch * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

int riga_row_dots(riga_ctx* ctx, const double* X_dev, int64_t ldx, const double* Y_dev, int64_t ldy, int64_t n,
                  int64_t nvec, double* out_dev) {
  RIGA_CHECK_ARG(ctx && X_dev && Y_dev && out_dev && n > 0 && nvec > 0, "bad arg");
  DeviceGuard g(ctx->device);
  k_row_dots<<<(unsigned)nvec, 256, 0, ctx->stream>>>(X_dev, ldx, Y_dev, ldy, n, out_dev);
  count_launch();
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

}  // extern "C"
