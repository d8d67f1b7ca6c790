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
// Reductions are two-phase with a fixed summation order (bitwise
// reproducible run to run).
#include <algorithm>
#include <cmath>
#include <cstring>

#include "internal.h"
#include "kernels.cuh"
#include "prof.h"

namespace riga {

constexpr int kChunk = 512;  // columns per CTA in the tall-skinny GEMV

struct Rows {  // up to two row blocks of one GEMV (basis + locked set)
  const double* a;
  int64_t na;
  const double* b;
  int64_t nb;
  int64_t ld;
};

// partial[blk * R + i] = sum_{c in chunk(blk)} row_i[c] * x[c],  R = na + nb
__global__ void __launch_bounds__(256) k_gemv_t(Rows A, int64_t n, const double* __restrict__ x,
                                                double* __restrict__ partial) {
  __shared__ double xs[kChunk];
  const int64_t c0 = (int64_t)blockIdx.x * kChunk;
  const int cn = (int)imin(kChunk, n - c0);
  for (int c = threadIdx.x; c < kChunk; c += blockDim.x) xs[c] = c < cn ? x[c0 + c] : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t R = A.na + A.nb;
  for (int64_t i = w; i < R; i += nw) {
    const double* row = (i < A.na ? A.a + i * A.ld : A.b + (i - A.na) * A.ld) + c0;
    double acc = 0.0;
    if (cn == kChunk) {
      const double2* r2 = reinterpret_cast<const double2*>(row);
#pragma unroll 4
      for (int c = lane; c < kChunk / 2; c += 32) {
        double2 v = __ldg(r2 + c);
        acc = fma(v.x, xs[2 * c], acc);
        acc = fma(v.y, xs[2 * c + 1], acc);
      }
    } else {
      for (int c = lane; c < cn; c += 32) acc = fma(row[c], xs[c], acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) partial[blockIdx.x * R + i] = acc;
  }
}

// coef[i] = sum_b partial[b * R + i]   (fixed order)
__global__ void k_reduce_rows(int64_t R, int nblk, const double* __restrict__ partial,
                              double* __restrict__ coef) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= R) return;
  double s = 0.0;
  for (int b = 0; b < nblk; ++b) s += partial[(int64_t)b * R + i];
  coef[i] = s;
}

// y[c] -= sum_i row_i[c] * coef[i]  over both row blocks; optionally also
// y2[c] -= sum_i row2_i[c] * coef[i] (the M-images, for locked projections)
__global__ void __launch_bounds__(256) k_gemv_n(Rows A, int64_t n, const double* __restrict__ coef,
                                                double* __restrict__ y, Rows A2,
                                                double* __restrict__ y2) {
  extern __shared__ double cs[];
  const int64_t R = A.na + A.nb;
  for (int64_t i = threadIdx.x; i < R; i += blockDim.x) cs[i] = coef[i];
  __syncthreads();
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  double acc = 0.0, acc2 = 0.0;
  int64_t i = 0;
  for (; i + 4 <= A.na; i += 4) {
    double v0 = __ldg(A.a + (i + 0) * A.ld + c), v1 = __ldg(A.a + (i + 1) * A.ld + c);
    double v2 = __ldg(A.a + (i + 2) * A.ld + c), v3 = __ldg(A.a + (i + 3) * A.ld + c);
    acc = fma(v0, cs[i], acc);
    acc = fma(v1, cs[i + 1], acc);
    acc = fma(v2, cs[i + 2], acc);
    acc = fma(v3, cs[i + 3], acc);
  }
  for (; i < A.na; ++i) acc = fma(__ldg(A.a + i * A.ld + c), cs[i], acc);
  for (int64_t j = 0; j < A.nb; ++j) acc = fma(__ldg(A.b + j * A.ld + c), cs[A.na + j], acc);
  y[c] -= acc;
  if (y2) {
    for (int64_t q = 0; q < A2.na; ++q) acc2 = fma(__ldg(A2.a + q * A2.ld + c), cs[q], acc2);
    for (int64_t j = 0; j < A2.nb; ++j) acc2 = fma(__ldg(A2.b + j * A2.ld + c), cs[A2.na + j], acc2);
    y2[c] -= acc2;
  }
}

// scal[0] = <a, b>, scal[1] = <c, d> (two dots in one pass), deterministic
__global__ void k_dot2(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                       const double* __restrict__ c, const double* __restrict__ d,
                       double* __restrict__ partial, unsigned* __restrict__ ticket,
                       double* __restrict__ out) {
  __shared__ double red[32];
  __shared__ bool last;
  double s0 = 0.0, s1 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    s0 = fma(a[i], b[i], s0);
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

// r = w - alpha v - sum_{i in [clo, k)} cpl[i] V[i]     (alpha = scal[0])
__global__ void k_residual(int64_t n, const double* __restrict__ w, const double* __restrict__ v,
                           const double* __restrict__ scal, const double* __restrict__ V,
                           int64_t ld, int64_t clo, int64_t k, const double* __restrict__ cpl,
                           double* __restrict__ r) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  double alpha = scal[0];
  double x = w[c] - alpha * v[c];
  if (clo < k) {
    double acc = 0.0;
    for (int64_t i = clo; i < k; ++i) acc = fma(V[i * ld + c], cpl[i], acc);
    x -= acc;
  }
  r[c] = x;
}

// dst = src * (1 / sqrt(s))  for two vector pairs, s = scal[idx]
__global__ void k_normalize2(int64_t n, const double* __restrict__ scal, int idx,
                             const double* __restrict__ a, double* __restrict__ da,
                             const double* __restrict__ b, double* __restrict__ db) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  double nrm = sqrt(fmax(scal[idx], 0.0));
  da[c] = a[c] / nrm;
  db[c] = b[c] / nrm;
}

// X[q][c] = sum_i W[i + q*k] * V[i][c]  for q < c_cnt (W column-major k x c)
template <int NQ>
__global__ void __launch_bounds__(256) k_lift(int64_t n, const double* __restrict__ V, int64_t ld,
                                              int64_t k, const double* __restrict__ W,
                                              int64_t q0, int64_t qn, double* __restrict__ X,
                                              int64_t ldx) {
  extern __shared__ double ws[];  // k * NQ
  for (int64_t t = threadIdx.x; t < k * NQ; t += blockDim.x) {
    int64_t i = t % k, q = t / k;
    ws[t] = (q0 + q < qn) ? W[(q0 + q) * k + i] : 0.0;
  }
  __syncthreads();
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  for (int64_t i = 0; i < k; ++i) {
    double v = __ldg(V + i * ld + c);
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = fma(ws[q * k + i], v, acc[q]);
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q)
    if (q0 + q < qn) X[(q0 + q) * ldx + c] = acc[q];
}

}  // namespace riga

using namespace riga;

struct riga_lanczos {
  riga_ctx* ctx = nullptr;
  riga_system* sys = nullptr;
  riga_factor* op = nullptr;
  int64_t n = 0, ld = 0, max_dim = 0, k = 0;
  int64_t nlocked = 0, cap = 0;
  DevBuf<double> V, MV, L, LM, w, r, Mr, coef, partial, scal, cpl, Wd, tmp;
  double* hbuf = nullptr;  // pinned readback
  int nblk = 0;
};

namespace {

int grow_locked(riga_lanczos* lz, int64_t need) {
  if (need <= lz->cap) return RIGA_OK;
  int64_t cap = std::max<int64_t>(8, lz->cap);
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
  // coefficient / partial buffers sized for basis + locked rows
  int64_t R = lz->max_dim + 1 + cap;
  RIGA_TRY(lz->coef.alloc(R, s));
  RIGA_TRY(lz->partial.alloc((int64_t)lz->nblk * R, s));
  return RIGA_OK;
}

// r -= V[:kk]^T (MV[:kk] r) + L^T (LM r), `passes` times (CGS2 when 2)
int cgs(riga_lanczos* lz, int64_t kk, double* r, int passes) {
  cudaStream_t s = lz->ctx->stream;
  int64_t R = kk + lz->nlocked;
  if (R == 0) return RIGA_OK;
  Rows dots{lz->MV.p, kk, lz->LM.p, lz->nlocked, lz->ld};
  Rows upd{lz->V.p, kk, lz->L.p, lz->nlocked, lz->ld};
  Rows none{nullptr, 0, nullptr, 0, lz->ld};
  for (int p = 0; p < passes; ++p) {
    ProfScope prof(kProfCgs, s, 2.0 * R * lz->n * 8.0);
    k_gemv_t<<<lz->nblk, 256, 0, s>>>(dots, lz->n, r, lz->partial.p); count_launch();
    k_reduce_rows<<<(unsigned)((R + 255) / 256), 256, 0, s>>>(R, lz->nblk, lz->partial.p, lz->coef.p); count_launch();
    k_gemv_n<<<(unsigned)((lz->n + 255) / 256), 256, R * 8, s>>>(upd, lz->n, lz->coef.p, r, none,
                                                                 nullptr); count_launch();
  }
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

// y = M x, or a copy for the Euclidean inner product (mass == NULL)
int mass_apply(riga_lanczos* lz, const double* x, double* y) {
  cudaStream_t s = lz->ctx->stream;
  if (lz->sys) return system_spmv(lz->sys, s, 1, 0.0, x, y);
  RIGA_CUDA(cudaMemcpyAsync(y, x, lz->n * 8, cudaMemcpyDeviceToDevice, s));
  return RIGA_OK;
}

int read_scal(riga_lanczos* lz, int count) {
  cudaStream_t s = lz->ctx->stream;
  RIGA_CUDA(cudaMemcpyAsync(lz->hbuf, lz->scal.p, count * 8, cudaMemcpyDeviceToHost, s));
  RIGA_CUDA(cudaStreamSynchronize(s));
  return RIGA_OK;
}

int dot2(riga_lanczos* lz, const double* a, const double* b, const double* c, const double* d,
         int slot) {
  cudaStream_t s = lz->ctx->stream;
  ProfScope prof(kProfVec, s, 32.0 * lz->n);
  int blocks = (int)std::min<int64_t>(296, (lz->n + 255) / 256);
  double* scratch = lz->scal.p + 16;
  k_dot2<<<blocks, 256, 0, s>>>(lz->n, a, b, c, d, scratch,
                                reinterpret_cast<unsigned*>(lz->scal.p + 15), lz->scal.p + slot); count_launch();
  RIGA_CUDA(cudaGetLastError());
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
  lz->sys = mass;
  lz->n = n;
  lz->ld = (n + 3) / 4 * 4;
  lz->max_dim = std::min<int64_t>(max_dim, n);
  lz->nblk = (int)((lz->n + kChunk - 1) / kChunk);
  int64_t rows = lz->max_dim + 1;
  cudaStream_t cs = ctx->stream;
  RIGA_TRY(lz->V.alloc(rows * lz->ld, cs));
  RIGA_TRY(lz->MV.alloc(rows * lz->ld, cs));
  RIGA_CUDA(cudaMemsetAsync(lz->V.p, 0, rows * lz->ld * 8, ctx->stream));
  RIGA_CUDA(cudaMemsetAsync(lz->MV.p, 0, rows * lz->ld * 8, ctx->stream));
  RIGA_TRY(lz->w.alloc(lz->ld, cs));
  RIGA_TRY(lz->r.alloc(lz->ld, cs));
  RIGA_TRY(lz->Mr.alloc(lz->ld, cs));
  RIGA_TRY(lz->tmp.alloc(lz->ld, cs));
  RIGA_TRY(lz->scal.alloc(16 + 2 * 296 + 16, cs));
  RIGA_CUDA(cudaMemsetAsync(lz->scal.p, 0, lz->scal.n * 8, ctx->stream));
  RIGA_TRY(lz->cpl.alloc(rows, cs));
  RIGA_TRY(grow_locked(lz.get(), 8));
  RIGA_CUDA(cudaMallocHost(&lz->hbuf, std::max<int64_t>(64, 3 * rows + 8) * 8));
  RIGA_CUDA(cudaStreamSynchronize(ctx->stream));
  *out = lz.release();
  return RIGA_OK;
}

int riga_lanczos_destroy(riga_lanczos* lz) {
  if (!lz) return RIGA_OK;
  DeviceGuard g(lz->ctx->device);
  cudaStreamSynchronize(lz->ctx->stream);
  if (lz->hbuf) cudaFreeHost(lz->hbuf);
  delete lz;
  return RIGA_OK;
}

int riga_lanczos_set_operator(riga_lanczos* lz, riga_factor* f) {
  RIGA_CHECK_ARG(lz && f, "null arg");
  RIGA_CHECK_ARG(f->sym->h.n == lz->n, "operator dimension mismatch");
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
  RIGA_CUDA(cudaMemcpyAsync(lz->r.p, r_host, lz->n * 8, cudaMemcpyHostToDevice, s));
  RIGA_TRY(mass_apply(lz, lz->r.p, lz->Mr.p));
  RIGA_TRY(dot2(lz, lz->r.p, lz->Mr.p, lz->r.p, lz->Mr.p, 0));
  RIGA_TRY(read_scal(lz, 1));
  if (!(std::sqrt(std::max(lz->hbuf[0], 0.0)) > 0.0)) {
    set_error("start vector has zero mass norm");
    return RIGA_BAD_ARG;
  }
  double* vk = lz->V.p + lz->k * lz->ld;
  double* mvk = lz->MV.p + lz->k * lz->ld;
  k_normalize2<<<(unsigned)((lz->n + 255) / 256), 256, 0, s>>>(lz->n, lz->scal.p, 0, lz->r.p, vk,
                                                               lz->Mr.p, mvk); count_launch();
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

int riga_lanczos_fresh(riga_lanczos* lz, const double* r_host, int* accepted) {
  RIGA_CHECK_ARG(lz && r_host && accepted, "null arg");
  DeviceGuard g(lz->ctx->device);
  cudaStream_t s = lz->ctx->stream;
  RIGA_CUDA(cudaMemcpyAsync(lz->r.p, r_host, lz->n * 8, cudaMemcpyHostToDevice, s));
  RIGA_TRY(mass_apply(lz, lz->r.p, lz->Mr.p));
  RIGA_TRY(dot2(lz, lz->r.p, lz->Mr.p, lz->r.p, lz->Mr.p, 4));  // ref norm^2 -> scal[4]
  RIGA_TRY(cgs(lz, lz->k, lz->r.p, 2));
  RIGA_TRY(mass_apply(lz, lz->r.p, lz->Mr.p));
  RIGA_TRY(dot2(lz, lz->r.p, lz->Mr.p, lz->r.p, lz->Mr.p, 0));
  RIGA_TRY(read_scal(lz, 6));
  double ref = std::sqrt(std::max(lz->hbuf[4], 0.0));
  double nrm = std::sqrt(std::max(lz->hbuf[0], 0.0));
  *accepted = nrm > 1e-8 * std::max(ref, 1e-300);
  if (*accepted) {
    double* vk = lz->V.p + lz->k * lz->ld;
    double* mvk = lz->MV.p + lz->k * lz->ld;
    k_normalize2<<<(unsigned)((lz->n + 255) / 256), 256, 0, s>>>(lz->n, lz->scal.p, 0, lz->r.p, vk,
                                                                 lz->Mr.p, mvk); count_launch();
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

}  // extern "C"

namespace {
// Second half of a step once w = H v is in lz->w (ref step :244-267).
// Returns RIGA_BREAKDOWN when beta is below the relative threshold.
int step_core(riga_lanczos* lz, int64_t clo, double breakdown_tol, double* a_out, double* b_out,
              double* w_out) {
  cudaStream_t s = lz->ctx->stream;
  const int64_t n = lz->n, ld = lz->ld, k = lz->k;
  const unsigned g1 = (unsigned)((n + 255) / 256);
  const double* v = lz->V.p + k * ld;
  const double* Mv = lz->MV.p + k * ld;
  RIGA_TRY(dot2(lz, Mv, lz->w.p, lz->w.p, lz->w.p, 0));  // alpha, |w|^2
  k_residual<<<g1, 256, 0, s>>>(n, lz->w.p, v, lz->scal.p, lz->V.p, ld, clo, k, lz->cpl.p, lz->r.p); count_launch();
  RIGA_TRY(cgs(lz, k + 1, lz->r.p, 2));
  RIGA_TRY(mass_apply(lz, lz->r.p, lz->Mr.p));
  RIGA_TRY(dot2(lz, lz->r.p, lz->Mr.p, lz->r.p, lz->Mr.p, 2));  // beta^2
  RIGA_TRY(read_scal(lz, 4));
  const double a = lz->hbuf[0], wn = std::sqrt(std::max(lz->hbuf[1], 0.0));
  const double b = std::sqrt(std::max(lz->hbuf[2], 0.0));
  *a_out = a;
  *w_out = wn;
  *b_out = b;
  lz->k = k + 1;
  if (b <= std::max(breakdown_tol, 1e-13 * wn)) return RIGA_BREAKDOWN;
  k_normalize2<<<g1, 256, 0, s>>>(n, lz->scal.p, 2, lz->r.p, lz->V.p + (k + 1) * ld, lz->Mr.p,
                                  lz->MV.p + (k + 1) * ld); count_launch();
  lz->hbuf[8] = b;  // next step's coupling: beta e_k
  RIGA_CUDA(cudaMemcpyAsync(lz->cpl.p + k, lz->hbuf + 8, 8, cudaMemcpyHostToDevice, s));
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

int first_coupling(riga_lanczos* lz, const double* coupling_host, int64_t* clo) {
  *clo = lz->k;
  if (coupling_host && lz->k > 0) {
    RIGA_CUDA(cudaMemcpyAsync(lz->cpl.p, coupling_host, lz->k * 8, cudaMemcpyHostToDevice,
                              lz->ctx->stream));
    *clo = 0;
  }
  return RIGA_OK;
}
}  // namespace

extern "C" {

int riga_lanczos_extend(riga_lanczos* lz, int64_t limit, const double* coupling_host,
                        double breakdown_tol, double* alpha, double* beta, double* wnorm,
                        int64_t* steps) {
  RIGA_CHECK_ARG(lz && alpha && beta && wnorm && steps, "null arg");
  RIGA_CHECK_ARG(lz->op, "no operator set");
  DeviceGuard g(lz->ctx->device);
  cudaStream_t s = lz->ctx->stream;
  limit = std::min(limit, lz->max_dim);
  *steps = 0;
  int64_t clo;
  RIGA_TRY(first_coupling(lz, coupling_host, &clo));
  int64_t i = 0;
  while (lz->k < limit) {
    const int64_t k = lz->k;
    RIGA_TRY(factor_solve(lz->op, s, lz->MV.p + k * lz->ld, lz->w.p));  // w = H v
    int rc = step_core(lz, clo, breakdown_tol, alpha + i, beta + i, wnorm + i);
    ++i;
    *steps = i;
    if (rc) return rc;
    clo = k;
  }
  return RIGA_OK;
}

int riga_lanczos_step_given(riga_lanczos* lz, const double* w_dev, const double* coupling_host,
                            double breakdown_tol, double* alpha, double* beta, double* wnorm) {
  RIGA_CHECK_ARG(lz && w_dev && alpha && beta && wnorm, "null arg");
  RIGA_CHECK_ARG(lz->k < lz->max_dim, "basis is full");
  DeviceGuard g(lz->ctx->device);
  int64_t clo;
  RIGA_TRY(first_coupling(lz, coupling_host, &clo));
  RIGA_CUDA(cudaMemcpyAsync(lz->w.p, w_dev, lz->n * 8, cudaMemcpyDeviceToDevice, lz->ctx->stream));
  return step_core(lz, clo, breakdown_tol, alpha, beta, wnorm);
}

static int lift_rows(riga_lanczos* lz, const double* Vb, int64_t k, const double* Wd, int64_t c,
                     double* X) {
  cudaStream_t s = lz->ctx->stream;
  ProfScope prof(kProfLift, s, 8.0 * (double)k * lz->n * ((c + 7) / 8));
  const unsigned g1 = (unsigned)((lz->n + 255) / 256);
  for (int64_t q0 = 0; q0 < c; q0 += 8) {
    k_lift<8><<<g1, 256, k * 8 * 8, s>>>(lz->n, Vb, lz->ld, k, Wd, q0, c, X, lz->ld); count_launch();
  }
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

int riga_lanczos_lift(riga_lanczos* lz, const double* W_host, int64_t c, double* X, double* MX) {
  RIGA_CHECK_ARG(lz && W_host && X && MX && c >= 0, "null arg");
  if (c == 0) return RIGA_OK;
  DeviceGuard g(lz->ctx->device);
  cudaStream_t s = lz->ctx->stream;
  int64_t k = lz->k;
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
  int64_t k = lz->k, ld = lz->ld;
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
    RIGA_CUDA(cudaStreamSynchronize(s));
  }
  // keep the pending direction: row k -> row c
  if (c != k) {
    RIGA_CUDA(cudaMemcpyAsync(lz->V.p + c * ld, lz->V.p + k * ld, ld * 8, cudaMemcpyDeviceToDevice, s));
    RIGA_CUDA(cudaMemcpyAsync(lz->MV.p + c * ld, lz->MV.p + k * ld, ld * 8, cudaMemcpyDeviceToDevice, s));
  }
  lz->k = c;
  return RIGA_OK;
}

int riga_lanczos_project_locked(riga_lanczos* lz, double* x, double* mx, int passes) {
  RIGA_CHECK_ARG(lz && x && mx, "null arg");
  if (!lz->nlocked) return RIGA_OK;
  DeviceGuard g(lz->ctx->device);
  cudaStream_t s = lz->ctx->stream;
  int64_t R = lz->nlocked;
  Rows dots{lz->LM.p, R, nullptr, 0, lz->ld};
  Rows upd{lz->L.p, R, nullptr, 0, lz->ld};
  Rows upd2{lz->LM.p, R, nullptr, 0, lz->ld};
  for (int p = 0; p < passes; ++p) {
    k_gemv_t<<<lz->nblk, 256, 0, s>>>(dots, lz->n, x, lz->partial.p); count_launch();
    k_reduce_rows<<<(unsigned)((R + 255) / 256), 256, 0, s>>>(R, lz->nblk, lz->partial.p, lz->coef.p); count_launch();
    k_gemv_n<<<(unsigned)((lz->n + 255) / 256), 256, R * 8, s>>>(upd, lz->n, lz->coef.p, x, upd2, mx); count_launch();
  }
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

int riga_lanczos_gram(riga_lanczos* lz, double* G) {
  RIGA_CHECK_ARG(lz && G, "null arg");
  DeviceGuard g(lz->ctx->device);
  cudaStream_t s = lz->ctx->stream;
  int64_t k = lz->k;
  if (!k) return RIGA_OK;
  Rows dots{lz->MV.p, k, nullptr, 0, lz->ld};
  std::vector<double> row(k);
  for (int64_t i = 0; i < k; ++i) {
    k_gemv_t<<<lz->nblk, 256, 0, s>>>(dots, lz->n, lz->V.p + i * lz->ld, lz->partial.p); count_launch();
    k_reduce_rows<<<(unsigned)((k + 255) / 256), 256, 0, s>>>(k, lz->nblk, lz->partial.p, lz->coef.p); count_launch();
    RIGA_CUDA(cudaMemcpyAsync(G + i * k, lz->coef.p, k * 8, cudaMemcpyDeviceToHost, s));
    RIGA_CUDA(cudaStreamSynchronize(s));
  }
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
