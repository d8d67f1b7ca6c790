#include <cstdlib>
// Context, device CSR system (upload / Kronecker assembly), SpMV, dots.
//
//  riga_system_assemble_kron  <- kron_assemble   ref assembly.py:139-186
//  riga_spmv / riga_csr_spmv  <- mass_matvec     ref sparsela.py:280-290
#include <map>
#include <mutex>
#include <unordered_map>
#include <cstring>
#include <mutex>

#include "internal.h"
#include "kernels.cuh"
#include "prof.h"

namespace riga {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
const char* last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------------------
// Kronecker assembly: one thread per nonzero of the d-dimensional pattern.
// Row r = (iz, iy, ix) (x fastest); 1D rows have contiguous column ranges, so
// the nnz of row r enumerate (jz, jy, jx) lexicographically = sorted columns.
// Values reproduce scipy's evaluation order exactly (no FMA contraction):
//   2D: K = my*kx + ky*mx                       M = my*mx
//   3D: K = ((mz*my)*kx + (mz*ky)*mx) + (kz*my)*mx    M = (mz*my)*mx
// ---------------------------------------------------------------------------
struct Kron1D {
  const int64_t* rp;
  const int32_t* ci;
  const double* k;
  const double* m;
  int64_t n;
};

__global__ void k_kron_rowptr(int dim, Kron1D x, Kron1D y, Kron1D z, int64_t n, int64_t* rowlen) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  int64_t ix = r % x.n, t = r / x.n;
  int64_t len = x.rp[ix + 1] - x.rp[ix];
  if (dim >= 2) {
    int64_t iy = t % y.n;
    t /= y.n;
    len *= y.rp[iy + 1] - y.rp[iy];
    if (dim == 3) len *= z.rp[t + 1] - z.rp[t];
  }
  rowlen[r] = len;
}

__global__ void k_kron_values(int dim, Kron1D x, Kron1D y, Kron1D z, int64_t n,
                              const int64_t* __restrict__ rowptr, int32_t* __restrict__ colidx,
                              double* __restrict__ K, double* __restrict__ M) {
  // one warp per row; lanes stride over the row's entries
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (warp >= n) return;
  int64_t r = warp;
  int64_t ix = r % x.n, t = r / x.n, iy = 0, iz = 0;
  if (dim >= 2) {
    iy = t % y.n;
    iz = t / y.n;
  }
  int64_t lx = x.rp[ix + 1] - x.rp[ix];
  int64_t ly = dim >= 2 ? y.rp[iy + 1] - y.rp[iy] : 1;
  int64_t base = rowptr[r], len = rowptr[r + 1] - base;
  for (int64_t e = lane; e < len; e += 32) {
    int64_t ex = e % lx, et = e / lx;
    int64_t qx = x.rp[ix] + ex;
    double kx = x.k[qx], mx = x.m[qx];
    int64_t col = x.ci[qx];
    double kv, mv;
    if (dim == 1) {
      kv = kx;
      mv = mx;
    } else {
      int64_t ey = et % ly, ez = et / ly;
      int64_t qy = y.rp[iy] + ey;
      double ky = y.k[qy], my = y.m[qy];
      col += (int64_t)y.ci[qy] * x.n;
      if (dim == 2) {
        kv = __dadd_rn(__dmul_rn(my, kx), __dmul_rn(ky, mx));
        mv = __dmul_rn(my, mx);
      } else {
        int64_t qz = z.rp[iz] + ez;
        double kz = z.k[qz], mz = z.m[qz];
        col += (int64_t)z.ci[qz] * x.n * y.n;
        double mzmy = __dmul_rn(mz, my);
        kv = __dadd_rn(__dadd_rn(__dmul_rn(mzmy, kx), __dmul_rn(__dmul_rn(mz, ky), mx)),
                       __dmul_rn(__dmul_rn(kz, my), mx));
        mv = __dmul_rn(mzmy, mx);
      }
    }
    colidx[base + e] = (int32_t)col;
    K[base + e] = kv;
    M[base + e] = mv;
  }
}

// ---------------------------------------------------------------------------
// CSR SpMV, LANES threads per row, fixed reduction order (deterministic).
// mode 0: y = A x;  mode 1: y = (K - sigma M) x with A = K, B = M.
// U elements per lane per round: chosen so one round covers a typical row.
// ---------------------------------------------------------------------------
template <int LANES, int U, int MODE>
__global__ void __launch_bounds__(256) k_spmv(int64_t n, const int64_t* __restrict__ rp,
                                              const int32_t* __restrict__ ci,
                                              const double* __restrict__ A,
                                              const double* __restrict__ B, double sigma,
                                              const double* __restrict__ x,
                                              double* __restrict__ y) {
  pdl_start();
  int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / LANES;
  int sub = threadIdx.x % LANES;
  if (row >= n) return;
  int64_t b = rp[row], e = rp[row + 1];
  double acc = 0.0;
  // U elements per lane per round: all value / index loads issued before the
  // dependent x gathers (one round trip each instead of one per element)
  for (int64_t q0 = b + sub; q0 < e; q0 += U * LANES) {
    double a[U];
    int32_t c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = q0 + u * LANES;
      const bool in = q < e;
      a[u] = in ? __ldg(A + q) : 0.0;
      if (MODE == 1) a[u] = in ? __dsub_rn(a[u], __dmul_rn(sigma, __ldg(B + q))) : 0.0;
      c[u] = in ? __ldg(ci + q) : 0;
    }
    double xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = __ldg(x + c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) acc = fma(a[u], xv[u], acc);
  }
#pragma unroll
  for (int o = LANES / 2; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o, LANES);
  if (sub == 0) y[row] = acc;
}

int csr_spmv_impl(cudaStream_t s, int64_t n, const int64_t* rp, const int32_t* ci, const double* A,
                  const double* B, double sigma, int mode, int64_t nnz, const double* x,
                  double* y) {
  if (n == 0) return RIGA_OK;
  ProfScope prof(kProfSpmv, s, 12.0 * nnz + 4.0 * (n + 1) + 16.0 * n);
  double avg = double(nnz) / double(n);
  // 16 lanes per row for the stencil rows of these pencils (avg 70-285 nnz);
  // U is the smallest of 4/6/8 whose one unrolled round covers a row 10 % above
  // the average, else 8.  Swept on cfg3/4/5 (tools/spmv_sweep.sh): 32 lanes or
  // 4-element rounds lose 5-30 % on the 3D pencils.
  int lanes = avg >= 40 ? 16 : (avg >= 16 ? 8 : 4);
  if (const char* e = getenv("RIGA_SPMV_LANES")) lanes = atoi(e);
  int per = (int)ceil(1.1 * avg / lanes);
  int U = per <= 4 ? 4 : (per <= 6 ? 6 : 8);
  if (const char* e = getenv("RIGA_SPMV_U")) U = atoi(e);
  int64_t threads = n * lanes;
  int blocks = (int)((threads + 255) / 256);
#define RIGA_SPMV_LAUNCH(L, UU)                                                            \
  if (mode == 0)                                                                           \
    k_spmv<L, UU, 0><<<blocks, 256, 0, s>>>(n, rp, ci, A, B, sigma, x, y);                 \
  else                                                                                     \
    k_spmv<L, UU, 1><<<blocks, 256, 0, s>>>(n, rp, ci, A, B, sigma, x, y);
#define RIGA_SPMV_CASE(L)                                                                  \
  case L:                                                                                  \
    if (U == 8) {                                                                          \
      RIGA_SPMV_LAUNCH(L, 8)                                                               \
    } else if (U == 6) {                                                                   \
      RIGA_SPMV_LAUNCH(L, 6)                                                               \
    } else {                                                                               \
      RIGA_SPMV_LAUNCH(L, 4)                                                               \
    }                                                                                      \
    break;
  switch (lanes) {
    RIGA_SPMV_CASE(4)
    RIGA_SPMV_CASE(8)
    RIGA_SPMV_CASE(16)
    RIGA_SPMV_CASE(32)
    default:
      set_error("spmv: RIGA_SPMV_LANES must be 4, 8, 16 or 32");
      return RIGA_BAD_ARG;
  }
#undef RIGA_SPMV_LAUNCH
#undef RIGA_SPMV_CASE
  count_launch();
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

int csr_spmv(cudaStream_t s, int64_t n, const int64_t* rowptr, const int32_t* colidx,
             const double* val, const double* x, double* y) {
  int64_t nnz = 0;
  RIGA_CUDA(cudaMemcpyAsync(&nnz, rowptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  RIGA_CUDA(stream_sync(s));
  return csr_spmv_impl(s, n, rowptr, colidx, val, nullptr, 0.0, 0, nnz, x, y);
}

int system_spmv(riga_system* sys, cudaStream_t s, int which, double sigma, const double* x,
                double* y) {
  switch (which) {
    case 0:
      return csr_spmv_impl(s, sys->n, sys->rowptr.p, sys->colidx.p, sys->K.p, nullptr, 0.0, 0,
                           sys->nnz, x, y);
    case 1:
      return csr_spmv_impl(s, sys->n, sys->rowptr.p, sys->colidx.p, sys->M.p, nullptr, 0.0, 0,
                           sys->nnz, x, y);
    case 2:
      return csr_spmv_impl(s, sys->n, sys->rowptr.p, sys->colidx.p, sys->K.p, sys->M.p, sigma, 1,
                           sys->nnz, x, y);
  }
  set_error("spmv: which must be 0 (K), 1 (M) or 2 (K - sigma M)");
  return RIGA_BAD_ARG;
}

// ---------------------------------------------------------------------------
// Kronecker mass product: M = M_z (x) M_y (x) M_x applied one axis at a time
// (out[.., i, ..] = sum_j m_axis[i][j] in[.., j, ..]), so a step reads the
// n-vector a few times instead of the nnz = prod(2 p + 1) n CSR entries.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void k_kron_axis_body(int64_t n, int64_t nax, int64_t stride, const int64_t* __restrict__ rp,
                            const int32_t* __restrict__ ci, const double* __restrict__ m,
                            const double* __restrict__ in, double* __restrict__ out) {
  pdl_start();
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t i = (r / stride) % nax;
  const int64_t base = r - i * stride;
  double acc = 0.0;
  for (int64_t q = rp[i]; q < rp[i + 1]; ++q) acc = fma(m[q], in[base + (int64_t)ci[q] * stride], acc);
  out[r] = acc;
}

__global__ void k_kron_axis(int64_t n, int64_t nax, int64_t stride, const int64_t* __restrict__ rp,
                            const int32_t* __restrict__ ci, const double* __restrict__ m,
                            const double* __restrict__ in, double* __restrict__ out) {
  k_kron_axis_body(n, nax, stride, rp, ci, m, in, out);
}

int kron_mass_apply(riga_system* sys, cudaStream_t s, const double* x, double* y, double* t1, double* t2) {
  const int d = sys->kdim;
  const int64_t n = sys->n;
  const unsigned g = (unsigned)((n + 255) / 256);
  const double* in = x;
  int64_t stride = 1;
  for (int t = 0; t < d; ++t) {
    double* out = t == d - 1 ? y : (t % 2 == 0 ? t1 : t2);
    const KronAxis& a = sys->kax[t];
    RIGA_CUDA(launch(k_kron_axis, g, 256, 0, s, n, a.n, stride, a.rp.p, a.ci.p, a.m.p, in, out));
    count_launch();
    in = out;
    stride *= a.n;
  }
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

// ---------------------------------------------------------------------------
// Dot product, deterministic: per-block partials + last-block final sum.
// ---------------------------------------------------------------------------
__global__ void k_dot(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
                      double* __restrict__ partial, unsigned* __restrict__ ticket,
                      double* __restrict__ out) {
  __shared__ double red[32];
  __shared__ bool last;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    acc = fma(x[i], y[i], acc);
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = acc;
    __threadfence();
    unsigned t = atomicAdd(ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (last) {
    double s = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) s += ((volatile double*)partial)[i];
    s = block_sum(s, red);
    if (threadIdx.x == 0) {
      *out = s;
      *ticket = 0u;
    }
  }
}

int launch_dot(cudaStream_t s, int64_t n, const double* x, const double* y, double* out_dev) {
  // scratch: partials (<= 592) + ticket live right after out_dev (caller
  // provides a buffer of at least kDotScratch doubles)
  int blocks = (int)std::min<int64_t>(592, std::max<int64_t>(1, (n + 255) / 256));
  double* partial = out_dev + 1;
  unsigned* ticket = reinterpret_cast<unsigned*>(out_dev + 1 + 592);
  k_dot<<<blocks, 256, 0, s>>>(n, x, y, partial, ticket, out_dev); count_launch();
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

// ---- context lifetime / pinned host cache --------------------------------
void ctx_release(riga_ctx* c) {
  if (!c) return;
  if (c->refs.fetch_sub(1) != 1) return;
  DeviceGuard g(c->device);
  stream_sync(c->stream);  // this stream only: pending reads into scratch_host
  for (auto& a : c->aux)
    if (a) {
      cudaStreamSynchronize(a);
      cudaStreamDestroy(a);
    }
  for (auto& e : c->aux_ev)
    if (e) cudaEventDestroy(e);
  if (c->scratch_dev) cudaFreeAsync(c->scratch_dev, c->stream);
  if (c->scratch_host) pinned_put(c->scratch_host);
  if (c->own_stream) cudaStreamDestroy(c->stream);  // released once its work drains
  delete c;
}

cudaError_t stream_sync(cudaStream_t s) {
  thread_local cudaEvent_t ev = nullptr;
  thread_local int ev_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!ev || ev_dev != dev) {
    cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventBlockingSync | cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
    ev_dev = dev;
  }
  cudaError_t e = cudaEventRecord(ev, s);
  if (e != cudaSuccess) return e;
  return cudaEventSynchronize(ev);
}

namespace {
std::mutex g_pin_mu;
std::multimap<size_t, void*> g_pin_free;
std::unordered_map<void*, size_t> g_pin_size;
}  // namespace

void* pinned_get(size_t bytes) {
  bytes = (bytes + 255) & ~size_t(255);
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    auto it = g_pin_free.lower_bound(bytes);
    if (it != g_pin_free.end() && it->first <= 2 * bytes) {
      void* p = it->second;
      g_pin_free.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_size[p] = bytes;
  return p;
}

void pinned_put(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  auto it = g_pin_size.find(p);
  if (it != g_pin_size.end()) g_pin_free.emplace(it->second, p);
}

}  // namespace riga

using namespace riga;

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* riga_last_error(void) { return riga::last_error(); }
int riga_version(void) { return 100; }

int riga_device_count(int* count) {
  RIGA_CHECK_ARG(count, "null count");
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    cudaGetLastError();
    c = 0;
  }
  *count = c;
  return RIGA_OK;
}

int riga_mem_info(int device, int reset_high, int64_t* out4) {
  RIGA_CHECK_ARG(out4, "null out");
  DeviceGuard g(device);
  cudaMemPool_t pool;
  RIGA_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  const cudaMemPoolAttr attrs[4] = {cudaMemPoolAttrReservedMemCurrent, cudaMemPoolAttrReservedMemHigh,
                                    cudaMemPoolAttrUsedMemCurrent, cudaMemPoolAttrUsedMemHigh};
  for (int i = 0; i < 4; ++i) {
    uint64_t v = 0;
    RIGA_CUDA(cudaMemPoolGetAttribute(pool, attrs[i], &v));
    out4[i] = (int64_t)v;
  }
  if (reset_high) {
    uint64_t z = 0;
    RIGA_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReservedMemHigh, &z));
    RIGA_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &z));
  }
  return RIGA_OK;
}

int riga_ctx_create(int device, void* stream_handle, riga_ctx** out) {
  RIGA_CHECK_ARG(out, "null out");
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess || c == 0) {
    cudaGetLastError();
    set_error("no CUDA device visible: the B200 engine has no CPU fallback");
    return RIGA_NO_DEVICE;
  }
  RIGA_CHECK_ARG(device >= 0 && device < c, "device index out of range");
  DeviceGuard g(device);
  {
    // keep freed stream-ordered allocations cached in the device pool
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  auto* ctx = new riga_ctx();
  ctx->device = device;
  if (stream_handle) {
    ctx->stream = (cudaStream_t)stream_handle;
  } else {
    cudaError_t e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete ctx;
      set_error(std::string("stream create: ") + cudaGetErrorString(e));
      return RIGA_CUDA_ERROR;
    }
    ctx->own_stream = true;
  }
  ctx->scratch_host = static_cast<double*>(pinned_get(4096 * sizeof(double)));
  cudaError_t e = ctx->scratch_host ? cudaSuccess : cudaErrorMemoryAllocation;
  if (e == cudaSuccess)
    e = cudaMallocAsync(reinterpret_cast<void**>(&ctx->scratch_dev), kDotScratch * 4 * sizeof(double), ctx->stream);
  if (e != cudaSuccess) {
    set_error(std::string("ctx scratch: ") + cudaGetErrorString(e));
    ctx_release(ctx);
    return RIGA_CUDA_ERROR;
  }
  cudaMemsetAsync(ctx->scratch_dev, 0, kDotScratch * 4 * sizeof(double), ctx->stream);
  ctx->scratch_dev_n = kDotScratch * 4;
  *out = ctx;
  return RIGA_OK;
}

int riga_ctx_destroy(riga_ctx* ctx) {
  ctx_release(ctx);
  return RIGA_OK;
}

int riga_ctx_synchronize(riga_ctx* ctx) {
  RIGA_CHECK_ARG(ctx, "null ctx");
  DeviceGuard g(ctx->device);
  RIGA_CUDA(stream_sync(ctx->stream));
  return RIGA_OK;
}

int riga_set_blocking_sync(int device, int on) {
  DeviceGuard g(device);
  unsigned flags = 0;
  RIGA_CUDA(cudaGetDeviceFlags(&flags));
  flags = (flags & ~(unsigned)cudaDeviceScheduleMask) | (on ? cudaDeviceScheduleBlockingSync : cudaDeviceScheduleAuto);
  const cudaError_t e = cudaSetDeviceFlags(flags & ~(unsigned)cudaDeviceMapHost);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error(std::string("cudaSetDeviceFlags: ") + cudaGetErrorString(e));
    return RIGA_CUDA_ERROR;
  }
  return RIGA_OK;
}

int riga_device_pool_reusable(int device, int64_t* bytes) {
  RIGA_CHECK_ARG(bytes, "null arg");
  *bytes = 0;
  DeviceGuard g(device);
  cudaMemPool_t pool;
  RIGA_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t reserved = 0, used = 0;
  RIGA_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
  RIGA_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
  *bytes = reserved > used ? (int64_t)(reserved - used) : 0;
  return RIGA_OK;
}

int riga_ctx_stream(riga_ctx* ctx, void** stream_out) {
  RIGA_CHECK_ARG(ctx && stream_out, "null arg");
  *stream_out = (void*)ctx->stream;
  return RIGA_OK;
}

int riga_system_upload(riga_ctx* ctx, int64_t n, int64_t nnz, const int64_t* rowptr,
                       const int32_t* colidx, const double* K, const double* M,
                       riga_system** out) {
  RIGA_CHECK_ARG(ctx && out && rowptr && colidx && K && M, "null arg");
  RIGA_CHECK_ARG(n > 0 && nnz >= 0 && rowptr[n] == nnz, "inconsistent CSR");
  RIGA_CHECK_ARG(nnz < (int64_t(1) << 31), "nnz must fit int32 slots");
  DeviceGuard g(ctx->device);
  auto sys = std::make_unique<riga_system>();
  sys->ctx = ctx;
  sys->ctxref.set(ctx);
  sys->n = n;
  sys->nnz = nnz;
  RIGA_TRY(sys->rowptr.upload(rowptr, n + 1, ctx->stream));
  RIGA_TRY(sys->colidx.upload(colidx, nnz, ctx->stream));
  RIGA_TRY(sys->K.upload(K, nnz, ctx->stream));
  RIGA_TRY(sys->M.upload(M, nnz, ctx->stream));
  RIGA_CUDA(stream_sync(ctx->stream));
  *out = sys.release();
  return RIGA_OK;
}

int riga_system_assemble_kron(riga_ctx* ctx, int dim, const int64_t* n1,
                              const int64_t* const* rowptr1, const int32_t* const* colidx1,
                              const double* const* k1, const double* const* m1,
                              riga_system** out) {
  RIGA_CHECK_ARG(ctx && out && n1 && rowptr1 && colidx1 && k1 && m1, "null arg");
  RIGA_CHECK_ARG(dim >= 1 && dim <= 3, "dim must be 1, 2 or 3");
  DeviceGuard g(ctx->device);
  cudaStream_t s = ctx->stream;
  DevBuf<int64_t> rp[3];
  DevBuf<int32_t> ci[3];
  DevBuf<double> kk[3], mm[3];
  Kron1D ax[3] = {};
  int64_t n = 1, nnz = 1;
  for (int t = 0; t < dim; ++t) {
    int64_t nt = n1[t], zt = rowptr1[t][nt];
    RIGA_CHECK_ARG(nt > 0, "empty 1D matrix");
    RIGA_TRY(rp[t].upload(rowptr1[t], nt + 1, s));
    RIGA_TRY(ci[t].upload(colidx1[t], zt, s));
    RIGA_TRY(kk[t].upload(k1[t], zt, s));
    RIGA_TRY(mm[t].upload(m1[t], zt, s));
    ax[t] = Kron1D{rp[t].p, ci[t].p, kk[t].p, mm[t].p, nt};
    n *= nt;
    nnz *= zt;
  }
  RIGA_CHECK_ARG(nnz < (int64_t(1) << 31), "nnz must fit int32 slots");
  auto sys = std::make_unique<riga_system>();
  sys->ctx = ctx;
  sys->ctxref.set(ctx);
  sys->n = n;
  sys->nnz = nnz;
  RIGA_TRY(sys->rowptr.alloc(n + 1, s));
  RIGA_TRY(sys->colidx.alloc(nnz, s));
  RIGA_TRY(sys->K.alloc(nnz, s));
  RIGA_TRY(sys->M.alloc(nnz, s));
  RIGA_CUDA(cudaMemsetAsync(sys->rowptr.p, 0, sizeof(int64_t), s));
  k_kron_rowptr<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(dim, ax[0], ax[1], ax[2], n,
                                                            sys->rowptr.p + 1); count_launch();
  RIGA_CUDA(cudaGetLastError());
  RIGA_TRY(inclusive_scan_i64(s, sys->rowptr.p + 1, n));
  k_kron_values<<<(unsigned)((n * 32 + 255) / 256), 256, 0, s>>>(
      dim, ax[0], ax[1], ax[2], n, sys->rowptr.p, sys->colidx.p, sys->K.p, sys->M.p); count_launch();
  RIGA_CUDA(cudaGetLastError());
  RIGA_CUDA(stream_sync(s));
  // keep the 1D factors: the Lanczos mass products run axis by axis
  sys->kdim = dim;
  for (int t = 0; t < dim; ++t) {
    sys->kax[t].n = n1[t];
    sys->kax[t].rp.swap(rp[t]);
    sys->kax[t].ci.swap(ci[t]);
    sys->kax[t].k.swap(kk[t]);
    sys->kax[t].m.swap(mm[t]);
  }
  *out = sys.release();
  return RIGA_OK;
}

int riga_system_set_kron(riga_system* sys, int dim, const int64_t* n1, const int64_t* const* rowptr1,
                         const int32_t* const* colidx1, const double* const* k1, const double* const* m1) {
  RIGA_CHECK_ARG(sys && n1 && rowptr1 && colidx1 && k1 && m1, "null arg");
  RIGA_CHECK_ARG(dim >= 1 && dim <= 3, "dim must be 1, 2 or 3");
  int64_t n = 1;
  for (int t = 0; t < dim; ++t) n *= n1[t];
  RIGA_CHECK_ARG(n == sys->n, "1D factor sizes do not multiply to the system size");
  DeviceGuard g(sys->ctx->device);
  cudaStream_t s = sys->ctx->stream;
  for (int t = 0; t < dim; ++t) {
    const int64_t nt = n1[t], zt = rowptr1[t][nt];
    sys->kax[t].n = nt;
    RIGA_TRY(sys->kax[t].rp.upload(rowptr1[t], nt + 1, s));
    RIGA_TRY(sys->kax[t].ci.upload(colidx1[t], zt, s));
    RIGA_TRY(sys->kax[t].k.upload(k1[t], zt, s));
    RIGA_TRY(sys->kax[t].m.upload(m1[t], zt, s));
  }
  RIGA_CUDA(stream_sync(s));
  sys->kdim = dim;
  return RIGA_OK;
}

int riga_system_info(riga_system* sys, int64_t* n, int64_t* nnz) {
  RIGA_CHECK_ARG(sys, "null system");
  if (n) *n = sys->n;
  if (nnz) *nnz = sys->nnz;
  return RIGA_OK;
}

int riga_system_download(riga_system* sys, int64_t* rowptr, int32_t* colidx, double* K,
                         double* M) {
  RIGA_CHECK_ARG(sys, "null system");
  DeviceGuard g(sys->ctx->device);
  cudaStream_t s = sys->ctx->stream;
  if (rowptr)
    RIGA_CUDA(cudaMemcpyAsync(rowptr, sys->rowptr.p, (sys->n + 1) * 8, cudaMemcpyDeviceToHost, s));
  if (colidx)
    RIGA_CUDA(cudaMemcpyAsync(colidx, sys->colidx.p, sys->nnz * 4, cudaMemcpyDeviceToHost, s));
  if (K) RIGA_CUDA(cudaMemcpyAsync(K, sys->K.p, sys->nnz * 8, cudaMemcpyDeviceToHost, s));
  if (M) RIGA_CUDA(cudaMemcpyAsync(M, sys->M.p, sys->nnz * 8, cudaMemcpyDeviceToHost, s));
  RIGA_CUDA(stream_sync(s));
  return RIGA_OK;
}

int riga_system_device_ptrs(riga_system* sys, const int64_t** rowptr, const int32_t** colidx,
                            const double** K, const double** M) {
  RIGA_CHECK_ARG(sys, "null system");
  if (rowptr) *rowptr = sys->rowptr.p;
  if (colidx) *colidx = sys->colidx.p;
  if (K) *K = sys->K.p;
  if (M) *M = sys->M.p;
  return RIGA_OK;
}

int riga_system_destroy(riga_system* sys) {
  if (!sys) return RIGA_OK;
  DeviceGuard g(sys->ctx->device);
  stream_sync(sys->ctx->stream);
  delete sys;
  return RIGA_OK;
}

int riga_spmv(riga_system* sys, int which, double sigma, const double* x, double* y) {
  RIGA_CHECK_ARG(sys && x && y, "null arg");
  DeviceGuard g(sys->ctx->device);
  return system_spmv(sys, sys->ctx->stream, which, sigma, x, y);
}

int riga_csr_spmv(riga_ctx* ctx, int64_t n, const int64_t* rowptr, const int32_t* colidx,
                  const double* val, const double* x, double* y) {
  RIGA_CHECK_ARG(ctx && rowptr && colidx && val && x && y && n >= 0, "null arg");
  DeviceGuard g(ctx->device);
  return csr_spmv(ctx->stream, n, rowptr, colidx, val, x, y);
}

int riga_dot(riga_ctx* ctx, int64_t n, const double* x, const double* y, double* out) {
  RIGA_CHECK_ARG(ctx && x && y && out, "null arg");
  DeviceGuard g(ctx->device);
  RIGA_TRY(launch_dot(ctx->stream, n, x, y, ctx->scratch_dev));
  RIGA_CUDA(cudaMemcpyAsync(ctx->scratch_host, ctx->scratch_dev, sizeof(double),
                            cudaMemcpyDeviceToHost, ctx->stream));
  RIGA_CUDA(stream_sync(ctx->stream));
  *out = ctx->scratch_host[0];
  return RIGA_OK;
}

}  // extern "C"
