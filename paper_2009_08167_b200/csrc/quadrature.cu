// Element-quadrature assembly of K and M: (p+1)^d Gauss points per element.
//
//  riga_system_assemble_quad <- assemble_1d + kron_assemble   ref assembly.py:72-111, :139-192
//
// The reference integrates 1D element matrices and composes them by Kronecker
// products.  Here every d-dimensional element is integrated directly with the
// tensor Gauss rule of (p+1)^d points (BASELINE's "(p+1)^d Gauss points per
// element"): for local bases a, b and points q,
//   K_e(a, b) = sum_q W_q grad N_a(x_q) . grad N_b(x_q),   M_e(a, b) = sum_q W_q N_a(x_q) N_b(x_q),
// with N_a(x_q) the product of the 1D B-spline values (and one derivative for
// each gradient component) that the host evaluates per element and direction
// (Cox-de Boor, bspline.eval_basis_span).  Equal to the Kronecker pencil up to
// roundoff (the tensor Gauss rule integrates these polynomial products exactly).
//
// One CTA per element: the (d+1) x (p+1)^d x (p+1)^d table of weighted basis
// values at the points is built in shared memory, then each thread owns
// (a <= b) pairs and accumulates both matrices over the points.  Elements are
// processed in (p+1)^d colour classes (element index mod p+1 per direction):
// two elements of one class share no basis function, so each CSR slot is
// updated by at most one CTA per launch and the colours run in a fixed order
// -- the result is deterministic without atomics.  A slot's CSR position is
// computed from the 1D patterns (rows of the Kronecker pattern enumerate
// (jz, jy, jx) lexicographically over contiguous 1D column ranges).
#include "internal.h"
#include "kernels.cuh"
#include "prof.h"

namespace riga {

struct QuadAxis {
  int64_t ne, n1;             // elements, Dirichlet-reduced basis count
  const int32_t* first;       // per element: global (full) index of its first basis function
  const double* w;            // [e][q] Gauss weights (scaled to the element)
  const double* N;            // [e][q][a] basis values
  const double* dN;           // [e][q][a] derivatives
  const int64_t* rp;          // reduced 1D CSR pattern
  const int32_t* ci;
};

struct QuadTab {
  QuadAxis ax[3];
};

template <int D, int P1>
__global__ void __launch_bounds__(256) k_quad_elem(QuadTab T, int3 color, int3 ncol, const int64_t* __restrict__ rowptr,
                                                   double* __restrict__ K, double* __restrict__ M) {
  constexpr int NB = D == 1 ? P1 : (D == 2 ? P1 * P1 : P1 * P1 * P1);  // local bases = points
  extern __shared__ double sm[];
  double* V = sm;                  // V[c][q][a], c = 0: value, 1..D: gradient components
  double* W = V + (D + 1) * NB * NB;  // weights per point
  double* tab = W + NB;               // per direction: w[P1], N[P1][P1], dN[P1][P1]
  __shared__ int64_t gidx[NB];        // reduced global index of each local basis (-1: eliminated)
  __shared__ int64_t rpos[NB];        // its CSR row start
  __shared__ int loc[NB][3];          // its 1D reduced indices
  // this block's element
  int64_t e[3] = {0, 0, 0};
  {
    int64_t b = blockIdx.x;
    const int cc[3] = {color.x, color.y, color.z};
    const int nc[3] = {ncol.x, ncol.y, ncol.z};
    for (int t = 0; t < D; ++t) {
      e[t] = cc[t] + (int64_t)P1 * (b % nc[t]);
      b /= nc[t];
    }
  }
  for (int t = 0; t < D; ++t)
    if (e[t] >= T.ax[t].ne) return;  // uniform over the block
  const int tid = threadIdx.x;
  for (int t = 0; t < D; ++t) {
    double* tb = tab + t * (P1 + 2 * P1 * P1);
    const QuadAxis& A = T.ax[t];
    for (int i = tid; i < P1; i += blockDim.x) tb[i] = A.w[e[t] * P1 + i];
    for (int i = tid; i < P1 * P1; i += blockDim.x) {
      tb[P1 + i] = A.N[e[t] * P1 * P1 + i];
      tb[P1 + P1 * P1 + i] = A.dN[e[t] * P1 * P1 + i];
    }
  }
  __syncthreads();
  // basis / point tables: q and a as multi-indices, x fastest
  for (int idx = tid; idx < NB * NB; idx += blockDim.x) {
    const int q = idx / NB, a = idx - q * NB;
    int qq = q, aa = a;
    double val = 1.0, wq = 1.0;
    double g[3] = {1.0, 1.0, 1.0};
    for (int t = 0; t < D; ++t) {
      const double* tb = tab + t * (P1 + 2 * P1 * P1);
      const int qt = qq % P1, at = aa % P1;
      qq /= P1;
      aa /= P1;
      const double nv = tb[P1 + qt * P1 + at], dv = tb[P1 + P1 * P1 + qt * P1 + at];
      for (int c = 0; c < D; ++c) g[c] *= (c == t) ? dv : nv;
      val *= nv;
      wq *= tb[qt];
    }
    V[q * NB + a] = val;
    for (int c = 0; c < D; ++c) V[(c + 1) * NB * NB + q * NB + a] = g[c];
    if (a == 0) W[q] = wq;
  }
  for (int a = tid; a < NB; a += blockDim.x) {
    int aa = a;
    int64_t g = 0, stride = 1;
    bool ok = true;
    for (int t = 0; t < D; ++t) {
      const int at = aa % P1;
      aa /= P1;
      const int64_t r = (int64_t)T.ax[t].first[e[t]] + at - 1;  // Dirichlet: full index 0 is eliminated
      ok = ok && r >= 0 && r < T.ax[t].n1;
      loc[a][t] = (int)r;
      g += r * stride;
      stride *= T.ax[t].n1;
    }
    gidx[a] = ok ? g : -1;
    rpos[a] = ok ? rowptr[g] : 0;
  }
  __syncthreads();
  // pairs a <= b: accumulate over the points, scatter to (a, b) and (b, a)
  constexpr int NP = NB * (NB + 1) / 2;
  for (int pidx = tid; pidx < NP; pidx += blockDim.x) {
    int a = 0, rem = pidx;
    while (rem >= NB - a) {
      rem -= NB - a;
      ++a;
    }
    const int b = a + rem;
    if (gidx[a] < 0 || gidx[b] < 0) continue;
    double kacc = 0.0, macc = 0.0;
#pragma unroll 4
    for (int q = 0; q < NB; ++q) {
      const double wq = W[q];
      double gg = 0.0;
#pragma unroll
      for (int c = 1; c <= D; ++c) gg = fma(V[c * NB * NB + q * NB + a], V[c * NB * NB + q * NB + b], gg);
      kacc = fma(wq, gg, kacc);
      macc = fma(wq, V[q * NB + a] * V[q * NB + b], macc);
    }
    // CSR slot of (row of a, column of b) and its transpose
    for (int sw = 0; sw < (a == b ? 1 : 2); ++sw) {
      const int ra = sw ? b : a, cb = sw ? a : b;
      int64_t off = 0;
      for (int t = D - 1; t >= 0; --t) {
        const QuadAxis& A = T.ax[t];
        const int64_t ir = loc[ra][t], jc = loc[cb][t];
        const int64_t beg = A.rp[ir], len = A.rp[ir + 1] - beg;
        off = off * len + (jc - A.ci[beg]);
      }
      const int64_t slot = rpos[ra] + off;
      K[slot] += kacc;
      M[slot] += macc;
    }
  }
}

template <int D, int P1>
static int run_quad(const QuadTab& T, cudaStream_t s, const int64_t* rowptr, double* K, double* M) {
  constexpr int NB = D == 1 ? P1 : (D == 2 ? P1 * P1 : P1 * P1 * P1);
  const size_t smem = ((size_t)(D + 1) * NB * NB + NB + (size_t)D * (P1 + 2 * P1 * P1)) * sizeof(double);
  RIGA_CUDA(cudaFuncSetAttribute(k_quad_elem<D, P1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int ncolors = 1;
  for (int t = 0; t < D; ++t) ncolors *= P1;
  for (int c = 0; c < ncolors; ++c) {
    int cc[3] = {0, 0, 0}, nc[3] = {1, 1, 1};
    int rem = c;
    int64_t blocks = 1;
    for (int t = 0; t < D; ++t) {
      cc[t] = rem % P1;
      rem /= P1;
      nc[t] = (int)((T.ax[t].ne - cc[t] + P1 - 1) / P1);
      blocks *= nc[t];
    }
    if (blocks <= 0) continue;
    k_quad_elem<D, P1><<<(unsigned)blocks, 256, smem, s>>>(T, make_int3(cc[0], cc[1], cc[2]),
                                                          make_int3(nc[0], nc[1], nc[2]), rowptr, K, M);
    count_launch();
  }
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

}  // namespace riga

using namespace riga;

extern "C" {

int riga_system_assemble_quad(riga_ctx* ctx, int dim, int p, const int64_t* ne, const int32_t* const* first,
                              const double* const* w, const double* const* N, const double* const* dN,
                              const int64_t* n1, const int64_t* const* rowptr1, const int32_t* const* colidx1,
                              const double* const* k1, const double* const* m1, riga_system** out) {
  RIGA_CHECK_ARG(ctx && out && ne && first && w && N && dN, "null arg");
  RIGA_CHECK_ARG(dim >= 1 && dim <= 3, "dim must be 1, 2 or 3");
  RIGA_CHECK_ARG(p >= 1 && p <= 5, "quadrature assembly supports degrees 1..5");
  DeviceGuard g(ctx->device);
  cudaStream_t s = ctx->stream;
  // the shared pattern (and scratch values) from the Kronecker path, then the values by quadrature
  riga_system* sys = nullptr;
  RIGA_TRY(riga_system_assemble_kron(ctx, dim, n1, rowptr1, colidx1, k1, m1, &sys));
  std::unique_ptr<riga_system> guard(sys);
  const int P1 = p + 1;
  DevBuf<int32_t> fb[3];
  DevBuf<double> wb[3], nb[3], db[3];
  QuadTab T{};
  for (int t = 0; t < dim; ++t) {
    RIGA_CHECK_ARG(ne[t] > 0, "empty axis");
    RIGA_TRY(fb[t].upload(first[t], ne[t], s));
    RIGA_TRY(wb[t].upload(w[t], ne[t] * P1, s));
    RIGA_TRY(nb[t].upload(N[t], ne[t] * P1 * P1, s));
    RIGA_TRY(db[t].upload(dN[t], ne[t] * P1 * P1, s));
    T.ax[t] = QuadAxis{ne[t], sys->kax[t].n, fb[t].p, wb[t].p, nb[t].p, db[t].p, sys->kax[t].rp.p, sys->kax[t].ci.p};
  }
  RIGA_CUDA(cudaMemsetAsync(sys->K.p, 0, sys->nnz * sizeof(double), s));
  RIGA_CUDA(cudaMemsetAsync(sys->M.p, 0, sys->nnz * sizeof(double), s));
  int rc = RIGA_BAD_ARG;
#define RIGA_QUAD_CASE(DD, PP) \
  if (dim == DD && P1 == PP) rc = run_quad<DD, PP>(T, s, sys->rowptr.p, sys->K.p, sys->M.p);
  RIGA_QUAD_CASE(1, 2) RIGA_QUAD_CASE(1, 3) RIGA_QUAD_CASE(1, 4) RIGA_QUAD_CASE(1, 5) RIGA_QUAD_CASE(1, 6)
  RIGA_QUAD_CASE(2, 2) RIGA_QUAD_CASE(2, 3) RIGA_QUAD_CASE(2, 4) RIGA_QUAD_CASE(2, 5) RIGA_QUAD_CASE(2, 6)
  RIGA_QUAD_CASE(3, 2) RIGA_QUAD_CASE(3, 3) RIGA_QUAD_CASE(3, 4)
#undef RIGA_QUAD_CASE
  if (rc != RIGA_OK) {
    if (rc == RIGA_BAD_ARG) set_error("quadrature assembly: unsupported (dim, degree)");
    return rc;
  }
  RIGA_CUDA(stream_sync(s));
  // M is not the Kronecker product of the 1D factors to the last bit: mass products use the CSR
  sys->kdim = 0;
  *out = guard.release();
  return RIGA_OK;
}

}  // extern "C"
