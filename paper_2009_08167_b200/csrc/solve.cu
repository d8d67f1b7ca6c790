// Supernodal forward/backward solves, level-synchronous with multi-CTA
// large supernodes.
//
//  riga_factor_solve <- solve_fb + _ldl_solve   ref sparsela.py:265-277, :162-175
//
// One launch per tree level and sweep; the CTAs of a launch take tasks from
// a per-level ticket (so a task only waits on tasks already running):
//   forward   WHOLE(s)   small supernode: one CTA pulls its front vector (b +
//                        children's update vectors through a precomputed pull
//                        map), dense triangular sweep, publishes its update
//                        vector;
//             CHAIN(s)   large supernode, pivot part: one CTA runs the 32-column
//                        block chain in shared memory (in-CTA syncs only) and
//                        publishes each solved block z_b with a release flag;
//             UPD(s,u)   32 update rows of a large supernode: consume z_b as the
//                        flags appear (overlapping the chain), write the update
//                        vector.
//   backward  COLDOT(s,b) large supernode: c_b = L21(:,b)^T x(update rows), the
//                        ancestors' values being final (previous launch);
//             CHAIN_T(s) waits for its COLDOTs, then the transposed block chain
//                        of the pivot part in shared memory;
//             WHOLE(s)   small supernode, transposed dense sweep.
// Cross-CTA data is read through L2 (ld.global.cg) after an acquire.
#include <algorithm>

#include "internal.h"
#include "kernels.cuh"
#include "prof.h"

namespace riga {

constexpr int kWholeMaxF = 320;  // max front rows of a WHOLE supernode
constexpr int kSolveThreads = 256;
constexpr int kSolveWarps = kSolveThreads / 32;

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_geq(const int* p, int target) {
  while (ld_acquire(p) < target) __nanosleep(20);
}

enum { kWhole = 0, kChain = 1, kUpd = 2, kColdot = 3, kChainT = 4 };

struct SolveDev {
  const int32_t* nbp;      // pivot blocks of a large supernode (0: small)
  const int32_t* flagoff;  // offset of its pivot-block flags
  const int64_t* gptr;     // pull map over front positions (rows_off indexing)
  const int32_t* gsrc;     // sources in the update-vector buffer
  int* flags;              // forward: z_b published (per large supernode, per block)
  int* coldone;            // backward: COLDOT tasks finished (per supernode)
};

__device__ __forceinline__ double gather_row(const SymDev& S, const SolveDev& T, int s, int64_t r,
                                             int64_t np, int64_t col0, const double* __restrict__ b,
                                             const double* __restrict__ upd) {
  double v = r < np ? b[S.order[col0 + r]] : 0.0;
  const int64_t g = S.rows_off[s] + r;
  for (int64_t q = T.gptr[g]; q < T.gptr[g + 1]; ++q) v += __ldcg(upd + T.gsrc[q]);
  return v;
}

// unit-lower 32x32 diagonal block solve by one warp; row `lane` of the block
// is preloaded so the substitution runs from registers
__device__ __forceinline__ double diag_solve(const double* __restrict__ P, int64_t f, int64_t kb,
                                             int nbk, int lane, double yi) {
  double lrow[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) lrow[k] = (k < lane && lane < nbk) ? P[(kb + k) * f + kb + lane] : 0.0;
#pragma unroll
  for (int k = 0; k < 32; ++k) yi = fma(-lrow[k], __shfl_sync(0xffffffffu, yi, k), yi);
  return yi;
}

__device__ __forceinline__ double diag_solve_t(const double* __restrict__ P, int64_t f, int64_t kb,
                                               int nbk, int lane, double xc) {
  double lcol[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) lcol[k] = (k > lane && k < nbk) ? P[(kb + lane) * f + kb + k] : 0.0;
#pragma unroll
  for (int k = 31; k >= 0; --k) xc = fma(-lcol[k], __shfl_sync(0xffffffffu, xc, k), xc);
  return xc;
}

__global__ void __launch_bounds__(kSolveThreads) k_fwd_level(SymDev S, SolveDev T, const int2* __restrict__ tasks,
                                                             int ntasks, int* ticket,
                                                             const double* __restrict__ panel,
                                                             const double* __restrict__ b,
                                                             double* __restrict__ xp,
                                                             double* __restrict__ upd) {
  extern __shared__ double y[];
  __shared__ int task_sh;
  __shared__ double part[kSolveWarps][32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) task_sh = atomicAdd(ticket, 1);
  __syncthreads();
  const int t = task_sh;
  if (t >= ntasks) return;
  const int2 task = tasks[t];
  const int s = task.x, type = task.y >> 24, j = task.y & 0x00ffffff;
  const int64_t f = S.front[s], np = S.ncol[s], col0 = S.col0[s];
  const double* P = panel + S.panel_off[s];
  if (type == kWhole) {
    for (int64_t r = tid; r < f; r += blockDim.x) y[r] = gather_row(S, T, s, r, np, col0, b, upd);
    __syncthreads();
    for (int64_t kb = 0; kb < np; kb += 32) {
      const int nbk = (int)imin(32, np - kb);
      if (w == 0) {
        double yi = lane < nbk ? y[kb + lane] : 0.0;
        yi = diag_solve(P, f, kb, nbk, lane, yi);
        if (lane < nbk) y[kb + lane] = yi;
      }
      __syncthreads();
      for (int64_t i = kb + nbk + tid; i < f; i += blockDim.x) {
        double acc = 0.0;
        for (int k = 0; k < nbk; ++k) acc = fma(P[(kb + k) * f + i], y[kb + k], acc);
        y[i] -= acc;
      }
      __syncthreads();
    }
    for (int64_t r = tid; r < np; r += blockDim.x) xp[col0 + r] = y[r];
    double* u = upd + S.upd_off[s];
    for (int64_t r = np + tid; r < f; r += blockDim.x) u[r - np] = y[r];
  } else if (type == kChain) {
    int* flags = T.flags + T.flagoff[s];
    for (int64_t r = tid; r < np; r += blockDim.x) y[r] = gather_row(S, T, s, r, np, col0, b, upd);
    __syncthreads();
    for (int64_t kb = 0; kb < np; kb += 32) {
      const int nbk = (int)imin(32, np - kb);
      if (w == 0) {
        double yi = lane < nbk ? y[kb + lane] : 0.0;
        yi = diag_solve(P, f, kb, nbk, lane, yi);
        if (lane < nbk) {
          y[kb + lane] = yi;
          xp[col0 + kb + lane] = yi;
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release(flags + kb / 32, 1);
      }
      __syncthreads();
      for (int64_t i = kb + nbk + tid; i < np; i += blockDim.x) {
        double acc = 0.0;
        if (nbk == 32) {
#pragma unroll
          for (int k = 0; k < 32; ++k) acc = fma(P[(kb + k) * f + i], y[kb + k], acc);
        } else {
          for (int k = 0; k < nbk; ++k) acc = fma(P[(kb + k) * f + i], y[kb + k], acc);
        }
        y[i] -= acc;
      }
      __syncthreads();
    }
  } else {  // kUpd
    const int* flags = T.flags + T.flagoff[s];
    const int nbp = T.nbp[s];
    const int64_t r0 = np + 32 * (int64_t)j, r1 = imin(r0 + 32, f), r = r0 + lane;
    const bool in = r < r1;
    double acc = 0.0;
    for (int cb = w; cb < nbp; cb += kSolveWarps) {
      if (lane == 0) wait_geq(flags + cb, 1);
      __syncwarp();
      const int64_t c0 = 32 * (int64_t)cb;
      const int nc = (int)imin(32, np - c0);
      const double zl = lane < nc ? __ldcg(xp + col0 + c0 + lane) : 0.0;
      if (nc == 32) {
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
          const double l = in ? P[(c0 + k) * f + r] : 0.0;
          acc = fma(l, __shfl_sync(0xffffffffu, zl, k), acc);
        }
      } else {
        for (int k = 0; k < nc; ++k) {
          const double l = in ? P[(c0 + k) * f + r] : 0.0;
          acc = fma(l, __shfl_sync(0xffffffffu, zl, k), acc);
        }
      }
    }
    part[w][lane] = acc;
    __syncthreads();
    if (w == 0 && in) {
      double v = gather_row(S, T, s, r, np, col0, b, upd);
#pragma unroll
      for (int q = 0; q < kSolveWarps; ++q) v -= part[q][lane];
      upd[S.upd_off[s] + r - np] = v;
    }
  }
}

__global__ void __launch_bounds__(kSolveThreads) k_bwd_level(SymDev S, SolveDev T, const int2* __restrict__ tasks,
                                                             int ntasks, int* ticket,
                                                             const double* __restrict__ panel,
                                                             const double* __restrict__ D,
                                                             double* __restrict__ xp,
                                                             double* __restrict__ cvec,
                                                             double* __restrict__ x) {
  extern __shared__ double y[];
  __shared__ int task_sh;
  __shared__ double part[kSolveWarps][32];
  // COLDOT tasks use the dynamic buffer as per-warp 32x33 transpose tiles
  double (*tile)[32][33] = reinterpret_cast<double (*)[32][33]>(y);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) task_sh = atomicAdd(ticket, 1);
  __syncthreads();
  const int t = task_sh;
  if (t >= ntasks) return;
  const int2 task = tasks[t];
  const int s = task.x, type = task.y >> 24, bj = task.y & 0x00ffffff;
  const int64_t f = S.front[s], np = S.ncol[s], col0 = S.col0[s];
  const double* P = panel + S.panel_off[s];
  const int32_t* rows = S.rows + S.rows_off[s];
  if (type == kWhole) {
    for (int64_t r = tid; r < f; r += blockDim.x)
      y[r] = r < np ? xp[col0 + r] / D[col0 + r] : __ldcg(xp + rows[r]);
    __syncthreads();
    const int64_t nblk = (np + 31) / 32;
    for (int64_t bi = nblk - 1; bi >= 0; --bi) {
      const int64_t kb = bi * 32;
      const int nbk = (int)imin(32, np - kb);
      for (int c = w; c < nbk; c += kSolveWarps) {
        const double* Pc = P + (kb + c) * f;
        double acc = 0.0;
        for (int64_t i = kb + nbk + lane; i < f; i += 32) acc = fma(Pc[i], y[i], acc);
        acc = warp_sum(acc);
        if (lane == 0) y[kb + c] -= acc;
      }
      __syncthreads();
      if (w == 0) {
        double xc = lane < nbk ? y[kb + lane] : 0.0;
        xc = diag_solve_t(P, f, kb, nbk, lane, xc);
        if (lane < nbk) y[kb + lane] = xc;
      }
      __syncthreads();
    }
    for (int64_t r = tid; r < np; r += blockDim.x) {
      xp[col0 + r] = y[r];
      x[S.order[col0 + r]] = y[r];
    }
  } else if (type == kColdot) {
    // c[col] = sum over update rows r of L[r][col] x[rows[r]], col in block bj
    const int64_t c0 = 32 * (int64_t)bj;
    const int nc = (int)imin(32, np - c0);
    const int nbu = (int)((f - np + 31) / 32);
    double acc = 0.0;
    for (int q = w; q < nbu; q += kSolveWarps) {
      const int64_t r0 = np + 32 * (int64_t)q, r1 = imin(r0 + 32, f), r = r0 + lane;
      const double xv = r < r1 ? __ldcg(xp + rows[r]) : 0.0;
      for (int k = 0; k < nc; ++k) tile[w][k][lane] = r < r1 ? P[(c0 + k) * f + r] : 0.0;
      __syncwarp();
      double a2 = 0.0;
#pragma unroll 8
      for (int rr = 0; rr < 32; ++rr) a2 = fma(tile[w][lane][rr], __shfl_sync(0xffffffffu, xv, rr), a2);
      acc += lane < nc ? a2 : 0.0;
      __syncwarp();
    }
    part[w][lane] = acc;
    __syncthreads();
    if (w == 0) {
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < kSolveWarps; ++q) v += part[q][lane];
      if (lane < nc) cvec[col0 + c0 + lane] = v;
      __threadfence();
      __syncwarp();
      if (lane == 0) atomicAdd(T.coldone + s, 1);
    }
  } else {  // kChainT
    const bool has_upd = f > np;
    if (tid == 0 && has_upd) wait_geq(T.coldone + s, T.nbp[s]);
    __syncthreads();
    for (int64_t r = tid; r < np; r += blockDim.x)
      y[r] = xp[col0 + r] / D[col0 + r] - (has_upd ? __ldcg(cvec + col0 + r) : 0.0);
    __syncthreads();
    const int64_t nblk = (np + 31) / 32;
    for (int64_t bi = nblk - 1; bi >= 0; --bi) {
      const int64_t kb = bi * 32;
      const int nbk = (int)imin(32, np - kb);
      if (w == 0) {
        double xc = lane < nbk ? y[kb + lane] : 0.0;
        xc = diag_solve_t(P, f, kb, nbk, lane, xc);
        if (lane < nbk) {
          y[kb + lane] = xc;
          xp[col0 + kb + lane] = xc;
          x[S.order[col0 + kb + lane]] = xc;
        }
      }
      __syncthreads();
      // y[i] -= sum_{r in block} L[kb+r][i] x[kb+r]  for all earlier columns i
      for (int64_t i = tid; i < kb; i += blockDim.x) {
        const double* Pi = P + i * f + kb;
        double acc = 0.0;
        if (nbk == 32) {
#pragma unroll
          for (int r = 0; r < 32; ++r) acc = fma(Pi[r], y[kb + r], acc);
        } else {
          for (int r = 0; r < nbk; ++r) acc = fma(Pi[r], y[kb + r], acc);
        }
        y[i] -= acc;
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// host: per-level task lists, pull map
// ---------------------------------------------------------------------------
int build_solve_plan(riga_symbolic* sym) {
  const SymbolicHost& h = sym->h;
  SolvePlanHost& L = sym->sp;
  const int64_t ns = h.nsuper;
  L = SolvePlanHost();
  L.nbp.assign(ns, 0);
  L.flagoff.assign(ns, 0);
  int32_t nflags = 0;
  auto large = [&](int64_t s) { return h.ncol[s] > 32 || h.front[s] > kWholeMaxF; };
  for (int64_t s = 0; s < ns; ++s) {
    if (!large(s)) continue;
    L.nbp[s] = (int32_t)((h.ncol[s] + 31) / 32);
    L.flagoff[s] = nflags;
    nflags += L.nbp[s];
  }
  L.nflags = nflags;
  L.fwd_ptr.assign(h.nlevels + 1, 0);
  L.bwd_ptr.assign(h.nlevels + 1, 0);
  L.fwd_smem.assign(h.nlevels, 0);
  L.bwd_smem.assign(h.nlevels, 0);
  auto code = [](int type, int j) { return (int32_t)((type << 24) | j); };
  for (int64_t l = 0; l < h.nlevels; ++l) {
    std::vector<int32_t> nodes(h.level_nodes.begin() + h.level_ptr[l],
                               h.level_nodes.begin() + h.level_ptr[l + 1]);
    std::stable_sort(nodes.begin(), nodes.end(), [&](int32_t a, int32_t b) {
      return h.ncol[a] * h.front[a] > h.ncol[b] * h.front[b];
    });
    int64_t sm_f = 0, sm_b = 0;
    for (int32_t s : nodes)
      if (large(s)) {
        L.fwd.push_back({s, code(kChain, 0)});
        sm_f = std::max<int64_t>(sm_f, h.ncol[s]);
        sm_b = std::max<int64_t>(sm_b, h.ncol[s]);
      }
    for (int32_t s : nodes)
      if (large(s)) {
        int64_t nbu = (h.front[s] - h.ncol[s] + 31) / 32;
        for (int64_t u = 0; u < nbu; ++u) L.fwd.push_back({s, code(kUpd, (int)u)});
        if (nbu > 0) {
          for (int32_t bb = 0; bb < L.nbp[s]; ++bb) L.bwd.push_back({s, code(kColdot, bb)});
          sm_b = std::max<int64_t>(sm_b, kSolveWarps * 32 * 33);
        }
      }
    for (int32_t s : nodes)
      if (large(s)) L.bwd.push_back({s, code(kChainT, 0)});
    for (int32_t s : nodes)
      if (!large(s)) {
        L.fwd.push_back({s, code(kWhole, 0)});
        L.bwd.push_back({s, code(kWhole, 0)});
        sm_f = std::max<int64_t>(sm_f, h.front[s]);
        sm_b = std::max<int64_t>(sm_b, h.front[s]);
      }
    L.fwd_ptr[l + 1] = (int64_t)L.fwd.size();
    L.bwd_ptr[l + 1] = (int64_t)L.bwd.size();
    L.fwd_smem[l] = std::max<int64_t>(sm_f, 1) * 8;
    L.bwd_smem[l] = std::max<int64_t>(sm_b, 1) * 8;
  }
  // pull map: front position -> sources in the update-vector buffer
  const int64_t nfront = h.rows_off[ns];
  std::vector<int64_t> cnt(nfront + 1, 0);
  for (int64_t p = 0; p < ns; ++p)
    for (int64_t q = h.child_ptr[p]; q < h.child_ptr[p + 1]; ++q) {
      int64_t c = h.child_list[q];
      for (int64_t t = 0; t < h.front[c] - h.ncol[c]; ++t)
        cnt[h.rows_off[p] + h.relpos[h.upd_off[c] + t] + 1]++;
    }
  for (int64_t i = 0; i < nfront; ++i) cnt[i + 1] += cnt[i];
  L.gptr = cnt;
  L.gsrc.assign(cnt[nfront], 0);
  std::vector<int64_t> fillp(cnt.begin(), cnt.end() - 1);
  for (int64_t p = 0; p < ns; ++p)
    for (int64_t q = h.child_ptr[p]; q < h.child_ptr[p + 1]; ++q) {
      int64_t c = h.child_list[q];
      for (int64_t t = 0; t < h.front[c] - h.ncol[c]; ++t)
        L.gsrc[fillp[h.rows_off[p] + h.relpos[h.upd_off[c] + t]]++] = (int32_t)(h.upd_off[c] + t);
    }
  // sync area: 2 tickets per level, pivot-block flags, COLDOT counters
  L.sync_ints = 2 * h.nlevels + nflags + ns;
  return RIGA_OK;
}

int upload_solve_plan(riga_symbolic* sym, cudaStream_t s) {
  SolvePlanHost& L = sym->sp;
  RIGA_TRY(sym->d_tfwd.upload(L.fwd.data(), L.fwd.size(), s));
  RIGA_TRY(sym->d_tbwd.upload(L.bwd.data(), L.bwd.size(), s));
  RIGA_TRY(sym->d_nbp.upload(L.nbp.data(), L.nbp.size(), s));
  RIGA_TRY(sym->d_flagoff.upload(L.flagoff.data(), L.flagoff.size(), s));
  RIGA_TRY(sym->d_gptr.upload(L.gptr.data(), L.gptr.size(), s));
  if (L.gsrc.empty())
    RIGA_TRY(sym->d_gsrc.alloc(1, s));
  else
    RIGA_TRY(sym->d_gsrc.upload(L.gsrc.data(), L.gsrc.size(), s));
  return RIGA_OK;
}

static int set_solve_attrs() {
  static bool done = false;
  if (done) return RIGA_OK;
  int dev = 0, maxsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa;
  RIGA_CUDA(cudaFuncGetAttributes(&fa, k_fwd_level));
  RIGA_CUDA(cudaFuncSetAttribute(k_fwd_level, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 maxsm - (int)fa.sharedSizeBytes));
  RIGA_CUDA(cudaFuncGetAttributes(&fa, k_bwd_level));
  RIGA_CUDA(cudaFuncSetAttribute(k_bwd_level, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 maxsm - (int)fa.sharedSizeBytes));
  done = true;
  return RIGA_OK;
}

int factor_solve(riga_factor* F, cudaStream_t st, const double* b, double* x) {
  riga_symbolic* sym = F->sym;
  const SymbolicHost& h = sym->h;
  const SolvePlanHost& L = sym->sp;
  ProfScope prof(kProfSolve, st, 16.0 * h.fill_nnz + 32.0 * h.n);
  RIGA_TRY(set_solve_attrs());
  SymDev S = sym->dev();
  if (!F->sync.p) RIGA_TRY(F->sync.alloc(L.sync_ints, st));
  if (!F->cvec.p) RIGA_TRY(F->cvec.alloc(h.n, st));
  int* tick = F->sync.p;
  SolveDev T{sym->d_nbp.p, sym->d_flagoff.p, sym->d_gptr.p, sym->d_gsrc.p,
             F->sync.p + 2 * h.nlevels, F->sync.p + 2 * h.nlevels + L.nflags};
  RIGA_CUDA(cudaMemsetAsync(F->sync.p, 0, L.sync_ints * sizeof(int), st));
  const int2* tf = reinterpret_cast<const int2*>(sym->d_tfwd.p);
  const int2* tb = reinterpret_cast<const int2*>(sym->d_tbwd.p);
  for (int64_t l = 0; l < h.nlevels; ++l) {
    int nt = (int)(L.fwd_ptr[l + 1] - L.fwd_ptr[l]);
    if (!nt) continue;
    k_fwd_level<<<nt, kSolveThreads, L.fwd_smem[l], st>>>(S, T, tf + L.fwd_ptr[l], nt, tick + 2 * l,
                                                          F->panel.p, b, F->xperm.p, F->upd.p);
    count_launch();
  }
  for (int64_t l = h.nlevels - 1; l >= 0; --l) {
    int nt = (int)(L.bwd_ptr[l + 1] - L.bwd_ptr[l]);
    if (!nt) continue;
    k_bwd_level<<<nt, kSolveThreads, L.bwd_smem[l], st>>>(S, T, tb + L.bwd_ptr[l], nt, tick + 2 * l + 1,
                                                          F->panel.p, F->D.p, F->xperm.p, F->cvec.p, x);
    count_launch();
  }
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

}  // namespace riga
