// Supernodal forward/backward solves, level-synchronous.
//
//  riga_factor_solve <- solve_fb + _ldl_solve   ref sparsela.py:265-277, :162-175
//
// Per tree level and sweep, two launches on the solve stream:
//   forward   k_chain_fwd  one CTA per large supernode: the 32-column block
//                          chain of its pivot part, warp-specialised (warp w
//                          owns blocks w mod 8; the owner of block b+1
//                          prefetches L[b+1,b] and its diagonal block into
//                          registers while z_b is produced, so a link is
//                          register math + an smem flag);
//             k_rest_fwd   WHOLE(s): small supernode in one CTA (front vector
//                          pulled from b and the children's update vectors
//                          through a precomputed map, dense sweep);
//                          UPD(s,u): 32 update rows of a large supernode,
//                          applying every z_b of the chain just finished.
//   backward  k_rest_bwd   COLDOT(s,b): c_b = L21(:,b)^T x(update rows), the
//                          ancestors being final; WHOLE(s) transposed sweep;
//             k_chain_bwd  transposed warp-specialised chain of each large
//                          supernode's pivot part.
// Stream order is the only synchronisation: no flags across CTAs.
#include <cstdlib>
#include <algorithm>

#include "internal.h"
#include "dmma.cuh"
#include "kernels.cuh"
#include "prof.h"

namespace riga {

constexpr int kWholeMaxF = 256;  // max front rows of a small (warp-task) supernode
constexpr int kWholeMaxNp = 64;  // max pivots of a small supernode (substitution mode)
constexpr int kGMaxNp = 128;     // max pivots of a G-mode supernode (any front size; 160 measured: no gain)
constexpr int kGRows = (kGMaxNp + 31) / 32;  // row strips of a lane in k_small_g
constexpr int kWarpPanel = 3328;  // doubles of a warp's staged panel (f * np <= this)
constexpr int kWarpSmem = kWholeMaxF + kWarpPanel;  // doubles of smem per warp task
constexpr int kSolveThreads = 256;
constexpr int kSolveWarps = kSolveThreads / 32;
constexpr int64_t kChainSmemMax = 232448 - 4096;  // staged chain panels must fit this

enum { kWholeGroup = 1, kUpd = 2, kColdot = 3, kGTiles = 4 };

// Update vectors of the forward sweep.  A supernode's update vector is stored where its parent reads it:
// child number k (< kUpdSlots) of parent p writes its entry for the parent's front row r to
// upd[k * nfront + rows_off[p] + r], and a row's gather is one mask byte plus up to kUpdSlots loads at
// addresses known from the row alone -- no index chain (the earlier pull map cost three dependent loads per
// row: gptr -> gsrc -> value).  Entries are written before they are read within a solve and only covered
// entries are read, so the slots are never cleared.  Children beyond kUpdSlots (none in the tensor-product
// dissections; general patterns can have them) keep the pull map over a tail region of the buffer; mask
// bit 7 flags a row with such sources.
constexpr int kUpdSlots = 4;
struct SolveDev {
  const uint8_t* cmask;   // per front row: bit k = child slot k contributes, bit 7 = overflow sources
  const int64_t* ubase;   // per supernode: k * nfront + rows_off[parent] (slot child), or -1
  const int64_t* gptr;    // overflow pull map over front positions (rows_off indexing)
  const int32_t* gsrc;    // its sources in the update-vector buffer
  int64_t nfront;         // front rows of all supernodes = the stride between slots
  int64_t otail;          // start of the overflow children's vectors (+ upd_off[c])
  int permuted;           // right-hand side already in elimination order
};

// where entry t of supernode s's update vector lives
__device__ __forceinline__ double* upd_slot(const SymDev& S, const SolveDev& T, int s, int64_t t, double* upd) {
  const int64_t ub = T.ubase[s];
  return ub >= 0 ? upd + ub + S.relpos[S.upd_off[s] + t] : upd + T.otail + S.upd_off[s] + t;
}

__device__ __forceinline__ double gather_row(const SymDev& S, const SolveDev& T, int s, int64_t r,
                                             int64_t np, int64_t col0, const double* __restrict__ b,
                                             const double* upd) {
  double v = r < np ? b[T.permuted ? col0 + r : S.order[col0 + r]] : 0.0;
  const int64_t g = S.rows_off[s] + r;
  const unsigned m = T.cmask[g];
  if (m == 0u) return v;
  const double* y = upd + g;
  double u[kUpdSlots];
#pragma unroll
  for (int k = 0; k < kUpdSlots; ++k) u[k] = (m >> k & 1u) ? y[k * T.nfront] : 0.0;
#pragma unroll
  for (int k = 0; k < kUpdSlots; ++k) v += u[k];
  if (m & 0x80u) {
    for (int64_t q = T.gptr[g]; q < T.gptr[g + 1]; ++q) v += upd[T.gsrc[q]];
  }
  return v;
}

// --- TMA bulk copy global -> shared, completion on an mbarrier --------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  unsigned ok = 0;
  while (!ok) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(b), "r"(phase)
        : "memory");
  }
}

// unit-lower 32x32 diagonal block solve by one warp, row `lane` in registers
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

// one warp: forward sweep of a small supernode (front in `yw`, <= kWholeMaxF rows).
// 32-bit local indexing; loops are specialised on the real block width so a
// tiny supernode (np = 7) does not pay for 32-wide predicated code.
__device__ __forceinline__ void warp_whole_fwd(const SymDev& S, const SolveDev& T, int s,
                                               const double* __restrict__ panel,
                                               const double* __restrict__ b, double* xp, double* upd,
                                               double* yw, int lane, uint64_t* bar) {
  const int f = (int)S.front[s], np = (int)S.ncol[s];
  const int64_t col0 = S.col0[s];
  const double* P = panel + S.panel_off[s];
  const bool staged = bar && f * np <= kWarpPanel;
  if (staged) {  // the whole panel to shared memory with one bulk copy, overlapping the gather
    double* sp = yw + kWholeMaxF;
    if (lane == 0) bulk_load(sp, P, (unsigned)(((f * np + 1) & ~1) * 8), bar);
    P = sp;
  }
  for (int r = lane; r < f; r += 32) yw[r] = gather_row(S, T, s, r, np, col0, b, upd);
  if (staged) mbar_wait(bar, 0);
  __syncwarp();
  for (int kb = 0; kb < np; kb += 32) {
    const int nbk = min(32, np - kb);
    double z = lane < nbk ? yw[kb + lane] : 0.0;
    if (nbk == 32) {
      z = diag_solve(P, f, kb, 32, lane, z);
    } else {
      const double* Pd = P + kb * f + kb + lane;
      for (int k = 0; k + 1 < nbk; ++k) {
        const double zk = __shfl_sync(0xffffffffu, z, k);
        if (lane > k && lane < nbk) z = fma(-Pd[k * f], zk, z);
      }
    }
    if (lane < nbk) yw[kb + lane] = z;
    __syncwarp();
    const double* Pc = P + kb * f;
    for (int i = kb + nbk + lane; i < f; i += 32) {
      double acc = 0.0;
      if (nbk == 32) {
#pragma unroll
        for (int k = 0; k < 32; ++k) acc = fma(Pc[k * f + i], yw[kb + k], acc);
      } else {
        for (int k = 0; k < nbk; ++k) acc = fma(Pc[k * f + i], yw[kb + k], acc);
      }
      yw[i] -= acc;
    }
    __syncwarp();
  }
  for (int r = lane; r < np; r += 32) xp[col0 + r] = yw[r];
  for (int r = np + lane; r < f; r += 32) *upd_slot(S, T, s, r - np, upd) = yw[r];
}

// one warp: backward sweep of a small supernode
__device__ __forceinline__ void warp_whole_bwd(const SymDev& S, int s, const double* __restrict__ panel,
                                               const double* __restrict__ D, double* xp, double* x,
                                               double* yw, int lane, uint64_t* bar) {
  const int f = (int)S.front[s], np = (int)S.ncol[s];
  const int64_t col0 = S.col0[s];
  const double* P = panel + S.panel_off[s];
  const int32_t* rows = S.rows + S.rows_off[s];
  const bool staged = bar && f * np <= kWarpPanel;
  if (staged) {
    double* sp = yw + kWholeMaxF;
    if (lane == 0) bulk_load(sp, P, (unsigned)(((f * np + 1) & ~1) * 8), bar);
    P = sp;
  }
  for (int r = lane; r < f; r += 32) yw[r] = r < np ? xp[col0 + r] / D[col0 + r] : xp[rows[r]];
  if (staged) mbar_wait(bar, 0);
  __syncwarp();
  const int nblk = (np + 31) / 32;
  for (int bi = nblk - 1; bi >= 0; --bi) {
    const int kb = bi * 32;
    const int nbk = min(32, np - kb);
    double red;  // lane c: sum over rows below the block of L[i][kb+c] y[i]
    if (nbk == 32) {
      double acc[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) acc[c] = 0.0;
      for (int i = kb + 32 + lane; i < f; i += 32) {
        const double yv = yw[i];
#pragma unroll
        for (int c = 0; c < 32; ++c) acc[c] = fma(P[(kb + c) * f + i], yv, acc[c]);
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
#pragma unroll
        for (int k = 0; k < o; ++k) {
          const bool hi = (lane & o) != 0;
          const double send = hi ? acc[k] : acc[k + o];
          const double recv = __shfl_xor_sync(0xffffffffu, send, o);
          acc[k] = (hi ? acc[k + o] : acc[k]) + recv;
        }
      }
      red = acc[0];
    } else {
      red = 0.0;
      for (int c = 0; c < nbk; ++c) {
        const double* Pc = P + (kb + c) * f;
        double a = 0.0;
        for (int i = kb + nbk + lane; i < f; i += 32) a = fma(Pc[i], yw[i], a);
        a = warp_sum(a);
        if (lane == c) red = a;
      }
    }
    double xc = lane < nbk ? yw[kb + lane] - red : 0.0;
    if (nbk == 32) {
      xc = diag_solve_t(P, f, kb, 32, lane, xc);
    } else {
      const double* Pd = P + (kb + lane) * f + kb;
      for (int k = nbk - 1; k >= 1; --k) {
        const double xk = __shfl_sync(0xffffffffu, xc, k);
        if (lane < k) xc = fma(-Pd[k], xk, xc);
      }
    }
    if (lane < nbk) yw[kb + lane] = xc;
    __syncwarp();
  }
  for (int r = lane; r < np; r += 32) {
    xp[col0 + r] = yw[r];
    x[S.order[col0 + r]] = yw[r];
  }
}

// ---------------------------------------------------------------------------
// small supernodes through G = [inv(L11); L21 inv(L11)] (f x np, ld f)
//
// Built once per factorisation (k_small_g), G turns a small supernode's
// whole sweep into one dense mat-vec with no serial dependence:
//     forward   z = G_top y1,  u = y2 - G_bot y1
//     backward  x1 = G^T [z ./ d ; -x2]
// G_top is lower triangular with explicit zeros above the diagonal.
// ---------------------------------------------------------------------------
// Layout: 32-row tiles, tile-major -- G(i, k) at g_off + (i / 32) * (32 np) + 32 k + (i % 32).  A forward
// warp task streams one contiguous np x 256 B block, a backward column group reads 2 KB contiguous per row
// strip; with the earlier column-major f x np layout every 256 B warp load came from a different DRAM page.
__host__ __device__ __forceinline__ int64_t g_doubles(int64_t f, int64_t np) { return (f + 31) / 32 * 32 * np; }

struct GDev {
  const double* g;        // all G blocks
  const int64_t* g_off;   // per supernode offset (-1: large supernode)
  const int2* tiles;      // warp tasks: (supernode, 32-row tile) forward / (supernode, 8-column group) backward
  int on;
  const double* D;        // pivots
  double* wz;             // z ./ d of the small supernodes (forward -> backward), so the
                          // backward column groups of one supernode never read the x
                          // another group of it is writing
};

// ---- static-operand prefetch (before the PDL wait) -------------------------
// Everything a level task reads that the previous kernels of the solve do
// not write -- task lists, front metadata, the pull map, G / inv(L11) /
// panel blocks -- is touched into L2 before griddepcontrol.wait, while the
// predecessor level drains; after the wait only the dynamic vectors (update
// vectors, z, x) are first touches, so a level's dependent-load chain runs
// at L2 latency.  Without a PDL launch the wait is a no-op and the prefetch
// simply runs first.
__device__ __forceinline__ void pf_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

__device__ __forceinline__ void pf_gather(const SymDev& S, const SolveDev& T, int s, int64_t r) {
  pf_l2(T.cmask + S.rows_off[s] + r);
}

// forward G tile (s, t): the G rows of the tile and the gather metadata
__device__ __forceinline__ void pf_gtile_fwd(const SymDev& S, const SolveDev& T, const GDev& GD, int2 task,
                                             int lane) {
  const int s = task.x;
  const int f = (int)S.front[s], np = (int)S.ncol[s];
  const double* G = GD.g + GD.g_off[s] + (int64_t)task.y * 32 * np;  // the tile: np x 32 doubles, contiguous
  for (int q = lane; q < 2 * np; q += 32) pf_l2(G + 16 * q);
  for (int r = lane; r < np; r += 32) pf_gather(S, T, s, r);
  const int i = 32 * task.y + lane;
  if (i >= np && i < f) pf_gather(S, T, s, i);
}

// backward G column group (s, g): its 8 G columns and the front rows
__device__ __forceinline__ void pf_gtile_bwd(const SymDev& S, const GDev& GD, int2 task, int lane) {
  const int s = task.x;
  const int f = (int)S.front[s], np = (int)S.ncol[s];
  const int c0 = 8 * task.y;
  const double* G = GD.g + GD.g_off[s];
  const int nc = min(8, np - c0);
  for (int r = (c0 & ~31) + 32 * (lane >> 3); r < f; r += 128)
    if ((lane & 7) < nc) pf_l2(G + (int64_t)(r >> 5) * 32 * np + 32 * (c0 + (lane & 7)));
  const int32_t* rows = S.rows + S.rows_off[s];
  for (int r = np + 32 * lane; r < f; r += 32 * 32) pf_l2(rows + r);
}

// panel block [c0, c0 + nc) x rows [r0, r1) of a chain supernode (kUpd / kColdot)
__device__ __forceinline__ void pf_panel(const double* P, int64_t f, int64_t c0, int nc, int64_t r0, int64_t r1,
                                         int tid, int nthreads) {
  const int64_t lines = (r1 - r0 + 31) / 32;
  for (int64_t q = tid; q < nc * lines; q += nthreads) {
    const int64_t c = c0 + q / lines, r = r0 + 32 * (q % lines);
    pf_l2(P + c * f + r);
  }
}

// one CTA per G-mode supernode (np <= 32 GR).  inv(L11) by column-oriented
// substitution: warp w owns columns w + 8 j (8 per round), lanes own rows
// lane + 32 ri; x_k is final at step k and broadcast by shuffle.  Then
// G_bot = L21 inv(L11) from inv(L11) in shared memory.  Instantiated per
// width class (GR = 1..4 row strips): shared memory and register work follow
// the class, so the narrow supernodes -- most of them -- run many CTAs per SM.
template <int GR>
__global__ void __launch_bounds__(256) k_small_g(SymDev S, const int32_t* __restrict__ nodes,
                                                 const double* __restrict__ panel,
                                                 const int64_t* __restrict__ g_off, double* __restrict__ gbuf) {
  constexpr int LD = 32 * GR + 1;
  extern __shared__ double Xs[];  // inv(L11) column-major, Xs[c * LD + r]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int s = nodes[blockIdx.x];
  const int f = (int)S.front[s], np = (int)S.ncol[s];
  const double* P = panel + S.panel_off[s];
  double* G = gbuf + g_off[s];
  for (int jb = 0; 64 * jb < np; ++jb) {
    double x[GR][8];
#pragma unroll
    for (int ri = 0; ri < GR; ++ri)
#pragma unroll
      for (int j = 0; j < 8; ++j) x[ri][j] = (lane + 32 * ri == w + 8 * (8 * jb + j)) ? 1.0 : 0.0;
    for (int k = 64 * jb; k + 1 < np; ++k) {
      const int kr = k >> 5, kl = k & 31;
      double l[GR];
#pragma unroll
      for (int ri = 0; ri < GR; ++ri) {
        const int r = lane + 32 * ri;
        l[ri] = (r > k && r < np) ? P[(int64_t)k * f + r] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        double own = x[0][j];
#pragma unroll
        for (int ri = 1; ri < GR; ++ri)
          if (kr == ri) own = x[ri][j];
        const double xk = __shfl_sync(0xffffffffu, own, kl);
#pragma unroll
        for (int ri = 0; ri < GR; ++ri) x[ri][j] = fma(-l[ri], xk, x[ri][j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = w + 8 * (8 * jb + j);
      if (c < np) {
#pragma unroll
        for (int ri = 0; ri < GR; ++ri) {
          const int r = lane + 32 * ri;
          if (r < np) {
            Xs[c * LD + r] = x[ri][j];
            G[(int64_t)ri * 32 * np + 32 * c + lane] = x[ri][j];
          }
        }
      }
    }
  }
  __syncthreads();
  for (int i0 = np; i0 < f; i0 += 32) {
    const int i = i0 + lane;
    for (int jb = 0; 64 * jb < np; ++jb) {
      if (w + 64 * jb >= np) continue;  // this warp's columns of the round are all past np
      double acc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = 0.0;
      for (int k = 64 * jb; k < np; ++k) {  // inv(L11)(k, c) = 0 for k < c
        const double l = i < f ? P[(int64_t)k * f + i] : 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int c = w + 8 * (8 * jb + j);
          acc[j] = fma(l, c < np ? Xs[c * LD + k] : 0.0, acc[j]);
        }
      }
      if (i < f) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int c = w + 8 * (8 * jb + j);
          if (c < np) G[(int64_t)(i >> 5) * 32 * np + 32 * c + (i & 31)] = acc[j];
        }
      }
    }
  }
}

// warp task (s, t): rows [32 t, 32 t + 32) of [z; u] = [0; y2] + [1; -1] .* (G y1)
__device__ __forceinline__ void warp_gtile_fwd(const SymDev& S, const SolveDev& T, const GDev& GD, int2 task,
                                               const double* __restrict__ b, double* xp, double* upd, double* yw,
                                               int lane) {
  const int s = task.x;
  const int f = (int)S.front[s], np = (int)S.ncol[s];
  const int64_t col0 = S.col0[s];
  const double* G = GD.g + GD.g_off[s];
  for (int r = lane; r < np; r += 32) yw[r] = gather_row(S, T, s, r, np, col0, b, upd);
  const int i = 32 * task.y + lane;
  const double yi = (i >= np && i < f) ? gather_row(S, T, s, i, np, col0, b, upd) : 0.0;
  __syncwarp();
  if (i >= f) return;
  // 4 partial sums, 16 independent G loads in flight per lane
  double a4[4] = {0.0, 0.0, 0.0, 0.0};
  const double* Gi = G + (int64_t)task.y * 32 * np + lane;  // the tile's np x 32 block, row `lane`
  int k = 0;
  for (; k + 16 <= np; k += 16) {
    double g[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) g[u] = Gi[(k + u) * 32];
#pragma unroll
    for (int u = 0; u < 16; ++u) a4[u & 3] = fma(g[u], yw[k + u], a4[u & 3]);
  }
#pragma unroll 8
  for (; k < np; ++k) a4[0] = fma(Gi[k * 32], yw[k], a4[0]);
  const double acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
  if (i < np) {
    xp[col0 + i] = acc;
    GD.wz[col0 + i] = acc / GD.D[col0 + i];
  } else {
    *upd_slot(S, T, s, i - np, upd) = yi - acc;
  }
}

// warp task (s, g): x1 for columns [8 g, 8 g + 8) = G^T [z ./ d ; -x2]
__device__ __forceinline__ void warp_gtile_bwd(const SymDev& S, const GDev& GD, int2 task,
                                               const double* __restrict__ D, double* xp, double* x, int lane) {
  const int s = task.x;
  const int f = (int)S.front[s], np = (int)S.ncol[s];
  const int64_t col0 = S.col0[s];
  const int c0 = 8 * task.y;
  const double* G = GD.g + GD.g_off[s];
  const int32_t* rows = S.rows + S.rows_off[s];
  double acc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c] = 0.0;
  const int nc = min(8, np - c0);
  int r = (c0 & ~31) + lane;  // G(r, c) = 0 above the diagonal
  for (; r + 32 < f; r += 64) {  // two row strips per round: 16 G loads in flight per lane
    const int r2 = r + 32;
    const double v1 = r < np ? GD.wz[col0 + r] : -xp[rows[r]];
    const double v2 = r2 < np ? GD.wz[col0 + r2] : -xp[rows[r2]];
    double g1[8], g2[8];
    const double* G1 = G + (int64_t)(r >> 5) * 32 * np + 32 * c0 + lane;  // strip r, columns c0 .. c0 + 8
    const double* G2 = G1 + 32 * np;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      g1[c] = c < nc ? G1[32 * c] : 0.0;
      g2[c] = c < nc ? G2[32 * c] : 0.0;
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = fma(g2[c], v2, fma(g1[c], v1, acc[c]));
  }
  if (r < f) {
    const double v = r < np ? GD.wz[col0 + r] : -xp[rows[r]];
#pragma unroll
    for (int c = 0; c < 8; ++c)
      acc[c] = fma(c < nc ? G[(int64_t)(r >> 5) * 32 * np + 32 * (c0 + c) + lane] : 0.0, v, acc[c]);
  }
#pragma unroll
  for (int o = 4; o >= 1; o >>= 1) {
#pragma unroll
    for (int k = 0; k < o; ++k) {
      const bool hi = (lane & o) != 0;
      const double send = hi ? acc[k] : acc[k + o];
      const double recv = __shfl_xor_sync(0xffffffffu, send, o);
      acc[k] = (hi ? acc[k + o] : acc[k]) + recv;
    }
  }
  double v = acc[0];
  v += __shfl_xor_sync(0xffffffffu, v, 8);
  v += __shfl_xor_sync(0xffffffffu, v, 16);
  const int c = c0 + lane;
  if (lane < 8 && c < np) {
    xp[col0 + c] = v;
    x[S.order[col0 + c]] = v;
  }
}

// ---------------------------------------------------------------------------
// bottom subtrees (G mode): one CTA per maximal subtree of small supernodes
// of height < sub_levels.  Its local levels run back to back separated by
// __syncthreads (CTA-scope visibility of the update vectors / x it wrote),
// so the bottom of the tree costs one launch per sweep instead of one per
// level, and each CTA's chain of small mat-vecs overlaps the others'.
// sub_ptr[i * (SL + 1) + j]: first task of local level j of subtree i.
// ---------------------------------------------------------------------------
// NT threads per subtree CTA (RIGA_SUB_THREADS: 256, 512 or 1024): the warps
// of a CTA stride over a local level's tiles, so a wider CTA keeps more of a
// subtree's loads in flight
template <int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) k_sub_fwd(SymDev S, SolveDev T, GDev GD,
                                                           const int32_t* __restrict__ sub_ptr, int SL,
                                                           const double* __restrict__ b, double* xp, double* upd) {
  constexpr int NW = NT / 32;
  pdl_start();
  __shared__ double y[NW * kGMaxNp];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int32_t* p = sub_ptr + blockIdx.x * (SL + 1);
  for (int j = 0; j < SL; ++j) {
    for (int t = p[j] + w; t < p[j + 1]; t += NW)
      warp_gtile_fwd(S, T, GD, GD.tiles[t], b, xp, upd, y + w * kGMaxNp, lane);
    __syncthreads();
  }
}

template <int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) k_sub_bwd(SymDev S, GDev GD, const int32_t* __restrict__ sub_ptr,
                                                           int SL, const double* __restrict__ D, double* xp,
                                                           double* x) {
  constexpr int NW = NT / 32;
  pdl_start();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int32_t* p = sub_ptr + blockIdx.x * (SL + 1);
  for (int j = SL - 1; j >= 0; --j) {
    for (int t = p[j] + w; t < p[j + 1]; t += NW) warp_gtile_bwd(S, GD, GD.tiles[t], D, xp, x, lane);
    __syncthreads();
  }
}

static int sub_threads() {
  static const int v = [] {
    const char* e = getenv("RIGA_SUB_THREADS");
    const int t = e ? atoi(e) : 256;
    return t >= 1024 ? 1024 : t >= 512 ? 512 : 256;
  }();
  return v;
}

// ---------------------------------------------------------------------------
// light kernels: WHOLE / UPD (forward), WHOLE / COLDOT (backward)
// ---------------------------------------------------------------------------
template <bool GT, int MINB = 4>
__device__ __forceinline__ void k_rest_fwd_body(SymDev S, SolveDev T,
                                                            const int2* __restrict__ tasks, int ntask,
                                                            const int32_t* __restrict__ wholes,
                                                            const double* __restrict__ panel,
                                                            const double* __restrict__ b,
                                                            double* __restrict__ xp,
                                                            double* __restrict__ upd, int stage, GDev GD) {
  extern __shared__ __align__(16) double y[];
  __shared__ double part[kSolveWarps][32];
  __shared__ uint64_t wbar[kSolveWarps];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (blockIdx.x < ntask) {  // static operands of this CTA's first task -> L2
    const int2 t0 = tasks[blockIdx.x];
    const int ty = t0.y >> 24, jj = t0.y & 0x00ffffff;
    if (GT && ty == kGTiles) {
      if (w < jj) pf_gtile_fwd(S, T, GD, GD.tiles[t0.x + w], lane);
    } else if (ty == kUpd) {
      const int64_t f = S.front[t0.x], np = S.ncol[t0.x];
      const int64_t r0 = np + 32 * (int64_t)jj;
      pf_panel(panel + S.panel_off[t0.x], f, 0, (int)np, r0, imin(r0 + 32, f), tid, blockDim.x);
      if (tid < 32 && r0 + tid < f) pf_gather(S, T, t0.x, r0 + tid);
    }
  }
  pdl_start();
  // grid-stride over the level's tasks (the grid may be capped below ntask)
  for (int ti = blockIdx.x; ti < ntask; ti += gridDim.x) {
  const int2 task = tasks[ti];
  const int type = task.y >> 24, j = task.y & 0x00ffffff;
  if (GT && type == kGTiles) {
    if (w < j) warp_gtile_fwd(S, T, GD, GD.tiles[task.x + w], b, xp, upd, y + w * kGMaxNp, lane);
    __syncwarp();
    continue;
  }
  if (!GT && type == kWholeGroup) {
    // warp w: small supernode wholes[task.x + w], whole front in a warp slice
    if (w < j) {
      if (stage && lane == 0) mbar_init(&wbar[w], 1);
      __syncwarp();
      warp_whole_fwd(S, T, wholes[task.x + w], panel, b, xp, upd, y + w * (stage ? kWarpSmem : kWholeMaxF), lane,
                     stage ? &wbar[w] : nullptr);
    }
    __syncwarp();
    continue;
  }
  const int s = task.x;
  const int64_t f = S.front[s], np = S.ncol[s], col0 = S.col0[s];
  const double* P = panel + S.panel_off[s];
  {
    // kUpd: rows [np + 32 j, ...) minus L21 z (all z final)
    const int nbp = (int)((np + 31) / 32);
    const int64_t r0 = np + 32 * (int64_t)j, r1 = imin(r0 + 32, f), r = r0 + lane;
    const bool in = r < r1;
    double acc = 0.0;
    for (int cb = w; cb < nbp; cb += kSolveWarps) {
      const int64_t c0 = 32 * (int64_t)cb;
      const int nc = (int)imin(32, np - c0);
      const double zl = lane < nc ? xp[col0 + c0 + lane] : 0.0;
#pragma unroll 8
      for (int k = 0; k < 32; ++k) {
        const double l = (in && k < nc) ? P[(c0 + k) * f + r] : 0.0;
        acc = fma(l, __shfl_sync(0xffffffffu, zl, k), acc);
      }
    }
    part[w][lane] = acc;
    __syncthreads();
    if (w == 0 && in) {
      double v = gather_row(S, T, s, r, np, col0, b, upd);
#pragma unroll
      for (int q = 0; q < kSolveWarps; ++q) v -= part[q][lane];
      *upd_slot(S, T, s, r - np, upd) = v;
    }
    __syncthreads();  // part[] is reused by the next task of this CTA
  }
  }
}

template <bool GT, int MINB = 4>
__global__ void __launch_bounds__(kSolveThreads, GT ? MINB : 2) k_rest_fwd(SymDev S, SolveDev T,
                                                            const int2* __restrict__ tasks, int ntask,
                                                            const int32_t* __restrict__ wholes,
                                                            const double* __restrict__ panel,
                                                            const double* __restrict__ b,
                                                            double* __restrict__ xp,
                                                            double* __restrict__ upd, int stage, GDev GD) {
  k_rest_fwd_body<GT, MINB>(S, T, tasks, ntask, wholes, panel, b, xp, upd, stage, GD);
}

template <bool GT, int MINB = 4>
__device__ __forceinline__ void k_rest_bwd_body(SymDev S, SolveDev T,
                                                            const int2* __restrict__ tasks, int ntask,
                                                            const int32_t* __restrict__ wholes,
                                                            const double* __restrict__ panel,
                                                            const double* __restrict__ D,
                                                            double* __restrict__ xp,
                                                            double* __restrict__ cvec,
                                                            double* __restrict__ x, int stage, int inv, GDev GD) {
  extern __shared__ __align__(16) double y[];
  __shared__ double part[kSolveWarps][32];
  __shared__ uint64_t wbar[kSolveWarps];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (blockIdx.x < ntask) {  // static operands of this CTA's first task -> L2
    const int2 t0 = tasks[blockIdx.x];
    const int ty = t0.y >> 24, jj = t0.y & 0x00ffffff;
    if (GT && ty == kGTiles) {
      if (w < jj) pf_gtile_bwd(S, GD, GD.tiles[t0.x + w], lane);
    } else if (ty == kColdot) {
      const int64_t f = S.front[t0.x], np = S.ncol[t0.x];
      const int64_t c0 = 32 * (int64_t)jj;
      pf_panel(panel + S.panel_off[t0.x], f, c0, (int)imin(32, np - c0), np, f, tid, blockDim.x);
      const int32_t* rows = S.rows + S.rows_off[t0.x];
      for (int64_t r = np + 32 * tid; r < f; r += 32 * (int64_t)blockDim.x) pf_l2(rows + r);
    }
  }
  pdl_start();
  for (int ti = blockIdx.x; ti < ntask; ti += gridDim.x) {
  const int2 task = tasks[ti];
  const int type = task.y >> 24, bj = task.y & 0x00ffffff;
  if (GT && type == kGTiles) {
    if (w < bj) warp_gtile_bwd(S, GD, GD.tiles[task.x + w], D, xp, x, lane);
    __syncwarp();
    continue;
  }
  if (!GT && type == kWholeGroup) {
    if (w < bj) {
      if (stage && lane == 0) mbar_init(&wbar[w], 1);
      __syncwarp();
      warp_whole_bwd(S, wholes[task.x + w], panel, D, xp, x, y + w * (stage ? kWarpSmem : kWholeMaxF), lane,
                     stage ? &wbar[w] : nullptr);
    }
    __syncwarp();
    continue;
  }
  const int s = task.x;
  const int64_t f = S.front[s], np = S.ncol[s], col0 = S.col0[s];
  const double* P = panel + S.panel_off[s];
  const int32_t* rows = S.rows + S.rows_off[s];
  {
    // kColdot: c[col] = sum_{update rows r} L[r][col] x[rows[r]], col in block bj;
    // warp w: 8-column group (w & 3) over every other 32-row strip (w >> 2),
    // fold-reduced across lanes, then the two row halves summed in order
    const int64_t c0 = 32 * (int64_t)bj + 8 * (w & 3);
    double acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = 0.0;
    for (int64_t r = np + 32 * (w >> 2) + lane; r < f; r += 64) {
      const double xv = xp[rows[r]];
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = fma(c0 + c < np ? P[(c0 + c) * f + r] : 0.0, xv, acc[c]);
    }
#pragma unroll
    for (int o = 4; o >= 1; o >>= 1) {
#pragma unroll
      for (int k = 0; k < o; ++k) {
        const bool hi = (lane & o) != 0;
        const double send = hi ? acc[k] : acc[k + o];
        const double recv = __shfl_xor_sync(0xffffffffu, send, o);
        acc[k] = (hi ? acc[k + o] : acc[k]) + recv;
      }
    }
    double v = acc[0];
    v += __shfl_xor_sync(0xffffffffu, v, 8);
    v += __shfl_xor_sync(0xffffffffu, v, 16);
    if (lane < 8) part[w][lane] = v;
    __syncthreads();
    if (w == 0) {
      const int g = lane >> 3, e = lane & 7;
      const int64_t col = 32 * (int64_t)bj + lane;
      if (col < np) {
        const double t = part[g][e] + part[g + 4][e];
        double* c = cvec + col0 + col;
        *c = inv ? *c - t : t;  // inverse path: cvec already holds z ./ d
      }
    }
    __syncthreads();  // part[] is reused by the next task of this CTA
  }
  }
}

template <bool GT, int MINB = 4>
__global__ void __launch_bounds__(kSolveThreads, GT ? MINB : 2) k_rest_bwd(SymDev S, SolveDev T,
                                                            const int2* __restrict__ tasks, int ntask,
                                                            const int32_t* __restrict__ wholes,
                                                            const double* __restrict__ panel,
                                                            const double* __restrict__ D,
                                                            double* __restrict__ xp,
                                                            double* __restrict__ cvec,
                                                            double* __restrict__ x, int stage, int inv, GDev GD) {
  k_rest_bwd_body<GT, MINB>(S, T, tasks, ntask, wholes, panel, D, xp, cvec, x, stage, inv, GD);
}

// ---------------------------------------------------------------------------
// chain kernels (one CTA per large supernode of the level)
//
// Right-looking over the 32-column pivot blocks.  The column panel a step
// needs -- L[kb : np, kb : kb+32], diagonal block included -- is staged in
// shared memory by cp.async one step ahead (double buffer, even/odd steps),
// so a step is: warp 0 solves the diagonal block from smem, then all
// threads update the rows below from smem.  When the two panels do not fit
// (np > ~460) the loop reads L directly.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// stage the panel of step kb (columns kb..kb+nbk, rows kb..np) into buf,
// layout buf[k * rows + (i - kb)]
__device__ __forceinline__ void stage_panel(double* buf, const double* __restrict__ P, int64_t f,
                                            int64_t np, int64_t kb) {
  const int nbk = (int)imin(32, np - kb);
  const int rows = (int)(np - kb);
  for (int k = 0; k < nbk; ++k) {
    const double* src = P + (kb + k) * f + kb;
    double* dst = buf + (int64_t)k * rows;
    for (int i = threadIdx.x; i < rows; i += blockDim.x) cp_async8(dst + i, src + i);
  }
  cp_async_commit();
}

__host__ __device__ __forceinline__ int64_t chain_panel_doubles(int64_t np) {
  // even steps (kb = 0, 64, ...) use buffer A (max at kb = 0), odd steps B (kb = 32)
  const int64_t a = np * imin(32, np);
  const int64_t b = np > 32 ? (np - 32) * imin(32, np - 32) : 0;
  return a + b;
}

__global__ void __launch_bounds__(kSolveThreads) k_chain_fwd(SymDev S, SolveDev T,
                                                             const int32_t* __restrict__ nodes,
                                                             int staged,
                                                             const double* __restrict__ panel,
                                                             const double* __restrict__ b,
                                                             double* __restrict__ xp,
                                                             const double* __restrict__ upd) {
  pdl_start();
  extern __shared__ double y[];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int s = nodes[blockIdx.x];
  const int64_t f = S.front[s], np = S.ncol[s], col0 = S.col0[s];
  const double* P = panel + S.panel_off[s];
  const bool st = staged && (np + chain_panel_doubles(np)) * 8 <= (int64_t)staged;
  double* bufA = y + np;
  double* bufB = bufA + np * imin(32, np);
  if (st) stage_panel(bufA, P, f, np, 0);
  for (int64_t r = tid; r < np; r += blockDim.x) y[r] = gather_row(S, T, s, r, np, col0, b, upd);
  int step = 0;
  for (int64_t kb = 0; kb < np; kb += 32, ++step) {
    const int nbk = (int)imin(32, np - kb);
    const int64_t rows = np - kb;
    double* cur = (step & 1) ? bufB : bufA;
    if (st) cp_async_wait_all();
    __syncthreads();
    if (st && kb + 32 < np) stage_panel((step & 1) ? bufA : bufB, P, f, np, kb + 32);
    if (w == 0) {
      double yi = lane < nbk ? y[kb + lane] : 0.0;
      if (st) {
        double lrow[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) lrow[k] = (k < lane && lane < nbk) ? cur[k * rows + lane] : 0.0;
#pragma unroll
        for (int k = 0; k < 32; ++k) yi = fma(-lrow[k], __shfl_sync(0xffffffffu, yi, k), yi);
      } else {
        yi = diag_solve(P, f, kb, nbk, lane, yi);
      }
      if (lane < nbk) {
        y[kb + lane] = yi;
        xp[col0 + kb + lane] = yi;
      }
    }
    __syncthreads();
    for (int64_t i = kb + nbk + tid; i < np; i += blockDim.x) {
      double acc = 0.0;
      if (st) {
        const double* c = cur + (i - kb);
#pragma unroll 8
        for (int k = 0; k < nbk; ++k) acc = fma(c[k * rows], y[kb + k], acc);
      } else if (nbk == 32) {
#pragma unroll
        for (int k = 0; k < 32; ++k) acc = fma(P[(kb + k) * f + i], y[kb + k], acc);
      } else {
        for (int k = 0; k < nbk; ++k) acc = fma(P[(kb + k) * f + i], y[kb + k], acc);
      }
      y[i] -= acc;
    }
  }
}

__global__ void __launch_bounds__(kSolveThreads) k_chain_bwd(SymDev S, const int32_t* __restrict__ nodes,
                                                             int staged,
                                                             const double* __restrict__ panel,
                                                             const double* __restrict__ D,
                                                             double* __restrict__ xp,
                                                             const double* __restrict__ cvec,
                                                             double* __restrict__ x) {
  pdl_start();
  extern __shared__ double y[];
  __shared__ double red[kSolveWarps][32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int s = nodes[blockIdx.x];
  const int64_t f = S.front[s], np = S.ncol[s], col0 = S.col0[s];
  const double* P = panel + S.panel_off[s];
  const bool has_upd = f > np;
  const int nblk = (int)((np + 31) / 32);
  const bool st = staged && (np + chain_panel_doubles(np)) * 8 <= (int64_t)staged;
  double* bufA = y + np;
  double* bufB = bufA + np * imin(32, np);
  // backward visits blocks last..0; block bi's panel goes to A if bi is even
  if (st) stage_panel(((nblk - 1) & 1) ? bufB : bufA, P, f, np, 32 * (int64_t)(nblk - 1));
  for (int64_t r = tid; r < np; r += blockDim.x)
    y[r] = xp[col0 + r] / D[col0 + r] - (has_upd ? cvec[col0 + r] : 0.0);
  for (int bi = nblk - 1; bi >= 0; --bi) {
    const int64_t kb = 32 * (int64_t)bi;
    const int nbk = (int)imin(32, np - kb);
    const int64_t rows = np - kb;
    double* cur = (bi & 1) ? bufB : bufA;
    if (st) cp_async_wait_all();
    __syncthreads();
    if (st && bi > 0) stage_panel(((bi - 1) & 1) ? bufB : bufA, P, f, np, kb - 32);
    // dots of the block's columns with the final x below the block (pivot
    // rows): every thread accumulates all 32 columns over its rows (loads
    // independent), then a 31-shuffle transpose-reduce leaves column c's
    // warp sum in lane c
    double acc[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) acc[c] = 0.0;
    for (int64_t i = kb + nbk + tid; i < np; i += blockDim.x) {
      const double yv = y[i];
      if (st) {
        const double* cc = cur + (i - kb);
#pragma unroll
        for (int c = 0; c < 32; ++c) acc[c] = fma(c < nbk ? cc[c * rows] : 0.0, yv, acc[c]);
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) acc[c] = fma(c < nbk ? P[(kb + c) * f + i] : 0.0, yv, acc[c]);
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
#pragma unroll
      for (int k = 0; k < o; ++k) {
        const bool hi = (lane & o) != 0;
        const double send = hi ? acc[k] : acc[k + o];
        const double recv = __shfl_xor_sync(0xffffffffu, send, o);
        acc[k] = (hi ? acc[k + o] : acc[k]) + recv;
      }
    }
    red[w][lane] = acc[0];
    __syncthreads();
    if (w == 0) {
      double xc = lane < nbk ? y[kb + lane] : 0.0;
#pragma unroll
      for (int q = 0; q < kSolveWarps; ++q) xc -= lane < nbk ? red[q][lane] : 0.0;
      if (st) {
        double lcol[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) lcol[k] = (k > lane && k < nbk) ? cur[lane * rows + k] : 0.0;
#pragma unroll
        for (int k = 31; k >= 0; --k) xc = fma(-lcol[k], __shfl_sync(0xffffffffu, xc, k), xc);
      } else {
        xc = diag_solve_t(P, f, kb, nbk, lane, xc);
      }
      if (lane < nbk) {
        y[kb + lane] = xc;
        xp[col0 + kb + lane] = xc;
        x[S.order[col0 + kb + lane]] = xc;
      }
    }
  }
}


// ---------------------------------------------------------------------------
// chain supernodes through the explicit inverse of their pivot block
//
// The pivot block L11 (np x np, unit lower) of every large supernode is
// inverted once per factorisation (k_trinv_diag + doubling GEMMs, part of the
// numeric factorisation), so the dependent 32-column chain of the solve
// becomes two parallel triangular mat-vecs:
//     forward   z  = inv(L11) y1                 (k_inv_fwd, 32-row tiles)
//     backward  x1 = inv(L11)^T (z ./ d - L21^T x2)  (k_inv_bwd, warp per row)
// spread over many CTAs instead of one CTA walking np/32 serial steps.
// Layout: inv(L11) column-major, ld np, at linv + inv_off[s]; entries above
// the diagonal inside a diagonal 32x32 block are zero (the tiles read them).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_trinv_diag(SymDev S, const int2* __restrict__ tasks, int ntask,
                                                    const double* __restrict__ panel,
                                                    const int64_t* __restrict__ inv_off, double* linv) {
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= ntask) return;
  const int s = tasks[t].x;
  const int f = (int)S.front[s], np = (int)S.ncol[s];
  const int j0 = 32 * tasks[t].y, nb = min(32, np - j0);
  const double* P = panel + S.panel_off[s];
  // lane c: column c of inv(L_bb), rows in order: x_r = [r == c] - sum_{c<=k<r} L(r,k) x_k
  double x[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    double v = r == lane ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < r; ++k) v = (k >= lane && r < nb) ? fma(-P[(int64_t)(j0 + k) * f + j0 + r], x[k], v) : v;
    x[r] = v;
  }
  if (lane < nb) {
    double* X = linv + inv_off[s] + (int64_t)(j0 + lane) * np + j0;
#pragma unroll
    for (int r = 0; r < 32; ++r)
      if (r < nb) X[r] = x[r];
  }
}

// Doubling: with inv(A) and inv(C) of two adjacent diagonal blocks of size
// s (A = [a0, a0+s), C = [c0, c0+sc), c0 = a0 + s) known,
//     inv([A 0; B C]) = [inv(A) 0; -inv(C) B inv(A)  inv(C)],
// so level s (s = 32, 64, 128, ...) fills every off-diagonal block X21 with
// two batched DMMA GEMMs: T = B inv(A) (K range skips inv(A)'s zero upper
// part), then X21 = -inv(C) T (K range stops at the tile's last row).
// Task (supernode, q): the pair starting at a0 = 2 q s.
__global__ void __launch_bounds__(128) k_trinv_gemm1(SymDev S, const int2* __restrict__ tasks, int sz,
                                                     const double* __restrict__ panel,
                                                     const int64_t* __restrict__ inv_off,
                                                     const int64_t* __restrict__ t_off, const double* linv,
                                                     double* tbuf) {
  const int2 task = tasks[blockIdx.y];
  const int s = task.x;
  const int64_t f = S.front[s], np = S.ncol[s];
  const int64_t a0 = 2 * (int64_t)task.y * sz, c0 = a0 + sz, sc = imin(sz, np - c0);
  const int64_t nti = (sc + 63) / 64, ntj = (sz + 63) / 64;
  if (blockIdx.x >= nti * ntj) return;
  const int64_t i0 = 64 * (blockIdx.x % nti), j0 = 64 * (blockIdx.x / nti);
  const double* B = panel + S.panel_off[s] + a0 * f + c0;   // B(i, t) = L(c0 + i, a0 + t)
  const double* Ai = linv + inv_off[s] + a0 * np + a0;      // inv(A)(t, j) at [j np + t]
  double* T = tbuf + t_off[blockIdx.y];                      // T(i, j) at [j sc + i]
  dmma_gemm_tile(B, f, Ai, np, j0, sz, i0, j0, sc, sz, T, sc, 1.0);
}

__global__ void __launch_bounds__(128) k_trinv_gemm2(SymDev S, const int2* __restrict__ tasks, int sz,
                                                     const int64_t* __restrict__ inv_off,
                                                     const int64_t* __restrict__ t_off, const double* tbuf,
                                                     double* linv) {
  const int2 task = tasks[blockIdx.y];
  const int s = task.x;
  const int64_t np = S.ncol[s];
  const int64_t a0 = 2 * (int64_t)task.y * sz, c0 = a0 + sz, sc = imin(sz, np - c0);
  const int64_t nti = (sc + 63) / 64, ntj = (sz + 63) / 64;
  if (blockIdx.x >= nti * ntj) return;
  const int64_t i0 = 64 * (blockIdx.x % nti), j0 = 64 * (blockIdx.x / nti);
  double* X = linv + inv_off[s];
  const double* Ci = X + c0 * np + c0;   // inv(C)(i, t) at [t np + i]
  const double* T = tbuf + t_off[blockIdx.y];  // T(t, j) at [j sc + t]
  dmma_gemm_tile(Ci, np, T, sc, 0, imin(i0 + 64, sc), i0, j0, sc, sz, X + a0 * np + c0, np, -1.0);
}

// forward: task (s, t) -> z rows [32t, 32t + 32) of supernode s
__device__ __forceinline__ void k_inv_fwd_body(SymDev S, SolveDev T, const int2* __restrict__ tasks,
                                                 const int64_t* __restrict__ inv_off,
                                                 const double* __restrict__ linv,
                                                 const double* __restrict__ D, const double* __restrict__ b,
                                                 double* __restrict__ xp, const double* __restrict__ upd,
                                                 double* __restrict__ cvec) {
  extern __shared__ double y[];
  __shared__ double part[8][32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int s = tasks[blockIdx.x].x;
  const int np = (int)S.ncol[s];
  const int64_t col0 = S.col0[s];
  {  // static operands -> L2: the 32-row strip of inv(L11), the gather metadata
    const int rr0 = 32 * tasks[blockIdx.x].y, rr1 = min(np, rr0 + 32);
    const double* A = linv + inv_off[s] + rr0;
    for (int k = tid; k < rr1; k += 256) {
      pf_l2(A + (int64_t)k * np);
      pf_gather(S, T, s, k);
    }
  }
  pdl_start();
  const int r0 = 32 * tasks[blockIdx.x].y, r1 = min(np, r0 + 32);
  for (int k = tid; k < r1; k += 256) y[k] = gather_row(S, T, s, k, np, col0, b, upd);
  __syncthreads();
  const int chunk = (r1 + 7) / 8;
  const int k0 = w * chunk, k1 = min(r1, k0 + chunk);
  const double* A = linv + inv_off[s] + r0 + lane;
  double acc = 0.0;
  if (r0 + lane < r1) {
#pragma unroll 4
    for (int k = k0; k < k1; ++k) acc = fma(A[(int64_t)k * np], y[k], acc);
  }
  part[w][lane] = acc;
  __syncthreads();
  if (w == 0 && r0 + lane < r1) {
    double z = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) z += part[q][lane];
    const int64_t g = col0 + r0 + lane;
    xp[g] = z;
    cvec[g] = z / D[g];  // backward right-hand side; COLDOT subtracts L21^T x2
  }
}

__global__ void __launch_bounds__(256) k_inv_fwd(SymDev S, SolveDev T, const int2* __restrict__ tasks,
                                                 const int64_t* __restrict__ inv_off,
                                                 const double* __restrict__ linv,
                                                 const double* __restrict__ D, const double* __restrict__ b,
                                                 double* __restrict__ xp, const double* __restrict__ upd,
                                                 double* __restrict__ cvec) {
  k_inv_fwd_body(S, T, tasks, inv_off, linv, D, b, xp, upd, cvec);
}

// backward: warp per pivot row r, x1[r] = sum_{k>=r} inv(L11)(k, r) w[k], w in cvec
__device__ __forceinline__ void k_inv_bwd_body(SymDev S, const int2* __restrict__ tasks,
                                                 const int64_t* __restrict__ inv_off,
                                                 const double* __restrict__ linv,
                                                 const double* __restrict__ cvec, double* __restrict__ xp,
                                                 double* __restrict__ x) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int s = tasks[blockIdx.x].x;
  const int np = (int)S.ncol[s];
  const int r = 8 * tasks[blockIdx.x].y + w;
  if (r < np) {  // static: this row of inv(L11) -> L2
    const double* A = linv + inv_off[s] + (int64_t)r * np;
    for (int k = (r & ~31) + 32 * lane; k < np; k += 32 * 32) pf_l2(A + k);
  }
  pdl_start();
  if (r >= np) return;
  const int64_t col0 = S.col0[s];
  const double* A = linv + inv_off[s] + (int64_t)r * np;
  const double* wv = cvec + col0;
  double acc = 0.0;
#pragma unroll 4
  for (int k = r + lane; k < np; k += 32) acc = fma(A[k], wv[k], acc);
  acc = warp_sum(acc);
  if (lane == 0) {
    xp[col0 + r] = acc;
    x[S.order[col0 + r]] = acc;
  }
}

__global__ void __launch_bounds__(256) k_inv_bwd(SymDev S, const int2* __restrict__ tasks,
                                                 const int64_t* __restrict__ inv_off,
                                                 const double* __restrict__ linv,
                                                 const double* __restrict__ cvec, double* __restrict__ xp,
                                                 double* __restrict__ x) {
  k_inv_bwd_body(S, tasks, inv_off, linv, cvec, xp, x);
}

// ---------------------------------------------------------------------------
// Chain supernodes: one step of local iterative refinement after each explicit
// inverse application.  Applying inv(L11) is not backward stable when L11 is
// ill-conditioned (unpivoted indefinite LDL^T): on cfg5 the inverse-only solve
// has backward error 1e-8 against 2e-11 for substitution, which caps the
// Lanczos residuals above north_star's 1e-8.  With z = inv~ y the correction
// z += inv~ (y - L11 z) leaves an error E L11 E y (quadratic in the inverse's
// error E): substitution-level accuracy for two extra sweeps over L11 / inv.
//   forward:  r = y - L11 z  (rows: warps split K, lanes = 32 rows, as k_inv_fwd)
//             z += inv(L11) r;  cvec = z / d
//   backward: r = w - L11^T x1  (warp per pivot row: column of L11, coalesced)
//             x1 += inv(L11)^T r
// ---------------------------------------------------------------------------
// Factor-time accuracy probe of each chain inverse: u = inv~ v for a fixed v, then
// err[s] = max_i |(L11 u)_i - v_i| / max|v| (the solve's local backward error on
// this supernode).  Supernodes above RIGA_INV_FIX_TOL (1e-11) get the refinement step.
__device__ __forceinline__ double chk_v(int k) {  // pseudo-random signs and magnitudes in [0.5, 1)
  const unsigned h = (unsigned)k * 2654435761u;
  return ((h >> 31) ? -1.0 : 1.0) * (0.5 + (double)((h >> 8) & 0xffff) / 131072.0);
}

__global__ void __launch_bounds__(256) k_inv_chk1(SymDev S, const int2* __restrict__ tasks,
                                                  const int64_t* __restrict__ inv_off,
                                                  const double* __restrict__ linv, double* __restrict__ u) {
  __shared__ double part[8][32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int s = tasks[blockIdx.x].x;
  const int np = (int)S.ncol[s];
  const int r0 = 32 * tasks[blockIdx.x].y, r1 = min(np, r0 + 32);
  const int chunk = (r1 + 7) / 8;
  const int k0 = w * chunk, k1 = min(r1, k0 + chunk);
  const double* A = linv + inv_off[s] + r0 + lane;
  double acc = 0.0;
  if (r0 + lane < r1)
    for (int k = k0; k < k1; ++k) acc = fma(A[(int64_t)k * np], chk_v(k), acc);
  part[w][lane] = acc;
  __syncthreads();
  if (w == 0 && r0 + lane < r1) {
    double z = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) z += part[q][lane];
    u[S.col0[s] + r0 + lane] = z;
  }
}

__global__ void __launch_bounds__(256) k_inv_chk2(SymDev S, const int2* __restrict__ tasks,
                                                  const double* __restrict__ panel, const double* __restrict__ u,
                                                  unsigned long long* __restrict__ err) {
  __shared__ double part[8][32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int s = tasks[blockIdx.x].x;
  const int np = (int)S.ncol[s];
  const int f = (int)S.front[s];
  const int64_t col0 = S.col0[s];
  const int r0 = 32 * tasks[blockIdx.x].y, r1 = min(np, r0 + 32);
  const int i = r0 + lane;
  const int chunk = (r1 + 7) / 8;
  const int k0 = w * chunk, k1 = min(r1, k0 + chunk);
  const double* P = panel + S.panel_off[s] + i;
  double acc = 0.0;
  if (i < r1) {
    const int kk1 = min(k1, i);
    for (int k = k0; k < kk1; ++k) acc = fma(P[(int64_t)k * f], u[col0 + k], acc);
  }
  part[w][lane] = acc;
  __syncthreads();
  if (w == 0) {
    double e = 0.0;
    if (i < r1) {
      double t = u[col0 + i];
#pragma unroll
      for (int q = 0; q < 8; ++q) t += part[q][lane];
      e = fabs(t - chk_v(i));  // max|v| < 1
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e = fmax(e, __shfl_xor_sync(0xffffffffu, e, o));
    if (lane == 0 && e > 0.0) atomicMax(err + s, (unsigned long long)__double_as_longlong(e));
  }
}

__global__ void __launch_bounds__(256) k_inv_fix_fwd_res(SymDev S, SolveDev T, const int2* __restrict__ tasks,
                                                         const int* __restrict__ flag, const double* __restrict__ panel,
                                                         const double* __restrict__ b, const double* __restrict__ xp,
                                                         const double* __restrict__ upd, double* __restrict__ rfix) {
  extern __shared__ double zsh[];
  __shared__ double part[8][32];
  pdl_start();
  if (flag && !flag[tasks[blockIdx.x].x]) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int s = tasks[blockIdx.x].x;
  const int np = (int)S.ncol[s];
  const int f = (int)S.front[s];
  const int64_t col0 = S.col0[s];
  const int r0 = 32 * tasks[blockIdx.x].y, r1 = min(np, r0 + 32);
  for (int k = tid; k < r1; k += 256) zsh[k] = xp[col0 + k];
  __syncthreads();
  const int i = r0 + lane;
  const int kend = r1 - 1;  // rows i of this tile use the columns k < i <= r1 - 1
  const int chunk = (kend + 7) / 8;
  const int k0 = w * chunk, k1 = min(kend, k0 + chunk);
  const double* P = panel + S.panel_off[s] + i;
  double acc = 0.0;
  if (i < r1) {
    const int kk1 = min(k1, i);
#pragma unroll 4
    for (int k = k0; k < kk1; ++k) acc = fma(P[(int64_t)k * f], zsh[k], acc);
  }
  part[w][lane] = acc;
  __syncthreads();
  if (w == 0 && i < r1) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) t += part[q][lane];
    const double y = gather_row(S, T, s, i, np, col0, b, upd);
    rfix[col0 + i] = (y - zsh[i]) - t;
  }
}

__global__ void __launch_bounds__(256) k_inv_fix_fwd_apply(SymDev S, const int2* __restrict__ tasks,
                                                           const int* __restrict__ flag,
                                                           const int64_t* __restrict__ inv_off,
                                                           const double* __restrict__ linv,
                                                           const double* __restrict__ D,
                                                           const double* __restrict__ rfix, double* __restrict__ xp,
                                                           double* __restrict__ cvec) {
  extern __shared__ double y[];
  __shared__ double part[8][32];
  pdl_start();
  if (flag && !flag[tasks[blockIdx.x].x]) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int s = tasks[blockIdx.x].x;
  const int np = (int)S.ncol[s];
  const int64_t col0 = S.col0[s];
  const int r0 = 32 * tasks[blockIdx.x].y, r1 = min(np, r0 + 32);
  for (int k = tid; k < r1; k += 256) y[k] = rfix[col0 + k];
  __syncthreads();
  const int chunk = (r1 + 7) / 8;
  const int k0 = w * chunk, k1 = min(r1, k0 + chunk);
  const double* A = linv + inv_off[s] + r0 + lane;
  double acc = 0.0;
  if (r0 + lane < r1) {
#pragma unroll 4
    for (int k = k0; k < k1; ++k) acc = fma(A[(int64_t)k * np], y[k], acc);
  }
  part[w][lane] = acc;
  __syncthreads();
  if (w == 0 && r0 + lane < r1) {
    double dz = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) dz += part[q][lane];
    const int64_t g = col0 + r0 + lane;
    const double z = xp[g] + dz;
    xp[g] = z;
    cvec[g] = z / D[g];
  }
}

__global__ void __launch_bounds__(256) k_inv_fix_bwd_res(SymDev S, const int2* __restrict__ tasks,
                                                         const int* __restrict__ flag, const double* __restrict__ panel,
                                                         const double* __restrict__ cvec,
                                                         const double* __restrict__ xp, double* __restrict__ rfix) {
  pdl_start();
  if (flag && !flag[tasks[blockIdx.x].x]) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int s = tasks[blockIdx.x].x;
  const int np = (int)S.ncol[s];
  const int r = 8 * tasks[blockIdx.x].y + w;
  if (r >= np) return;
  const int f = (int)S.front[s];
  const int64_t col0 = S.col0[s];
  const double* P = panel + S.panel_off[s] + (int64_t)r * f;  // column r of L11
  const double* xv = xp + col0;
  double acc = 0.0;
#pragma unroll 4
  for (int k = r + 1 + lane; k < np; k += 32) acc = fma(P[k], xv[k], acc);
  acc = warp_sum(acc);
  if (lane == 0) rfix[col0 + r] = (cvec[col0 + r] - xv[r]) - acc;
}

__global__ void __launch_bounds__(256) k_inv_fix_bwd_apply(SymDev S, const int2* __restrict__ tasks,
                                                           const int* __restrict__ flag,
                                                           const int64_t* __restrict__ inv_off,
                                                           const double* __restrict__ linv,
                                                           const double* __restrict__ rfix, double* __restrict__ xp,
                                                           double* __restrict__ x) {
  pdl_start();
  if (flag && !flag[tasks[blockIdx.x].x]) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int s = tasks[blockIdx.x].x;
  const int np = (int)S.ncol[s];
  const int r = 8 * tasks[blockIdx.x].y + w;
  if (r >= np) return;
  const int64_t col0 = S.col0[s];
  const double* A = linv + inv_off[s] + (int64_t)r * np;
  const double* rv = rfix + col0;
  double acc = 0.0;
#pragma unroll 4
  for (int k = r + lane; k < np; k += 32) acc = fma(A[k], rv[k], acc);
  acc = warp_sum(acc);
  if (lane == 0) {
    const double v = xp[col0 + r] + acc;
    xp[col0 + r] = v;
    x[S.order[col0 + r]] = v;
  }
}

// ---------------------------------------------------------------------------
// host: per-level task lists, pull map
// ---------------------------------------------------------------------------
static int env_flag(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

// bottom subtrees of G supernodes below this height run as one CTA each
// (k_sub_fwd/bwd).  cfg3 A/B of the solve: 6 is best for a few concurrent
// slices, 7 for 16 (+12 % solves/s, lone solve +1 %; 8: +9 %, lone +23 %);
// riga_set_solve_sub_levels picks it per run (slicing.solve_sub_levels),
// RIGA_SUB_LEVELS overrides.  Read when a symbolic analysis builds its solve plan.
static int g_sub_levels = 6;

int build_solve_plan(riga_symbolic* sym) {
  const SymbolicHost& h = sym->h;
  SolvePlanHost& L = sym->sp;
  const int64_t ns = h.nsuper;
  L = SolvePlanHost();
  // TMA staging of small panels (a 229 KB block per 8 warps) only pays for a
  // solve running alone; concurrent slice streams want small blocks that
  // co-reside, so it is opt-in (RIGA_WARP_STAGE=1)
  L.warp_stage = env_flag("RIGA_WARP_STAGE", 0);
  // chain supernodes through inv(L11) (default) or the serial chain kernels
  L.chain_inv = env_flag("RIGA_CHAIN_INV", 1);
  // one local refinement step after every inv(L11) application (backward stability; RIGA_INV_FIX=0 off)
  L.inv_fix = env_flag("RIGA_INV_FIX", 1);
  // small supernodes through G = [inv(L11); L21 inv(L11)] (default) or substitution
  L.small_g = env_flag("RIGA_SMALL_G", 1);
  L.occ = env_flag("RIGA_REST_OCC", 4);  // CTAs per SM the G-mode level kernels are register-bounded for
  L.rest_cap = env_flag("RIGA_REST_CAP", 1 << 30);  // CTAs per level launch (grid-stride over the tasks)
  L.g_off.assign(ns, -1);
  L.inv_off.assign(ns, -1);
  L.ifwd_ptr.assign(h.nlevels + 1, 0);
  L.ibwd_ptr.assign(h.nlevels + 1, 0);
  L.ifwd_smem.assign(h.nlevels, 8);
  auto large = [&](int64_t s) {
    return L.small_g ? h.ncol[s] > kGMaxNp : (h.ncol[s] > kWholeMaxNp || h.front[s] > kWholeMaxF);
  };
  // bottom subtrees (G mode): maximal subtrees of small supernodes of height
  // < sub_levels; supernodes are numbered in postorder, so a subtree is a
  // contiguous range
  L.sub_levels = L.small_g ? env_flag("RIGA_SUB_LEVELS", g_sub_levels) : 0;
  std::vector<char> in_sub(ns, 0);
  if (L.sub_levels > 0) {
    const int SL = L.sub_levels;
    std::vector<int32_t> size(ns, 1);
    std::vector<char> ok(ns, 1);
    for (int64_t s = 0; s < ns; ++s) {
      if (large(s) || h.level[s] >= SL) ok[s] = 0;
      for (int64_t q = h.child_ptr[s]; q < h.child_ptr[s + 1]; ++q) {
        const int32_t c = h.child_list[q];
        size[s] += size[c];
        if (!ok[c]) ok[s] = 0;
      }
    }
    for (int64_t s = 0; s < ns; ++s) {
      const int32_t par = h.sparent[s];
      if (!ok[s] || (par >= 0 && ok[par])) continue;  // not a maximal subtree root
      std::vector<std::vector<int32_t>> byl(SL);
      for (int64_t q = s - size[s] + 1; q <= s; ++q) {
        byl[h.level[q]].push_back((int32_t)q);
        in_sub[q] = 1;
        L.g_off[q] = L.g_total;
        L.g_total += g_doubles(h.front[q], h.ncol[q]);
        L.wholes.push_back((int32_t)q);
      }
      for (int j = 0; j < SL; ++j) {
        L.sub_fptr.push_back((int32_t)L.sub_ftiles.size());
        L.sub_bptr.push_back((int32_t)L.sub_btiles.size());
        for (int32_t q : byl[j]) {
          for (int32_t t = 0; t < (int32_t)((h.front[q] + 31) / 32); ++t) L.sub_ftiles.push_back({q, t});
          for (int32_t g = 0; g < (int32_t)((h.ncol[q] + 7) / 8); ++g) L.sub_btiles.push_back({q, g});
        }
      }
      L.sub_fptr.push_back((int32_t)L.sub_ftiles.size());
      L.sub_bptr.push_back((int32_t)L.sub_btiles.size());
      L.sub_maxsn = std::max(L.sub_maxsn, size[s]);
      ++L.nsub;
    }
  }
  L.fwd_ptr.assign(h.nlevels + 1, 0);
  L.bwd_ptr.assign(h.nlevels + 1, 0);
  L.chain_ptr.assign(h.nlevels + 1, 0);
  L.fwd_smem.assign(h.nlevels, 8);
  L.bwd_smem.assign(h.nlevels, 8);
  L.chf_smem.assign(h.nlevels, 8);
  L.chb_smem.assign(h.nlevels, 8);
  auto code = [](int type, int j) { return (int32_t)((type << 24) | j); };
  for (int64_t l = 0; l < h.nlevels; ++l) {
    std::vector<int32_t> nodes(h.level_nodes.begin() + h.level_ptr[l],
                               h.level_nodes.begin() + h.level_ptr[l + 1]);
    std::stable_sort(nodes.begin(), nodes.end(), [&](int32_t a, int32_t b) {
      return h.ncol[a] * h.front[a] > h.ncol[b] * h.front[b];
    });
    int64_t smf = 1, smb = 1, scf = 1, scb = 1;
    std::vector<int32_t> small;
    for (int32_t s : nodes) {
      if (in_sub[s]) continue;
      if (large(s)) {
        const int64_t np = h.ncol[s], nblk = (np + 31) / 32;
        L.chains.push_back(s);
        L.inv_off[s] = L.inv_total;
        L.inv_total += np * np;
        for (int64_t t = 0; t < nblk; ++t) {
          L.ifwd.push_back({s, (int32_t)t});
          L.idiag.push_back({s, (int32_t)t});
        }
        for (int64_t g = 0; g < (np + 7) / 8; ++g) L.ibwd.push_back({s, (int32_t)g});
        L.ifwd_smem[l] = std::max<int64_t>(L.ifwd_smem[l], np * 8);
        const int64_t want = np + chain_panel_doubles(np);
        const int64_t fit = want * 8 <= kChainSmemMax ? want : np;
        scf = std::max<int64_t>(scf, fit);
        scb = std::max<int64_t>(scb, fit);
        const int64_t nbu = (h.front[s] - np + 31) / 32;
        for (int64_t u = 0; u < nbu; ++u) L.fwd.push_back({s, code(kUpd, (int)u)});
        if (nbu > 0) {
          for (int64_t bb = 0; bb < nblk; ++bb) L.bwd.push_back({s, code(kColdot, (int)bb)});
        }
      } else {
        small.push_back(s);
        L.g_off[s] = L.g_total;
        L.g_total += g_doubles(h.front[s], h.ncol[s]);
      }
    }
    if (L.small_g) {
      // small supernodes through G: warp tasks (32-row tiles forward,
      // 8-column groups backward), 8 per CTA
      std::vector<I2> tf, tb;
      for (int32_t s : small) {
        for (int32_t t = 0; t < (int32_t)((h.front[s] + 31) / 32); ++t) tf.push_back({s, t});
        for (int32_t g = 0; g < (int32_t)((h.ncol[s] + 7) / 8); ++g) tb.push_back({s, g});
      }
      for (size_t q = 0; q < tf.size(); q += kSolveWarps) {
        const int cnt = (int)std::min<size_t>(kSolveWarps, tf.size() - q);
        L.fwd.push_back({(int32_t)(L.gfwd.size() + q), code(kGTiles, cnt)});
      }
      for (size_t q = 0; q < tb.size(); q += kSolveWarps) {
        const int cnt = (int)std::min<size_t>(kSolveWarps, tb.size() - q);
        L.bwd.push_back({(int32_t)(L.gbwd.size() + q), code(kGTiles, cnt)});
      }
      L.gfwd.insert(L.gfwd.end(), tf.begin(), tf.end());
      L.gbwd.insert(L.gbwd.end(), tb.begin(), tb.end());
    } else {
      // small supernodes: groups of 8, one warp each
      for (size_t q = 0; q < small.size(); q += kSolveWarps) {
        const int cnt = (int)std::min<size_t>(kSolveWarps, small.size() - q);
        const int32_t first = (int32_t)L.wholes.size() + (int32_t)q;
        L.fwd.push_back({first, code(kWholeGroup, cnt)});
        L.bwd.push_back({first, code(kWholeGroup, cnt)});
      }
    }
    L.wholes.insert(L.wholes.end(), small.begin(), small.end());
    if (!small.empty()) {
      const int64_t per = L.small_g ? kGMaxNp : L.warp_stage ? kWarpSmem : kWholeMaxF;
      smf = std::max<int64_t>(smf, kSolveWarps * per);
      smb = std::max<int64_t>(smb, kSolveWarps * per);
    }
    L.fwd_ptr[l + 1] = (int64_t)L.fwd.size();
    L.bwd_ptr[l + 1] = (int64_t)L.bwd.size();
    L.chain_ptr[l + 1] = (int64_t)L.chains.size();
    L.ifwd_ptr[l + 1] = (int64_t)L.ifwd.size();
    L.ibwd_ptr[l + 1] = (int64_t)L.ibwd.size();
    L.fwd_smem[l] = smf * 8;
    L.bwd_smem[l] = smb * 8;
    L.chf_smem[l] = scf * 8;
    L.chb_smem[l] = scb * 8;
  }
  // G-mode supernodes by width class for k_small_g<GR> (np <= 32 GR), large fronts first inside a class
  L.gnodes = L.wholes;
  std::stable_sort(L.gnodes.begin(), L.gnodes.end(), [&](int32_t a, int32_t b) {
    const int64_t ca = (h.ncol[a] + 31) / 32, cb = (h.ncol[b] + 31) / 32;
    return ca != cb ? ca < cb : h.front[a] > h.front[b];
  });
  for (int c = 0; c <= 4; ++c)
    L.gcls_ptr[c] = std::lower_bound(L.gnodes.begin(), L.gnodes.end(), c,
                                     [&](int32_t a, int cls) { return (h.ncol[a] + 31) / 32 <= cls; }) -
                    L.gnodes.begin();
  // doubling levels of the pivot-block inversions: level l pairs adjacent
  // diagonal blocks of size 32 << l; T scratch offsets per task
  for (int64_t sz = 32, lev = 0;; sz *= 2, ++lev) {
    std::vector<I2> tk;
    std::vector<int64_t> toff;
    int64_t tt = 0, maxt = 0;
    for (int32_t s : L.chains) {
      const int64_t np = h.ncol[s];
      for (int64_t q = 0; 2 * q * sz + sz < np; ++q) {
        const int64_t sc = std::min<int64_t>(sz, np - (2 * q * sz + sz));
        tk.push_back({s, (int32_t)q});
        toff.push_back(tt);
        tt += sc * sz;
        maxt = std::max<int64_t>(maxt, ((sc + 63) / 64) * ((sz + 63) / 64));
      }
    }
    if (tk.empty()) break;
    L.dbl_size.push_back(sz);
    L.dbl_ptr.push_back((int64_t)L.dbl_tasks.size());
    L.dbl_tiles.push_back(maxt);
    L.dbl_tasks.insert(L.dbl_tasks.end(), tk.begin(), tk.end());
    L.dbl_toff.insert(L.dbl_toff.end(), toff.begin(), toff.end());
    L.dbl_tmax = std::max(L.dbl_tmax, tt);
  }
  L.dbl_ptr.push_back((int64_t)L.dbl_tasks.size());
  // update-vector slots: child number k < kUpdSlots of a parent writes straight into the parent's front
  // rows of slot k; later children keep a pull map over a tail region (SolveDev)
  const int64_t nfront = h.rows_off[ns];
  L.nfront = nfront;
  L.otail = (int64_t)kUpdSlots * nfront;
  L.cmask.assign(nfront, 0);
  L.ubase.assign(ns, -1);
  std::vector<int64_t> cnt(nfront + 1, 0);
  bool overflow = false;
  for (int64_t p = 0; p < ns; ++p)
    for (int64_t q = h.child_ptr[p]; q < h.child_ptr[p + 1]; ++q) {
      const int64_t c = h.child_list[q], k = q - h.child_ptr[p];
      if (k < kUpdSlots) L.ubase[c] = k * nfront + h.rows_off[p];
      for (int64_t t = 0; t < h.front[c] - h.ncol[c]; ++t) {
        const int64_t g = h.rows_off[p] + h.relpos[h.upd_off[c] + t];
        if (k < kUpdSlots) {
          L.cmask[g] |= (uint8_t)(1u << k);
        } else {
          L.cmask[g] |= 0x80u;
          cnt[g + 1]++;
          overflow = true;
        }
      }
    }
  L.upd_doubles = L.otail + (overflow ? h.upd_total : 0);
  for (int64_t i = 0; i < nfront; ++i) cnt[i + 1] += cnt[i];
  L.gptr = cnt;
  L.gsrc.assign(cnt[nfront], 0);
  if (overflow) {
    std::vector<int64_t> fillp(cnt.begin(), cnt.end() - 1);
    for (int64_t p = 0; p < ns; ++p)
      for (int64_t q = h.child_ptr[p] + kUpdSlots; q < h.child_ptr[p + 1]; ++q) {
        const int64_t c = h.child_list[q];
        for (int64_t t = 0; t < h.front[c] - h.ncol[c]; ++t)
          L.gsrc[fillp[h.rows_off[p] + h.relpos[h.upd_off[c] + t]]++] = (int32_t)(L.otail + h.upd_off[c] + t);
      }
  }
  return RIGA_OK;
}

int upload_solve_plan(riga_symbolic* sym, cudaStream_t s) {
  SolvePlanHost& L = sym->sp;
  if (!L.fwd.empty()) RIGA_TRY(sym->d_tfwd.upload(L.fwd.data(), L.fwd.size(), s));
  if (!L.bwd.empty()) RIGA_TRY(sym->d_tbwd.upload(L.bwd.data(), L.bwd.size(), s));
  if (!L.chains.empty()) RIGA_TRY(sym->d_chains.upload(L.chains.data(), L.chains.size(), s));
  if (!L.wholes.empty()) RIGA_TRY(sym->d_wholes.upload(L.wholes.data(), L.wholes.size(), s));
  if (!L.gnodes.empty()) RIGA_TRY(sym->d_gnodes.upload(L.gnodes.data(), L.gnodes.size(), s));
  if (L.nsub) {
    RIGA_TRY(sym->d_sub_fptr.upload(L.sub_fptr.data(), L.sub_fptr.size(), s));
    RIGA_TRY(sym->d_sub_bptr.upload(L.sub_bptr.data(), L.sub_bptr.size(), s));
    RIGA_TRY(sym->d_sub_ftiles.upload(L.sub_ftiles.data(), L.sub_ftiles.size(), s));
    RIGA_TRY(sym->d_sub_btiles.upload(L.sub_btiles.data(), L.sub_btiles.size(), s));
  }
  RIGA_TRY(sym->d_gptr.upload(L.gptr.data(), L.gptr.size(), s));
  RIGA_TRY(sym->d_cmask.upload(L.cmask.data(), std::max<size_t>(L.cmask.size(), 1), s));
  RIGA_TRY(sym->d_ubase.upload(L.ubase.data(), L.ubase.size(), s));
  if (L.small_g && L.g_total) {
    RIGA_TRY(sym->d_g_off.upload(L.g_off.data(), L.g_off.size(), s));
    RIGA_TRY(sym->d_gfwd.upload(L.gfwd.data(), L.gfwd.size(), s));
    RIGA_TRY(sym->d_gbwd.upload(L.gbwd.data(), L.gbwd.size(), s));
  }
  if (L.chain_inv && L.inv_total) {
    RIGA_TRY(sym->d_inv_off.upload(L.inv_off.data(), L.inv_off.size(), s));
    RIGA_TRY(sym->d_ifwd.upload(L.ifwd.data(), L.ifwd.size(), s));
    RIGA_TRY(sym->d_ibwd.upload(L.ibwd.data(), L.ibwd.size(), s));
    RIGA_TRY(sym->d_idiag.upload(L.idiag.data(), L.idiag.size(), s));
    if (!L.dbl_tasks.empty()) {
      RIGA_TRY(sym->d_dbl_tasks.upload(L.dbl_tasks.data(), L.dbl_tasks.size(), s));
      RIGA_TRY(sym->d_dbl_toff.upload(L.dbl_toff.data(), L.dbl_toff.size(), s));
    }
  }
  if (L.gsrc.empty())
    RIGA_TRY(sym->d_gsrc.alloc(1, s));
  else
    RIGA_TRY(sym->d_gsrc.upload(L.gsrc.data(), L.gsrc.size(), s));
  return RIGA_OK;
}

template <typename K>
static int raise_smem(K kernel, int maxsm) {
  cudaFuncAttributes fa;
  RIGA_CUDA(cudaFuncGetAttributes(&fa, kernel));
  RIGA_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 maxsm - (int)fa.sharedSizeBytes));
  return RIGA_OK;
}

static int set_solve_attrs() {
  static bool done = false;
  if (done) return RIGA_OK;
  int dev = 0, maxsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  RIGA_TRY(raise_smem(k_rest_fwd<false>, maxsm));
  RIGA_TRY(raise_smem(k_rest_bwd<false>, maxsm));
  RIGA_TRY(raise_smem(k_rest_fwd<true, 4>, maxsm));
  RIGA_TRY(raise_smem(k_rest_bwd<true, 4>, maxsm));
  RIGA_TRY(raise_smem(k_rest_fwd<true, 6>, maxsm));
  RIGA_TRY(raise_smem(k_rest_bwd<true, 6>, maxsm));
  RIGA_TRY(raise_smem(k_rest_fwd<true, 8>, maxsm));
  RIGA_TRY(raise_smem(k_rest_bwd<true, 8>, maxsm));
  RIGA_TRY(raise_smem(k_chain_fwd, maxsm));
  RIGA_TRY(raise_smem(k_chain_bwd, maxsm));
  RIGA_TRY(raise_smem(k_inv_fwd, maxsm));
  RIGA_TRY(raise_smem(k_inv_fix_fwd_res, maxsm));
  RIGA_TRY(raise_smem(k_inv_fix_fwd_apply, maxsm));
  done = true;
  return RIGA_OK;
}

int prepare_solve() { return set_solve_attrs(); }

// G = [inv(L11); L21 inv(L11)] of every G-mode supernode; needs only those supernodes' finished panels, so
// the factorization launches it on a side stream once their last tree level is done (gsmall must already
// be allocated in an order the stream respects)
template <int GR>
static int launch_small_g(riga_factor* F, cudaStream_t st, const int32_t* nodes, int count) {
  if (count <= 0) return RIGA_OK;
  constexpr int smem = 32 * GR * (32 * GR + 1) * 8;
  static bool attr = false;
  if (!attr) {
    RIGA_CUDA(cudaFuncSetAttribute(k_small_g<GR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  riga_symbolic* sym = F->sym;
  k_small_g<GR><<<count, 256, smem, st>>>(sym->dev(), nodes, F->panel.p, sym->d_g_off.p, F->gsmall.p);
  count_launch();
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

int build_small_g(riga_factor* F, cudaStream_t st) {
  riga_symbolic* sym = F->sym;
  const SolvePlanHost& L = sym->sp;
  if (!(L.small_g && L.g_total)) return RIGA_OK;
  // the G-mode supernodes sorted by width class (np <= 32, 64, 96, 128), widest first
  const int32_t* nodes = sym->d_gnodes.p;
  RIGA_TRY(launch_small_g<4>(F, st, nodes + L.gcls_ptr[3], (int)(L.gcls_ptr[4] - L.gcls_ptr[3])));
  RIGA_TRY(launch_small_g<3>(F, st, nodes + L.gcls_ptr[2], (int)(L.gcls_ptr[3] - L.gcls_ptr[2])));
  RIGA_TRY(launch_small_g<2>(F, st, nodes + L.gcls_ptr[1], (int)(L.gcls_ptr[2] - L.gcls_ptr[1])));
  RIGA_TRY(launch_small_g<1>(F, st, nodes + L.gcls_ptr[0], (int)(L.gcls_ptr[1] - L.gcls_ptr[0])));
  return RIGA_OK;
}

// highest tree level holding a G-mode supernode (-1: none)
int64_t small_g_top_level(const riga_symbolic* sym) {
  const SolvePlanHost& L = sym->sp;
  if (!(L.small_g && L.g_total)) return -1;
  int64_t top = -1;
  for (int32_t s : L.wholes) top = std::max<int64_t>(top, sym->h.level[s]);
  return top;
}

int build_chain_inverse(riga_factor* F, cudaStream_t st) {
  riga_symbolic* sym = F->sym;
  const SolvePlanHost& L = sym->sp;
  SymDev S = sym->dev();
  if (!L.chain_inv || !L.inv_total) return RIGA_OK;
  if (!F->linv.p) RIGA_TRY(F->linv.alloc(L.inv_total, st));
  if (L.inv_fix && !F->rfix.p) RIGA_TRY(F->rfix.alloc(sym->h.n, st));
  if (L.inv_fix && !F->inv_err.p) RIGA_TRY(F->inv_err.alloc(sym->h.nsuper, st));
  // the doubling GEMMs read whole diagonal blocks: the upper triangles must be zero
  RIGA_CUDA(cudaMemsetAsync(F->linv.p, 0, L.inv_total * sizeof(double), st));
  const int nd = (int)L.idiag.size();
  k_trinv_diag<<<(nd + 7) / 8, 256, 0, st>>>(S, reinterpret_cast<const int2*>(sym->d_idiag.p), nd, F->panel.p,
                                             sym->d_inv_off.p, F->linv.p);
  count_launch();
  if (!L.dbl_tasks.empty()) {
    DevBuf<double> tbuf;
    RIGA_TRY(tbuf.alloc(std::max<int64_t>(L.dbl_tmax, 1), st));
    const int2* dt = reinterpret_cast<const int2*>(sym->d_dbl_tasks.p);
    for (size_t l = 0; l < L.dbl_size.size(); ++l) {
      const int64_t t0 = L.dbl_ptr[l], nt = L.dbl_ptr[l + 1] - t0;
      const dim3 g((unsigned)L.dbl_tiles[l], (unsigned)nt);
      k_trinv_gemm1<<<g, 128, 0, st>>>(S, dt + t0, (int)L.dbl_size[l], F->panel.p, sym->d_inv_off.p,
                                       sym->d_dbl_toff.p + t0, F->linv.p, tbuf.p);
      k_trinv_gemm2<<<g, 128, 0, st>>>(S, dt + t0, (int)L.dbl_size[l], sym->d_inv_off.p, sym->d_dbl_toff.p + t0,
                                       tbuf.p, F->linv.p);
      count_launch(2);
    }
  }
  if (L.inv_fix && !L.ifwd.empty()) {
    const int nt = (int)L.ifwd.size();
    const int2* it = reinterpret_cast<const int2*>(sym->d_ifwd.p);
    RIGA_CUDA(cudaMemsetAsync(F->inv_err.p, 0, sym->h.nsuper * sizeof(unsigned long long), st));
    k_inv_chk1<<<nt, 256, 0, st>>>(S, it, sym->d_inv_off.p, F->linv.p, F->rfix.p);
    k_inv_chk2<<<nt, 256, 0, st>>>(S, it, F->panel.p, F->rfix.p, F->inv_err.p);
    count_launch(2);
  }
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}


}  // namespace riga

extern "C" int riga_set_solve_sub_levels(int levels) {
  RIGA_CHECK_ARG(levels >= 0 && levels <= 64, "sub levels out of range");
  riga::g_sub_levels = levels;
  return RIGA_OK;
}

namespace riga {

int factor_solve(riga_factor* F, cudaStream_t st, const double* b, double* x, bool b_permuted, bool accurate) {
  riga_symbolic* sym = F->sym;
  const SymbolicHost& h = sym->h;
  const SolvePlanHost& L = sym->sp;
  ProfScope prof(kProfSolve, st, 16.0 * h.fill_nnz + 32.0 * h.n);
  RIGA_TRY(set_solve_attrs());
  SymDev S = sym->dev();
  SolveDev T{sym->d_cmask.p, sym->d_ubase.p, sym->d_gptr.p, sym->d_gsrc.p, L.nfront, L.otail, b_permuted ? 1 : 0};
  const int gon = L.small_g && L.g_total ? 1 : 0;
  const GDev GDf{F->gsmall.p, sym->d_g_off.p, reinterpret_cast<const int2*>(sym->d_gfwd.p), gon, F->D.p,
                 F->cvec.p};
  const GDev GDb{F->gsmall.p, sym->d_g_off.p, reinterpret_cast<const int2*>(sym->d_gbwd.p), gon, F->D.p,
                 F->cvec.p};
  const int2* tf = reinterpret_cast<const int2*>(sym->d_tfwd.p);
  const int2* tb = reinterpret_cast<const int2*>(sym->d_tbwd.p);
  if (L.nsub && gon) {
    const GDev Gs{F->gsmall.p, sym->d_g_off.p, reinterpret_cast<const int2*>(sym->d_sub_ftiles.p), 1, F->D.p,
                  F->cvec.p};
    const int nt = sub_threads();
    RIGA_CUDA(launch(nt == 1024 ? k_sub_fwd<1024> : nt == 512 ? k_sub_fwd<512> : k_sub_fwd<256>,
                     (unsigned)L.nsub, nt, 0,
                     st, S, T, Gs, sym->d_sub_fptr.p, L.sub_levels, b, F->xperm.p,
                                                          F->upd.p));
    count_launch();
  }
  for (int64_t l = 0; l < h.nlevels; ++l) {
    const int nc = (int)(L.chain_ptr[l + 1] - L.chain_ptr[l]);
    const int ni = (int)(L.ifwd_ptr[l + 1] - L.ifwd_ptr[l]);
    if (L.chain_inv && ni) {
      const int2* it = reinterpret_cast<const int2*>(sym->d_ifwd.p) + L.ifwd_ptr[l];
      RIGA_CUDA(launch(k_inv_fwd, ni, 256, L.ifwd_smem[l], st, S, T, it, sym->d_inv_off.p, F->linv.p, F->D.p, b,
                       F->xperm.p, F->upd.p, F->cvec.p));
      count_launch();
      if (L.inv_fix && (accurate || F->fix_level[l])) {
        const int* fl = accurate ? nullptr : F->fix_flag.p;
        RIGA_CUDA(launch(k_inv_fix_fwd_res, ni, 256, L.ifwd_smem[l], st, S, T, it, fl, F->panel.p, b,
                         F->xperm.p, F->upd.p, F->rfix.p));
        RIGA_CUDA(launch(k_inv_fix_fwd_apply, ni, 256, L.ifwd_smem[l], st, S, it, fl, sym->d_inv_off.p,
                         F->linv.p, F->D.p, F->rfix.p, F->xperm.p, F->cvec.p));
        count_launch(2);
      }
    } else if (nc) {
      RIGA_CUDA(launch(k_chain_fwd, nc, kSolveThreads, L.chf_smem[l], st, S, T, sym->d_chains.p + L.chain_ptr[l],
                                                            (int)L.chf_smem[l], F->panel.p, b, F->xperm.p,
                                                            F->upd.p));
      count_launch();
    }
    const int nt = (int)(L.fwd_ptr[l + 1] - L.fwd_ptr[l]);
    if (nt) {
      RIGA_CUDA(launch((gon ? (L.occ == 8 ? k_rest_fwd<true, 8> : L.occ == 6 ? k_rest_fwd<true, 6> : k_rest_fwd<true, 4>)
           : k_rest_fwd<false>), std::min(nt, L.rest_cap), kSolveThreads, L.fwd_smem[l], st, S, T, tf + L.fwd_ptr[l], nt, sym->d_wholes.p,
                                                           F->panel.p, b, F->xperm.p, F->upd.p, L.warp_stage, GDf));
      count_launch();
    }
  }
  for (int64_t l = h.nlevels - 1; l >= 0; --l) {
    const int nt = (int)(L.bwd_ptr[l + 1] - L.bwd_ptr[l]);
    if (nt) {
      RIGA_CUDA(launch((gon ? (L.occ == 8 ? k_rest_bwd<true, 8> : L.occ == 6 ? k_rest_bwd<true, 6> : k_rest_bwd<true, 4>)
           : k_rest_bwd<false>), std::min(nt, L.rest_cap), kSolveThreads, L.bwd_smem[l], st, S, T, tb + L.bwd_ptr[l], nt, sym->d_wholes.p,
                                                           F->panel.p, F->D.p, F->xperm.p, F->cvec.p, x, L.warp_stage,
                                                           L.chain_inv, GDb));
      count_launch();
    }
    const int nc = (int)(L.chain_ptr[l + 1] - L.chain_ptr[l]);
    const int ni = (int)(L.ibwd_ptr[l + 1] - L.ibwd_ptr[l]);
    if (L.chain_inv && ni) {
      const int2* it = reinterpret_cast<const int2*>(sym->d_ibwd.p) + L.ibwd_ptr[l];
      RIGA_CUDA(launch(k_inv_bwd, ni, 256, 0, st, S, it, sym->d_inv_off.p, F->linv.p, F->cvec.p, F->xperm.p, x));
      count_launch();
      if (L.inv_fix && (accurate || F->fix_level[l])) {
        const int* fl = accurate ? nullptr : F->fix_flag.p;
        RIGA_CUDA(launch(k_inv_fix_bwd_res, ni, 256, 0, st, S, it, fl, F->panel.p, F->cvec.p, F->xperm.p,
                         F->rfix.p));
        RIGA_CUDA(launch(k_inv_fix_bwd_apply, ni, 256, 0, st, S, it, fl, sym->d_inv_off.p, F->linv.p,
                         F->rfix.p, F->xperm.p, x));
        count_launch(2);
      }
    } else if (nc) {
      RIGA_CUDA(launch(k_chain_bwd, nc, kSolveThreads, L.chb_smem[l], st, S, sym->d_chains.p + L.chain_ptr[l],
                                                            (int)L.chb_smem[l], F->panel.p, F->D.p,
                                                            F->xperm.p, F->cvec.p, x));
      count_launch();
    }
  }
  if (L.nsub && gon) {
    const GDev Gs{F->gsmall.p, sym->d_g_off.p, reinterpret_cast<const int2*>(sym->d_sub_btiles.p), 1, F->D.p,
                  F->cvec.p};
    const int nt = sub_threads();
    RIGA_CUDA(launch(nt == 1024 ? k_sub_bwd<1024> : nt == 512 ? k_sub_bwd<512> : k_sub_bwd<256>,
                     (unsigned)L.nsub, nt, 0,
                     st, S, Gs, sym->d_sub_bptr.p, L.sub_levels, F->D.p,
                                                          F->xperm.p, x));
    count_launch();
  }
  RIGA_CUDA(cudaGetLastError());
  return RIGA_OK;
}

}  // namespace riga
