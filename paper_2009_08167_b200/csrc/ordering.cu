// Separator ordering of the tensor-product box (ref sparsela.py:319-392, separator_ordering).
//
//  riga_separator_boxes  the dissection tree: every box is cut at the C0 plane nearest its middle (width one,
//                        longest axis with a candidate first), without one at a width-p slab in the middle of
//                        its longest axis; boxes no longer than max(2p, 8) are leaves.  A few thousand boxes:
//                        host, microseconds.  Output order = elimination order of the blocks: leaves in
//                        recursion order, then separators deepest level first.
//  riga_separator_emit   the permutation itself, O(n): one thread per elimination position finds its block
//                        (binary search over the block offsets) and decodes the lexicographic cell (axis 0
//                        fastest, as the reference's emit()).  Device.
#include <algorithm>
#include <vector>

#include "common.h"
#include "riga_b200.h"

namespace riga {
namespace {

struct Box {
  int64_t lo[3], hi[3];
};

struct Dissector {
  int d = 0, p = 0;
  int64_t leaf = 0;
  std::vector<int64_t> lines[3];
  std::vector<Box> leaves;
  std::vector<std::vector<Box>> seps;  // per recursion depth

  void run(const Box& b, size_t depth) {
    int64_t w[3] = {1, 1, 1};
    for (int t = 0; t < d; ++t) w[t] = b.hi[t] - b.lo[t];
    // axes by decreasing extent (stable: the lower axis first on ties)
    int ax[3] = {0, 1, 2};
    std::stable_sort(ax, ax + d, [&](int x, int y) { return w[x] > w[y]; });
    int ct = -1;
    int64_t s0 = 0, s1 = 0;
    for (int q = 0; q < d && ct < 0; ++q) {
      const int t = ax[q];
      const int64_t a = b.lo[t], e = b.hi[t];
      // candidates a + 1 <= c <= e - 2; nearest to (a + e - 1) / 2, the smaller one on ties
      auto it0 = std::lower_bound(lines[t].begin(), lines[t].end(), a + 1);
      auto it1 = std::upper_bound(lines[t].begin(), lines[t].end(), e - 2);
      int64_t best = -1, bestd = 0;
      for (auto it = it0; it < it1; ++it) {
        const int64_t dd = std::llabs(2 * *it - (a + e - 1));
        if (best < 0 || dd < bestd) {
          best = *it;
          bestd = dd;
        }
      }
      if (best >= 0) {
        ct = t;
        s0 = best;
        s1 = best + 1;
      }
    }
    if (ct < 0) {
      int t = 0;
      for (int q = 1; q < d; ++q)
        if (w[q] > w[t]) t = q;
      if (w[t] <= leaf) {
        leaves.push_back(b);
        return;
      }
      const int64_t a = b.lo[t], e = b.hi[t];
      s0 = std::min(std::max(a + (w[t] - p) / 2, a + 1), e - 1 - p);
      s1 = s0 + p;
      ct = t;
    }
    Box lo = b, hi = b, mid = b;
    lo.hi[ct] = s0;
    hi.lo[ct] = s1;
    mid.lo[ct] = s0;
    mid.hi[ct] = s1;
    run(lo, depth + 1);
    run(hi, depth + 1);
    if (seps.size() <= depth) seps.resize(depth + 1);
    seps[depth].push_back(mid);
  }
};

__global__ void k_emit_order(int64_t n, int64_t nchunks, const int64_t* __restrict__ chunks, int64_t s1, int64_t s2,
                             int64_t* __restrict__ perm) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  int64_t a = 0, b = nchunks - 1;  // last chunk with off <= k
  while (a < b) {
    const int64_t m = (a + b + 1) >> 1;
    if (chunks[7 * m] <= k) a = m;
    else b = m - 1;
  }
  const int64_t* c = chunks + 7 * a;
  int64_t j = k - c[0];
  const int64_t j0 = j % c[4];
  j /= c[4];
  const int64_t j1 = j % c[5];
  const int64_t j2 = j / c[5];
  perm[k] = (c[1] + j0) + (c[2] + j1) * s1 + (c[3] + j2) * s2;
}

}  // namespace
}  // namespace riga

using namespace riga;

extern "C" {

int riga_separator_boxes(int d, const int64_t* ext, int degree, const int64_t* lines, const int64_t* nlines,
                         int64_t cap, int64_t* nchunks, int64_t* chunks) {
  RIGA_CHECK_ARG(d >= 1 && d <= 3 && ext && degree >= 1 && nlines && nchunks, "bad arg");
  Dissector D;
  D.d = d;
  D.p = degree;
  D.leaf = std::max<int64_t>(2 * degree, 8);
  Box root{};
  int64_t at = 0;
  for (int t = 0; t < 3; ++t) {
    root.lo[t] = 0;
    root.hi[t] = t < d ? ext[t] : 1;
    if (t < d) {
      RIGA_CHECK_ARG(ext[t] >= 1 && nlines[t] >= 0 && (nlines[t] == 0 || lines), "bad extents / lines");
      D.lines[t].assign(lines + at, lines + at + nlines[t]);
      RIGA_CHECK_ARG(std::is_sorted(D.lines[t].begin(), D.lines[t].end()), "C0 lines must be ascending");
      at += nlines[t];
    }
  }
  D.run(root, 0);
  std::vector<const Box*> order;
  for (const Box& b : D.leaves) order.push_back(&b);
  for (size_t lv = D.seps.size(); lv-- > 0;)
    for (const Box& b : D.seps[lv]) order.push_back(&b);
  *nchunks = (int64_t)order.size();
  if (!chunks || cap < *nchunks) return RIGA_OK;  // size query
  int64_t off = 0;
  for (size_t c = 0; c < order.size(); ++c) {
    int64_t* o = chunks + 7 * c;
    o[0] = off;
    int64_t cells = 1;
    for (int t = 0; t < 3; ++t) {
      o[1 + t] = order[c]->lo[t];
      o[4 + t] = order[c]->hi[t] - order[c]->lo[t];
      cells *= o[4 + t];
    }
    off += cells;
  }
  return RIGA_OK;
}

int riga_separator_emit(riga_ctx* ctx, int d, const int64_t* ext, int64_t nchunks, const int64_t* chunks_host,
                        int64_t n, int64_t* perm_dev) {
  RIGA_CHECK_ARG(ctx && d >= 1 && d <= 3 && ext && nchunks >= 1 && chunks_host && n >= 1 && perm_dev, "bad arg");
  const int64_t* last = chunks_host + 7 * (nchunks - 1);
  RIGA_CHECK_ARG(last[0] + last[4] * last[5] * last[6] == n, "blocks do not enumerate n cells");
  DeviceGuard g(ctx->device);
  DevBuf<int64_t> dc;
  RIGA_TRY(dc.alloc(7 * nchunks, ctx->stream));
  RIGA_CUDA(cudaMemcpyAsync(dc.p, chunks_host, 7 * nchunks * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
  const int64_t s1 = ext[0], s2 = d > 1 ? ext[0] * ext[1] : ext[0];
  k_emit_order<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(n, nchunks, dc.p, s1, s2, perm_dev);
  RIGA_CUDA(cudaGetLastError());
  RIGA_CUDA(cudaStreamSynchronize(ctx->stream));  // chunks_host may be released by the caller
  return RIGA_OK;
}

}  // extern "C"
