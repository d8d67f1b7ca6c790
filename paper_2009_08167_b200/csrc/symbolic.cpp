// Host symbolic analysis for the supernodal multifrontal LDL^T.
//
// Replaces what the reference redoes inside every factor_ldl call
// (/root/reference/pkg/src/rigaeig/sparsela.py:239-250: permute, triu,
// _etree_counts :100-115) with a once-per-pattern analysis whose products
// the device factorization and solves reuse for every shift sigma:
//
//   1. elimination tree of P A P^T (ancestor path compression),
//   2. postorder of the tree (an equivalent ordering: same fill, same
//      column counts, same factor_flops as the caller's perm),
//   3. exact column counts (row-subtree marking, the reference's count),
//   4. fundamental supernodes, then relaxed amalgamation (nrelax/zrelax
//      thresholds in the CHOLMOD style) so that deep 3D trees become
//      shallow trees of dense fronts,
//   5. frontal row structures, extend-add relative positions, the scatter
//      map of original entries into fronts, and tree levels for the
//      level-batched device schedule.
#include "symbolic.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <numeric>
#include <string>
#include <thread>

namespace riga {

namespace {

// Host threads for the pattern sweeps (column counts, front structures, the
// scatter map): RIGA_SYM_THREADS, default min(16, hardware threads).
int sym_threads(int64_t work) {
  static const int t = [] {
    const char* e = std::getenv("RIGA_SYM_THREADS");
    const int h = (int)std::thread::hardware_concurrency();
    return std::max(1, e ? std::atoi(e) : std::min(16, std::max(1, h)));
  }();
  return work < 4096 ? 1 : t;
}

template <class F>
void par_run(int nt, F&& f) {  // f(thread index), joined before returning
  if (nt <= 1) {
    f(0);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(nt - 1);
  for (int t = 1; t < nt; ++t) th.emplace_back([&f, t] { f(t); });
  f(0);
  for (auto& x : th) x.join();
}

// Dynamic chunks of [0, n) over nt threads: f(thread, begin, end).
template <class F>
void par_chunks(int nt, int64_t n, int64_t chunk, F&& f) {
  std::atomic<int64_t> next{0};
  par_run(nt, [&](int t) {
    for (;;) {
      const int64_t b = next.fetch_add(chunk);
      if (b >= n) break;
      f(t, b, std::min(n, b + chunk));
    }
  });
}

// widest supernode kept in one piece (RIGA_SN_MAXCOLS, default 2048; 0 = never split)
static int64_t max_sn_cols() {
  static const int64_t v = [] {
    const char* e = std::getenv("RIGA_SN_MAXCOLS");
    const int64_t w = e && *e ? std::atoll(e) : 2048;
    return w <= 0 ? INT64_MAX : std::max<int64_t>(w, 256);
  }();
  return v;
}

struct Relax {
  int64_t nrelax[3] = {4, 16, 48};
  double zrelax[3] = {0.8, 0.1, 0.05};
};

}  // namespace

int analyze(int64_t n, const int64_t* rowptr, const int32_t* colidx, const int64_t* perm,
            SymbolicHost& S, std::string& err, bool with_asm_map) {
  S = SymbolicHost();
  S.n = n;
  // RIGA_SYM_TIME=1: wall time of every phase on stderr
  static const bool timed = std::getenv("RIGA_SYM_TIME") != nullptr;
  auto tprev = std::chrono::steady_clock::now();
  auto phase = [&](const char* name) {
    if (!timed) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[riga] analyze %-18s %8.2f ms\n", name,
                 std::chrono::duration<double, std::milli>(now - tprev).count());
    tprev = now;
  };
  if (n <= 0) {
    err = "empty matrix";
    return 1;
  }
  S.nnz = rowptr[n];
  // ---- caller permutation and its inverse -------------------------------
  std::vector<int32_t> ip(n, -1);
  for (int64_t k = 0; k < n; ++k) {
    int64_t o = perm[k];
    if (o < 0 || o >= n || ip[o] != -1) {
      err = "ordering is not a permutation of 0..n-1";
      return 1;
    }
    ip[o] = (int32_t)k;
  }
  // ---- 1. elimination tree in the caller's order ------------------------
  // upper entries of column k of PAP^T = neighbours c of perm[k] with ip[c] < k
  // The permuted upper pattern is filtered in parallel first, so the serial
  // ancestor walk reads only the entries it uses.
  std::vector<int64_t> uptr(n + 1, 0);
  std::vector<int32_t> upat;
  {
    const int nt = sym_threads(n);
    par_chunks(nt, n, 2048, [&](int, int64_t k0, int64_t k1) {
      for (int64_t k = k0; k < k1; ++k) {
        const int64_t o = perm[k];
        int64_t c = 0;
        for (int64_t q = rowptr[o]; q < rowptr[o + 1]; ++q) c += ip[colidx[q]] < k;
        uptr[k + 1] = c;
      }
    });
    for (int64_t k = 0; k < n; ++k) uptr[k + 1] += uptr[k];
    upat.resize(uptr[n]);
    par_chunks(nt, n, 2048, [&](int, int64_t k0, int64_t k1) {
      for (int64_t k = k0; k < k1; ++k) {
        const int64_t o = perm[k];
        int64_t w = uptr[k];
        for (int64_t q = rowptr[o]; q < rowptr[o + 1]; ++q) {
          const int32_t i = ip[colidx[q]];
          if (i < k) upat[w++] = i;
        }
      }
    });
  }
  std::vector<int64_t> parent(n, -1), anc(n, -1);
  for (int64_t k = 0; k < n; ++k) {
    for (int64_t q = uptr[k]; q < uptr[k + 1]; ++q) {
      int64_t i = upat[q];
      while (i != -1 && i < k) {
        int64_t nxt = anc[i];
        anc[i] = k;
        if (nxt == -1) parent[i] = k;
        i = nxt;
      }
    }
  }
  phase("etree");
  // ---- 2. postorder ------------------------------------------------------
  std::vector<int64_t> head(n, -1), next(n, -1);
  for (int64_t j = n - 1; j >= 0; --j) {
    if (parent[j] != -1) {
      next[j] = head[parent[j]];
      head[parent[j]] = j;
    }
  }
  std::vector<int64_t> post;
  post.reserve(n);
  {
    std::vector<int64_t> stack;
    for (int64_t r = 0; r < n; ++r) {
      if (parent[r] != -1) continue;
      stack.push_back(r);
      while (!stack.empty()) {
        int64_t p = stack.back();
        int64_t c = head[p];
        if (c == -1) {
          stack.pop_back();
          post.push_back(p);
        } else {
          head[p] = next[c];
          stack.push_back(c);
        }
      }
    }
  }
  if ((int64_t)post.size() != n) {
    err = "postorder failed";
    return 1;
  }
  std::vector<int64_t> ipost(n);
  for (int64_t k = 0; k < n; ++k) ipost[post[k]] = k;
  S.post = post;
  S.order.resize(n);
  S.iorder.resize(n);
  for (int64_t k = 0; k < n; ++k) {
    S.order[k] = perm[post[k]];
    S.iorder[S.order[k]] = (int32_t)k;
  }
  std::vector<int64_t> par(n, -1);  // tree in postorder numbering
  for (int64_t k = 0; k < n; ++k) par[k] = parent[post[k]] == -1 ? -1 : ipost[parent[post[k]]];
  const std::vector<int32_t>& io = S.iorder;

  phase("postorder");
  // ---- 3. exact column counts (row subtrees) -----------------------------
  // Row k of L is the union of the tree paths from A's entries (i < k) up to
  // k; rows are independent, so threads take row chunks with private marks
  // and counts, summed afterwards.
  S.colcount.assign(n, 1);
  {
    const int nt = sym_threads(n);
    std::vector<std::vector<int32_t>> cnt(nt), marks(nt);
    par_chunks(nt, n, 1024, [&](int t, int64_t k0, int64_t k1) {
      if (cnt[t].empty()) {
        cnt[t].assign(n, 0);
        marks[t].assign(n, -1);
      }
      int32_t* c = cnt[t].data();
      int32_t* mark = marks[t].data();
      for (int64_t k = k0; k < k1; ++k) {
        mark[k] = (int32_t)k;
        const int64_t o = S.order[k];
        for (int64_t q = rowptr[o]; q < rowptr[o + 1]; ++q) {
          int64_t i = io[colidx[q]];
          if (i >= k) continue;
          while (mark[i] != (int32_t)k) {
            mark[i] = (int32_t)k;
            c[i] += 1;
            i = par[i];
          }
        }
      }
    });
    par_chunks(nt, n, 16384, [&](int, int64_t b, int64_t e) {
      for (const auto& c : cnt)
        if (!c.empty())
          for (int64_t i = b; i < e; ++i) S.colcount[i] += c[i];
    });
  }
  S.fill_nnz = 0;
  S.factor_flops = 0;
  for (int64_t j = 0; j < n; ++j) {
    S.fill_nnz += S.colcount[j];
    S.factor_flops += S.colcount[j] * S.colcount[j];
  }
  // fill_nnz = nnz(strict L) + n  (ref sparsela.py:257) == sum of counts
  {
    std::vector<int64_t> h(n, 0);
    for (int64_t j = 0; j < n; ++j)
      if (par[j] != -1) h[par[j]] = std::max(h[par[j]], h[j] + 1);
    S.tree_height = 0;
    for (int64_t j = 0; j < n; ++j) S.tree_height = std::max(S.tree_height, h[j] + 1);
  }

  phase("colcounts");
  // ---- 4a. fundamental supernodes ------------------------------------------
  std::vector<int64_t> nchild(n, 0);
  for (int64_t j = 0; j < n; ++j)
    if (par[j] != -1) nchild[par[j]]++;
  std::vector<int64_t> sfirst;  // first column of each fundamental supernode
  for (int64_t j = 0; j < n; ++j) {
    bool merge = j > 0 && par[j - 1] == j && S.colcount[j - 1] == S.colcount[j] + 1 &&
                 nchild[j] == 1;
    if (!merge) sfirst.push_back(j);
  }
  int64_t nf = (int64_t)sfirst.size();
  S.fundamental = nf;
  sfirst.push_back(n);
  std::vector<int64_t> col2sn(n);
  for (int64_t s = 0; s < nf; ++s)
    for (int64_t j = sfirst[s]; j < sfirst[s + 1]; ++j) col2sn[j] = s;
  // ---- 4b. relaxed amalgamation ------------------------------------------
  // Each fundamental supernode s: ncol, front size f = colcount(first col),
  // true nonzeros, stored entries.  Merge s into its parent p when s is the
  // last child in postorder (columns contiguous) and the zero fraction of
  // the merged dense front is within the thresholds.
  std::vector<int64_t> g_first(nf), g_ncol(nf), g_f(nf), g_true(nf), g_rep(nf);
  for (int64_t s = 0; s < nf; ++s) {
    g_first[s] = sfirst[s];
    g_ncol[s] = sfirst[s + 1] - sfirst[s];
    g_f[s] = S.colcount[sfirst[s]];
    int64_t t = 0;
    for (int64_t j = sfirst[s]; j < sfirst[s + 1]; ++j) t += S.colcount[j];
    g_true[s] = t;
    g_rep[s] = s;
  }
  auto find = [&](int64_t s) {
    while (g_rep[s] != s) {
      g_rep[s] = g_rep[g_rep[s]];
      s = g_rep[s];
    }
    return s;
  };
  auto stored = [](int64_t ncol, int64_t f) { return ncol * f - ncol * (ncol - 1) / 2; };
  Relax R;
  std::vector<int64_t> sp_f(nf, -1);  // fundamental parent supernode
  for (int64_t s = 0; s < nf; ++s) {
    int64_t last = sfirst[s + 1] - 1;
    sp_f[s] = par[last] == -1 ? -1 : col2sn[par[last]];
  }
  for (int64_t s = nf - 1; s >= 0; --s) {
    if (sp_f[s] == -1) continue;
    int64_t p = find(sp_f[s]);
    int64_t cs = find(s);
    if (cs != s) continue;
    if (g_first[p] != g_first[s] + g_ncol[s]) continue;  // not contiguous
    int64_t ncol = g_ncol[s] + g_ncol[p];
    int64_t f = g_ncol[s] + g_f[p];
    int64_t st = stored(ncol, f);
    int64_t tr = g_true[s] + g_true[p];
    double z = st > 0 ? double(st - tr) / double(st) : 0.0;
    bool ok = ncol <= R.nrelax[0] || (ncol <= R.nrelax[1] && z <= R.zrelax[0]) ||
              (ncol <= R.nrelax[2] && z <= R.zrelax[1]) || z <= R.zrelax[2];
    if (!ok) continue;
    // small fronts must stay small enough for the shared-memory path or
    // be genuinely large; never grow a front past 2x its parent's columns
    g_rep[s] = p;
    g_first[p] = g_first[s];
    g_ncol[p] = ncol;
    g_f[p] = f;
    g_true[p] = tr;
  }
  // collect final supernodes in column order
  std::vector<int64_t> fin;
  for (int64_t s = 0; s < nf; ++s)
    if (find(s) == s) fin.push_back(s);
  std::sort(fin.begin(), fin.end(), [&](int64_t a, int64_t b) { return g_first[a] < g_first[b]; });
  // Very wide supernodes (the top separators of a 3D dissection) are cut into a chain of equal pieces of
  // at most max_sn_cols() columns: piece k's front is the old front minus the earlier pieces' columns and
  // its parent is piece k + 1, so everything downstream (front structures, extend-add maps, levels) sees
  // ordinary supernodes.  What it buys: the solve keeps an explicit inv(L11) per chain supernode, and
  // inverting one 7526-column block (cfg5's root) costs as many flops as factoring its front -- four
  // 1882-column pieces cost 1/16 of that and the off-diagonal blocks are applied from the panel instead.
  S.col0.clear();
  S.ncol.clear();
  const int64_t wmax = max_sn_cols();
  for (int64_t q = 0; q < (int64_t)fin.size(); ++q) {
    const int64_t first = g_first[fin[q]], nc = g_ncol[fin[q]];
    const int64_t pieces = nc > wmax ? (nc + wmax - 1) / wmax : 1;
    for (int64_t k = 0; k < pieces; ++k) {
      const int64_t a = first + nc * k / pieces, b = first + nc * (k + 1) / pieces;
      S.col0.push_back(a);
      S.ncol.push_back(b - a);
    }
  }
  int64_t ns = (int64_t)S.col0.size();
  S.nsuper = ns;
  std::vector<int64_t> c2s(n);
  for (int64_t s = 0; s < ns; ++s)
    for (int64_t j = S.col0[s]; j < S.col0[s] + S.ncol[s]; ++j) c2s[j] = s;
  S.sparent.assign(ns, -1);
  for (int64_t s = 0; s < ns; ++s) {
    int64_t last = S.col0[s] + S.ncol[s] - 1;
    S.sparent[s] = par[last] == -1 ? -1 : (int32_t)c2s[par[last]];
  }
  // children lists
  S.child_ptr.assign(ns + 1, 0);
  for (int64_t s = 0; s < ns; ++s)
    if (S.sparent[s] >= 0) S.child_ptr[S.sparent[s] + 1]++;
  for (int64_t s = 0; s < ns; ++s) S.child_ptr[s + 1] += S.child_ptr[s];
  S.child_list.resize(S.child_ptr[ns]);
  {
    std::vector<int64_t> fillp(S.child_ptr.begin(), S.child_ptr.end() - 1);
    for (int64_t s = 0; s < ns; ++s)
      if (S.sparent[s] >= 0) S.child_list[fillp[S.sparent[s]]++] = (int32_t)s;
  }

  phase("supernodes");
  // ---- 5a. front structures ---------------------------------------------
  // struct(s) = cols(s) U {rows > last(s) of A's lower columns in s}
  //           U {update rows of children > last(s)}, sorted.
  // Supernodes of one tree level are independent (children sit at lower
  // levels), so each level is one parallel sweep.
  S.level.assign(ns, 0);
  int32_t maxlev = 0;
  for (int64_t s = 0; s < ns; ++s) {  // children precede parents
    if (S.sparent[s] >= 0)
      S.level[S.sparent[s]] = std::max(S.level[S.sparent[s]], S.level[s] + 1);
    maxlev = std::max(maxlev, S.level[s]);
  }
  S.nlevels = maxlev + 1;
  S.level_ptr.assign(S.nlevels + 1, 0);
  for (int64_t s = 0; s < ns; ++s) S.level_ptr[S.level[s] + 1]++;
  for (int64_t l = 0; l < S.nlevels; ++l) S.level_ptr[l + 1] += S.level_ptr[l];
  S.level_nodes.resize(ns);
  {
    std::vector<int64_t> fillp(S.level_ptr.begin(), S.level_ptr.end() - 1);
    for (int64_t s = 0; s < ns; ++s) S.level_nodes[fillp[S.level[s]]++] = (int32_t)s;
  }
  S.front.resize(ns);
  S.rows_off.resize(ns + 1);
  {
    std::vector<std::vector<int32_t>> fr(ns);
    const int nt = sym_threads(n);
    std::vector<std::vector<int32_t>> marks(nt);
    auto one = [&](int32_t* mark, int64_t s) {
      const int64_t a = S.col0[s], e = S.col0[s] + S.ncol[s] - 1;
      std::vector<int32_t>& out = fr[s];
      out.clear();
      for (int64_t j = a; j <= e; ++j) out.push_back((int32_t)j);
      const size_t head = out.size();
      for (int64_t j = a; j <= e; ++j) mark[j] = (int32_t)s;
      for (int64_t j = a; j <= e; ++j) {
        const int64_t o = S.order[j];
        for (int64_t q = rowptr[o]; q < rowptr[o + 1]; ++q) {
          const int64_t i = io[colidx[q]];
          if (i > e && mark[i] != (int32_t)s) {
            mark[i] = (int32_t)s;
            out.push_back((int32_t)i);
          }
        }
      }
      for (int64_t t = S.child_ptr[s]; t < S.child_ptr[s + 1]; ++t) {
        const std::vector<int32_t>& rc = fr[S.child_list[t]];
        for (size_t u = S.ncol[S.child_list[t]]; u < rc.size(); ++u) {
          const int64_t i = rc[u];
          if (i > e && mark[i] != (int32_t)s) {
            mark[i] = (int32_t)s;
            out.push_back((int32_t)i);
          }
        }
      }
      std::sort(out.begin() + head, out.end());
      S.front[s] = (int64_t)out.size();
    };
    for (int64_t l = 0; l < S.nlevels; ++l) {
      const int64_t b = S.level_ptr[l], cnt = S.level_ptr[l + 1] - b;
      const int ntl = cnt < 64 ? 1 : nt;
      par_chunks(ntl, cnt, 8, [&](int t, int64_t q0, int64_t q1) {
        if (marks[t].empty()) marks[t].assign(n, -1);
        for (int64_t q = q0; q < q1; ++q) one(marks[t].data(), S.level_nodes[b + q]);
      });
    }
    S.rows_off[0] = 0;
    for (int64_t s = 0; s < ns; ++s) S.rows_off[s + 1] = S.rows_off[s] + S.front[s];
    S.rows.resize(S.rows_off[ns]);
    par_chunks(nt, ns, 64, [&](int, int64_t s0, int64_t s1) {
      for (int64_t s = s0; s < s1; ++s) std::copy(fr[s].begin(), fr[s].end(), S.rows.begin() + S.rows_off[s]);
    });
  }
  phase("fronts");
  // ---- 5b. storage offsets, statistics -------------------------------------
  S.panel_off.resize(ns);
  S.cb_off.resize(ns);
  S.upd_off.resize(ns + 1);
  S.panel_total = S.cb_total = S.upd_total = S.stored_L = 0;
  S.max_front = S.max_ncol = S.relaxed_flops = 0;
  // large fronts first in both regions so one memset covers them
  for (int pass = 0; pass < 2; ++pass) {
    for (int64_t s = 0; s < ns; ++s) {
      bool large = S.front[s] > kSmallFront;
      if ((pass == 0) != large) continue;
      int64_t f = S.front[s], np = S.ncol[s], nu = f - np;
      S.panel_off[s] = S.panel_total;
      S.panel_total += (f * np + 1) & ~int64_t(1);  // 16-byte aligned panels (TMA bulk copies)
      (void)nu;
    }
    if (pass == 0) S.panel_large = S.panel_total;
  }
  for (int64_t s = 0; s < ns; ++s) {
    int64_t f = S.front[s], np = S.ncol[s], nu = f - np;
    S.upd_off[s] = S.upd_total;
    S.upd_total += nu;
    S.stored_L += stored(np, f) - np;  // strict lower entries incl. relaxation zeros
    S.max_front = std::max(S.max_front, f);
    S.max_ncol = std::max(S.max_ncol, np);
    for (int64_t k = 0; k < np; ++k) S.relaxed_flops += (f - k) * (f - k);
  }
  S.upd_off[ns] = S.upd_total;
  phase("offsets");
  // ---- 5c. extend-add relative positions (update rows -> parent front) ----
  S.relpos.assign(S.upd_total, -1);
  {
    std::vector<int32_t> pos(n, -1);
    for (int64_t p = 0; p < ns; ++p) {
      const int32_t* rp = &S.rows[S.rows_off[p]];
      for (int64_t u = 0; u < S.front[p]; ++u) pos[rp[u]] = (int32_t)u;
      for (int64_t t = S.child_ptr[p]; t < S.child_ptr[p + 1]; ++t) {
        int64_t c = S.child_list[t];
        const int32_t* rc = &S.rows[S.rows_off[c]];
        for (int64_t u = S.ncol[c]; u < S.front[c]; ++u) {
          int32_t q = pos[rc[u]];
          if (q < 0) {
            err = "extend-add row missing from parent structure";
            return 1;
          }
          S.relpos[S.upd_off[c] + u - S.ncol[c]] = q;
        }
      }
      for (int64_t u = 0; u < S.front[p]; ++u) pos[rp[u]] = -1;
    }
  }
  phase("relpos");
  // ---- 5d. original-entry scatter map (lower triangle, by supernode) ------
  // Two parallel passes over supernodes: count, then fill at the prefix sums.
  if (with_asm_map) S.asm_ptr.assign(ns + 1, 0);
  if (with_asm_map) {
    const int nt = sym_threads(n);
    par_chunks(nt, ns, 32, [&](int, int64_t s0, int64_t s1) {
      for (int64_t s = s0; s < s1; ++s) {
        int64_t c = 0;
        for (int64_t j = S.col0[s]; j < S.col0[s] + S.ncol[s]; ++j) {
          const int64_t o = S.order[j];
          for (int64_t q = rowptr[o]; q < rowptr[o + 1]; ++q) c += io[colidx[q]] >= j;
        }
        S.asm_ptr[s + 1] = c;
      }
    });
    for (int64_t s = 0; s < ns; ++s) S.asm_ptr[s + 1] += S.asm_ptr[s];
    S.asm_slot.resize(S.asm_ptr[ns]);
    S.asm_local.resize(S.asm_ptr[ns]);
    std::vector<std::vector<int32_t>> poss(nt);
    std::atomic<int> bad{0};
    par_chunks(nt, ns, 32, [&](int t, int64_t s0, int64_t s1) {
      if (poss[t].empty()) poss[t].assign(n, -1);
      int32_t* pos = poss[t].data();
      for (int64_t s = s0; s < s1; ++s) {
        const int32_t* rs = &S.rows[S.rows_off[s]];
        const int64_t f = S.front[s];
        int64_t w = S.asm_ptr[s];
        for (int64_t u = 0; u < f; ++u) pos[rs[u]] = (int32_t)u;
        for (int64_t j = S.col0[s]; j < S.col0[s] + S.ncol[s]; ++j) {
          const int64_t o = S.order[j];
          for (int64_t q = rowptr[o]; q < rowptr[o + 1]; ++q) {
            const int64_t i = io[colidx[q]];
            if (i < j) continue;
            const int32_t r = pos[i];
            if (r < 0) {
              bad = 1;
              continue;
            }
            S.asm_slot[w] = q;
            S.asm_local[w++] = (int32_t)((j - S.col0[s]) * f + r);
          }
        }
        for (int64_t u = 0; u < f; ++u) pos[rs[u]] = -1;
      }
    });
    if (bad) {
      err = "original entry outside its front";
      return 1;
    }
  }
  S.nnz_lower = (int64_t)S.asm_slot.size();
  phase("asm map");
  // ---- 5e. levels (computed in 5a): small fronts first within a level -------
  S.level_nsmall.assign(S.nlevels, 0);
  for (int64_t l = 0; l < S.nlevels; ++l) {
    auto b = S.level_nodes.begin() + S.level_ptr[l], e = S.level_nodes.begin() + S.level_ptr[l + 1];
    std::stable_sort(b, e, [&](int32_t x, int32_t y) {
      bool lx = S.front[x] > kSmallFront, ly = S.front[y] > kSmallFront;
      if (lx != ly) return !lx;
      return S.front[x] < S.front[y];
    });
    int64_t cnt = 0;
    for (auto it = b; it != e; ++it)
      if (S.front[*it] <= kSmallFront) cnt++;
    S.level_nsmall[l] = cnt;
  }
  phase("levels");
  // ---- 5f. update-block memory plan ------------------------------------------
  // A front's update block is written at its own level and consumed (extend-
  // add) at its parent's level, so it is live on [level(s), level(parent)].
  // First-fit offsets over that liveness: cb_total is the high-water mark, not
  // the sum of all update blocks (cfg5: 26 GB summed).
  {
    std::map<int64_t, int64_t> freel;  // offset -> length of free gaps below the top
    int64_t top = 0;
    auto take = [&](int64_t need) {
      for (auto it = freel.begin(); it != freel.end(); ++it) {
        if (it->second >= need) {
          const int64_t off = it->first, rest = it->second - need;
          freel.erase(it);
          if (rest) freel[off + need] = rest;
          return off;
        }
      }
      const int64_t off = top;
      top += need;
      return off;
    };
    auto give = [&](int64_t off, int64_t len) {
      auto it = freel.emplace(off, len).first;
      auto nx = std::next(it);
      if (nx != freel.end() && it->first + it->second == nx->first) {
        it->second += nx->second;
        freel.erase(nx);
      }
      if (it != freel.begin()) {
        auto pv = std::prev(it);
        if (pv->first + pv->second == it->first) {
          pv->second += it->second;
          freel.erase(it);
          it = pv;
        }
      }
      if (it->first + it->second == top) {
        top = it->first;
        freel.erase(it);
      }
    };
    std::vector<std::vector<int32_t>> consumed(S.nlevels);
    for (int64_t l = 0; l < S.nlevels; ++l) {
      for (int64_t q = S.level_ptr[l]; q < S.level_ptr[l + 1]; ++q) {
        const int32_t s = S.level_nodes[q];
        const int64_t nu = S.front[s] - S.ncol[s];
        S.cb_off[s] = 0;
        if (nu <= 0) continue;
        S.cb_off[s] = take((nu * nu + 1) & ~int64_t(1));
        if (S.sparent[s] >= 0) consumed[S.level[S.sparent[s]]].push_back(s);
      }
      S.cb_total = std::max(S.cb_total, top);
      for (int32_t c : consumed[l]) {
        const int64_t nu = S.front[c] - S.ncol[c];
        give(S.cb_off[c], (nu * nu + 1) & ~int64_t(1));
      }
    }
    S.cb_large = 0;
  }
  phase("cb plan");
  return 0;
}

}  // namespace riga
