// Handle definitions shared by the translation units of libriga_b200.so.
#pragma once

#include <cstring>
#include <memory>

#include "common.h"
#include "symbolic.h"

// 1D factor of a Kronecker-assembled system (x = axis 0 is fastest)
struct KronAxis {
  int64_t n = 0;
  riga::DevBuf<int64_t> rp;
  riga::DevBuf<int32_t> ci;
  riga::DevBuf<double> k, m;
};

struct riga_system {
  riga::CtxRef ctxref;
  riga_ctx* ctx = nullptr;
  int64_t n = 0, nnz = 0;
  riga::DevBuf<int64_t> rowptr;
  riga::DevBuf<int32_t> colidx;
  riga::DevBuf<double> K, M;
  int kdim = 0;      // > 0: M = M_z (x) M_y (x) M_x is applied axis by axis
  KronAxis kax[3];
};

// Device copy of the symbolic analysis (read-only, shared by all factors).
struct SymDev {
  const int64_t *col0, *ncol, *front, *rows_off, *panel_off, *cb_off, *upd_off;
  const int64_t *child_ptr, *asm_ptr;
  const int32_t *sparent, *rows, *relpos, *child_list, *asm_slot, *asm_local;
  const int32_t *level_nodes, *order;
};

namespace riga {
// device recurrence state of one Lanczos run (lanczos.cu)
struct LzDev {
  int k;        // basis size; the pending direction sits in row k
  int clo;      // coupling window [clo, k) applied by the next step
  int nlocked;  // locked rows
  int stop;     // 1 = breakdown, 2 = limit reached (later replays are no-ops)
  int limit;    // extend target
  int steps;    // steps executed since the last upload
  int pad[2];
  double btol;     // breakdown tolerance
  double scal[8];  // [0] alpha, [1] |w|^2, [2] beta^2, [4] ref norm^2
};

}  // namespace riga

struct LevelPlan {
  int64_t begin = 0, nsmall = 0, nlarge = 0;  // offsets into level_nodes
  // small fronts: contiguous classes [cls_begin[c], cls_begin[c+1]) with max front cls_f[c]
  std::vector<int64_t> cls_begin;
  std::vector<int32_t> cls_f;
  int64_t max_np_large = 0, max_f_large = 0, max_nu_large = 0;
  // extend-add rounds into large parents: ranges into ea_items (device)
  std::vector<int64_t> ea_round_begin;  // size rounds+1
  std::vector<int64_t> ea_round_maxnu;
  int64_t max_f = 0, max_np = 0;
};

struct I2 {
  int32_t x, y;
};

// Task lists and pull map of the level-scheduled solve kernels (solve.cu).
struct SolvePlanHost {
  int warp_stage = 0, chain_inv = 1, small_g = 1, occ = 4, rest_cap = 1 << 30;
  int inv_fix = 1;  // local refinement step after each inv(L11) application
  int64_t g_total = 0;                 // doubles of G = [inv(L11); L21 inv(L11)] of the small supernodes
  std::vector<int64_t> g_off;          // per supernode offset into gsmall (-1: large)
  std::vector<I2> gfwd, gbwd;          // G warp tasks: (supernode, row tile) / (supernode, column group)
  int64_t inv_total = 0;               // doubles of the inv(L11) blocks of the chain supernodes
  std::vector<int64_t> inv_off;        // per supernode offset into linv (-1: none)
  std::vector<I2> ifwd, ibwd, idiag;  // (supernode, 32-row tile / 8-row group / 32-col block)
  std::vector<I2> dbl_tasks;            // doubling inversion pairs (supernode, q), by level
  std::vector<int64_t> dbl_ptr, dbl_size, dbl_tiles, dbl_toff;
  int64_t dbl_tmax = 0;                 // doubles of T scratch (largest level)
  std::vector<int64_t> ifwd_ptr, ibwd_ptr, ifwd_smem;
  std::vector<I2> fwd, bwd;        // light tasks grouped by level
  std::vector<int32_t> chains;     // large supernodes grouped by level
  std::vector<int32_t> wholes;     // small supernodes (warp tasks) grouped by level
  std::vector<int32_t> gnodes;     // the same sorted by width class (k_small_g<GR>)
  int64_t gcls_ptr[5] = {0, 0, 0, 0, 0};  // class c (np <= 32 c) is gnodes[gcls_ptr[c-1] .. gcls_ptr[c])
  int sub_levels = 0, nsub = 0;        // bottom subtrees: height bound, count
  int sub_maxsn = 0;                   // most supernodes in one bottom subtree
  std::vector<int32_t> sub_fptr, sub_bptr;  // per subtree (sub_levels + 1) local-level task bounds
  std::vector<I2> sub_ftiles, sub_btiles;   // their G warp tasks (row tiles / column groups)
  std::vector<int64_t> fwd_ptr, bwd_ptr, chain_ptr;
  std::vector<int64_t> fwd_smem, bwd_smem, chf_smem, chb_smem;  // bytes per level launch
  std::vector<int32_t> gsrc;            // overflow pull map (children beyond the update-vector slots)
  std::vector<int64_t> gptr;
  std::vector<uint8_t> cmask;           // per front row: contributing child slots (solve.cu SolveDev)
  std::vector<int64_t> ubase;           // per supernode: base of its update vector's slot (-1: overflow child)
  int64_t nfront = 0, otail = 0, upd_doubles = 1;  // slot stride, overflow region start, buffer size
};

struct riga_symbolic {
  riga::CtxRef ctxref;
  riga_ctx* ctx = nullptr;
  riga_system* sys = nullptr;  // may be null (host-only analysis)
  riga::SymbolicHost h;
  std::vector<LevelPlan> plan;
  std::vector<int32_t> ea_items_host;  // child ids, grouped by (level, round)
  std::vector<int32_t> large_host;     // all large fronts (for k_asm_large)
  bool on_device = false;
  // device arrays
  riga::DevBuf<int64_t> d_col0, d_ncol, d_front, d_rows_off, d_panel_off, d_cb_off, d_upd_off;
  riga::DevBuf<int64_t> d_child_ptr, d_asm_ptr;
  riga::DevBuf<int32_t> d_sparent, d_rows, d_relpos, d_child_list, d_asm_slot, d_asm_local;
  riga::DevBuf<int32_t> d_level_nodes, d_order, d_ea_items, d_large_nodes;
  int64_t n_large = 0;
  SolvePlanHost sp;
  riga::DevBuf<I2> d_tfwd, d_tbwd;
  riga::DevBuf<int32_t> d_chains, d_wholes, d_gnodes, d_gsrc, d_sub_fptr, d_sub_bptr;
  riga::DevBuf<int64_t> d_gptr, d_inv_off, d_g_off, d_ubase;
  riga::DevBuf<uint8_t> d_cmask;
  riga::DevBuf<I2> d_ifwd, d_ibwd, d_idiag, d_dbl_tasks, d_gfwd, d_gbwd, d_sub_ftiles, d_sub_btiles;
  riga::DevBuf<int64_t> d_dbl_toff;
  SymDev dev() const {
    return SymDev{d_col0.p,     d_ncol.p,      d_front.p,      d_rows_off.p,   d_panel_off.p,
                  d_cb_off.p,   d_upd_off.p,   d_child_ptr.p,  d_asm_ptr.p,    d_sparent.p,
                  d_rows.p,     d_relpos.p,    d_child_list.p, d_asm_slot.p,   d_asm_local.p,
                  d_level_nodes.p, d_order.p};
  }
};

struct riga_factor {
  riga::CtxRef ctxref;
  riga_ctx* ctx = nullptr;
  riga_symbolic* sym = nullptr;
  double sigma = 0.0;
  riga::DevBuf<double> panel;  // all L panels (f x np, ld f)
  riga::DevBuf<double> D;      // pivots in elimination order
  riga::DevBuf<double> xperm;  // solve workspace (n)
  riga::DevBuf<double> upd;    // solve contribution vectors (sum n_u)
  riga::DevBuf<int64_t> stat;  // [0] n_negative, [1] first bad pivot (n if none)
  riga::DevBuf<double> cvec;   // backward L21^T x partial sums
  riga::DevBuf<double> tol;    // [0] max|A|, [1] zero_tol
  riga::DevBuf<double> linv;   // inv(L11) of the chain supernodes (solve.cu)
  riga::DevBuf<double> gsmall; // G of the small supernodes (solve.cu)
  riga::DevBuf<double> rfix;   // chain-supernode refinement residuals (n)
  riga::DevBuf<unsigned long long> inv_err;  // per supernode: inverse accuracy probe (double bits)
  riga::DevBuf<int> fix_flag;  // per supernode: 1 = refine after the inverse application
  std::vector<char> fix_level; // per level: any flagged chain supernode
  int n_fix = 0;               // flagged chain supernodes
  float factor_ms = 0.f;
};

namespace riga {
// kernels shared between translation units
int launch_dot(cudaStream_t s, int64_t n, const double* x, const double* y, double* out_dev);
int system_spmv(riga_system* sys, cudaStream_t s, int which, double sigma, const double* x, double* y);
// y = M x through the 1D factors (kdim > 0); t1, t2: n-vector scratch
int kron_mass_apply(riga_system* sys, cudaStream_t s, const double* x, double* y, double* t1, double* t2);
int csr_spmv(cudaStream_t s, int64_t n, const int64_t* rowptr, const int32_t* colidx,
             const double* val, const double* x, double* y);
// accurate: every chain supernode takes the local refinement step (the API
// solves); otherwise only those the factor-time probe flagged (the Lanczos
// steps, whose accuracy the residual gate covers)
int factor_solve(riga_factor* f, cudaStream_t s, const double* b, double* x, bool b_permuted = false,
                 bool accurate = false);
int build_solve_plan(riga_symbolic* sym);
int prepare_solve();
int upload_solve_plan(riga_symbolic* sym, cudaStream_t s);
int build_chain_inverse(riga_factor* F, cudaStream_t s);  // inv(L11) of the chain supernodes + accuracy probe
int build_small_g(riga_factor* F, cudaStream_t s);        // G blocks of the small supernodes
int64_t small_g_top_level(const riga_symbolic* sym);
int flag_inverse_refinement(riga_factor* F, cudaStream_t s);
inline double __longlong_as_double_host(long long v) {
  double d;
  memcpy(&d, &v, sizeof d);
  return d;
}
}  // namespace riga
