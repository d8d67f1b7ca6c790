// Host-side symbolic analysis of P A P^T for the multifrontal LDL^T.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace riga {

// Fronts with f <= kSmallFront are factored by one CTA in shared memory
// (f*f doubles <= 200 KB); larger ones by the batched multi-CTA path.
constexpr int kSmallFront = 160;

struct SymbolicHost {
  int64_t n = 0, nnz = 0, nnz_lower = 0;
  std::vector<int64_t> order;    // position -> original index (postordered perm)
  std::vector<int32_t> iorder;   // original index -> position
  std::vector<int64_t> post;     // position in the postorder -> position in the caller perm
  std::vector<int64_t> colcount; // per position, diagonal included (exact, unamalgamated)
  int64_t fill_nnz = 0, factor_flops = 0, fundamental = 0, tree_height = 0;

  // supernodes (relaxed), numbered in postorder (children before parents)
  int64_t nsuper = 0;
  std::vector<int64_t> col0, ncol, front, rows_off, panel_off, cb_off, upd_off;
  std::vector<int32_t> sparent;  // -1 for roots
  std::vector<int32_t> level;    // 0 = leaf
  std::vector<int32_t> rows;     // concatenated front row structures (positions)
  std::vector<int32_t> relpos;   // per supernode: its update rows -> position in parent's front
  std::vector<int64_t> child_ptr;   // CSR of supernode children
  std::vector<int32_t> child_list;
  int64_t panel_total = 0, cb_total = 0, upd_total = 0, stored_L = 0;
  int64_t panel_large = 0, cb_large = 0;  // large fronts occupy [0, *_large)
  int64_t max_front = 0, max_ncol = 0, relaxed_flops = 0;

  // original entries of the lower triangle, grouped by supernode:
  // asm_ptr[s]..asm_ptr[s+1]; slot = CSR slot in A; local = col_in_front*f + row_pos
  std::vector<int64_t> asm_ptr, asm_slot;
  std::vector<int32_t> asm_local;

  // levels (bottom-up): level_ptr over level_nodes; within a level: small
  // fronts first (sorted by f), then large fronts
  int64_t nlevels = 0;
  std::vector<int64_t> level_ptr;
  std::vector<int32_t> level_nodes;
  std::vector<int64_t> level_nsmall;  // count of small fronts at the head of each level
};

// Returns 0 on success; message in err otherwise.  with_asm_map = false leaves the scatter map of the
// original entries (asm_ptr / asm_slot / asm_local, nnz_lower) empty: a device analysis builds it on the
// device instead (factor.cu, build_asm_map_device).
int analyze(int64_t n, const int64_t* rowptr, const int32_t* colidx, const int64_t* perm,
            SymbolicHost& out, std::string& err, bool with_asm_map = true);

}  // namespace riga
