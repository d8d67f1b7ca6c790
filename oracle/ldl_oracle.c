/*
 * ORACLE — test infrastructure only.  Never linked into the product path.
 *
 * Plain-C restatement of the reference's sparse LDL^T kernels, used by
 * tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg as the
 * checker.  Algorithm follows the reference's numba kernels:
 *
 *   oracle_etree_counts  <- _etree_counts   /root/reference/pkg/src/rigaeig/sparsela.py:100-115
 *   oracle_ldl_numeric   <- _ldl_numeric    sparsela.py:118-159
 *   oracle_ldl_solve     <- _ldl_solve      sparsela.py:162-175
 *
 * Input convention (sparsela.py:239-243): the upper triangle of P A P^T in
 * compressed-column form, diagonal included (Ap int64[n+1], Ai int32).
 * The up-looking column algorithm (Liu's elimination tree with path
 * marking; row pattern of L by a reach in the etree) is restated here with
 * the same floating-point operation order so that, compiled without FMA
 * contraction, D and L come out bit-identical to the reference's.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* Elimination tree and strict-lower column counts of L.
 * For each column k, every upper entry (i, k) with i < k walks i -> parent(i)
 * until it meets a node already visited in this column; each step marks the
 * node, counts one nonzero L(k, i) and fills in missing parents.            */
void oracle_etree_counts(int64_t n, const int64_t* Ap, const int32_t* Ai,
                         int32_t* parent, int64_t* lnz) {
  int64_t* mark = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t j = 0; j < n; ++j) { parent[j] = -1; mark[j] = -1; lnz[j] = 0; }
  for (int64_t k = 0; k < n; ++k) {
    mark[k] = k;
    for (int64_t q = Ap[k]; q < Ap[k + 1]; ++q) {
      int64_t node = Ai[q];
      for (; mark[node] != k; node = parent[node]) {
        if (parent[node] == -1) parent[node] = (int32_t)k;
        mark[node] = k;
        lnz[node] += 1;
      }
    }
  }
  free(mark);
}

/* Numeric up-looking LDL^T without pivoting.  Column lists Lp (from the
 * counts) are filled in increasing row order.  Returns -1, or the first
 * column k with |D[k]| < zero_tol (the factorization stops there, as in
 * the reference).                                                          */
int64_t oracle_ldl_numeric(int64_t n, const int64_t* Ap, const int32_t* Ai,
                           const double* Ax, const int32_t* parent,
                           const int64_t* Lp, int32_t* Li, double* Lx,
                           double* D, double zero_tol) {
  size_t nn = (size_t)(n > 0 ? n : 1);
  double* work = (double*)calloc(nn, sizeof(double));
  int64_t* stack = (int64_t*)malloc(sizeof(int64_t) * nn);
  int64_t* walk = (int64_t*)malloc(sizeof(int64_t) * nn);
  int64_t* mark = (int64_t*)malloc(sizeof(int64_t) * nn);
  int64_t* used = (int64_t*)calloc(nn, sizeof(int64_t));
  int64_t failed = -1;
  for (int64_t j = 0; j < n; ++j) mark[j] = -1;

  for (int64_t k = 0; k < n && failed < 0; ++k) {
    /* scatter column k of the upper triangle into work[], collect the
     * nonzero pattern of row k of L as a topologically ordered stack    */
    int64_t top = n;
    mark[k] = k;
    work[k] = 0.0;
    for (int64_t q = Ap[k]; q < Ap[k + 1]; ++q) {
      int64_t node = Ai[q];
      work[node] += Ax[q];
      int64_t len = 0;
      for (; mark[node] != k; node = parent[node]) {
        walk[len++] = node;
        mark[node] = k;
      }
      while (len > 0) stack[--top] = walk[--len];
    }
    /* sparse triangular solve for row k, accumulating the diagonal */
    double dk = work[k];
    work[k] = 0.0;
    for (int64_t s = top; s < n; ++s) {
      int64_t i = stack[s];
      double yi = work[i];
      work[i] = 0.0;
      int64_t end = Lp[i] + used[i];
      for (int64_t q = Lp[i]; q < end; ++q) work[Li[q]] -= Lx[q] * yi;
      double lki = yi / D[i];
      dk -= lki * yi;
      Li[end] = (int32_t)k;
      Lx[end] = lki;
      used[i] += 1;
    }
    D[k] = dk;
    if (fabs(dk) < zero_tol) failed = k;
  }
  free(work); free(stack); free(walk); free(mark); free(used);
  return failed;
}

/* In-place x <- L^{-T} D^{-1} L^{-1} x (column-oriented forward sweep that
 * skips zero entries, diagonal scale, dot-product backward sweep).       */
void oracle_ldl_solve(int64_t n, const int64_t* Lp, const int32_t* Li,
                      const double* Lx, const double* D, double* x) {
  for (int64_t j = 0; j < n; ++j) {
    double xj = x[j];
    if (xj == 0.0) continue;
    for (int64_t q = Lp[j]; q < Lp[j + 1]; ++q) x[Li[q]] -= Lx[q] * xj;
  }
  for (int64_t j = 0; j < n; ++j) x[j] /= D[j];
  for (int64_t j = n - 1; j >= 0; --j) {
    double acc = 0.0;
    for (int64_t q = Lp[j]; q < Lp[j + 1]; ++q) acc += Lx[q] * x[Li[q]];
    x[j] -= acc;
  }
}
