/*
 * riga_b200.h — C ABI of libriga_b200.so, the B200 (sm_100a) engine behind
 * the drop-in Python API of paper_2009_08167_b200.
 *
 * The reference (rigaeig v0.1.0, /root/reference/pkg/src/rigaeig) has no FFI:
 * its boundary is the set of Python functions in sparsela.py/eigensolver.py,
 * one level above three numba kernels.  Each entry point below names the
 * reference interface it replaces.  ctypes binds this header
 * (paper_2009_08167_b200/_lib.py; INTEGRATION.md shows the binding).
 *
 * Conventions
 *  - every call returns an int status (never throws across the ABI):
 *      0 RIGA_OK, 1 RIGA_ZERO_PIVOT, 2 RIGA_BAD_ARG, 3 RIGA_CUDA_ERROR,
 *      4 RIGA_OOM, 5 RIGA_BREAKDOWN (Lanczos invariant subspace), 6 RIGA_NO_DEVICE;
 *    riga_last_error() gives the message of the last failure (thread-local).
 *  - "host" pointers are plain CPU memory; "dev" pointers are device memory
 *    on the handle's device (e.g. torch tensor data_ptr()).
 *  - handles are opaque, owned by the library, freed by riga_*_destroy; each
 *    handle is bound to one device and one CUDA stream and must not be used
 *    from two host threads at once; different handles may run concurrently.
 *  - indices: CSR row pointers int64, column indices int32; permutations
 *    int64 with position k holding the original index eliminated k-th
 *    (reference separator_ordering convention, sparsela.py:319-330).
 */
#ifndef RIGA_B200_H
#define RIGA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  RIGA_OK = 0,
  RIGA_ZERO_PIVOT = 1,
  RIGA_BAD_ARG = 2,
  RIGA_CUDA_ERROR = 3,
  RIGA_OOM = 4,
  RIGA_BREAKDOWN = 5,
  RIGA_NO_DEVICE = 6
};

typedef struct riga_ctx riga_ctx;
typedef struct riga_system riga_system;
typedef struct riga_symbolic riga_symbolic;
typedef struct riga_factor riga_factor;
typedef struct riga_lanczos riga_lanczos;

/* ---- library / context ------------------------------------------------ */
const char* riga_last_error(void);
int riga_version(void);
/* Number of CUDA devices visible (0 on a CPU-only host). */
int riga_device_count(int* count);
/* Stream-ordered pool of `device` (where every engine buffer lives):
 * out[0] reserved bytes, out[1] reserved high-water, out[2] used bytes,
 * out[3] used high-water.  reset_high != 0 resets both high-water marks. */
int riga_mem_info(int device, int reset_high, int64_t* out4);
/* Context = (device, stream).  stream_handle: 0 -> create a private
 * non-blocking stream; otherwise a cudaStream_t owned by the caller. */
int riga_ctx_create(int device, void* stream_handle, riga_ctx** out);
int riga_ctx_destroy(riga_ctx* ctx);
int riga_ctx_synchronize(riga_ctx* ctx);
/* Bytes the device's default stream-ordered pool holds but no allocation
 * uses (freed engine buffers and torch tensors kept for reuse): memory
 * planners count them as available.                                       */
int riga_device_pool_reusable(int device, int64_t* bytes);
/* Host threads waiting on the device block (on = 1) instead of spinning
 * (cudaDeviceScheduleBlockingSync on the device's primary context): with a
 * host thread per slice, spinning waiters compete for the host cores.      */
int riga_set_blocking_sync(int device, int on);
/* Raw cudaStream_t of the context (for torch.cuda.ExternalStream). */
int riga_ctx_stream(riga_ctx* ctx, void** stream_out);

/* ---- system: device CSR of K and M on one shared pattern ------------------
 * Replaces the scipy CSR pair of DiscreteSystem (ref assembly.py:24-62).   */
int riga_system_upload(riga_ctx* ctx, int64_t n, int64_t nnz, const int64_t* rowptr_host,
                       const int32_t* colidx_host, const double* K_host, const double* M_host,
                       riga_system** out);
/* Device assembly of the Kronecker-composed Dirichlet-reduced pencil from
 * 1D banded CSR matrices (ref assembly.py:139-192 kron_assemble).  dim in
 * {1,2,3}; per direction t (x, y, z): n1[t], rowptr1[t], colidx1[t],
 * k1[t], m1[t] (host).  Values are bit-identical to scipy's kron/+ (product
 * and sum order fixed, no FMA contraction).                                 */
int riga_system_assemble_kron(riga_ctx* ctx, int dim, const int64_t* n1,
                              const int64_t* const* rowptr1, const int32_t* const* colidx1,
                              const double* const* k1, const double* const* m1,
                              riga_system** out);
/* Device element-quadrature assembly (ref assembly.py:72-111 integrated in d
 * dimensions): every element of the tensor mesh with (p+1)^d Gauss points.
 * Per direction t: ne[t] elements; first[t][e] = global (full) index of the
 * element's first basis function (span - p); w[t][e][q] scaled Gauss
 * weights; N[t][e][q][a], dN[t][e][q][a] basis values / derivatives at the
 * points (host).  n1 / rowptr1 / colidx1 / k1 / m1: the Dirichlet-reduced 1D
 * matrices as for riga_system_assemble_kron (they define the shared CSR
 * pattern).  Values equal the Kronecker pencil to roundoff; deterministic
 * (element colour classes, no atomics).  dim 1-3, degree 1-5 (3D: 1-3).    */
int riga_system_assemble_quad(riga_ctx* ctx, int dim, int p, const int64_t* ne, const int32_t* const* first,
                              const double* const* w, const double* const* N, const double* const* dN,
                              const int64_t* n1, const int64_t* const* rowptr1, const int32_t* const* colidx1,
                              const double* const* k1, const double* const* m1, riga_system** out);
/* Attach 1D factors to an uploaded pencil whose M is M_z (x) M_y (x) M_x
 * (arguments as riga_system_assemble_kron; n must equal prod n1): the
 * Lanczos mass products then run axis by axis instead of over the CSR.
 * The caller asserts the Kronecker structure (DiscreteSystem.m1d).        */
int riga_system_set_kron(riga_system* sys, int dim, const int64_t* n1,
                         const int64_t* const* rowptr1, const int32_t* const* colidx1,
                         const double* const* k1, const double* const* m1);
int riga_system_info(riga_system* sys, int64_t* n, int64_t* nnz);
int riga_system_download(riga_system* sys, int64_t* rowptr_host, int32_t* colidx_host,
                         double* K_host, double* M_host);
/* Device pointers (for callers that keep data on the device). */
int riga_system_device_ptrs(riga_system* sys, const int64_t** rowptr, const int32_t** colidx,
                            const double** K, const double** M);
int riga_system_destroy(riga_system* sys);

/* y = A x on the device, A = K (which=0), M (which=1) or K - sigma M (2).
 * Replaces mass_matvec (ref sparsela.py:280-290, scipy csr_matvec).        */
int riga_spmv(riga_system* sys, int which, double sigma, const double* x_dev, double* y_dev);
/* Y[j] = A X[j] for nvec device vectors (rows, leading dimensions ldx /
 * ldy >= n), A as riga_spmv, on ctx's stream (NULL = the system's).       */
int riga_spmv_many(riga_ctx* ctx, riga_system* sys, int which, double sigma, const double* X_dev, int64_t ldx,
                   int64_t nvec, double* Y_dev, int64_t ldy);
/* Generic device CSR SpMV on caller arrays (any square CSR, e.g. a plain
 * scipy matrix handed to mass_matvec).                                     */
int riga_csr_spmv(riga_ctx* ctx, int64_t n, const int64_t* rowptr_dev, const int32_t* colidx_dev,
                  const double* val_dev, const double* x_dev, double* y_dev);

/* ---- separator ordering (ref sparsela.py:319-392 separator_ordering) -----
 * Nested dissection aligned with the C0 planes of the tensor-product box of
 * `d` axes with ext[t] cells (Dirichlet-reduced basis counts) and degree p.
 * lines: the C0 plane indices of all axes concatenated (ascending per axis),
 * nlines[t] of them on axis t (ref _direction_c0 :313-316).
 * riga_separator_boxes builds the dissection tree on the host (a few
 * thousand boxes) and returns the blocks in elimination order: leaves in
 * recursion order, then separators deepest level first (ref :386-389).
 * chunks: cap x 7 int64 (offset, lo[3], extent[3]); with chunks == NULL or
 * cap too small only *nchunks is set (size query).
 * riga_separator_emit writes the permutation on the device (one thread per
 * elimination position; cells of a block in the reference's emit() order,
 * axis 0 fastest): perm_dev[k] = original index eliminated k-th.           */
int riga_separator_boxes(int d, const int64_t* ext, int degree, const int64_t* lines, const int64_t* nlines,
                         int64_t cap, int64_t* nchunks, int64_t* chunks);
int riga_separator_emit(riga_ctx* ctx, int d, const int64_t* ext, int64_t nchunks, const int64_t* chunks_host,
                        int64_t n, int64_t* perm_dev);

/* ---- symbolic analysis (host C++ and, for the scatter map of the original
 * entries, device kernels; once per pattern + ordering) ------------------
 * Replaces the per-call permute/triu/_etree_counts of factor_ldl
 * (ref sparsela.py:239-250, _etree_counts :100-115): elimination tree,
 * postorder, column counts, fundamental + relaxed supernodes, frontal row
 * structures, extend-add maps, tree levels.  fill_nnz and factor_flops
 * are the reference's exact (unamalgamated) counts: nnz(L)+n and
 * sum (colcount)^2 (ref sparsela.py:257-258).                              */
int riga_symbolic_create(riga_system* sys, const int64_t* perm_host, riga_symbolic** out);
/* Host-only analysis of a pattern (no device needed; used by CPU tests). */
int riga_symbolic_analyze(int64_t n, const int64_t* rowptr_host, const int32_t* colidx_host,
                          const int64_t* perm_host, riga_symbolic** out);
/* stats[0..15]: fill_nnz, factor_flops, n_supernodes, max_front, n_levels,
 * panel_entries, cb_entries, max_ncol, fundamental_supernodes,
 * stored_L_entries, n_small_fronts, n_large_fronts, nnz_lower,
 * tree_height, relaxed_flops (padded dense-front flop count), reserved. */
int riga_symbolic_stats(riga_symbolic* sym, int64_t* stats16);
/* Elimination order actually used (postordered copy of perm), int64[n]. */
int riga_symbolic_order(riga_symbolic* sym, int64_t* order_host);
/* Exact column counts of L (diagonal included) in the caller's perm order. */
int riga_symbolic_colcounts(riga_symbolic* sym, int64_t* counts_host);
/* Scatter map of the original lower-triangle entries into the fronts, grouped
 * by supernode: asm_ptr[n_supernodes + 1], then per entry the CSR slot and the
 * position col_in_front * f + row_pos in the supernode's panel.  A device
 * analysis (riga_symbolic_create) builds it on the device, a host analysis on
 * the host; *count = entries (stats nnz_lower); with the three arrays NULL
 * only *count is set.  For tests.                                            */
int riga_symbolic_asm_map(riga_symbolic* sym, int64_t* count, int64_t* asm_ptr_host, int32_t* slot_host,
                          int32_t* local_host);
/* Supernode table (relaxed supernodes in postorder, n_supernodes entries
 * each): first column, column count, front size, parent (-1 root), tree
 * level (0 = leaf).  For analysis and tests.                              */
int riga_symbolic_supernodes(riga_symbolic* sym, int64_t* col0, int64_t* ncol, int64_t* front,
                             int64_t* parent, int64_t* level);
int riga_symbolic_destroy(riga_symbolic* sym);

/* ---- numeric multifrontal LDL^T of K - sigma M --------------------------
 * Replaces factor_ldl + _ldl_numeric (ref sparsela.py:212-262, :118-159):
 * unpivoted, zero_tol = rel_zero_tol * max|K - sigma M| computed on the
 * device; inertia from the signs of D.  Status RIGA_ZERO_PIVOT when some
 * |d_k| < zero_tol; *bad_pivot = the smallest such elimination position.
 * ctx selects the stream (NULL = the symbolic handle's context); the
 * factor stays bound to that context.                                      */
int riga_factor_create(riga_ctx* ctx, riga_symbolic* sym, double sigma, double rel_zero_tol,
                       riga_factor** out, int64_t* n_negative, int64_t* bad_pivot);
/* x = A^{-1} b, b and x device vectors in ORIGINAL numbering (may alias).
 * Replaces solve_fb + _ldl_solve (ref sparsela.py:265-277, :162-175).      */
int riga_factor_solve(riga_factor* f, const double* b_dev, double* x_dev);
/* Block solve X[:, j] = A^{-1} B[:, j] for nrhs device vectors stored with
 * leading dimensions ldb / ldx (>= n), on ctx's stream (NULL = the
 * factor's; ordered after the factor's own stream).
 * solve(fact, x, nrhs); used by the residual-gate refinement.             */
int riga_factor_solve_many(riga_ctx* ctx, riga_factor* f, const double* B_dev, int64_t ldb, int64_t nrhs,
                           double* X_dev, int64_t ldx);
/* Timing of the last numeric factorization on the device (ms). */
int riga_factor_time_ms(riga_factor* f, float* ms);
/* D in elimination order (host double[n]). */
int riga_factor_D(riga_factor* f, double* D_host);
/* Supernodal L as CSC (unit diagonal excluded) in elimination order
 * riga_symbolic_order(); Lp int64[n+1]; sizes from stats[9]
 * (stored_L_entries).  For the reference's LDLFactorization.l_matrix()
 * test hooks (ref sparsela.py:199-203).                                    */
int riga_factor_export(riga_factor* f, int64_t* Lp_host, int32_t* Li_host, double* Lx_host);
int riga_factor_destroy(riga_factor* f);

/* ---- device Lanczos (shift-invert, CGS2 full reorthogonalisation) ------
 * Replaces LanczosState / lanczos_extend / lift / thick_restart
 * (ref eigensolver.py:140-357).  The basis V, its mass products MV
 * (row-major, max_dim+1 rows of n) and the locked set live on the device;
 * the host keeps T, coupling and all decisions.  mass = NULL selects the
 * Euclidean inner product (ref LanczosState(mass=None)).                   */
int riga_lanczos_create(riga_ctx* ctx, riga_system* mass, int64_t n, int64_t max_dim,
                        riga_lanczos** out);
int riga_lanczos_destroy(riga_lanczos* lz);
/* Empty the state for reuse by a new LanczosState with the same n and
 * max_dim (k = 0, no locked rows; buffers are kept, so a reused state
 * allocates nothing) and bind `mass` (same n; NULL = Euclidean).           */
int riga_lanczos_reset(riga_lanczos* lz, riga_system* mass);
/* Operator for the next extend: H = (K - shift M)^{-1} M via factor f.     */
int riga_lanczos_set_operator(riga_lanczos* lz, riga_factor* f);
/* Current basis size k (host view). */
int riga_lanczos_k(riga_lanczos* lz, int64_t* k);
/* Set the pending direction r from a host vector: Mr = M r, M-normalise.
 * Status RIGA_BAD_ARG when the mass norm is zero (ref :188-195).          */
int riga_lanczos_set_start(riga_lanczos* lz, const double* r_host);
/* Fresh random direction (host-drawn r, ref _fresh_direction :214-227):
 * ref_norm = sqrt(r M r); CGS2 against V[:k] and the locked set; accept if
 * the new mass norm > 1e-8 max(ref_norm, 1e-300).  *accepted = 0/1.       */
int riga_lanczos_fresh(riga_lanczos* lz, const double* r_host, int* accepted);
/* Append a locked pair (device vectors x, Mx of length n). */
int riga_lanczos_lock(riga_lanczos* lz, const double* x_dev, const double* mx_dev);
int riga_lanczos_locked_count(riga_lanczos* lz, int64_t* count);
/* Run Lanczos steps until k == limit or a breakdown (ref step :235-268).
 * coupling_host: the arrowhead row coupling[:k] to apply on the first step
 * (NULL = none).  Per executed step i: alpha[i], beta[i], wnorm[i] (host).
 * *steps = steps executed; status RIGA_BREAKDOWN if the last step broke
 * down (k already advanced, as in the reference).                          */
int riga_lanczos_extend(riga_lanczos* lz, int64_t limit, const double* coupling_host,
                        double breakdown_tol, double* alpha, double* beta, double* wnorm,
                        int64_t* steps);
/* Device milliseconds of the last extend's step replays (CUDA events on
 * the state's stream around the replayed step graphs; 0 if none ran).      */
int riga_lanczos_last_extend_ms(riga_lanczos* lz, float* ms);
/* One step with a caller-computed w = H v (device vector of length n), for
 * operators that are not a device factor (ref LanczosState(apply_op=...)
 * with an arbitrary callable).  Outputs as riga_lanczos_extend (1 step).   */
int riga_lanczos_step_given(riga_lanczos* lz, const double* w_dev, const double* coupling_host,
                            double breakdown_tol, double* alpha, double* beta, double* wnorm);
/* X = V[:k]^T W, MX = MV[:k]^T W for c weight columns (W host, k x c,
 * column-major), written as c rows of n into X_dev / MX_dev (ref lift
 * :270-274, batched over the converged pairs of a cycle).                 */
int riga_lanczos_lift(riga_lanczos* lz, const double* W_host, int64_t c, double* X_dev, double* MX_dev);
/* Thick restart: V[:c] <- (V[:k]^T W)^T, MV likewise, k <- c; the pending
 * residual direction is kept (ref thick_restart :326-357).                 */
int riga_lanczos_restart(riga_lanczos* lz, const double* W_host, int64_t c);
/* In-place projection of (x, mx) against the locked set, `passes` times:
 * c = LM x; x -= L^T c; mx -= LM^T c (ref _sweep locking block :491-505).  */
int riga_lanczos_project_locked(riga_lanczos* lz, double* x_dev, double* mx_dev, int passes);
/* Lock c converged pairs (rows of X / MX, row stride ldx, device) in order,
 * exactly as the reference's locking loop (ref _sweep :483-523): M-normalise,
 * two projections against the locked set (which grows by the pairs accepted
 * earlier in the batch), reject when the projected norm is < 0.3, else
 * re-normalise and append.  X / MX are updated in place; accepted[q] = 0/1
 * (host).  One host synchronisation for the whole batch.                  */
int riga_lanczos_lock_batch(riga_lanczos* lz, double* X_dev, double* MX_dev, int64_t c, int64_t ldx,
                            int* accepted);
/* Block form of the same locking (one pass over the locked set per 8 pairs
 * instead of per pair): M-normalise the c rows, then twice project against
 * the locked set and against the earlier rows of the batch; returns the
 * projected x.Mx per row (host) for the accept / 0.3 decision.  Equal to
 * the sequential order to second order in the (1e-10-level) couplings.    */
int riga_lanczos_lock_block(riga_lanczos* lz, double* X_dev, double* MX_dev, int64_t c, int64_t ldx,
                            double* nrm2_host);
/* Append c rows to the locked set, dividing row q by sqrt(nrm2[q]) first
 * when scale[q] != 0.                                                     */
int riga_lanczos_append_rows(riga_lanczos* lz, double* X_dev, double* MX_dev, int64_t c, int64_t ldx,
                             const double* nrm2_host, const int* scale_host);
/* Measurement hook: `passes` Gram-Schmidt passes of x against V[:k] and the
 * locked set (the step's CGS kernels, launched directly on the context
 * stream so CUDA events can bracket them); *rows = k + locked.            */
int riga_lanczos_cgs_probe(riga_lanczos* lz, double* x_dev, int passes, int64_t* rows);
/* Measurement hook: the step's delayed-CGS2 sweeps (one dots sweep of the
 * pending row and w over V[:k+1] + locked, one update sweep) with w = w_dev;
 * writes only scratch.  *rows = k + 1 + locked.                           */
int riga_lanczos_dcgs_probe(riga_lanczos* lz, const double* w_dev, int64_t* rows);
/* Gram matrix G = V[:k] MV[:k]^T to host (k x k row-major) for the
 * DEBUG_INVARIANTS checks (ref check_invariants :276-282).                 */
int riga_lanczos_gram(riga_lanczos* lz, double* G_host);
/* Device bytes the state holds (basis, locked rows at their current
 * capacity, scratch): memory planners count pooled idle states with it.   */
int riga_lanczos_bytes(riga_lanczos* lz, int64_t* bytes);
/* Device pointers of V and MV (row-major, leading dimension *ld). */
int riga_lanczos_basis(riga_lanczos* lz, double** V, double** MV, int64_t* ld);

/* ---- measurement ---------------------------------------------------------
 * Kernel launches issued by the engine since load (bench.py gpu_launches). */
int riga_launch_count(int64_t* count);
/* Per-category device timing with CUDA events on the launching stream:
 * 0 factor (work = factor_flops), 1 solve (bytes 16 fill_nnz + 32 n),
 * 2 SpMV (bytes 12 nnz + 4 (n+1) + 16 n), 3 CGS pass (bytes 2 rows n 8),
 * 4 vector ops, 5 lift/restart.  read: ms, work, scope counts per category. */
int riga_prof_enable(int on);
/* Programmatic dependent launch of the step kernels on (1) / off (0) for
 * graphs captured from now on (default: RIGA_PDL env, off).  It shortens a
 * lone slice's step (~10 %); with many concurrent slice streams the waiting
 * CTAs cost more than they hide, so the slicing driver enables it only with
 * few slices per GPU.                                                       */
int riga_set_pdl(int on);
/* Height bound of the bottom subtrees whose solve runs as one CTA each, for
 * symbolic analyses created from now on (default 6; RIGA_SUB_LEVELS
 * overrides).  Few concurrent slices per GPU: 6 (latency); 16: 8.          */
int riga_set_solve_sub_levels(int levels);
int riga_prof_read(double* ms, double* work, int64_t* scopes, int ncat);
int riga_prof_reset(void);

/* ---- eigenpair residuals (north-star gate) ---------------------------------
 * For nvec device vectors x_v (rows of X, leading dimension ldx >= n) and
 * host eigenvalues lam[v]: out[3 v + 0] = ||K x - lam M x||^2,
 * out[3 v + 1] = ||M x||^2, out[3 v + 2] = ||K x||^2 (host), one fused
 * pass over the CSR of K and M per 8 vectors, fixed-order reductions.
 * Replaces the residual loop of solve_spectrum (ref eigensolver.py:784-792)
 * and evaluates north_star's ||Ku - lam Mu|| / (|lam| ||Mu||) for every
 * returned pair.  ctx selects the stream (NULL = the system's).            */
int riga_residuals(riga_ctx* ctx, riga_system* sys, const double* X_dev, int64_t ldx, int64_t nvec,
                   const double* lam_host, double* out_host);

/* ---- tensor-product evaluation of the eigen-error study (verify.py) -------
 * riga_tp_contract replaces one direction of ErrorEvaluator._contract (ref
 * verify.py:218-225): in is an (outer, n_in, inner) row-major tensor,
 *   out[o, q, i] = s[o / outer_per_batch] * sum_{j < p1} vals[q p1 + j] * in[o, first[q] + j - off, i]
 * with rows outside [0, n_in) read as zero (off = 1 embeds the reduced
 * coefficient tensor between its Dirichlet layers, ref :136-148);
 * bscale_dev may be NULL.  A collocation matrix has p1 = p + 1 non-zeros per
 * quadrature point (first[q] = its first basis index), so the contraction is
 * a banded gather, HBM-bound.
 * riga_tp_reduce replaces ErrorEvaluator.integrate of (u_h - u)^2 (mode 0) or
 * u_h u (mode 1) or of the grid itself (mode 2) (ref :227-255) for nbatch grids G (nbatch, q_z, q_y, q_x)
 * against the exact modes u = prod_t sqrt(2) sin(k_t pi x_t) (ref :105-133;
 * direction `deriv` >= 0: that factor's derivative), formed on the fly from
 * kidx_dev[b dim + t]; nq_host, x_dev, w_dev: points and weights per
 * direction (x first); gsign_dev (may be NULL) multiplies G in mode 0;
 * out_dev[nbatch].  Fixed-order reductions.
 * riga_row_dots: out[v] = X[v, :] . Y[v, :] (the c^T M c normalisations).   */
int riga_tp_contract(riga_ctx* ctx, const double* in_dev, double* out_dev, int64_t outer, int64_t n_in,
                     int64_t n_out, int64_t inner, int p1, int off, const int32_t* first_dev,
                     const double* vals_dev, const double* bscale_dev, int64_t outer_per_batch);
int riga_tp_reduce(riga_ctx* ctx, const double* G_dev, int64_t nbatch, int dim, const int64_t* nq_host,
                   const double* const* x_dev, const double* const* w_dev, const int32_t* kidx_dev, int deriv,
                   int mode, const double* gsign_dev, double* out_dev);
int riga_row_dots(riga_ctx* ctx, const double* X_dev, int64_t ldx, const double* Y_dev, int64_t ldy, int64_t n,
                  int64_t nvec, double* out_dev);

/* ---- dense vector helpers on the device (stream of ctx) ----------------- */
int riga_dot(riga_ctx* ctx, int64_t n, const double* x_dev, const double* y_dev, double* out_host);

#ifdef __cplusplus
}
#endif
#endif /* RIGA_B200_H */
