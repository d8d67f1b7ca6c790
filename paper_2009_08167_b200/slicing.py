"""Uniform spectrum slicing across streams and GPUs.

Additive to the reference API (it has only the adaptive ``_march``):

* ``uniform_shifts(lam_e, S)``        sigma_k = k lam_e / S
* ``kronecker_spectrum(system)``      exact discrete spectrum from the 1D
                                      pencils (identity of ref
                                      tests/test_assembly.py:64-72)
* ``choose_lambda_e(system, N0)``     lam_e in the first spectral gap at or
                                      after N0
* ``solve_uniform_slices(...)``       every slice (sigma_k, sigma_k+1] with
                                      reference ``solve_slice`` semantics
                                      (fresh pool, rng seed_k, m = 2 count_k),
                                      but each boundary shift is factored
                                      once, slices run concurrently on
                                      several CUDA streams of a GPU, and
                                      across ranks (one process per GPU) the
                                      slices are partitioned by LPT on their
                                      inertia counts.  The only collectives
                                      are all-gathers of the boundary
                                      inertias and of the eigenvalues (plus
                                      boundary pairs for de-duplication).
"""
from __future__ import annotations

import math
import threading
import time
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import torch

from . import device as _dev
from .eigensolver import (CountMismatch, SolverOptions, _Boundary, _Pencil, _Pool, _solve_interval,
                          residual_gate)
from .sparsela import CostCounters, Symbolic, mass_matvec, separator_ordering


def uniform_shifts(lam_e: float, S: int) -> np.ndarray:
    return np.array([k * lam_e / S for k in range(S + 1)])


def kronecker_spectrum(system) -> np.ndarray:
    """Sorted discrete eigenvalues from the Dirichlet-reduced 1D pencils."""
    mus = [scipy.linalg.eigh(k.toarray(), m.toarray(), eigvals_only=True, driver="gvd")
           for k, m in zip(system.k1d, system.m1d)]
    lam = mus[0]
    for mu in mus[1:]:
        lam = np.add.outer(mu, lam).ravel()
    return np.sort(lam)


def choose_lambda_e(system, n0: int, lam: np.ndarray | None = None):
    """(lam_e, count): midpoint of the first gap at or after the n0-th
    eigenvalue; gaps within 1e-8 relative are cluster-internal."""
    lam = kronecker_spectrum(system) if lam is None else lam
    i = n0 - 1
    while i + 1 < lam.size and lam[i + 1] - lam[i] <= 1e-8 * lam[i + 1]:
        i += 1
    if i + 1 >= lam.size:
        return float(lam[-1] * (1 + 1e-6)), int(lam.size)
    return 0.5 * float(lam[i] + lam[i + 1]), i + 1


def lpt_assign(counts, world: int) -> list:
    """Longest-processing-time assignment of slices to ranks."""
    load = [0] * world
    out = [[] for _ in range(world)]
    for k in sorted(range(len(counts)), key=lambda k: (-counts[k], k)):
        r = min(range(world), key=lambda r: (load[r], r))
        out[r].append(k)
        load[r] += max(counts[k], 1)
    return [sorted(v) for v in out]


@dataclass
class SlicesResult:
    shifts: np.ndarray            # boundaries actually used (after ZeroPivot nudges)
    nu: np.ndarray                # inertia nu(sigma_k)
    expected: np.ndarray          # per-slice counts from inertia
    found: np.ndarray             # per-slice counts found (all ranks)
    eigenvalues: np.ndarray       # all ranks, sorted
    local_slices: list            # slice ids solved on this rank
    local_eigenvalues: dict       # slice id -> eigenvalues
    local_vectors: dict           # slice id -> vectors (rows; torch on device or numpy)
    counters: CostCounters
    timings: dict = field(default_factory=dict)
    factor_ms: list = field(default_factory=list)
    residuals: dict = field(default_factory=dict)  # slice id -> north-star residuals of its pairs
    max_residual: float = 0.0                       # over all ranks
    gate_rounds: dict = field(default_factory=dict)  # slice id -> refinement rounds the gate needed


def boundary_dedup(entries: list, scale: float):
    """De-duplicate pairs gathered from both sides of internal slice boundaries.

    ``entries``: (slice k, index j, lam, x, M x) with x M-normalised, host arrays, every rank's pairs
    within 1e-7 max(|lam|, 1) of an internal shift.  The rules are the reference's, applied in its
    sequential slice order (k ascending):

    * ``_Pool.add`` (ref eigensolver.py:407-420): a pair is a copy of an accepted one when
      |lam_a - lam| <= 1e-7 max(|lam|, 1) and |x_a^T M x| > 0.1; the later copy is dropped;
    * ``_dedup_and_orthonormalize`` (ref :670-712): accepted pairs cluster when consecutive gaps are
      <= 1e-8 max(scale, |lam|); inside a cluster a member with |G_ab| > 1 - 1e-9 is dropped, then a
      Loewdin step G^{-1/2} X re-orthonormalises the cluster when ||G - I||_max > 1e-10.

    Returns (drop: set of (k, j), updates: {(k, j): (x, M x)}).  Pure host code: every rank computes
    the same answer from the same gathered list.
    """
    drop = set()
    acc = []  # accepted entries in slice order
    for e in sorted(entries, key=lambda t: (t[0], t[1])):
        k, j, lam, x, mx = e
        close = 1e-7 * max(abs(lam), 1.0)
        if any(abs(a[2] - lam) <= close and abs(float(np.dot(a[3], mx))) > 0.1 for a in acc):
            drop.add((k, j))
            continue
        acc.append(e)
    upd = {}
    acc.sort(key=lambda t: t[2])
    i = 0
    while i < len(acc):
        t = i + 1
        while t < len(acc) and acc[t][2] - acc[t - 1][2] <= 1e-8 * max(scale, abs(acc[t][2])):
            t += 1
        cl = acc[i:t]
        if len(cl) > 1:
            X = np.stack([c[3] for c in cl])
            MX = np.stack([c[4] for c in cl])
            G = X @ MX.T
            dup = set()
            for a in range(len(cl)):
                if a in dup:
                    continue
                for b in range(a + 1, len(cl)):
                    if abs(G[a, b]) > 1.0 - 1e-9:
                        dup.add(b)
            for b in sorted(dup):
                drop.add((cl[b][0], cl[b][1]))
            keep = [a for a in range(len(cl)) if a not in dup]
            cl = [cl[a] for a in keep]
            G = G[np.ix_(keep, keep)]
            if len(cl) > 1 and np.abs(G - np.eye(len(cl))).max() > 1e-10:
                ev, evec = np.linalg.eigh(0.5 * (G + G.T))
                T = evec @ np.diag(np.clip(ev, 1e-30, None) ** -0.5) @ evec.T
                Xn, MXn = T @ X[keep], T @ MX[keep]
                for a, c in enumerate(cl):
                    upd[(c[0], c[1])] = (Xn[a], MXn[a])
        i = t
    return drop, upd


_ctx_cache: dict = {}
_ctx_lock = threading.Lock()
_ctx_busy: set = set()


def _take_ctx(device: int, key, priority: int = 0):
    """The worker context (own stream) for `key` -- ("slice", k) or
    ("boundary", i) -- reused across calls with the same key: slice k always
    runs on the same stream, so its pooled Lanczos state (device buffers and
    captured step graph, eigensolver._state_pool) is hit on every call and
    torch's per-stream block cache does not fragment."""
    with _ctx_lock:
        ck = (device, key, priority)
        ctx = _ctx_cache.get(ck)
        if ctx is None or ck in _ctx_busy:  # a concurrent call holds it: a private one
            ctx = _dev.Context(device, priority=priority)
            if ck not in _ctx_cache:
                _ctx_cache[ck] = ctx
        if _ctx_cache.get(ck) is ctx:
            _ctx_busy.add(ck)
        ctx._cache_key = ck
        return ctx


def _give_ctx(ctx) -> None:
    ctx.synchronize()
    with _ctx_lock:
        ck = getattr(ctx, "_cache_key", None)
        if ck is not None and _ctx_cache.get(ck) is ctx:
            _ctx_busy.discard(ck)


def _priorities(work: list) -> list:
    """Stream priority per slice: the slices with the most work get the
    higher of two priorities, so the block scheduler lets them run ahead and
    the others fill the gaps.  The high class is 3/8 of the slices: it
    finishes first, and the tail of the run then still has 10 of 16 streams
    busy (a B200 needs >= 12 concurrent cfg3 slices to run at its aggregate
    step rate; cfg3 A/B: equal halves 1.715 s, 6 + 10 1.673 s, none 1.73 s).
    RIGA_SLICE_PRIORITY=0: one class; RIGA_PRIO_HIGH=k: k slices in the high class."""
    import os

    if not work or os.environ.get("RIGA_SLICE_PRIORITY", "1") == "0":
        return [0] * len(work)
    least, greatest = torch.cuda.Stream.priority_range()  # e.g. (0, -5)
    greatest = max(greatest, least - 1) if greatest < least else greatest
    env = os.environ.get("RIGA_PRIO_HIGH", "")
    nhigh = int(env) if env else (3 * len(work) + 4) // 8
    order = sorted(range(len(work)), key=lambda i: (-work[i], i))
    pr = [least] * len(work)
    for rank, i in enumerate(order):
        if rank < nhigh:
            pr[i] = greatest
    return pr


_sync_mode_set: set = set()


def _blocking_sync(device: int) -> None:
    """Device waits of the slice threads block instead of spinning (RIGA_BLOCKING_SYNC=1); once per device."""
    import os

    if device in _sync_mode_set or os.environ.get("RIGA_BLOCKING_SYNC", "0") != "1":
        return
    from . import _lib as _L

    _sync_mode_set.add(device)
    _L.lib().riga_set_blocking_sync(device, 1)  # best effort: an active context may refuse the change


class _blas_threads:
    """Limit the BLAS/OpenMP pools for the duration of a block (None: no-op)."""

    def __init__(self, n):
        self.n, self.ctl = n, None

    def __enter__(self):
        if self.n is not None:
            from threadpoolctl import threadpool_limits

            self.ctl = threadpool_limits(limits=self.n)
        return self

    def __exit__(self, *exc):
        if self.ctl is not None:
            self.ctl.restore_original_limits()
        return False


def _allgather(obj, group_world):
    if group_world <= 1:
        return [obj]
    import torch.distributed as dist

    out = [None] * group_world
    dist.all_gather_object(out, obj)
    return out


def solve_sub_levels(slices_per_gpu: int) -> int:
    """Subtree height of the solve plan for a run with this many concurrent
    slices per GPU (riga_set_solve_sub_levels).  cfg3 solves/s at 1 / 7 / 10 / 16
    streams (tools/concurrency_probe.py --what solve): height 6 2.46 k / 11.2 k /
    13.5 k / 15.0 k, height 7 2.43 k / 10.8 k / 13.8 k / 16.8 k, height 8 2.00 k /
    9.5 k / 12.4 k / 16.4 k.  7 replaced 8 in session 5: as fast with 16 streams and
    15 % faster once only 7 slices are still running (the tail of a step)."""
    return 7 if slices_per_gpu >= 12 else 6


class solve_plan:
    """Symbolic analyses created inside the block use `sub_levels`."""

    def __init__(self, sub_levels: int):
        self.levels = sub_levels

    def __enter__(self):
        from . import _lib as _L

        _L.lib().riga_set_solve_sub_levels(int(self.levels))
        return self

    def __exit__(self, *exc):
        from . import _lib as _L

        _L.lib().riga_set_solve_sub_levels(6)
        return False


def solve_uniform_slices(system, shifts, seeds=None, m_factor: int = 2, streams: int = 4,
                         rank: int = 0, world: int = 1, vectors_to_host: bool = True,
                         pencil_symbolic: Symbolic | None = None, perm=None, m_fixed: int | None = None,
                         **opts) -> SlicesResult:
    """Solve every slice (shifts[k], shifts[k+1]] (see module docstring).  The Lanczos basis of slice k has
    m = m_factor x count_k vectors (the BASELINE protocol), or m_fixed for every slice (solve_spectrum's
    SolverOptions.m)."""
    t_all = time.perf_counter()
    shifts = np.asarray(shifts, dtype=np.float64)
    S = shifts.size - 1
    seeds = list(range(S)) if seeds is None else list(seeds)
    counters = CostCounters()
    base_ctx = _dev.current()
    _blocking_sync(base_ctx.device)
    if perm is None:
        perm = separator_ordering(system)
    if pencil_symbolic is None:
        with solve_plan(solve_sub_levels(min(streams, -(-S // max(world, 1))))):
            sym = Symbolic.on_device(system.device, perm)
    else:
        sym = pencil_symbolic

    def make_pencil(ctx, cnt):
        p = _Pencil.__new__(_Pencil)
        p.system, p.ctx, p.M, p.n = system, ctx, system.M, system.dof_count
        p.perm, p.counters, p.symbolic = perm, cnt, sym
        return p

    # --- memory plan: per-factor bytes (panels + inverse/G companions) and the
    # transient update blocks; keep boundary factors only when they all fit,
    # and cap the concurrent slices by what one slice needs ----------------
    st_ = sym.stats
    n = system.dof_count
    fac_bytes = 8.0 * (1.35 * st_.get("panel_entries", 0) + 6 * n)
    cb_bytes = 8.0 * st_.get("cb_entries", 0)
    free_b, total_b = torch.cuda.mem_get_info(base_ctx.device)
    # memory the stream-ordered pool keeps for reuse (freed buffers of earlier calls) and idle pooled Lanczos
    # states (reused by the slice streams) is available to this call too
    import ctypes

    from . import _lib as _L0
    from . import eigensolver as _E0

    reuse = ctypes.c_int64(0)
    _L0.check(_L0.lib().riga_device_pool_reusable(base_ctx.device, ctypes.byref(reuse)), "pool")
    # idle Lanczos states of another problem size will never be reused by this call: free them first
    _E0.trim_state_pool(base_ctx.device, lambda n_, m_: n_ == n)
    free_b += reuse.value + _E0.pooled_state_bytes(base_ctx.device, n)
    budget = 0.85 * free_b
    keep_factors = (S + 1) * fac_bytes <= 0.35 * budget

    # --- 1. boundary pass: each rank factors its share of the S+1 shifts ---
    t0 = time.perf_counter()
    mine_b = [k for k in range(S + 1) if k % world == rank]
    bnd = {}
    # ZeroPivot nudges and the bisection floor use the slice width, as the reference's solve_slice
    # (ref eigensolver.py:645 scale = hi_req - lo_req); a shared boundary takes the narrower adjacent slice
    widths = np.diff(shifts) if S else np.ones(1)

    def bscale(k):
        return float(min(widths[max(k - 1, 0)], widths[min(k, S - 1)])) if S else 1.0
    bcnt = CostCounters()
    kept = {}
    # independent factorizations on several streams at once (a small front
    # tree leaves most of the GPU idle); concurrency capped by the transient
    # update-block memory each one needs
    import os

    nbw_cap = int(os.environ.get("RIGA_BOUNDARY_STREAMS", "8"))
    nbw = int(max(1, min(nbw_cap, len(mine_b), (0.5 * budget) // max(fac_bytes + cb_bytes, 1.0))))
    bq = list(mine_b)
    blk = threading.Lock()
    berr = []

    def bworker(bi):
        ctx = _take_ctx(base_ctx.device, ("boundary", bi), 0)
        cnt = CostCounters()
        pen = make_pencil(ctx, cnt)
        with ctx:
            while True:
                with blk:
                    if not bq or berr:
                        break
                    k = bq.pop(0)
                try:
                    sig, fact = pen.factor(float(shifts[k]), bscale(k))
                    with blk:
                        bnd[k] = (sig, fact.n_negative, fact.device_ms)
                        if k < S and keep_factors:
                            kept[k] = (sig, fact)
                    del fact
                except Exception as e:  # surfaced after join
                    with blk:
                        berr.append(e)
        with blk:
            bcnt.merge(cnt)
        _give_ctx(ctx)

    bth = [threading.Thread(target=bworker, args=(i,)) for i in range(nbw)]
    for t in bth:
        t.start()
    for t in bth:
        t.join()
    if berr:
        raise berr[0]
    counters.merge(bcnt)
    counters.nsh += len(mine_b)
    allb = {}
    for part in _allgather(bnd, world):
        allb.update(part)
    sig_used = np.array([allb[k][0] for k in range(S + 1)])
    nu = np.array([allb[k][1] for k in range(S + 1)], dtype=np.int64)
    expected = np.diff(nu)
    t_bnd = time.perf_counter() - t0

    # --- 2. LPT assignment of slices to ranks -------------------------------
    assign = lpt_assign(list(expected), world)
    my = assign[rank]
    # pooled states of basis sizes this call does not use are stale: free them before the slices allocate
    def slice_m(k):
        want = m_fixed if m_fixed is not None else m_factor * int(expected[k])
        return max(2, min(want, system.dof_count))

    m_used = {slice_m(k) for k in my}
    _E0.trim_state_pool(base_ctx.device, lambda n_, m_: n_ == n and min(m_, n) in m_used)
    # drop factors this rank does not need
    kept = {k: v for k, v in kept.items() if k in my}

    # --- 3. solve my slices concurrently on `streams` CUDA streams ----------
    gate = opts.get("residual_gate", SolverOptions.residual_gate)
    results = {}
    slice_times = {}
    errors = []
    lock = threading.Lock()
    factor_lock = threading.Lock()
    queue = sorted(my, key=lambda k: -expected[k])
    order = list(queue)
    m_max = max([slice_m(k) for k in my] + [2])
    # per slice: its factor (unless kept), V + MV and the locked set L + LM
    # (capacity >= m rows each), lifted/locking temporaries and pool vectors
    per_slice = 1.2 * (fac_bytes * (0 if keep_factors else 1) + 16.0 * (m_max + 1) * n * 2
                       + 8.0 * (3 * m_max + 16) * n)
    kept_bytes = fac_bytes * len(kept)
    cap = int(max(1, (budget - kept_bytes - cb_bytes) // max(per_slice, 1)))
    nthreads = max(1, min(streams, len(my), cap))
    one_per_thread = len(my) <= nthreads
    # few concurrent slices: each one's step latency is the bound -> PDL on
    # (RIGA_PDL=0/1 overrides); many: off (waiting CTAs crowd the others)
    import os

    pdl_env = os.environ.get("RIGA_PDL")
    from . import _lib as _L

    _L.lib().riga_set_pdl(int(pdl_env == "1") if pdl_env in ("0", "1") else int(nthreads <= 4))
    # one slice per stream: stream priorities by expected work; otherwise a
    # shared queue (largest first) on default-priority streams
    prio = _priorities([int(expected[k]) for k in order]) if one_per_thread else [0] * len(order)
    def worker(widx):
        ctx = _take_ctx(base_ctx.device, ("slice", order[widx] if one_per_thread else widx), prio[widx])
        cnt = CostCounters()
        mine = [order[widx]] if one_per_thread else None
        with ctx:
            while True:
                with lock:
                    if mine is not None:
                        if not mine:
                            break
                        k = mine.pop()
                    else:
                        if not queue:
                            break
                        k = queue.pop(0)
                try:
                    t_start = time.perf_counter()
                    pen = make_pencil(ctx, cnt)
                    lo, hi = float(sig_used[k]), float(sig_used[k + 1])
                    if k in kept:
                        lob = _Boundary(lo, int(nu[k]), kept[k][1])
                    else:
                        # one refactorization at a time: its transient update
                        # blocks (cb_bytes) are budgeted once
                        with factor_lock:
                            s2, f2 = pen.factor(lo, hi - lo)
                            ctx.synchronize()
                        lob = _Boundary(s2, f2.n_negative, f2)
                        cnt.nsh += 1
                    hib = _Boundary(hi, int(nu[k + 1]), None)
                    count = int(expected[k])
                    pool = _Pool()
                    if count > 0:
                        m = slice_m(k)
                        so = SolverOptions(m=m, **opts)
                        rng = np.random.default_rng(seeds[k])
                        _solve_interval(pen, lob, hib, pool, so, rng, hi - lo)
                    t_col = time.perf_counter()
                    idx = sorted((i for i, lam in enumerate(pool.lams) if lob.sigma < lam <= hib.sigma),
                                 key=lambda i: pool.lams[i])
                    lams = np.array([pool.lams[i] for i in idx])
                    res, rounds = np.empty(0), None
                    if idx:
                        X = torch.stack([pool.vecs[i] for i in idx])
                        # north-star residual gate (device residuals; block refinement with this slice's
                        # midpoint factor for any slice with a pair above the bound)
                        _tg = time.perf_counter()
                        def fac_mid(sg, pen=pen, lo=lo, hi=hi):
                            with factor_lock:  # transient update blocks budgeted once
                                f = pen.factor(sg, hi - lo)[1]
                                ctx.synchronize()
                            cnt.nsh += 1
                            return f

                        lams, X, res, _, rounds = residual_gate(system, fac_mid, (lo, hi), lams, X, ctx, gate,
                                                                counters=cnt)
                        cnt.phase("residual_gate", time.perf_counter() - _tg)
                        if vectors_to_host:
                            # pinned staging (torch's caching host allocator)
                            # + async copy on the slice stream: a pageable
                            # .cpu() would serialise the slices
                            _tp = time.perf_counter()
                            H = torch.empty(X.shape, dtype=X.dtype, pin_memory=True)
                            cnt.phase("collect_pin", time.perf_counter() - _tp)
                            H.copy_(X, non_blocking=True)
                            ctx.synchronize()
                            X = H.numpy()
                    else:
                        X = np.empty((0, system.dof_count))
                    ctx.synchronize()
                    cnt.phase("collect", time.perf_counter() - t_col)
                    with lock:
                        results[k] = (lams, X, res, rounds)
                        slice_times[k] = (t_start - t0, time.perf_counter() - t0, cnt.nfb)
                except Exception as e:  # surfaced after join
                    with lock:
                        errors.append((k, e))
        with lock:
            counters.merge(cnt)
        _give_ctx(ctx)

    t0 = time.perf_counter()
    threads = [threading.Thread(target=worker, args=(i,)) for i in range(nthreads)]
    # the host side of each slice (Rayleigh-Ritz eigh, small dense algebra)
    # runs in its own thread: one BLAS thread each, not nthreads x cores
    with _blas_threads(1 if nthreads > 1 else None):
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    if errors:
        k, e = errors[0]
        raise RuntimeError(f"slice {k} failed on rank {rank}: {e}") from e
    t_sl = time.perf_counter() - t0

    def _refill(k, drop, bnear):
        lams_k, X_k, _, _ = results[k]
        pen = make_pencil(base_ctx, counters)
        lo, hi = float(sig_used[k]), float(sig_used[k + 1])
        dev = f"cuda:{base_ctx.device}"
        with base_ctx:
            s2, f2 = pen.factor(lo, hi - lo)
            counters.nsh += 1
            lob = _Boundary(s2, int(nu[k]), f2)
            hib = _Boundary(hi, int(nu[k + 1]), None)
            pool = _Pool()
            for lam, x in zip(lams_k, X_k):
                pool.lams.append(float(lam))
                pool.vecs.append(torch.as_tensor(np.asarray(x) if isinstance(X_k, np.ndarray) else x, device=dev))
            for kk, j, lam, x, _mx in bnear:
                if kk != k and (kk, j) not in drop:
                    pool.lams.append(float(lam))
                    pool.vecs.append(torch.as_tensor(x, device=dev))
            so = SolverOptions(m=slice_m(k), **opts)
            _solve_interval(pen, lob, hib, pool, so, np.random.default_rng(seeds[k] + 104729), hi - lo)
            idx = sorted((i for i, lam in enumerate(pool.lams) if lo < lam <= hi), key=lambda i: pool.lams[i])
            lams = np.array([pool.lams[i] for i in idx])
            X = torch.stack([pool.vecs[i] for i in idx])
            lams, X, res, _, rounds = residual_gate(system, lambda sg: pen.factor(sg, hi - lo)[1], (lo, hi),
                                                    lams, X, base_ctx, gate, counters=counters)
            if vectors_to_host:
                X = X.cpu().numpy()
        return lams, X, res, rounds

    # --- 4. boundary de-duplication + global eigenvalue gather --------------
    # pairs within 1e-7 max(|lam|, 1) of an internal boundary travel with their M-normalised vectors
    # (host copies; none exist at the BASELINE configs, whose shifts sit >= 1e-4 relative from the
    # spectrum); every rank applies the reference's _Pool.add / _dedup_and_orthonormalize rules to the
    # same gathered set and patches its own slices
    _td = time.perf_counter()
    near = []
    for k in my:
        lams_k, X_k = results[k][0], results[k][1]
        for j, lam in enumerate(lams_k):
            if any(0 < b < S and abs(lam - sig_used[b]) <= 1e-7 * max(abs(lam), 1.0) for b in (k, k + 1)):
                xk = X_k[j] if isinstance(X_k, np.ndarray) else X_k[j].cpu().numpy()
                mxk = mass_matvec(system.M, xk)
                near.append((int(k), int(j), float(lam), np.asarray(xk), np.asarray(mxk)))
    scale_all = max([float(np.max(np.abs(results[k][0]))) for k in my if results[k][0].size] + [1.0])
    gathered = _allgather(({k: results[k][0] for k in my}, near, scale_all), world)
    bnear = sorted((e for _, nr, _ in gathered for e in nr), key=lambda e: (e[0], e[1]))
    scale_all = max(g[2] for g in gathered)
    drop, upd = boundary_dedup(bnear, scale_all)
    for k in my:
        lams_k, X_k, res_k, rr_k = results[k]
        mine_upd = {j: v for (kk, j), v in upd.items() if kk == k}
        mine_drop = sorted(j for (kk, j) in drop if kk == k)
        if mine_upd:
            for j, (xn, _mxn) in mine_upd.items():
                if isinstance(X_k, np.ndarray):
                    X_k[j] = xn
                else:
                    X_k[j] = torch.as_tensor(xn, device=X_k.device)
        if mine_drop:
            keep = np.setdiff1d(np.arange(lams_k.size), mine_drop)
            lams_k = lams_k[keep]
            X_k = X_k[keep] if isinstance(X_k, np.ndarray) else X_k[torch.as_tensor(keep, device=X_k.device)]
            res_k = res_k[keep] if res_k.size else res_k
            if rr_k is not None and rr_k.ref_residuals is not None and rr_k.ref_residuals.size:
                rr_k.ref_residuals = rr_k.ref_residuals[keep]
        results[k] = (lams_k, X_k, res_k, rr_k)
        if lams_k.size < expected[k]:
            # a dropped copy took the place of one of this slice's own pairs: search (lo, hi] again with
            # every known pair deflated (the reference's shared pool gives its sweeps the same window)
            results[k] = _refill(k, drop, bnear)
    local_eigs = {k: results[k][0] for k in my}
    if drop:
        local_eigs_g = _allgather(local_eigs, world)
    else:
        local_eigs_g = [g[0] for g in gathered]
    t_dedup = time.perf_counter() - _td
    found = np.zeros(S, dtype=np.int64)
    all_eigs = []
    for le in local_eigs_g:
        for k, v in le.items():
            found[k] = v.size
            all_eigs.append(v)
    for k in range(S):
        if found[k] != expected[k]:
            raise CountMismatch(f"slice {k} expected {expected[k]} found {found[k]}",
                                interval=(sig_used[k], sig_used[k + 1]), expected=int(expected[k]),
                                found=int(found[k]))
    max_res = max([float(results[k][2].max()) for k in my if results[k][2].size] + [0.0])
    max_res = max(_allgather(max_res, world))
    eig = np.sort(np.concatenate(all_eigs)) if all_eigs else np.empty(0)
    res = SlicesResult(sig_used, nu, expected, found, eig, my, local_eigs,
                       {k: results[k][1] for k in my}, counters)
    res.residuals = {k: results[k][2] for k in my}
    res.max_residual = max_res
    res.gate_rounds = {k: (results[k][3].rounds if results[k][3] is not None else 0) for k in my}
    res.gate_info = {k: results[k][3] for k in my}
    res.timings = {"boundary_s": t_bnd, "slices_s": t_sl, "total_s": time.perf_counter() - t_all,
                   "dedup_s": t_dedup, "streams_used": nthreads, "kept_boundary_factors": bool(keep_factors),
                   "boundary_pairs": len(bnear), "boundary_duplicates": len(drop),
                   "slice_wall": {int(k): [round(a, 3), round(b, 3)] for k, (a, b, _) in slice_times.items()},
                   "slice_nfb": {int(k): int(nf) for k, (_, _, nf) in slice_times.items()}}
    res.factor_ms = [allb[k][2] for k in range(S + 1)]
    return res


# ---------------------------------------------------------------------------
# solve_spectrum on concurrent streams
# ---------------------------------------------------------------------------


def factor_inertias(system, sigmas, scale: float, streams: int = 8, sym=None, perm=None):
    """Inertia nu(sigma) of every shift, the factorizations on concurrent streams (factors discarded).
    ZeroPivot nudges follow ref _Pencil.factor (sigma += 1e-8 scale, x10, <= 12 tries).  Returns
    [(sigma_used, nu)] in input order and the CostCounters of the factorizations."""
    base_ctx = _dev.current()
    if perm is None:
        perm = separator_ordering(system)
    if sym is None:
        sym = Symbolic.on_device(system.device, perm)
    sigmas = [float(x) for x in sigmas]
    out = [None] * len(sigmas)
    todo = list(range(len(sigmas)))
    lock = threading.Lock()
    errs = []
    total = CostCounters()

    def work(widx):
        ctx = _take_ctx(base_ctx.device, ("inertia", widx), 0)
        cnt = CostCounters()
        pen = _Pencil.__new__(_Pencil)
        pen.system, pen.ctx, pen.M, pen.n = system, ctx, system.M, system.dof_count
        pen.perm, pen.counters, pen.symbolic = perm, cnt, sym
        with ctx:
            while True:
                with lock:
                    if not todo or errs:
                        break
                    i = todo.pop(0)
                try:
                    sg, f = pen.factor(sigmas[i], scale)
                    with lock:
                        out[i] = (sg, f.n_negative)
                    del f
                except Exception as e:  # surfaced after join
                    with lock:
                        errs.append(e)
        with lock:
            total.merge(cnt)
        _give_ctx(ctx)

    th = [threading.Thread(target=work, args=(w,)) for w in range(max(1, min(streams, len(sigmas))))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    total.nsh += len(sigmas)
    return out, total


def spectrum_shifts(system, count=None, interval=None, target: int = 30, streams: int = 8, sym=None, perm=None):
    """Shift placement for solve_spectrum by a speculative inertia pre-pass instead of the reference's
    sequential march (ref _march eigensolver.py:579-633, lowest-count start :756-773).  Trial shifts are
    factored a batch at a time on concurrent streams; where they go is predicted from the inertia counts
    already known with Weyl's law for the d-dimensional Laplacian, nu(sigma) ~ C sigma^(d/2): the first probe
    calibrates C, every slice is aimed at `target` eigenvalues (the march's width rule), and a slice that
    still holds more than 4 target (the march's acceptance bound) is split again between its measured
    endpoints.  Returns (shifts, nus, counters): shifts[0] = sigma0 = -0.1 lambda_1-bound for a count
    request (as the reference) or lo for an interval; the last shift covers `count` (or is hi)."""
    from .eigensolver import _lambda1_upper_bound

    counters = CostCounters()
    if perm is None:
        perm = separator_ordering(system)
    if sym is None:
        sym = Symbolic.on_device(system.device, perm)
    e = 0.5 * system.dim  # Weyl exponent

    def probe(sig, scale):
        res, c = factor_inertias(system, sig, scale, streams, sym, perm)
        counters.merge(c)
        return res

    def split(a, na, b, nb_, k):
        """k - 1 shifts in (a, b) at equal predicted counts (power law through the endpoints, from 0 for a
        lower end below the spectrum of the positive definite Laplacian pencil)."""
        if b <= 0.0:
            return [a + (b - a) * j / k for j in range(1, k)]
        ua, ub = max(a, 0.0) ** e, b ** e
        out = [(ua + (ub - ua) * j / k) ** (1.0 / e) for j in range(1, k)]
        return [x for x in out if a < x < b]

    if interval is not None:
        lo, hi = float(interval[0]), float(interval[1])
        scale = hi - lo
        pts = probe([lo, hi], scale)
    else:
        lam1 = _lambda1_upper_bound(system)
        scale = lam1
        sigma0 = -0.1 * lam1
        for _ in range(8):
            (s0, nu0), = probe([sigma0], scale)
            if nu0 == 0:
                break
            counters.retries += 1
            sigma0 = s0 * 10.0
        pts = [(s0, nu0)]
        # Weyl's law on [0, 1]^d, nu(sigma) ~ c sigma^e (c = 1/pi, 1/(4 pi), 1/(6 pi^2)), recalibrated from
        # every batch: a batch aims at count j/8 (j = 1..8) and 1.05 count until count is covered
        c_fit = {1: 1.0 / math.pi, 2: 1.0 / (4.0 * math.pi), 3: 1.0 / (6.0 * math.pi ** 2)}[system.dim]
        for _ in range(20):
            want = [((nu0 + count * j / 8.0) / c_fit) ** (1.0 / e) for j in range(1, 9)]
            want.append(((nu0 + 1.05 * count) / c_fit) ** (1.0 / e))
            pts = sorted(pts + probe(want, scale))
            if max(nu for _, nu in pts) - nu0 >= count:
                break
            sa, na = max(pts, key=lambda t: (t[1], t[0]))
            c_fit = (na - nu0) / sa ** e if na > nu0 else c_fit / 4.0

    def cut(pts):
        # a count request keeps the shifts up to the first that covers `count`
        if interval is not None:
            return pts
        base = pts[0][1]
        i = next(i for i, (_, nu) in enumerate(pts) if nu - base >= count)
        return pts[: i + 1]

    pts = cut(pts)
    # aim every slice at `target`; split again any slice above 4 target (the march's acceptance bound)
    first = True
    for _ in range(40):
        new = []
        for (a, na), (b, nb_) in zip(pts[:-1], pts[1:]):
            c = nb_ - na
            if c > (target if first else 4 * target):
                new += split(a, na, b, nb_, -(-c // target))
        first = False
        if not new:
            break
        pts = cut(sorted(pts + probe(new, scale)))
    shifts = np.array([p_[0] for p_ in pts])
    nus = np.array([p_[1] for p_ in pts], dtype=np.int64)
    return shifts, nus, counters


def solve_spectrum_sliced(system, count=None, interval=None, seed: int = 0, device: bool = False, streams: int = 16,
                          **kwargs):
    """solve_spectrum (ref eigensolver.py:715-799) with every slice on its own CUDA stream: the shifts come from
    the concurrent inertia pre-pass (spectrum_shifts), the slices run through solve_uniform_slices with the
    caller's SolverOptions (basis m fixed, as the reference's slices; residual gate and boundary
    de-duplication per slice), then the reference's selection of the lowest `count` (or every pair of the
    interval).  Slice k uses seed + k (its own RNG stream; the sequential driver shares one).  Same results as
    the sequential driver: counts exact, eigenvalues to 1e-10."""
    from .eigensolver import EigenResult

    if (count is None) == (interval is None):
        raise ValueError("request either the lowest `count` or an `interval`")
    opts = SolverOptions(**kwargs)
    if interval is not None:
        if not float(interval[0]) < float(interval[1]):
            raise ValueError("empty interval")
    elif not 1 <= count <= system.dof_count:
        raise ValueError(f"requested {count} of {system.dof_count} eigenpairs")
    _ta = time.perf_counter()
    perm = separator_ordering(system)
    with solve_plan(solve_sub_levels(streams)):
        sym = Symbolic.on_device(system.device, perm)
    t_sym = time.perf_counter() - _ta
    _t0 = time.perf_counter()
    shifts, nus, pre = spectrum_shifts(system, count, interval, opts.target, min(streams, 8), sym, perm)
    t_shifts = time.perf_counter() - _t0
    sopts = {k: v for k, v in kwargs.items() if k != "m"}
    S = shifts.size - 1
    # host vectors come back per slice (pinned, asynchronous, overlapping the other slices); pairs of two
    # slices in one eigenvalue cluster can only meet at a shared shift, where solve_uniform_slices' boundary
    # de-duplication applies the reference's _Pool.add / _dedup_and_orthonormalize rules, and a slice's own
    # locked pairs are M-orthonormal by construction, so the final cluster pass of the sequential driver
    # has nothing left to do here
    res = solve_uniform_slices(system, shifts, seeds=[seed + k for k in range(S)], streams=streams,
                               vectors_to_host=not device, pencil_symbolic=sym, perm=perm, m_fixed=opts.m, **sopts)
    counters = res.counters
    counters.merge(pre)
    counters.phase("spectrum_shifts", t_shifts)
    counters.phase("spectrum_slices", res.timings.get("total_s", 0.0))
    counters.phase("spectrum_probes", float(pre.nsh))
    counters.phase("spectrum_symbolic", t_sym)
    _tf = time.perf_counter()
    want = count if interval is None else int(nus[-1] - nus[0])
    lam_l, vec_l, north_l, ref_l, sid_l = [], [], [], [], []
    taken = 0
    for k in range(S):  # slices in ascending order; a count request stops at `count`
        ev = res.local_eigenvalues.get(k, np.empty(0))
        if ev.size == 0:
            continue
        take = ev.size if interval is not None else min(ev.size, want - taken)
        if take <= 0:
            break
        info = res.gate_info.get(k)
        lam_l.append(ev[:take])
        vec_l.append(res.local_vectors[k][:take])
        north_l.append(res.residuals[k][:take])
        ref_l.append(info.ref_residuals[:take] if info is not None and info.ref_residuals is not None
                     else np.full(take, np.nan))
        sid_l.append(np.full(take, k))
        taken += take
    if taken != want:
        raise CountMismatch(f"slices returned {taken} of {want} eigenpairs", expected=want, found=taken)
    lams_arr = np.concatenate(lam_l) if lam_l else np.empty(0)
    north = np.concatenate(north_l) if north_l else np.empty(0)
    residuals = np.concatenate(ref_l) if ref_l else np.empty(0)
    slice_ids = np.concatenate(sid_l) if sid_l else np.empty(0, dtype=int)
    slices = [(float(res.shifts[k]), float(res.shifts[k + 1]), int(res.expected[k])) for k in range(S)]
    n = system.dof_count
    if device:
        Xout = torch.cat(vec_l).T if vec_l else torch.empty((n, 0), dtype=torch.float64)
    else:
        Xout = np.concatenate(vec_l).T if vec_l else np.empty((n, 0))
    gate = max(res.gate_rounds.values(), default=0)
    counters.phase("spectrum_finish", time.perf_counter() - _tf)
    return EigenResult(lams_arr, Xout, residuals, slice_ids, slices, counters, north, gate)
