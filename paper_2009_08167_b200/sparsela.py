"""Sparse symmetric LDL^T, solves and mass products on the B200 engine.

API mirror of /root/reference/pkg/src/rigaeig/sparsela.py (same names,
argument meaning, exceptions and counter conventions):

* factor_ldl   -> riga_symbolic_* (host C++, once per pattern) +
                  riga_factor_create (multifrontal supernodal LDL^T on the
                  device, FP64 tensor-core Schur updates, inertia from D)
* solve_fb     -> riga_factor_solve (supernodal forward/backward sweeps)
* mass_matvec  -> riga_spmv / riga_csr_spmv (CSR SpMV kernel)
* separator_ordering / nested_dissection_graph stay on the host.

FLOP conventions are the reference's (sparsela.py:1-17): factorization
sum_j colcount_j^2 on the exact unamalgamated structure, solves
2 fill_nnz, mat-vec 2 nnz.  ``LDLFactorization.permutation`` is the
elimination order actually used: a postorder of the requested ordering's
elimination tree (same fill, same column counts, same factor_flops).
"""
from __future__ import annotations

import ctypes
import os
import threading
import time
import weakref
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from . import device as _dev
from .assembly import DeviceSystem, DiscreteSystem, SymSparseMatrix
from .bspline import separator_basis_indices

_TRACE = os.environ.get("RIGA_TRACE") == "1"


class ZeroPivot(Exception):
    """Pivot at or numerically at zero: the shift hit an eigenvalue."""


class NegativeNorm(Exception):
    """v^T M v < 0 for the mass inner product: M is not positive definite."""


@dataclass
class OpCounter:
    flops: int = 0
    calls: int = 0
    seconds: float = 0.0

    def add(self, flops: int, seconds: float) -> None:
        self.flops += int(flops)
        self.calls += 1
        self.seconds += seconds

    def merge(self, other: "OpCounter") -> None:
        self.flops += other.flops
        self.calls += other.calls
        self.seconds += other.seconds


@dataclass
class CostCounters:
    fact: OpCounter = field(default_factory=OpCounter)
    fb: OpCounter = field(default_factory=OpCounter)
    matvec: OpCounter = field(default_factory=OpCounter)
    nsh: int = 0
    nit: int = 0
    retries: int = 0
    steps_per_iteration: list = field(default_factory=list)
    phase_s: dict = field(default_factory=dict)  # host wall seconds per driver phase (engine extension)

    trace: list | None = None  # (phase, t_start, t_end, thread) when RIGA_TRACE=1

    def phase(self, name: str, dt: float, steps: int = 0) -> None:
        self.phase_s[name] = self.phase_s.get(name, 0.0) + dt
        if _TRACE and name != "cgs_rows":
            t1 = time.perf_counter()
            if self.trace is None:
                self.trace = []
            self.trace.append((name, t1 - dt, t1, threading.get_ident(), steps))

    @property
    def nfa(self) -> int:
        return self.fact.calls

    @property
    def nfb(self) -> int:
        return self.fb.calls

    @property
    def nmv(self) -> int:
        return self.matvec.calls

    def merge(self, other: "CostCounters") -> None:
        self.fact.merge(other.fact)
        self.fb.merge(other.fb)
        self.matvec.merge(other.matvec)
        self.nsh += other.nsh
        self.nit += other.nit
        self.retries += other.retries
        self.steps_per_iteration.extend(other.steps_per_iteration)
        for k, v in other.phase_s.items():
            self.phase_s[k] = self.phase_s.get(k, 0.0) + v
        if other.trace:
            self.trace = (self.trace or []) + other.trace


# ---------------------------------------------------------------------------
# symbolic analysis (host C++ in the engine)
# ---------------------------------------------------------------------------

STAT_NAMES = ("fill_nnz", "factor_flops", "n_supernodes", "max_front", "n_levels",
              "panel_entries", "cb_entries", "max_ncol", "fundamental_supernodes",
              "stored_L_entries", "n_small_fronts", "n_large_fronts", "nnz_lower",
              "tree_height", "relaxed_flops")


class Symbolic:
    """riga_symbolic handle: ordering + supernodal structure of one pattern."""

    def __init__(self, handle, device_system: DeviceSystem | None, n: int):
        self.handle = handle
        self.system = device_system  # keeps the device pattern alive
        self.n = n
        st = np.zeros(16, np.int64)
        _lib.check(_lib.lib().riga_symbolic_stats(handle, _lib.ptr(st)))
        self.stats = {k: int(v) for k, v in zip(STAT_NAMES, st)}
        self._order = None

    @classmethod
    def on_device(cls, dsys: DeviceSystem, perm: np.ndarray) -> "Symbolic":
        perm = np.ascontiguousarray(perm, dtype=np.int64)
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().riga_symbolic_create(dsys.handle, _lib.ptr(perm), ctypes.byref(h)),
                   "symbolic")
        return cls(h, dsys, dsys.n)

    @classmethod
    def host_only(cls, A, perm: np.ndarray) -> "Symbolic":
        A = sp.csr_array(A)
        A.sort_indices()
        perm = np.ascontiguousarray(perm, dtype=np.int64)
        rp = np.ascontiguousarray(A.indptr, np.int64)
        ci = np.ascontiguousarray(A.indices, np.int32)
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().riga_symbolic_analyze(A.shape[0], _lib.ptr(rp), _lib.ptr(ci),
                                                    _lib.ptr(perm), ctypes.byref(h)), "symbolic")
        return cls(h, None, A.shape[0])

    @property
    def order(self) -> np.ndarray:
        if self._order is None:
            o = np.empty(self.n, np.int64)
            _lib.check(_lib.lib().riga_symbolic_order(self.handle, _lib.ptr(o)))
            self._order = o
        return self._order

    def supernodes(self) -> dict:
        """Relaxed supernode table: col0, ncol, front, parent, level."""
        ns = self.stats["n_supernodes"]
        arrs = {k: np.empty(ns, np.int64) for k in ("col0", "ncol", "front", "parent", "level")}
        _lib.check(_lib.lib().riga_symbolic_supernodes(self.handle, *[_lib.ptr(arrs[k]) for k in
                                                                     ("col0", "ncol", "front", "parent", "level")]))
        return arrs

    def colcounts(self) -> np.ndarray:
        c = np.empty(self.n, np.int64)
        _lib.check(_lib.lib().riga_symbolic_colcounts(self.handle, _lib.ptr(c)))
        return c

    def __del__(self):
        try:
            if self.handle:
                _lib.lib().riga_symbolic_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


# ---------------------------------------------------------------------------
# factorization
# ---------------------------------------------------------------------------


class LDLFactorization:
    """P A P^T = L diag(D) L^T on the device (ref sparsela.py:178-203).

    Attributes read by reference callers: ``n``, ``n_negative``,
    ``inertia``, ``fill_nnz``, ``factor_flops``, ``permutation``, ``D``,
    ``Lp``/``Li``/``Lx`` and ``l_matrix()`` (the latter materialised lazily
    from the device panels).
    """

    def __init__(self, handle, symbolic: Symbolic, ctx, n_negative: int, sigma: float):
        self.handle = handle
        self.symbolic = symbolic
        self.ctx = ctx
        self.sigma = sigma
        n = symbolic.n
        self.inertia = (int(n_negative), 0, int(n - n_negative))
        self.fill_nnz = symbolic.stats["fill_nnz"]
        self.factor_flops = symbolic.stats["factor_flops"]
        self._D = None
        self._L = None
        ms = ctypes.c_float(0)
        _lib.lib().riga_factor_time_ms(handle, ctypes.byref(ms))
        self.device_ms = float(ms.value)

    @property
    def n(self) -> int:
        return self.symbolic.n

    @property
    def n_negative(self) -> int:
        return self.inertia[0]

    @property
    def permutation(self) -> np.ndarray:
        return self.symbolic.order

    @property
    def D(self) -> np.ndarray:
        if self._D is None:
            D = np.empty(self.n, np.float64)
            _lib.check(_lib.lib().riga_factor_D(self.handle, _lib.ptr(D)))
            self._D = D
        return self._D

    def _export(self):
        if self._L is None:
            m = self.symbolic.stats["stored_L_entries"]
            Lp = np.empty(self.n + 1, np.int64)
            Li = np.empty(m, np.int32)
            Lx = np.empty(m, np.float64)
            _lib.check(_lib.lib().riga_factor_export(self.handle, _lib.ptr(Lp), _lib.ptr(Li), _lib.ptr(Lx)))
            self._L = (Lp, Li, Lx)
        return self._L

    @property
    def Lp(self):
        return self._export()[0]

    @property
    def Li(self):
        return self._export()[1]

    @property
    def Lx(self):
        return self._export()[2]

    def l_matrix(self) -> sp.csc_array:
        Lp, Li, Lx = self._export()
        n = self.n
        L = sp.csc_array((Lx, Li, Lp), shape=(n, n))
        return sp.csc_array(L + sp.eye_array(n, format="csc"))

    def solve_device(self, b: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        out = torch.empty_like(b) if out is None else out
        _lib.check(_lib.lib().riga_factor_solve(self.handle, _lib.ptr(b), _lib.ptr(out)), "solve")
        return out

    def __del__(self):
        try:
            if self.handle:
                _lib.lib().riga_factor_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def numeric_factor(symbolic: Symbolic, sigma: float, ctx=None, rel_zero_tol: float = 1e-14):
    """Device LDL^T of K - sigma M on the symbolic's pattern; raises ZeroPivot."""
    ctx = ctx or _dev.current()
    h = ctypes.c_void_p()
    neg = ctypes.c_int64(0)
    bad = ctypes.c_int64(0)
    st = _lib.lib().riga_factor_create(ctx.handle, symbolic.handle, float(sigma), rel_zero_tol,
                                       ctypes.byref(h), ctypes.byref(neg), ctypes.byref(bad))
    if st == _lib.ZERO_PIVOT:
        msg = _lib.last_error()
        if h.value:
            _lib.lib().riga_factor_destroy(h)
        raise ZeroPivot(msg)
    _lib.check(st, "factor")
    return LDLFactorization(h, symbolic, ctx, neg.value, sigma)


def _as_csr(A) -> sp.csr_array:
    if isinstance(A, SymSparseMatrix):
        return A.csr
    return sp.csr_array(A)


def factor_ldl(A, ordering="nd", counters: CostCounters | None = None) -> LDLFactorization:
    """Factor symmetric A as P A P^T = L D L^T without pivoting (ref :212-262).

    ``ordering``: "natural", "nd" or an explicit permutation.  Raises
    ZeroPivot on a pivot below 1e-14 max|A|, ValueError on bad arguments.
    """
    t0 = time.perf_counter()
    if isinstance(A, SymSparseMatrix) and A.device is not None:
        n = A.dimension
    else:
        A = _as_csr(A)
        n = A.shape[0]
    if isinstance(ordering, str):
        if ordering == "natural":
            perm = np.arange(n, dtype=np.int64)
        elif ordering == "nd":
            perm = nested_dissection_graph(_as_csr(A))
        else:
            raise ValueError(f"unknown ordering strategy {ordering!r}")
    else:
        perm = np.asarray(ordering, dtype=np.int64)
        if perm.shape != (n,):
            raise ValueError("permutation length does not match matrix dimension")
    ctx = _dev.current()
    if isinstance(A, SymSparseMatrix) and A.device is not None and A.which == 0:
        dsys, sigma = A.device, 0.0
    else:
        csr = _as_csr(A)
        if csr.nnz == 0 or not np.any(csr.data):
            raise ZeroPivot("matrix is identically zero")
        dsys, sigma = DeviceSystem.upload(ctx, csr), 0.0
    sym = Symbolic.on_device(dsys, perm)
    fact = numeric_factor(sym, sigma, ctx)
    if counters is not None:
        counters.fact.add(fact.factor_flops, time.perf_counter() - t0)
    return fact


def solve_fb(fact: LDLFactorization, b, counters: CostCounters | None = None):
    """A^{-1} b (ref :265-277).  numpy in -> numpy out; torch CUDA in -> torch out."""
    is_t = isinstance(b, torch.Tensor)
    shape = tuple(b.shape) if is_t else np.shape(b)
    if shape != (fact.n,):
        raise ValueError(f"rhs has shape {shape}, expected ({fact.n},)")
    t0 = time.perf_counter()
    bd = _dev.to_device(b, fact.ctx)
    with torch.cuda.stream(fact.ctx.stream):
        x = fact.solve_device(bd)
        out = x if is_t else _dev.to_host(x)
    if counters is not None:
        counters.fb.add(2 * fact.fill_nnz, time.perf_counter() - t0)
    return out


# device copies of host matrices handed to mass_matvec (keyed by id, weakly)
_upload_cache: dict = {}


def _device_matrix(M, ctx):
    """(DeviceSystem, which) for a SymSparseMatrix or host CSR."""
    if isinstance(M, SymSparseMatrix) and M.device is not None:
        return M.device, M.which
    csr = _as_csr(M)
    key = (id(M), ctx.device)
    hit = _upload_cache.get(key)
    if hit is not None and hit[0]() is M:
        return hit[1], 0
    dsys = DeviceSystem.upload(ctx, csr)
    try:
        wr = weakref.ref(M)
    except TypeError:
        return dsys, 0
    _upload_cache[key] = (wr, dsys)
    return dsys, 0


def mass_matvec(M, v, counters: CostCounters | None = None):
    """y = M v on the device; charges 2 nnz(M) (ref :280-290)."""
    is_t = isinstance(v, torch.Tensor)
    n = M.dimension if isinstance(M, SymSparseMatrix) else _as_csr(M).shape[0]
    shape = tuple(v.shape) if is_t else np.shape(v)
    if shape != (n,):
        raise ValueError(f"vector has shape {shape}, expected ({n},)")
    ctx = _dev.current()
    t0 = time.perf_counter()
    dsys, which = _device_matrix(M, ctx)
    vd = _dev.to_device(v, ctx)
    with torch.cuda.stream(ctx.stream):
        y = torch.empty_like(vd)
        _lib.check(_lib.lib().riga_spmv(dsys.handle, which, 0.0, _lib.ptr(vd), _lib.ptr(y)), "spmv")
        out = y if is_t else _dev.to_host(y)
    if counters is not None:
        counters.matvec.add(2 * dsys.nnz, time.perf_counter() - t0)
    return out


def _rows(X: torch.Tensor) -> torch.Tensor:
    if X.dim() != 2 or X.stride(1) != 1:
        X = X.contiguous()
    return X


def solve_many(fact: LDLFactorization, B: torch.Tensor, ctx=None, counters: CostCounters | None = None):
    """Rows X[j] = A^{-1} B[j] of a device block (SURVEY §8b solve(fact, x, nrhs); ref solve_fb :265-277
    applied per column), on ctx's stream."""
    ctx = ctx or _dev.current()
    B = _rows(B)
    with torch.cuda.stream(ctx.stream):
        X = torch.empty_like(B)
    _lib.check(_lib.lib().riga_factor_solve_many(ctx.handle, fact.handle, _lib.ptr(B), B.stride(0), B.shape[0],
                                                 _lib.ptr(X), X.stride(0)), "solve_many")
    if counters is not None:
        for _ in range(B.shape[0]):
            counters.fb.add(2 * fact.fill_nnz, 0.0)
    return X


def spmv_many(system, which: int, X: torch.Tensor, ctx=None, counters: CostCounters | None = None):
    """Rows Y[j] = A X[j], A = K (0) or M (1) of a device pencil (ref mass_matvec :280-290 per row)."""
    ctx = ctx or _dev.current()
    dsys = system.device
    X = _rows(X)
    with torch.cuda.stream(ctx.stream):
        Y = torch.empty_like(X)
    _lib.check(_lib.lib().riga_spmv_many(ctx.handle, dsys.handle, which, 0.0, _lib.ptr(X), X.stride(0), X.shape[0],
                                         _lib.ptr(Y), Y.stride(0)), "spmv_many")
    if counters is not None:
        for _ in range(X.shape[0]):
            counters.matvec.add(2 * dsys.nnz, 0.0)
    return Y


def pair_residuals(system, X: torch.Tensor, lams, ctx=None):
    """Residuals of eigenpairs (rows of device block X, eigenvalues lams) on the device, one fused pass over
    K and M per 8 pairs (riga_residuals):

    * north_star: ||K x - lam M x|| / (|lam| ||M x||)
    * reference:  ||K x - lam M x|| / ||K x||  (ref eigensolver.py:784-792)
    """
    ctx = ctx or _dev.current()
    lams = np.ascontiguousarray(np.asarray(lams, dtype=np.float64))
    c = lams.size
    if c == 0:
        return np.empty(0), np.empty(0)
    X = _rows(X)
    out = np.empty(3 * c)
    _lib.check(_lib.lib().riga_residuals(ctx.handle, system.device.handle, _lib.ptr(X), X.stride(0), c,
                                         _lib.ptr(lams), _lib.ptr(out)), "residuals")
    out = out.reshape(c, 3)
    num = np.sqrt(out[:, 0])
    north = num / np.maximum(np.abs(lams) * np.sqrt(out[:, 1]), 1e-300)
    ref = num / np.maximum(np.sqrt(out[:, 2]), 1e-300)
    return north, ref


def m_inner(u, v, M=None) -> float:
    """v^T M u (Euclidean when M is None); ref :293-297."""
    if M is None:
        if isinstance(u, torch.Tensor) or isinstance(v, torch.Tensor):
            return float(torch.dot(_dev.to_device(v), _dev.to_device(u)))
        return float(np.dot(v, u))
    Mu = mass_matvec(M, u)
    if isinstance(Mu, torch.Tensor):
        return float(torch.dot(_dev.to_device(v), Mu))
    return float(np.dot(v, Mu))


def m_norm(v, M=None) -> float:
    sq = m_inner(v, v, M)
    if sq < -1e-12:
        raise NegativeNorm(f"v^T M v = {sq} < 0")
    return float(np.sqrt(max(sq, 0.0)))


# ---------------------------------------------------------------------------
# orderings (host)
# ---------------------------------------------------------------------------


def _c0_lines(system: DiscreteSystem):
    return [separator_basis_indices(s) - 1 for s in system.spaces]


def separator_blocks(system: DiscreteSystem) -> np.ndarray:
    """The dissection tree of ``separator_ordering`` as blocks in elimination order: one row
    (offset, lo[3], extent[3]) per leaf / separator box (engine: riga_separator_boxes, host C++)."""
    ext = np.array([s.basis_count - 2 for s in system.spaces], dtype=np.int64)
    lines = [np.ascontiguousarray(l, dtype=np.int64) for l in _c0_lines(system)]
    nlines = np.array([l.size for l in lines], dtype=np.int64)
    flat = np.concatenate(lines) if lines else np.zeros(0, np.int64)
    flat = np.ascontiguousarray(flat if flat.size else np.zeros(1, np.int64))
    L = _lib.lib()
    nch = ctypes.c_int64(0)
    p = int(system.spaces[0].degree)
    _lib.check(L.riga_separator_boxes(system.dim, _lib.ptr(ext), p, _lib.ptr(flat), _lib.ptr(nlines), 0,
                                      ctypes.byref(nch), None), "separator_boxes")
    chunks = np.zeros((nch.value, 7), dtype=np.int64)
    _lib.check(L.riga_separator_boxes(system.dim, _lib.ptr(ext), p, _lib.ptr(flat), _lib.ptr(nlines), nch.value,
                                      ctypes.byref(nch), _lib.ptr(chunks)), "separator_boxes")
    return chunks


def separator_ordering(system: DiscreteSystem) -> np.ndarray:
    """Nested dissection aligned with the rIGA C0 planes (ref :319-392).

    Each box is cut at the C0 interface nearest its middle (width one,
    longest axis with a candidate first); without one, at a width-p slab in
    the middle of its longest axis; boxes no longer than max(2p, 8) are
    leaves.  Order: leaves (recursion order), then separators deepest first.

    The tree (a few thousand boxes) is built by the engine on the host; the
    permutation itself is written by a device kernel when the system lives on
    a device (riga_separator_emit), else block by block with numpy.
    """
    chunks = separator_blocks(system)
    ext = np.array([s.basis_count - 2 for s in system.spaces], dtype=np.int64)
    n = system.dof_count
    if int(chunks[-1, 0] + np.prod(chunks[-1, 4:7])) != n:
        raise AssertionError("dissection did not enumerate every DOF")
    dev = getattr(system, "device", None)
    if dev is not None:
        ctx = dev.ctx
        with ctx:
            perm = torch.empty(n, dtype=torch.int64, device=f"cuda:{ctx.device}")
            _lib.check(_lib.lib().riga_separator_emit(ctx.handle, system.dim, _lib.ptr(ext), chunks.shape[0],
                                                      _lib.ptr(chunks), n, _lib.ptr(perm)), "separator_emit")
            return perm.cpu().numpy()
    strides = np.ones(3, dtype=np.int64)
    for t in range(1, system.dim):
        strides[t] = strides[t - 1] * ext[t - 1]
    order = np.empty(n, dtype=np.int64)
    for off, l0, l1, l2, e0, e1, e2 in chunks:
        a0 = (l0 + np.arange(e0, dtype=np.int64)) * strides[0]
        a1 = (l1 + np.arange(e1, dtype=np.int64)) * strides[1]
        a2 = (l2 + np.arange(e2, dtype=np.int64)) * strides[2]
        order[off:off + e0 * e1 * e2] = (a2[:, None, None] + a1[None, :, None] + a0[None, None, :]).ravel()
    return order


def nested_dissection_graph(pattern, leaf: int = 16) -> np.ndarray:
    """BFS level-set nested dissection for non-tensor patterns (ref :395-447)."""
    A = _as_csr(pattern)
    n = A.shape[0]
    ip, ix = A.indptr, A.indices
    out = []
    todo = [np.arange(n, dtype=np.int64)]
    # process as the reference's recursion does: depth-first, low part first,
    # separator appended after both halves -> emulate with an explicit stack
    stack = [("visit", todo[0])]
    while stack:
        kind, vs = stack.pop()
        if kind == "emit":
            out.append(vs)
            continue
        if vs.size <= leaf:
            out.append(vs)
            continue
        loc = np.full(n, -1, dtype=np.int64)
        loc[vs] = np.arange(vs.size)
        lev = np.full(vs.size, -1, dtype=np.int64)
        lev[0] = 0
        front, depth = [int(vs[0])], 0
        while front:
            nxt = []
            for u in front:
                for w in ix[ip[u]:ip[u + 1]]:
                    lw = loc[w]
                    if lw >= 0 and lev[lw] < 0:
                        lev[lw] = depth + 1
                        nxt.append(int(w))
            front, depth = nxt, depth + 1
        seen = lev >= 0
        if not seen.all():
            stack.append(("visit", vs[~seen]))
            stack.append(("visit", vs[seen]))
            continue
        t = int(np.median(lev))
        lo, hi = vs[lev < t], vs[lev > t]
        if lo.size == 0 or hi.size == 0:
            out.append(vs)
            continue
        stack.append(("emit", vs[lev == t]))
        stack.append(("visit", hi))
        stack.append(("visit", lo))
    return np.concatenate(out)
