"""Galerkin assembly: host 1D Gauss-Legendre tables, device Kronecker CSR.

API mirror of /root/reference/pkg/src/rigaeig/assembly.py.  The 1D
element integrals stay on the host (a few hundred tiny element matrices,
computed with the reference's own numpy expressions so the 1D tables are
bit-identical); the d-dimensional K and M -- up to 1e8 nonzeros for
config 5 -- are assembled on the device by ``riga_system_assemble_kron``
(k_kron_values: one warp per row, products and sums in scipy's order with
no FMA contraction, so every value is bit-identical to the reference's
``sp.kron`` chains).  ``DiscreteSystem.K.csr`` materialises host scipy
copies lazily, only when a caller asks for them.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import scipy.io
import scipy.sparse as sp

from . import _lib
from .bspline import SplineSpace, element_spans, eval_basis_span, make_spline_space


class DeviceSystem:
    """Owner of one device CSR pencil (riga_system)."""

    def __init__(self, handle, ctx, n: int, nnz: int):
        self.handle, self.ctx, self.n, self.nnz = handle, ctx, n, nnz
        self._host = None

    def attach_kron(self, k1d, m1d) -> None:
        """Declare M = M_z (x) M_y (x) M_x (1D factors in x-fastest order, as
        DiscreteSystem.k1d / m1d): Lanczos mass products then run axis by axis
        (riga_system_set_kron)."""
        d = len(m1d)
        parts_k = [_csr_parts(sp.csr_array(k)) for k in k1d]
        parts_m = [_csr_parts(sp.csr_array(m)) for m in m1d]
        n1 = np.array([m.shape[0] for m in m1d], dtype=np.int64)
        P = ctypes.c_void_p * d
        rps = P(*[_lib.ptr(q[0]).value for q in parts_m])
        cis = P(*[_lib.ptr(q[1]).value for q in parts_m])
        kvs = P(*[_lib.ptr(q[2]).value for q in parts_k])
        mvs = P(*[_lib.ptr(q[2]).value for q in parts_m])
        _lib.check(_lib.lib().riga_system_set_kron(self.handle, d, _lib.ptr(n1), rps, cis, kvs, mvs), "set_kron")

    def host_arrays(self):
        if self._host is None:
            rp = np.empty(self.n + 1, np.int64)
            ci = np.empty(self.nnz, np.int32)
            K = np.empty(self.nnz, np.float64)
            M = np.empty(self.nnz, np.float64)
            _lib.check(_lib.lib().riga_system_download(self.handle, _lib.ptr(rp), _lib.ptr(ci),
                                                       _lib.ptr(K), _lib.ptr(M)), "download")
            self._host = (rp, ci, K, M)
        return self._host

    @classmethod
    def upload(cls, ctx, A, B=None):
        """Device copy of host CSR A (and B on the same pattern, else zeros)."""
        A = A if isinstance(A, sp.csr_array) else sp.csr_array(A)
        A.sort_indices()
        n = A.shape[0]
        rp = np.ascontiguousarray(A.indptr, dtype=np.int64)
        ci = np.ascontiguousarray(A.indices, dtype=np.int32)
        av = np.ascontiguousarray(A.data, dtype=np.float64)
        if B is None:
            bv = np.zeros_like(av)
        else:
            B = B if isinstance(B, sp.csr_array) else sp.csr_array(B)
            same = B.indptr is A.indptr and B.indices is A.indices  # one pattern object (sorted with A)
            if not same:
                B.sort_indices()
            if not same and not (np.array_equal(B.indptr, A.indptr) and np.array_equal(B.indices, A.indices)):
                raise ValueError("K and M must share one sparsity pattern")
            bv = np.ascontiguousarray(B.data, dtype=np.float64)
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().riga_system_upload(ctx.handle, n, int(rp[-1]), _lib.ptr(rp), _lib.ptr(ci),
                                                 _lib.ptr(av), _lib.ptr(bv), ctypes.byref(h)), "upload")
        return cls(h, ctx, n, int(rp[-1]))

    def __del__(self):
        try:
            if self.handle:
                _lib.lib().riga_system_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


@dataclass(frozen=True)
class SymSparseMatrix:
    """Symmetric sparse matrix, full pattern (ref assembly.py:24-45).

    Either host-backed (``csr`` given) or one half of a device pencil
    (``device`` + ``which`` 0 = K, 1 = M) with a lazily built host copy.
    """

    _csr: object = None
    device: DeviceSystem | None = None
    which: int = 0
    _cache: dict = field(default_factory=dict, compare=False, repr=False)

    @property
    def csr(self) -> sp.csr_array:
        if self._csr is not None:
            return self._csr
        if "csr" not in self._cache:
            rp, ci, K, M = self.device.host_arrays()
            vals = K if self.which == 0 else M
            self._cache["csr"] = sp.csr_array((vals, ci, rp), shape=(self.device.n, self.device.n))
        return self._cache["csr"]

    @property
    def dimension(self) -> int:
        return self.device.n if self.device is not None else self._csr.shape[0]

    @property
    def nnz(self) -> int:
        return self.device.nnz if self.device is not None else self._csr.nnz

    def toarray(self) -> np.ndarray:
        return self.csr.toarray()


@dataclass(frozen=True)
class DiscreteSystem:
    """Dirichlet-reduced pencil (K, M) on [0,1]^d (ref assembly.py:48-62)."""

    K: SymSparseMatrix
    M: SymSparseMatrix
    spaces: tuple
    dim: int
    dof_count: int
    k1d: tuple
    m1d: tuple
    device: DeviceSystem | None = None


def gauss_points(nq: int, a: float, b: float):
    x, w = np.polynomial.legendre.leggauss(nq)
    half = 0.5 * (b - a)
    return a + half * (x + 1.0), half * w


def assemble_1d(space: SplineSpace, n_quad: int | None = None):
    """Full-basis 1D K1, M1 with n_quad (default p+1) Gauss points per element
    (ref assembly.py:72-111; same element-matrix expressions)."""
    p, n = space.degree, space.basis_count
    nq = p + 1 if n_quad is None else n_quad
    rows, cols, kv, mv = [], [], [], []
    for mu, a, b in element_spans(space):
        pts, wts = gauss_points(nq, a, b)
        vals, ders = eval_basis_span(space, mu, pts)
        ke = ders.T @ (ders * wts[:, None])
        me = vals.T @ (vals * wts[:, None])
        ke = 0.5 * (ke + ke.T)
        me = 0.5 * (me + me.T)
        idx = np.arange(mu - p, mu + 1)
        rr, cc = np.meshgrid(idx, idx, indexing="ij")
        rows.append(rr.ravel()); cols.append(cc.ravel())
        kv.append(ke.ravel()); mv.append(me.ravel())
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    K = sp.coo_array((np.concatenate(kv), (rows, cols)), shape=(n, n)).tocsr()
    M = sp.coo_array((np.concatenate(mv), (rows, cols)), shape=(n, n)).tocsr()
    return SymSparseMatrix(K), SymSparseMatrix(M)


def apply_dirichlet(K1: SymSparseMatrix, M1: SymSparseMatrix):
    n = K1.dimension
    if n < 3:
        raise ValueError("no interior degrees of freedom left after elimination")
    keep = np.arange(1, n - 1)
    return SymSparseMatrix(K1.csr[keep][:, keep]), SymSparseMatrix(M1.csr[keep][:, keep])


def _csr_parts(A):
    A = sp.csr_array(A)
    A.sort_indices()
    return (np.ascontiguousarray(A.indptr, np.int64), np.ascontiguousarray(A.indices, np.int32),
            np.ascontiguousarray(A.data, np.float64))


def kron_assemble(spaces, stiffness_only: bool = False, ctx=None) -> DiscreteSystem:
    """d-dimensional Dirichlet-reduced system, x fastest (ref assembly.py:139-186),
    assembled on the device."""
    from . import device as _dev

    spaces = tuple(spaces)
    d = len(spaces)
    if d not in (1, 2, 3):
        raise ValueError(f"dimension must be 1, 2 or 3, got {d}")
    if len({s.degree for s in spaces}) != 1:
        raise ValueError("per-direction degrees must match")
    k1d, m1d = [], []
    for s in spaces:
        K1, M1 = apply_dirichlet(*assemble_1d(s))
        k1d.append(K1.csr); m1d.append(M1.csr)
    ctx = ctx or _dev.current()
    parts_k = [_csr_parts(k) for k in k1d]
    parts_m = [_csr_parts(m) for m in m1d]
    for (rk, ck, _), (rm, cm, _) in zip(parts_k, parts_m):
        if not (np.array_equal(rk, rm) and np.array_equal(ck, cm)):
            raise ValueError("1D K and M patterns differ")
    n1 = np.array([k.shape[0] for k in k1d], dtype=np.int64)
    P = ctypes.c_void_p * d
    rps = P(*[_lib.ptr(p[0]).value for p in parts_k])
    cis = P(*[_lib.ptr(p[1]).value for p in parts_k])
    kvs = P(*[_lib.ptr(p[2]).value for p in parts_k])
    mvs = P(*[_lib.ptr(p[2]).value for p in parts_m])
    h = ctypes.c_void_p()
    _lib.check(_lib.lib().riga_system_assemble_kron(ctx.handle, d, _lib.ptr(n1), rps, cis, kvs, mvs,
                                                    ctypes.byref(h)), "assemble")
    n = int(np.prod(n1))
    nnz = int(np.prod([p[0][-1] for p in parts_k]))
    dev = DeviceSystem(h, ctx, n, nnz)
    K = SymSparseMatrix(device=dev, which=0)
    if stiffness_only:
        M = SymSparseMatrix(sp.csr_array((n, n)))
    else:
        M = SymSparseMatrix(device=dev, which=1)
    return DiscreteSystem(K, M, spaces, d, n, tuple(k1d), tuple(m1d), dev)


def quadrature_tables(space: SplineSpace):
    """Per element of one direction: first global basis index (span - p), the (p+1) Gauss weights scaled to
    the element, and the (p+1) x (p+1) basis values / derivatives at the points ([e][q][a]).  Host side of
    the device quadrature assembly (the 1D ingredients of ref assembly.py:72-111)."""
    p = space.degree
    first, ws, Ns, dNs = [], [], [], []
    for mu, a, b in element_spans(space):
        pts, wts = gauss_points(p + 1, a, b)
        vals, ders = eval_basis_span(space, mu, pts)
        first.append(mu - p)
        ws.append(wts)
        Ns.append(vals)
        dNs.append(ders)
    return (np.ascontiguousarray(first, np.int32), np.ascontiguousarray(np.stack(ws), np.float64),
            np.ascontiguousarray(np.stack(Ns), np.float64), np.ascontiguousarray(np.stack(dNs), np.float64))


def quadrature_assemble(spaces, ctx=None) -> DiscreteSystem:
    """d-dimensional Dirichlet-reduced system by element quadrature on the device: (p+1)^d Gauss points
    per d-dimensional element (BASELINE configs), the same CSR pattern and x-fastest numbering as
    ``kron_assemble``; values equal the Kronecker pencil to roundoff (riga_system_assemble_quad)."""
    from . import device as _dev

    spaces = tuple(spaces)
    d = len(spaces)
    if d not in (1, 2, 3):
        raise ValueError(f"dimension must be 1, 2 or 3, got {d}")
    if len({s.degree for s in spaces}) != 1:
        raise ValueError("per-direction degrees must match")
    p = spaces[0].degree
    k1d, m1d, tabs = [], [], []
    for s in spaces:
        K1, M1 = apply_dirichlet(*assemble_1d(s))
        k1d.append(K1.csr); m1d.append(M1.csr)
        tabs.append(quadrature_tables(s))
    ctx = ctx or _dev.current()
    parts_k = [_csr_parts(k) for k in k1d]
    parts_m = [_csr_parts(m) for m in m1d]
    n1 = np.array([k.shape[0] for k in k1d], dtype=np.int64)
    ne = np.array([t[0].size for t in tabs], dtype=np.int64)
    P = ctypes.c_void_p * d
    arr = lambda xs: P(*[_lib.ptr(x).value for x in xs])  # noqa: E731
    h = ctypes.c_void_p()
    _lib.check(_lib.lib().riga_system_assemble_quad(
        ctx.handle, d, p, _lib.ptr(ne), arr([t[0] for t in tabs]), arr([t[1] for t in tabs]),
        arr([t[2] for t in tabs]), arr([t[3] for t in tabs]), _lib.ptr(n1), arr([q[0] for q in parts_k]),
        arr([q[1] for q in parts_k]), arr([q[2] for q in parts_k]), arr([q[2] for q in parts_m]),
        ctypes.byref(h)), "assemble_quad")
    n = int(np.prod(n1))
    nnz = int(np.prod([q[0][-1] for q in parts_k]))
    dev = DeviceSystem(h, ctx, n, nnz)
    return DiscreteSystem(SymSparseMatrix(device=dev, which=0), SymSparseMatrix(device=dev, which=1), spaces, d, n,
                          tuple(k1d), tuple(m1d), dev)


def build_system(d: int, ne: int, p: int, level: int = 0, assembly: str = "kron", **kw) -> DiscreteSystem:
    """ref assembly.py:189-192.  ``assembly`` (engine extension): "kron" (default) composes the device CSR
    from the 1D matrices in the reference's own product and sum order (bit-identical K and M);
    "quadrature" integrates every d-dimensional element with (p+1)^d Gauss points on the device."""
    spaces = (make_spline_space(ne, p, level),) * d
    if assembly == "kron":
        return kron_assemble(spaces, **kw)
    if assembly == "quadrature":
        return quadrature_assemble(spaces, **kw)
    raise ValueError(f"unknown assembly {assembly!r}")


def dof_count(ne: int, p: int, level: int, d: int) -> int:
    per = ne + p - 2 if level == 0 else ne + 2**level * (p - 1) - 1
    return per**d


def nnz_mass_formula(ne: int, p: int, level: int, d: int) -> int:
    if level == 0:
        per = ne * (2 * p + 1) + p * p
    else:
        per = 2**level * (ne * (2 * p + 1) // 2**level + p * p - 1)
    return per**d


def write_matrix_market(path, matrix: SymSparseMatrix) -> None:
    scipy.io.mmwrite(path, sp.coo_matrix(sp.tril(matrix.csr)), symmetry="symmetric")
