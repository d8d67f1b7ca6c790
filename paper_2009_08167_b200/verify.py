"""Exact Laplace spectra and eigen-error metrics (EV, EFL, EFE).

Drop-in for /root/reference/pkg/src/rigaeig/verify.py:
same names, arguments, dataclasses and exceptions.  The exact pairs on the
unit box with zero boundary values are lambda = pi^2 (i^2 + j^2 + ...) with
products of sqrt(2) sin(k pi x); discrete pairs are matched positionally
after sorting (ref :1-17), and

    EV  = (lambda_h - lambda) / lambda
    EFL = || u_h - u ||_L2^2      (modes whose exact eigenfunction is unique)
    EFE = EV + EFL

Device side: ``error_table`` evaluates every eigenfunction error of a solve
at once with engine kernels (csrc/verify.cu): the coefficient tensors of all
unique-eigenfunction modes go through one banded tensor-product contraction
per direction (``riga_tp_contract``; ref ErrorEvaluator._contract :218-225 --
a collocation matrix has p + 1 non-zeros per point, so this is HBM-bound
gather work, not a GEMM), the M-normalisations use the engine's batched mass
product and row dots, and the quadrature sums against the exact modes, formed
on the fly, are fixed-order reductions (``riga_tp_reduce``); the reference
loops over modes on the host.  The per-mode methods of ``ErrorEvaluator`` are
kept for API parity and run the same kernels on one mode.  There is no host
path: without a CUDA device the evaluator raises.
"""
from __future__ import annotations

import ctypes
import itertools
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .assembly import DiscreteSystem, gauss_points
from .bspline import element_spans, eval_basis, eval_basis_span

PI2 = math.pi * math.pi


@dataclass(frozen=True)
class ExactMode:
    """One continuous eigenmode (ref verify.py:35-52)."""

    indices: tuple
    lam: float
    cluster_id: int
    cluster_size: int
    cluster_rank: int

    @property
    def diagonal(self) -> bool:
        return len(set(self.indices)) == 1

    @property
    def unique_eigenfunction(self) -> bool:
        return self.diagonal and self.cluster_size == 1


def exact_spectrum(d: int, count: int | None = None, interval=None) -> list:
    """Exact eigenvalues ascending, ties lexicographic (ref :54-102): the
    first ``count`` modes or all modes inside the closed ``interval``."""
    if d not in (1, 2, 3):
        raise ValueError(f"dimension must be 1, 2 or 3, got {d}")
    if (count is None) == (interval is None):
        raise ValueError("request either `count` or `interval`")
    if interval is not None:
        lo, hi = float(interval[0]), float(interval[1])
        kmax = int(math.sqrt(max(hi / PI2 - (d - 1), 0.0))) + 1
        cand = [(PI2 * sum(i * i for i in ix), ix) for ix in itertools.product(range(1, kmax + 1), repeat=d)]
        cand = sorted((lam, ix) for lam, ix in cand if lo <= lam <= hi)
    else:
        kmax = max(2, int(round(count ** (1.0 / d))) + 2)
        while True:
            # any tuple with an index > kmax exceeds pi^2 ((kmax+1)^2 + d - 1)
            cut = PI2 * ((kmax + 1) ** 2 + (d - 1))
            cand = [(PI2 * sum(i * i for i in ix), ix) for ix in itertools.product(range(1, kmax + 1), repeat=d)]
            cand = [(lam, ix) for lam, ix in cand if lam < cut]
            if len(cand) >= count:
                cand = sorted(cand)[:count]
                break
            kmax *= 2
    modes, i, cid = [], 0, 0
    while i < len(cand):
        j = i + 1
        while j < len(cand) and abs(cand[j][0] - cand[i][0]) < 1e-9 * cand[i][0]:
            j += 1
        for rank, (lam, ix) in enumerate(cand[i:j]):
            modes.append(ExactMode(ix, lam, cid, j - i, rank))
        cid += 1
        i = j
    return modes


def _sine_factors(mode: ExactMode, axes, deriv: int | None = None):
    out = []
    for t, (k, ax) in enumerate(zip(mode.indices, axes)):
        if t == deriv:
            out.append(math.sqrt(2.0) * k * math.pi * np.cos(k * math.pi * ax))
        else:
            out.append(math.sqrt(2.0) * np.sin(k * math.pi * ax))
    return out


def _outer(factors):
    """Grid from per-direction factors (x first) with the last axis fastest."""
    out = np.ones(())
    for f in reversed(factors):  # z ... x
        out = np.multiply.outer(out, f)
    return out


def exact_eigenfunction(mode: ExactMode, axes) -> np.ndarray:
    """ref :105-118: on the tensor grid of ``axes`` (x first), x fastest."""
    return _outer(_sine_factors(mode, axes))


def exact_eigenfunction_deriv(mode: ExactMode, axes, t: int) -> np.ndarray:
    """ref :121-133: partial derivative along direction t."""
    return _outer(_sine_factors(mode, axes, deriv=t))


def _embed_coefficients(system: DiscreteSystem, coeffs: np.ndarray) -> np.ndarray:
    """Reduced vector -> full control tensor (z, y, x), zero boundary layers (ref :136-148)."""
    if coeffs.shape != (system.dof_count,):
        raise ValueError(f"coefficient vector has shape {coeffs.shape}, expected ({system.dof_count},)")
    red = [s.basis_count - 2 for s in reversed(system.spaces)]
    full = [s.basis_count for s in reversed(system.spaces)]
    U = np.zeros(full)
    U[tuple(slice(1, n - 1) for n in full)] = coeffs.reshape(red)
    return U


def evaluate_eigenfunction(system: DiscreteSystem, coeffs, points) -> np.ndarray:
    """Discrete eigenfunction at arbitrary points of [0,1]^d (ref :151-178)."""
    U = _embed_coefficients(system, np.asarray(coeffs, dtype=np.float64))
    pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
    if system.dim == 1 and pts.shape[0] == 1 and pts.shape[1] != 1:
        pts = pts.T
    if pts.shape[1] != system.dim:
        raise ValueError(f"points have dimension {pts.shape[1]}, system is {system.dim}D")
    d = system.dim
    out = np.empty(pts.shape[0])
    for q, x in enumerate(pts):
        ev = [eval_basis(system.spaces[t], float(x[t])) for t in range(d)]
        block = U[tuple(slice(ev[t].first_index, ev[t].first_index + len(ev[t].values)) for t in reversed(range(d)))]
        for t in range(d):  # contract x (the last axis) first
            block = block @ ev[t].values
        out[q] = float(block)
    return out


class ErrorEvaluator:
    """Per-direction Gauss rules (degree + 2 points per element by default)
    and collocation tables, built once on the host (ref :181-216) and kept on
    the device in banded form: a quadrature point sees p + 1 basis functions,
    so each direction is ``first`` (their first index) and a (points, p + 1)
    value table.  Every contraction and quadrature sum is an engine kernel
    (``riga_tp_contract`` / ``riga_tp_reduce``); there is no host path."""

    def __init__(self, system: DiscreteSystem, n_quad: int | None = None, ctx=None):
        from . import device as _dev

        self.system = system
        self.dim = system.dim
        self.ctx = ctx or _dev.current()
        self.device = torch.device(f"cuda:{self.ctx.device}")
        self.axes, self.weights, self.first, self.vals, self.ders = [], [], [], [], []
        for space in system.spaces:
            nq = (space.degree + 2) if n_quad is None else n_quad
            pts, wts, rows_v, rows_d, firsts = [], [], [], [], []
            for mu, a, b in element_spans(space):
                x, w = gauss_points(nq, a, b)
                v, dv = eval_basis_span(space, mu, x)
                pts.append(x)
                wts.append(w)
                rows_v.append(v)
                rows_d.append(dv)
                firsts.append(np.full(nq, mu - space.degree))
            self.axes.append(np.concatenate(pts))
            self.weights.append(np.concatenate(wts))
            self.first.append(np.concatenate(firsts).astype(np.int32))
            self.vals.append(np.ascontiguousarray(np.concatenate(rows_v)))
            self.ders.append(np.ascontiguousarray(np.concatenate(rows_d)))
        up = lambda a: _dev.to_device(a, self.ctx)  # noqa: E731
        with torch.cuda.stream(self.ctx.stream):
            self._first = [torch.from_numpy(f).to(self.device) for f in self.first]
        self._vals = [up(v) for v in self.vals]
        self._ders = [up(v) for v in self.ders]
        self._w = [up(w) for w in self.weights]
        self._ax = [up(a) for a in self.axes]
        self._nq = np.array([a.size for a in self.axes], dtype=np.int64)
        self._red = [s.basis_count - 2 for s in system.spaces]  # x first
        PP = ctypes.c_void_p * self.dim
        self._axp = PP(*[a.data_ptr() for a in self._ax])
        self._wp = PP(*[w.data_ptr() for w in self._w])

    # -- batched device kernels (leading batch axis) ---------------------
    def _contract_b(self, C: torch.Tensor, deriv: int | None = None, scale: torch.Tensor | None = None):
        """Reduced coefficient rows C (B, dof_count) -> values of u_h (or its partial derivative along
        ``deriv``) on the quadrature grid, (B, q_z, q_y, q_x); rows optionally scaled by ``scale`` (B,)."""
        if C.dim() != 2 or C.shape[1] != self.system.dof_count:
            raise ValueError(f"coefficient block has shape {tuple(C.shape)}, expected (B, {self.system.dof_count})")
        L = _lib.lib()
        B = C.shape[0]
        cur = C if (C.is_contiguous() and C.dtype == torch.float64) else C.to(torch.float64).contiguous()
        shape = [B] + list(reversed(self._red))  # (B, n_z, n_y, n_x)
        with torch.cuda.stream(self.ctx.stream):
            for t in range(self.dim):  # x (the last axis) first
                ax = len(shape) - 1 - t
                outer = int(np.prod(shape[:ax]))
                inner = int(np.prod(shape[ax + 1:]))
                tab = self._ders[t] if t == deriv else self._vals[t]
                p1 = tab.shape[1]
                out = torch.empty(outer * int(self._nq[t]) * inner, dtype=torch.float64, device=self.device)
                sc = scale if (t == 0 and scale is not None) else None
                _lib.check(L.riga_tp_contract(self.ctx.handle, _lib.ptr(cur), _lib.ptr(out), outer, shape[ax],
                                              int(self._nq[t]), inner, p1, 1, _lib.ptr(self._first[t]),
                                              _lib.ptr(tab), _lib.ptr(sc), outer // B), "tp_contract")
                shape[ax] = int(self._nq[t])
                cur = out
        return cur.reshape(shape)

    def _reduce_b(self, G: torch.Tensor, modes, kind: int, deriv: int | None = None,
                  gsign: torch.Tensor | None = None) -> torch.Tensor:
        """Quadrature sums over the grid per batch member: kind 0 = (g G - u)^2, 1 = G u, 2 = G, with
        u the exact mode (or its partial derivative along ``deriv``) formed on the device."""
        B = G.shape[0]
        G = G if G.is_contiguous() else G.contiguous()
        ks = np.ascontiguousarray([m.indices for m in modes] if modes else np.ones((B, self.dim)), dtype=np.int32)
        with torch.cuda.stream(self.ctx.stream):
            kd = torch.from_numpy(ks).to(self.device)
            out = torch.empty(B, dtype=torch.float64, device=self.device)
        _lib.check(_lib.lib().riga_tp_reduce(self.ctx.handle, _lib.ptr(G), B, self.dim, _lib.ptr(self._nq),
                                             self._axp, self._wp, _lib.ptr(kd), -1 if deriv is None else deriv,
                                             kind, _lib.ptr(gsign), _lib.ptr(out)), "tp_reduce")
        return out

    # -- per-mode API (ref :218-255) ---------------------------------------
    def _one(self, coeffs) -> torch.Tensor:
        from . import device as _dev

        c = np.asarray(coeffs, dtype=np.float64)
        if c.shape != (self.system.dof_count,):
            raise ValueError(f"coefficient vector has shape {tuple(c.shape)}, expected ({self.system.dof_count},)")
        return _dev.to_device(c, self.ctx)[None]

    def uh_values(self, coeffs) -> np.ndarray:
        return self._contract_b(self._one(coeffs))[0].cpu().numpy()

    def uh_deriv(self, coeffs, t: int) -> np.ndarray:
        return self._contract_b(self._one(coeffs), deriv=t)[0].cpu().numpy()

    def integrate(self, grid) -> float:
        from . import device as _dev

        g = _dev.to_device(np.asarray(grid, dtype=np.float64), self.ctx)
        if tuple(g.shape) != tuple(int(n) for n in reversed(self._nq)):
            raise ValueError(f"grid has shape {tuple(g.shape)}, expected {tuple(reversed(self._nq.tolist()))}")
        return float(self._reduce_b(g[None], None, 2)[0])

    def l2_error_sq(self, coeffs, mode: ExactMode) -> float:
        return float(self._reduce_b(self._contract_b(self._one(coeffs)), [mode], 0)[0])

    def energy_error_sq(self, coeffs, mode: ExactMode) -> float:
        C = self._one(coeffs)
        return sum(float(self._reduce_b(self._contract_b(C, deriv=t), [mode], 0, deriv=t)[0])
                   for t in range(self.dim))

    def inner_with_exact(self, coeffs, mode: ExactMode) -> float:
        return float(self._reduce_b(self._contract_b(self._one(coeffs)), [mode], 1)[0])


@dataclass
class AlignedMode:
    """ref :258-265."""

    mode: ExactMode
    position: int
    lam_h: float
    coeffs: np.ndarray | None


@dataclass
class ErrorRecord:
    """ref :268-276."""

    position: int
    indices: tuple
    ev: float
    efl: float
    efe: float
    diagonal: bool


def _mass_norms(system: DiscreteSystem, C: torch.Tensor, ctx) -> torch.Tensor:
    """sqrt(c^T M c) of each row of the device block C: batched engine mass product + row dots."""
    from .sparsela import spmv_many

    MC = spmv_many(system, 1, C, ctx=ctx)
    with torch.cuda.stream(ctx.stream):
        out = torch.empty(C.shape[0], dtype=torch.float64, device=C.device)
    _lib.check(_lib.lib().riga_row_dots(ctx.handle, _lib.ptr(C), C.stride(0), _lib.ptr(MC), MC.stride(0), C.shape[1],
                                        C.shape[0], _lib.ptr(out)), "row_dots")
    with torch.cuda.stream(ctx.stream):
        return torch.sqrt(torch.clamp(out, min=0.0))


def _aligned_batch(lams, vectors, modes, system, evaluator):
    """Positional match; unique-eigenfunction modes M-normalised and signed to a nonnegative inner
    product with the exact mode, all at once (ref :279-313).  Returns the raw coefficient rows C,
    their scale (sign / M-norm) and the grid values G of the M-normalised, unsigned functions."""
    n = min(lams.size, len(modes))
    uniq = [i for i in range(n) if modes[i].unique_eigenfunction]
    C = scale = G = None
    if uniq:
        from . import device as _dev

        ctx = evaluator.ctx
        V = vectors if isinstance(vectors, torch.Tensor) else np.asarray(vectors, dtype=np.float64)
        C = _dev.to_device(np.ascontiguousarray(V[:, uniq].T) if not isinstance(V, torch.Tensor) else V[:, uniq].T, ctx)
        nrm = _mass_norms(system, C, ctx)
        with torch.cuda.stream(ctx.stream):
            inv = 1.0 / torch.where(nrm > 0, nrm, torch.ones_like(nrm))
        G = evaluator._contract_b(C, scale=inv)
        inner = evaluator._reduce_b(G, [modes[i] for i in uniq], 1)
        with torch.cuda.stream(ctx.stream):
            sgn = torch.where(inner < 0, -1.0, 1.0).to(torch.float64)
            scale = inv * sgn
    return n, uniq, C, scale, G


def match_and_normalize(eigenvalues, vectors, modes, system: DiscreteSystem,
                        evaluator: ErrorEvaluator | None = None) -> list:
    """ref :279-313."""
    lams = np.asarray(eigenvalues, dtype=np.float64)
    n = min(lams.size, len(modes))
    if evaluator is None and any(modes[i].unique_eigenfunction for i in range(n)):
        evaluator = ErrorEvaluator(system)
    n, uniq, C, scale, _ = _aligned_batch(lams, vectors, modes, system, evaluator) if evaluator else (n, [], None, None, None)
    Ch = (C * scale[:, None]).cpu().numpy() if C is not None else None
    where = {i: q for q, i in enumerate(uniq)}
    return [AlignedMode(modes[i], i, float(lams[i]), Ch[where[i]] if i in where else None) for i in range(n)]


def error_metrics(aligned: AlignedMode, system: DiscreteSystem,
                  evaluator: ErrorEvaluator | None = None) -> ErrorRecord:
    """ref :316-329."""
    mode = aligned.mode
    ev = (aligned.lam_h - mode.lam) / mode.lam
    if aligned.coeffs is None:
        return ErrorRecord(aligned.position, mode.indices, ev, math.nan, math.nan, mode.diagonal)
    if evaluator is None:
        evaluator = ErrorEvaluator(system)
    efl = evaluator.l2_error_sq(aligned.coeffs, mode)
    return ErrorRecord(aligned.position, mode.indices, ev, efl, ev + efl, mode.diagonal)


def error_table(result_eigenvalues, result_vectors, system: DiscreteSystem) -> list:
    """Error records of a whole solve against the exact spectrum (ref
    :332-338); every EFL of the solve in one batched device evaluation: one
    tensor-product contraction of all unique-eigenfunction modes, the sign
    and the squared L2 error from the same grid values."""
    lams = np.asarray(result_eigenvalues, dtype=np.float64)
    modes = exact_spectrum(system.dim, count=lams.size)
    ev = ErrorEvaluator(system)
    n, uniq, C, scale, G = _aligned_batch(lams, result_vectors, modes, system, ev)
    efl = {}
    if uniq:
        with torch.cuda.stream(ev.ctx.stream):
            sgn = torch.sign(scale)
        vals = ev._reduce_b(G, [modes[i] for i in uniq], 0, gsign=sgn).cpu().numpy()
        efl = {i: float(v) for i, v in zip(uniq, vals)}
    out = []
    for i in range(n):
        m = modes[i]
        e = (float(lams[i]) - m.lam) / m.lam
        if i in efl:
            out.append(ErrorRecord(i, m.indices, e, efl[i], e + efl[i], m.diagonal))
        else:
            out.append(ErrorRecord(i, m.indices, e, math.nan, math.nan, m.diagonal))
    return out
