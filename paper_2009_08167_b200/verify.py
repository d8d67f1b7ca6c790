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
at once -- the coefficient tensors of all unique-eigenfunction modes are
contracted with the per-direction collocation matrices as batched FP64
GEMMs on the GPU (tensor-product evaluation, ref ErrorEvaluator._contract
:218-225), the M-normalisations use the engine's mass product, and the
quadrature sums are batched reductions; the reference loops over modes on
the host.  The per-mode methods of ``ErrorEvaluator`` are kept for API
parity and run the same contractions on one mode.
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass

import numpy as np
import torch

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
    and dense collocation matrices, built once (ref :181-216); contractions
    on the device."""

    def __init__(self, system: DiscreteSystem, n_quad: int | None = None, device=None):
        self.system = system
        self.dim = system.dim
        self.device = torch.device(device if device is not None else
                                   ("cuda" if torch.cuda.is_available() else "cpu"))
        self.axes, self.weights, self.bval, self.bder = [], [], [], []
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
            pts = np.concatenate(pts)
            p1 = space.degree + 1
            bv = np.zeros((pts.size, space.basis_count))
            bd = np.zeros_like(bv)
            f0 = np.concatenate(firsts)
            rv, rd = np.concatenate(rows_v), np.concatenate(rows_d)
            rr = np.repeat(np.arange(pts.size), p1)
            cc = (f0[:, None] + np.arange(p1)[None, :]).ravel()
            bv[rr, cc] = rv.ravel()
            bd[rr, cc] = rd.ravel()
            self.axes.append(pts)
            self.weights.append(np.concatenate(wts))
            self.bval.append(bv)
            self.bder.append(bd)
        dev = self.device
        self._bval = [torch.as_tensor(b, device=dev) for b in self.bval]
        self._bder = [torch.as_tensor(b, device=dev) for b in self.bder]
        self._w = [torch.as_tensor(w, device=dev) for w in self.weights]
        self._ax = [torch.as_tensor(a, device=dev) for a in self.axes]

    # -- batched device kernels (leading batch axis) ---------------------
    def _contract_b(self, U: torch.Tensor, mats) -> torch.Tensor:
        """U (B, n_z, n_y, n_x) -> values on the quadrature grid (B, q_z, q_y, q_x)."""
        out = U
        for t in range(self.dim):  # x is the last axis
            ax = out.dim() - 1 - t
            out = torch.movedim(torch.movedim(out, ax, -1) @ mats[t].T, -1, ax)
        return out

    def _integrate_b(self, G: torch.Tensor) -> torch.Tensor:
        out = G
        for t in range(self.dim):
            out = out @ self._w[t]  # contracts the current last axis (x, then y, then z)
        return out

    def _exact_b(self, modes, deriv: int | None = None) -> torch.Tensor:
        ks = torch.as_tensor([m.indices for m in modes], dtype=torch.float64, device=self.device)
        out = None
        for t in reversed(range(self.dim)):  # z ... x: x fastest
            arg = math.pi * ks[:, t:t + 1] * self._ax[t][None, :]
            f = math.sqrt(2.0) * (ks[:, t:t + 1] * math.pi * torch.cos(arg) if t == deriv else torch.sin(arg))
            out = f if out is None else out[..., None] * f.reshape(f.shape[0], *([1] * (out.dim() - 1)), f.shape[1])
        return out

    def _embed_b(self, C: torch.Tensor) -> torch.Tensor:
        red = [s.basis_count - 2 for s in reversed(self.system.spaces)]
        full = [s.basis_count for s in reversed(self.system.spaces)]
        U = torch.zeros((C.shape[0], *full), dtype=torch.float64, device=self.device)
        U[(slice(None),) + tuple(slice(1, n - 1) for n in full)] = C.reshape(C.shape[0], *red)
        return U

    # -- per-mode API (ref :218-255) ---------------------------------------
    def _one(self, coeffs) -> torch.Tensor:
        c = torch.as_tensor(np.asarray(coeffs, dtype=np.float64), device=self.device)
        if c.shape != (self.system.dof_count,):
            raise ValueError(f"coefficient vector has shape {tuple(c.shape)}, expected ({self.system.dof_count},)")
        return self._embed_b(c[None])

    def uh_values(self, coeffs) -> np.ndarray:
        return self._contract_b(self._one(coeffs), self._bval)[0].cpu().numpy()

    def uh_deriv(self, coeffs, t: int) -> np.ndarray:
        mats = [self._bder[s] if s == t else self._bval[s] for s in range(self.dim)]
        return self._contract_b(self._one(coeffs), mats)[0].cpu().numpy()

    def integrate(self, grid) -> float:
        g = torch.as_tensor(np.asarray(grid, dtype=np.float64), device=self.device)
        return float(self._integrate_b(g[None])[0])

    def l2_error_sq(self, coeffs, mode: ExactMode) -> float:
        diff = self._contract_b(self._one(coeffs), self._bval) - self._exact_b([mode])
        return float(self._integrate_b(diff * diff)[0])

    def energy_error_sq(self, coeffs, mode: ExactMode) -> float:
        U = self._one(coeffs)
        tot = 0.0
        for t in range(self.dim):
            mats = [self._bder[s] if s == t else self._bval[s] for s in range(self.dim)]
            diff = self._contract_b(U, mats) - self._exact_b([mode], deriv=t)
            tot += float(self._integrate_b(diff * diff)[0])
        return tot

    def inner_with_exact(self, coeffs, mode: ExactMode) -> float:
        G = self._contract_b(self._one(coeffs), self._bval)
        return float(self._integrate_b(G * self._exact_b([mode]))[0])


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


def _mass_norms(system: DiscreteSystem, C: torch.Tensor) -> torch.Tensor:
    """sqrt(c^T M c) of each row of C (device mass product per vector)."""
    from .sparsela import mass_matvec

    out = torch.empty(C.shape[0], dtype=torch.float64, device=C.device)
    for i in range(C.shape[0]):
        mc = mass_matvec(system.M, C[i])
        mc = torch.as_tensor(mc, device=C.device) if not isinstance(mc, torch.Tensor) else mc
        out[i] = torch.dot(C[i], mc)
    return torch.sqrt(torch.clamp(out, min=0.0))


def _aligned_batch(lams, vectors, modes, system, evaluator):
    """Positional match; unique-eigenfunction modes M-normalised and signed
    to a nonnegative inner product with the exact mode, all at once."""
    n = min(lams.size, len(modes))
    uniq = [i for i in range(n) if modes[i].unique_eigenfunction]
    C = None
    if uniq:
        V = vectors if isinstance(vectors, torch.Tensor) else torch.as_tensor(np.asarray(vectors, dtype=np.float64))
        C = V[:, uniq].T.to(device=evaluator.device, dtype=torch.float64).contiguous()
        nrm = _mass_norms(system, C) if evaluator.device.type == "cuda" else torch.as_tensor(
            [math.sqrt(max(float(c @ (system.M.csr @ c)), 0.0)) for c in C.cpu().numpy()])
        C = C / torch.where(nrm > 0, nrm, torch.ones_like(nrm))[:, None].to(C.device)
        G = evaluator._contract_b(evaluator._embed_b(C), evaluator._bval)
        E = evaluator._exact_b([modes[i] for i in uniq])
        sgn = torch.where(evaluator._integrate_b(G * E) < 0, -1.0, 1.0)
        C = C * sgn[:, None]
    return n, uniq, C


def match_and_normalize(eigenvalues, vectors, modes, system: DiscreteSystem,
                        evaluator: ErrorEvaluator | None = None) -> list:
    """ref :279-313."""
    lams = np.asarray(eigenvalues, dtype=np.float64)
    n = min(lams.size, len(modes))
    if evaluator is None and any(modes[i].unique_eigenfunction for i in range(n)):
        evaluator = ErrorEvaluator(system)
    n, uniq, C = _aligned_batch(lams, vectors, modes, system, evaluator) if evaluator else (n, [], None)
    Ch = C.cpu().numpy() if C is not None else None
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
    :332-338); every EFL of the solve in one batched device evaluation."""
    lams = np.asarray(result_eigenvalues, dtype=np.float64)
    modes = exact_spectrum(system.dim, count=lams.size)
    ev = ErrorEvaluator(system)
    n, uniq, C = _aligned_batch(lams, result_vectors, modes, system, ev)
    efl = {}
    if uniq:
        diff = ev._contract_b(ev._embed_b(C), ev._bval) - ev._exact_b([modes[i] for i in uniq])
        vals = ev._integrate_b(diff * diff).cpu().numpy()
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
