"""CPU restatement of the reference's eigen-error evaluation (TEST INFRASTRUCTURE).

Restates rigaeig v0.1.0 ``verify.py`` with numpy, one mode at a time as the
reference does: ErrorEvaluator tables (ref verify.py:181-216), tensor-product
contraction (:218-225), quadrature (:227-231), the exact modes (:105-133),
match_and_normalize (:279-313) and error_table (:332-338).  Only ``tests/``
imports this module; the product path (paper_2009_08167_b200/verify.py) runs
engine kernels on the device and never imports it.

Pinned: tests/test_verify.py checks it against tests/golden/verify_golden.json,
records produced by the reference itself (tests/golden/make_verify_golden.py).
"""
from __future__ import annotations

import itertools
import math

import numpy as np

from . import rigaeig_port as O

PI2 = math.pi * math.pi


def exact_modes(d: int, count: int):
    """(lambda, indices, unique_eigenfunction) ascending, ties lexicographic (ref :54-102)."""
    kmax = max(2, int(round(count ** (1.0 / d))) + 2)
    while True:
        cut = PI2 * ((kmax + 1) ** 2 + (d - 1))
        cand = [(PI2 * sum(i * i for i in ix), ix) for ix in itertools.product(range(1, kmax + 1), repeat=d)]
        cand = [c for c in cand if c[0] < cut]
        if len(cand) >= count:
            cand = sorted(cand)[:count]
            break
        kmax *= 2
    out, i = [], 0
    while i < len(cand):
        j = i + 1
        while j < len(cand) and abs(cand[j][0] - cand[i][0]) < 1e-9 * cand[i][0]:
            j += 1
        for lam, ix in cand[i:j]:
            out.append((lam, ix, len(set(ix)) == 1 and j - i == 1))
        i = j
    return out


def gauss(n: int, a: float, b: float):
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (b - a) * x + 0.5 * (a + b), 0.5 * (b - a) * w


class Evaluator:
    """Dense collocation matrices per direction, degree + 2 Gauss points per element (ref :181-216)."""

    def __init__(self, system: O.System):
        self.system = system
        self.axes, self.weights, self.bval = [], [], []
        for space in system.spaces:
            nq = space.degree + 2
            pts, wts = [], []
            for _, a, b in O.spans(space):
                x, w = gauss(nq, a, b)
                pts.append(x)
                wts.append(w)
            pts = np.concatenate(pts)
            bv = np.zeros((pts.size, space.basis_count))
            for r, x in enumerate(pts):
                first, vals, _ = O.basis_at(space, float(x))
                bv[r, first:first + len(vals)] = vals
            self.axes.append(pts)
            self.weights.append(np.concatenate(wts))
            self.bval.append(bv)

    def embed(self, c):
        red = [s.basis_count - 2 for s in reversed(self.system.spaces)]
        full = [s.basis_count for s in reversed(self.system.spaces)]
        U = np.zeros(full)
        U[tuple(slice(1, n - 1) for n in full)] = np.asarray(c).reshape(red)
        return U

    def values(self, c):
        out = self.embed(c)
        d = len(self.bval)
        for t in range(d):  # x is the last axis (ref :218-225)
            ax = out.ndim - 1 - t
            out = np.moveaxis(np.moveaxis(out, ax, -1) @ self.bval[t].T, -1, ax)
        return out

    def integrate(self, G):
        out = G
        for t in range(len(self.weights)):
            out = out @ self.weights[t]
        return float(out)

    def exact(self, ix):
        out = np.ones(())
        for k, ax in reversed(list(zip(ix, self.axes))):
            out = np.multiply.outer(out, math.sqrt(2.0) * np.sin(k * math.pi * ax))
        return out


def error_table(lams, vectors, system: O.System):
    """[(position, indices, ev, efl or None)] (ref :279-338)."""
    lams = np.asarray(lams, dtype=np.float64)
    modes = exact_modes(system.dim, lams.size)
    ev = Evaluator(system)
    out = []
    for i, (lam, ix, uniq) in enumerate(modes):
        e = (float(lams[i]) - lam) / lam
        efl = None
        if uniq:
            c = np.asarray(vectors[:, i], dtype=np.float64)
            nrm = math.sqrt(max(float(c @ (system.M @ c)), 0.0))
            c = c / nrm if nrm > 0 else c
            G, E = ev.values(c), ev.exact(ix)
            if ev.integrate(G * E) < 0:
                G = -G
            efl = ev.integrate((G - E) ** 2)
        out.append((i, ix, e, efl))
    return out
