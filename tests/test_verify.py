"""verify: exact spectra and EV/EFL/EFE against the
reference's own error_table records (tests/golden/verify_golden.json, made
by tests/golden/make_verify_golden.py from rigaeig v0.1.0).  The CPU tests
run the same batched contractions on the host; the GPU test runs them on the
device with the engine's mass products."""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg

from oracle import rigaeig_port as O
from paper_2009_08167_b200 import verify as V
from paper_2009_08167_b200.assembly import DiscreteSystem, SymSparseMatrix
from paper_2009_08167_b200.bspline import make_spline_space

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "verify_golden.json")))


def host_system(d, ne, p, lv):
    """The reference pencil (oracle port, bit-identical K, M) with this
    package's spline spaces, no device."""
    so = O.build_system(d, ne, p, lv)
    spaces = tuple(make_spline_space(ne, p, lv) for _ in range(d))
    return DiscreteSystem(SymSparseMatrix(so.K), SymSparseMatrix(so.M), spaces, d, so.K.shape[0], (), (), None)


def inputs(s):
    return scipy.linalg.eigh(s.K.csr.toarray(), s.M.csr.toarray(), driver="gvd")


def check(records, case):
    ref = case["records"]
    assert len(records) == len(ref)
    for r, g in zip(records, ref):
        assert r.position == g["position"] and list(r.indices) == g["indices"] and r.diagonal == g["diagonal"]
        assert math.isclose(r.ev, g["ev"], rel_tol=1e-9, abs_tol=1e-14)
        if g["efl"] is None:
            assert math.isnan(r.efl) and math.isnan(r.efe)
        else:
            assert math.isclose(r.efl, g["efl"], rel_tol=1e-8, abs_tol=1e-15)
            assert math.isclose(r.efe, r.ev + r.efl, rel_tol=1e-12)


def test_exact_spectrum_counts_clusters_and_errors():
    m = V.exact_spectrum(2, count=6)
    assert [x.indices for x in m] == [(1, 1), (1, 2), (2, 1), (2, 2), (1, 3), (3, 1)]
    assert m[1].cluster_size == 2 and m[0].unique_eigenfunction and not m[1].unique_eigenfunction
    assert math.isclose(m[0].lam, 2 * math.pi ** 2)
    inter = V.exact_spectrum(3, interval=(0.0, 3 * math.pi ** 2 + 1e-9))
    assert [x.indices for x in inter] == [(1, 1, 1)]
    with pytest.raises(ValueError):
        V.exact_spectrum(4, count=3)
    with pytest.raises(ValueError):
        V.exact_spectrum(2)


@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: f"d{c['d']}_ne{c['ne']}_p{c['p']}_l{c['level']}")
def test_error_table_matches_reference_host(case):
    s = host_system(case["d"], case["ne"], case["p"], case["level"])
    lam, X = inputs(s)
    n = case["count"]
    import torch

    ev = V.ErrorEvaluator(s, device="cpu")
    n_, uniq, C = V._aligned_batch(lam[:n], X[:, :n], V.exact_spectrum(s.dim, count=n), s, ev)
    recs = []
    modes = V.exact_spectrum(s.dim, count=n)
    efl = {}
    if uniq:
        diff = ev._contract_b(ev._embed_b(C), ev._bval) - ev._exact_b([modes[i] for i in uniq])
        efl = dict(zip(uniq, ev._integrate_b(diff * diff).numpy()))
    for i in range(n):
        e = (lam[i] - modes[i].lam) / modes[i].lam
        f = float(efl[i]) if i in efl else math.nan
        recs.append(V.ErrorRecord(i, modes[i].indices, e, f, e + f, modes[i].diagonal))
    check(recs, case)
    # per-mode API agrees with the batched one
    if uniq:
        i = uniq[0]
        c = C[0].numpy()
        assert math.isclose(ev.l2_error_sq(c, modes[i]), float(efl[i]), rel_tol=1e-10)
        grid = ev.uh_values(c)
        assert grid.shape == tuple(len(a) for a in reversed(ev.axes))
        assert math.isclose(ev.integrate(grid * V.exact_eigenfunction(modes[i], ev.axes)),
                            ev.inner_with_exact(c, modes[i]), rel_tol=1e-12)
        # energy seminorm: EFE identity EV + EFL vs the integrated |grad(u_h - u)|^2 / lambda
        lam_ex = modes[i].lam
        assert math.isclose(ev.energy_error_sq(c, modes[i]) / lam_ex, (lam[i] - lam_ex) / lam_ex + float(efl[i]),
                            rel_tol=1e-3)
    assert torch is not None


def test_evaluate_eigenfunction_points():
    s = host_system(2, 8, 2, 0)
    lam, X = inputs(s)
    c = X[:, 0]
    pts = np.array([[0.3, 0.7], [0.5, 0.5], [0.0, 0.2]])
    vals = V.evaluate_eigenfunction(s, c, pts)
    ev = V.ErrorEvaluator(s, device="cpu")
    # at the quadrature points the point evaluation equals the tensor contraction
    g = ev.uh_values(c)
    q = (ev.axes[0][3], ev.axes[1][5])
    assert math.isclose(V.evaluate_eigenfunction(s, c, np.array([q]))[0], g[5, 3], rel_tol=1e-12)
    assert vals[2] == 0.0 or abs(vals[2]) < 1e-14  # boundary: zero
    with pytest.raises(ValueError):
        V.evaluate_eigenfunction(s, c, np.zeros((2, 3)))


@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: f"d{c['d']}_ne{c['ne']}_p{c['p']}_l{c['level']}")
def test_error_table_matches_reference_device(case):
    import paper_2009_08167_b200 as P

    s = P.build_system(case["d"], case["ne"], case["p"], case["level"])
    lam, X = scipy.linalg.eigh(s.K.toarray(), s.M.toarray(), driver="gvd")
    n = case["count"]
    check(V.error_table(lam[:n], X[:, :n], s), case)
