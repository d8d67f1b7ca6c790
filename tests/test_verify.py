"""verify: exact spectra and EV/EFL/EFE against the
reference's own error_table records (tests/golden/verify_golden.json, made
by tests/golden/make_verify_golden.py from rigaeig v0.1.0).  The CPU tests
pin the numpy restatement (oracle/verify_port.py) to those records and cover
the host-side pieces; the GPU tests run the product path -- engine kernels
for the tensor-product contractions, quadrature sums and mass products --
against the records and against the restatement."""
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
def test_oracle_error_table_pinned_to_reference(case):
    """The numpy restatement (oracle/verify_port.py) against the reference's own records."""
    from oracle import verify_port as VP

    so = O.build_system(case["d"], case["ne"], case["p"], case["level"])
    lam, X = scipy.linalg.eigh(so.K.toarray(), so.M.toarray(), driver="gvd")
    n = case["count"]
    recs = [V.ErrorRecord(i, ix, e, math.nan if f is None else f, math.nan if f is None else e + f,
                          len(set(ix)) == 1)
            for i, ix, e, f in VP.error_table(lam[:n], X[:, :n], so)]
    check(recs, case)


def test_evaluator_has_no_host_path():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        V.ErrorEvaluator(host_system(2, 8, 2, 0))


def test_evaluate_eigenfunction_points():
    s = host_system(2, 8, 2, 0)
    lam, X = inputs(s)
    c = X[:, 0]
    pts = np.array([[0.3, 0.7], [0.5, 0.5], [0.0, 0.2]])
    vals = V.evaluate_eigenfunction(s, c, pts)
    # at a quadrature point the point evaluation equals the oracle's tensor contraction
    from oracle import verify_port as VP

    so = O.build_system(2, 8, 2, 0)
    ev = VP.Evaluator(so)
    g = ev.values(c)
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


@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD["cases"][:3], ids=lambda c: f"d{c['d']}_ne{c['ne']}_p{c['p']}_l{c['level']}")
def test_engine_evaluator_matches_oracle_per_mode(case):
    """Per-mode API through the engine kernels (riga_tp_contract / riga_tp_reduce) against the numpy
    restatement: grid values, derivative grids, quadrature, L2 / energy errors, inner products."""
    import paper_2009_08167_b200 as P
    from oracle import verify_port as VP

    s = P.build_system(case["d"], case["ne"], case["p"], case["level"])
    so = O.build_system(case["d"], case["ne"], case["p"], case["level"])
    lam, X = scipy.linalg.eigh(so.K.toarray(), so.M.toarray(), driver="gvd")
    modes = V.exact_spectrum(s.dim, count=case["count"])
    i = next(k for k, m in enumerate(modes) if m.unique_eigenfunction)
    c = X[:, i] / math.sqrt(X[:, i] @ (so.M @ X[:, i]))
    ev, ov = V.ErrorEvaluator(s), VP.Evaluator(so)
    G = ev.uh_values(c)
    Go = ov.values(c)
    assert G.shape == Go.shape == tuple(len(a) for a in reversed(ev.axes))
    assert np.allclose(G, Go, rtol=1e-12, atol=1e-14)
    E = ov.exact(modes[i].indices)
    assert math.isclose(ev.integrate(G * E), ov.integrate(Go * E), rel_tol=1e-11)
    assert math.isclose(ev.inner_with_exact(c, modes[i]), ov.integrate(Go * E), rel_tol=1e-11)
    sg = 1.0 if ov.integrate(Go * E) >= 0 else -1.0
    assert math.isclose(ev.l2_error_sq(sg * c, modes[i]), ov.integrate((sg * Go - E) ** 2), rel_tol=1e-8, abs_tol=1e-18)
    # derivative grids: finite-difference check of the contraction along each direction is overkill here;
    # the EFE identity EV + EFL = |grad(u_h - u)|^2 / lambda ties them to the eigenvalue error instead
    lam_ex = modes[i].lam
    assert math.isclose(ev.energy_error_sq(sg * c, modes[i]) / lam_ex,
                        (lam[i] - lam_ex) / lam_ex + ev.l2_error_sq(sg * c, modes[i]), rel_tol=1e-3)
    with pytest.raises(ValueError):
        ev.uh_values(c[:-1])
    al = V.match_and_normalize(lam[:case["count"]], X[:, :case["count"]], modes, s, ev)
    a = al[i]
    assert a.coeffs is not None and math.isclose(abs(a.coeffs @ (so.M @ a.coeffs)), 1.0, rel_tol=1e-12)
    assert ev.inner_with_exact(a.coeffs, modes[i]) >= 0
    rec = V.error_metrics(a, s, ev)
    assert math.isclose(rec.efl, ev.l2_error_sq(a.coeffs, modes[i]), rel_tol=1e-12)
