"""CPU-only checks: the C-ABI library loads and exports every declared
symbol, the host-side pieces of the product (B-splines, 1D assembly,
ordering, C++ symbolic analysis, LPT assignment) agree with the golden
fixtures / the oracle.  No compute call needs a GPU here."""
import hashlib
import os
import re

import numpy as np
import pytest

from conftest import ROOT

import paper_2009_08167_b200 as P
from paper_2009_08167_b200 import _lib
from paper_2009_08167_b200.slicing import lpt_assign


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "riga_b200.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(riga_\w+)\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    names = header_symbols()
    assert len(names) >= 40
    for name in names:
        assert hasattr(L, name), name
    # the ctypes table binds exactly the declared API
    assert set(_lib.SIGNATURES) | {"riga_last_error"} == set(names)


def test_no_device_fails_loudly():
    import ctypes

    if _lib.device_count() > 0:
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    st = _lib.lib().riga_ctx_create(0, None, ctypes.byref(h))
    assert st == _lib.NO_DEVICE
    assert "no CPU fallback" in _lib.last_error()


class _HostSystem:
    """Just what the ordering needs (spaces, dim, dof_count)."""

    def __init__(self, d, ne, p, lv):
        self.spaces = (P.make_spline_space(ne, p, lv),) * d
        self.dim = d
        n1 = self.spaces[0].basis_count - 2
        self.dof_count = n1**d


SMALL = [(1, 16, 2, 0), (1, 32, 3, 1), (2, 8, 2, 0), (2, 8, 3, 1), (3, 4, 2, 1), (2, 16, 2, 0)]


@pytest.mark.parametrize("d,ne,p,lv", SMALL)
def test_ordering_matches_reference(golden_arrays, d, ne, p, lv):
    perm = P.separator_ordering(_HostSystem(d, ne, p, lv))
    np.testing.assert_array_equal(perm, golden_arrays[f"s{d}_{ne}_{p}_{lv}/perm"])


@pytest.mark.parametrize("name", ["cfg1", "cfg2_riga", "cfg2_iga", "cfg3_riga", "cfg4_riga", "cfg4_iga"])
def test_ordering_matches_reference_configs(golden, name):
    c = golden["configs"][name]
    perm = P.separator_ordering(_HostSystem(c["d"], c["ne"], c["p"], c["level"]))
    assert sha(perm.astype(np.int64)) == golden["systems"][name]["perm"]


@pytest.mark.parametrize("ne,p,lv", [(16, 2, 0), (32, 3, 1), (8, 2, 0), (64, 3, 3), (256, 4, 4)])
def test_1d_tables_bit_identical(ne, p, lv):
    from oracle import rigaeig_port as O

    sp1 = P.make_spline_space(ne, p, lv)
    K1, M1 = P.apply_dirichlet(*P.assemble_1d(sp1))
    Ko, Mo = O.dirichlet_1d(*O.matrices_1d(O.make_space(ne, p, lv)))
    np.testing.assert_array_equal(K1.csr.data, Ko.data)
    np.testing.assert_array_equal(M1.csr.data, Mo.data)
    np.testing.assert_array_equal(K1.csr.indices, Ko.indices)


def test_1d_reference_systems_bit_identical(golden):
    for key in ("s1_16_2_0", "s1_32_3_1"):
        _, ne, p, lv = map(int, key[1:].split("_"))
        K1, M1 = P.apply_dirichlet(*P.assemble_1d(P.make_spline_space(ne, p, lv)))
        assert sha(K1.csr.data) == golden["systems"][key]["K_data"]
        assert sha(M1.csr.data) == golden["systems"][key]["M_data"]


def test_bspline_api_errors():
    with pytest.raises(ValueError):
        P.make_spline_space(12, 2, 1)  # not a power of two
    with pytest.raises(ValueError):
        P.eval_basis(P.make_spline_space(4, 2), 1.5)
    sp1 = P.make_spline_space(8, 3, 3)
    assert P.separator_basis_indices(sp1).size == 7
    b = P.eval_basis(sp1, 0.3)
    assert abs(b.values.sum() - 1.0) < 1e-14


@pytest.mark.parametrize("name", ["cfg1", "cfg2_riga", "cfg2_iga", "cfg3_riga", "cfg4_riga", "cfg4_iga"])
def test_symbolic_counts_match_reference(golden, name):
    """Engine host symbolic: exact fill_nnz / factor_flops of the reference."""
    from oracle import rigaeig_port as O

    c = golden["configs"][name]
    g = golden["systems"][name]
    s = O.build_system(c["d"], c["ne"], c["p"], c["level"], stiffness_only=True)
    perm = P.separator_ordering(_HostSystem(c["d"], c["ne"], c["p"], c["level"]))
    sym = P.sparsela.Symbolic.host_only(s.K, perm)
    fill = g["fill_nnz"] if "fill_nnz" in g else g["factors"][0]["fill_nnz"]
    flops = g["factor_flops"] if "factor_flops" in g else g["factors"][0]["factor_flops"]
    assert sym.stats["fill_nnz"] == fill
    assert sym.stats["factor_flops"] == flops
    # the postordered elimination order is a permutation with the same counts
    order = sym.order
    assert np.array_equal(np.sort(order), np.arange(s.dof_count))
    assert sym.stats["stored_L_entries"] >= fill - s.dof_count


def test_symbolic_colcounts_equal_oracle():
    from oracle import rigaeig_port as O

    s = O.build_system(2, 16, 3, 1)
    perm = O.separator_ordering(s)
    Ap, Ai, _ = O.permuted_upper_csc(s.K, perm)
    _, lnz = O.symbolic(s.dof_count, Ap, Ai)
    sym = P.sparsela.Symbolic.host_only(s.K, perm)
    np.testing.assert_array_equal(sym.colcounts(), lnz + 1)


def test_symbolic_parallel_sweeps_match_one_thread():
    """The host analysis's threaded sweeps (column counts, front structures, scatter map) give the same
    supernodes, structures and counts as one thread (RIGA_SYM_THREADS=1 in a child process)."""
    import json
    import os
    import subprocess
    import sys

    from oracle import rigaeig_port as O

    code = r"""
import json, sys
sys.path.insert(0, %r)
import numpy as np
import paper_2009_08167_b200 as P
from oracle import rigaeig_port as O
s = O.build_system(2, 64, 3, 2)
perm = O.separator_ordering(s)
sym = P.sparsela.Symbolic.host_only(s.K, perm)
sn = sym.supernodes()
print(json.dumps({"stats": {k: int(v) for k, v in sym.stats.items()}, "order": sym.order.tolist(),
                  "cc": sym.colcounts().tolist(), "sn": {k: v.tolist() for k, v in sn.items()}}))
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for threads in ("1", "8"):
        env = dict(os.environ, RIGA_SYM_THREADS=threads)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert len(outs[0]["order"]) >= 4096  # large enough for the threaded paths
    assert outs[0] == outs[1]


def test_lpt_assignment():
    counts = [115, 125, 123, 125, 124, 126, 123, 126, 130, 127, 121, 128, 125, 125, 129, 128]
    for world in (1, 2, 4, 8):
        a = lpt_assign(counts, world)
        assert sorted(sum(a, [])) == list(range(16))
        loads = [sum(counts[k] for k in r) for r in a]
        assert max(loads) - min(loads) <= max(counts)
    assert lpt_assign([96, 17, 31], 2) == [[0], [1, 2]]


def test_quadrature_tables_reproduce_kronecker_pencil():
    """Host side of the device element-quadrature assembly: integrating the 2D elements with the tensor
    Gauss rule from quadrature_tables (numpy restatement of the device kernel's sums) reproduces the
    Kronecker-composed K and M to roundoff (ref assembly.py:72-111, :162-177)."""
    import scipy.sparse as sp

    from paper_2009_08167_b200.assembly import apply_dirichlet, assemble_1d, quadrature_tables
    from paper_2009_08167_b200.bspline import make_spline_space

    ne, p, lv = 8, 3, 1
    s = make_spline_space(ne, p, lv)
    K1, M1 = apply_dirichlet(*assemble_1d(s))
    n1 = K1.dimension
    Kk = sp.kron(M1.csr, K1.csr) + sp.kron(K1.csr, M1.csr)
    Mk = sp.kron(M1.csr, M1.csr)
    first, w, N, dN = quadrature_tables(s)
    n = n1 * n1
    Kq = np.zeros((n, n))
    Mq = np.zeros((n, n))
    for ey in range(first.size):
        for ex in range(first.size):
            W = np.outer(w[ey], w[ex]).ravel()  # q = (qy, qx), x fastest
            v = np.einsum("ya,xb->yxab", N[ey], N[ex]).reshape(-1, (p + 1) ** 2)
            gx = np.einsum("ya,xb->yxab", N[ey], dN[ex]).reshape(-1, (p + 1) ** 2)
            gy = np.einsum("ya,xb->yxab", dN[ey], N[ex]).reshape(-1, (p + 1) ** 2)
            ke = gx.T @ (W[:, None] * gx) + gy.T @ (W[:, None] * gy)
            me = v.T @ (W[:, None] * v)
            iy = first[ey] + np.arange(p + 1) - 1
            ix = first[ex] + np.arange(p + 1) - 1
            g = (iy[:, None] * n1 + ix[None, :]).ravel()
            ok = ((iy[:, None] >= 0) & (iy[:, None] < n1) & (ix[None, :] >= 0) & (ix[None, :] < n1)).ravel()
            sel = np.flatnonzero(ok)
            Kq[np.ix_(g[sel], g[sel])] += ke[np.ix_(sel, sel)]
            Mq[np.ix_(g[sel], g[sel])] += me[np.ix_(sel, sel)]
    assert np.abs(Kq - Kk.toarray()).max() <= 1e-13 * np.abs(Kk.toarray()).max()
    assert np.abs(Mq - Mk.toarray()).max() <= 1e-13 * np.abs(Mk.toarray()).max()
    assert np.array_equal(Kq != 0, Kk.toarray() != 0)
