"""Pin the CPU oracle (oracle/rigaeig_port.py + oracle/ldl_oracle.c) to the
reference's own outputs, recorded by tests/golden/make_golden.py which
imported the reference package itself.  CPU only."""
import hashlib

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import rigaeig_port as O


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


SMALL = [(1, 16, 2, 0), (1, 32, 3, 1), (2, 8, 2, 0), (2, 8, 3, 1), (3, 4, 2, 1), (2, 16, 2, 0)]


@pytest.mark.parametrize("d,ne,p,lv", SMALL)
def test_small_systems_bit_identical(golden, golden_arrays, d, ne, p, lv):
    key = f"s{d}_{ne}_{p}_{lv}"
    g = golden["systems"][key]
    s = O.build_system(d, ne, p, lv)
    assert s.dof_count == g["N"] and s.K.nnz == g["nnz"]
    assert sha(s.K.data) == g["K_data"] and sha(s.M.data) == g["M_data"]
    assert sha(s.K.indptr.astype(np.int64)) == g["indptr"]
    assert sha(s.K.indices.astype(np.int32)) == g["indices"]
    perm = O.separator_ordering(s)
    np.testing.assert_array_equal(perm, golden_arrays[f"{key}/perm"])
    for j, fr in enumerate(g["factors"]):
        f = O.factor_ldl(s.K - fr["sigma"] * s.M, ordering=perm)
        assert list(f.inertia) == fr["inertia"]
        assert f.fill_nnz == fr["fill_nnz"] and f.factor_flops == fr["factor_flops"]
        # same operation order as the reference's numba kernel: bitwise D
        np.testing.assert_array_equal(f.D, golden_arrays[f"{key}/D{j}"])
        x = O.solve_fb(f, golden_arrays[f"{key}/b{j}"])
        np.testing.assert_array_equal(x, golden_arrays[f"{key}/x{j}"])


@pytest.mark.parametrize("name", ["cfg1", "cfg2_riga", "cfg2_iga"])
def test_config_structure_and_inertia(golden, name):
    g = golden["systems"][name]
    c = golden["configs"][name]
    s = O.build_system(c["d"], c["ne"], c["p"], c["level"])
    assert s.dof_count == g["N"] and s.K.nnz == g["nnz"]
    assert sha(s.K.data) == g["K_data"] and sha(s.M.data) == g["M_data"]
    perm = O.separator_ordering(s)
    assert sha(perm.astype(np.int64)) == g["perm"]
    for fr in g["factors"]:
        f = O.factor_ldl(s.K - fr["sigma"] * s.M, ordering=perm)
        assert list(f.inertia) == fr["inertia"]
        assert f.fill_nnz == fr["fill_nnz"] and f.factor_flops == fr["factor_flops"]
        assert sha(f.D) == fr["D"]


@pytest.mark.parametrize("name", ["cfg1", "cfg2_riga"])
def test_oracle_slices_match_reference(golden, golden_arrays, name):
    c = golden["configs"][name]
    s = O.build_system(c["d"], c["ne"], c["p"], c["level"])
    for k in range(c["S"]):
        g = golden["slices"][f"{name}/{k}"]
        res = O.solve_slice(s, (c["shifts"][k], c["shifts"][k + 1]), seed=k, m=g["m"])
        assert res.expected_count == g["expected"] == res.eigenvalues.size
        np.testing.assert_allclose(res.eigenvalues, golden_arrays[f"{name}/slice{k}/eig"], rtol=1e-12)
        assert res.counters.nfb == g["nfb"] and res.counters.nmv == g["nmv"]


def test_kronecker_spectrum_and_lambda_e(golden, golden_arrays):
    for name in ("cfg1", "cfg2_riga", "cfg2_iga", "cfg4_riga"):
        c = golden["configs"][name]
        lam = O.kronecker_spectrum(c["d"], c["ne"], c["p"], c["level"])
        le, cnt = O.lambda_e_for(lam, c["N0"])
        assert cnt == c["count"]
        assert le == pytest.approx(c["lambda_e"], rel=1e-14)
        np.testing.assert_allclose(lam[: cnt + 8], golden_arrays[f"{name}/lam_first"], rtol=1e-13)
        nu = [int(np.sum(lam < sg)) for sg in c["shifts"]]
        assert nu == c["nu"]


def test_kronecker_counts_equal_oracle_inertia_cfg2(golden):
    c = golden["configs"]["cfg2_riga"]
    s = O.build_system(c["d"], c["ne"], c["p"], c["level"])
    perm = O.separator_ordering(s)
    for sg, nu in zip(c["shifts"], c["nu"]):
        assert O.factor_ldl(s.K - sg * s.M, ordering=perm).n_negative == nu


def test_known_answers():
    # single-DOF 2D system: K = 8/3, M = 1/9, lambda = 24 (ref tests/test_assembly.py:53-61)
    s = O.build_system(2, 2, 1)
    assert s.dof_count == 1
    assert s.K.toarray()[0, 0] == pytest.approx(8 / 3)
    assert s.M.toarray()[0, 0] == pytest.approx(1 / 9)
    # diagonal inertia, zero pivot (ref tests/test_sparsela.py:46-81)
    f = O.factor_ldl(sp.csr_array(sp.diags_array([2.0, -3.0, 5.0])), ordering="natural")
    assert f.inertia == (1, 0, 2)
    with pytest.raises(O.ZeroPivot):
        O.factor_ldl(sp.csr_array(sp.diags_array([1.0, 1e-20, 3.0])), ordering="natural")
    with pytest.raises(ValueError):
        O.factor_ldl(sp.csr_array(sp.eye_array(3)), ordering="bogus")
