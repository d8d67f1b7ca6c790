"""GPU parity: assembly, SpMV, LDL^T inertia / reconstruction / solves through
the drop-in API, against the oracle and the reference's golden fixtures.
Mirrors the reference's tests/test_sparsela.py cases."""
import hashlib

import numpy as np
import pytest
import scipy.linalg
import scipy.sparse as sp

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2009_08167_b200")
from paper_2009_08167_b200.sparsela import Symbolic, numeric_factor  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def dense_eig(system):
    return scipy.linalg.eigh(system.K.toarray(), system.M.toarray(), eigvals_only=True, driver="gvd")


def random_spd(n, seed, density=0.2):
    rng = np.random.default_rng(seed)
    A = sp.random_array((n, n), density=density, rng=rng)
    A = A + A.T + sp.diags_array(np.full(n, n * 1.0))
    return sp.csr_array(A)


@pytest.mark.parametrize("name", ["cfg1", "cfg2_riga", "cfg2_iga", "cfg3_riga", "cfg4_riga", "cfg4_iga"])
def test_device_assembly_bit_identical(golden, name):
    c = golden["configs"][name]
    g = golden["systems"][name]
    s = P.build_system(c["d"], c["ne"], c["p"], c["level"])
    assert s.dof_count == g["N"] and s.K.nnz == g["nnz"]
    assert sha(s.K.csr.data) == g["K_data"]
    assert sha(s.M.csr.data) == g["M_data"]


@pytest.mark.parametrize("name", ["cfg1", "cfg2_riga", "cfg2_iga", "cfg3_riga", "cfg4_riga", "cfg4_iga", "cfg5_riga"])
def test_device_separator_ordering_equals_reference(golden, name):
    """separator_ordering (ref sparsela.py:319-392) with the permutation written by the device kernel
    (riga_separator_emit over the engine's dissection blocks): identical to the reference's ordering, and
    to the host emission of the same blocks."""
    import types

    c = golden["configs"][name]
    s = P.build_system(c["d"], c["ne"], c["p"], c["level"])
    assert s.device is not None
    perm = P.separator_ordering(s)
    assert perm.dtype == np.int64 and perm.shape == (s.dof_count,)
    assert sha(perm) == golden["systems"][name]["perm"]
    host = types.SimpleNamespace(spaces=s.spaces, dim=s.dim, dof_count=s.dof_count, device=None)
    assert np.array_equal(P.separator_ordering(host), perm)


@pytest.mark.parametrize("d,ne,p,lv", [(1, 16, 2, 0), (1, 32, 3, 1), (2, 8, 2, 0), (2, 8, 3, 1), (3, 4, 2, 1), (2, 16, 2, 0)])
def test_device_separator_ordering_small_systems(golden_arrays, d, ne, p, lv):
    """Device-written permutation on the small systems of the CPU test (1D, 2D and 3D, with and without C0
    lines): equal to the reference's recorded ordering."""
    s = P.build_system(d, ne, p, lv)
    assert s.device is not None
    np.testing.assert_array_equal(P.separator_ordering(s), golden_arrays[f"s{d}_{ne}_{p}_{lv}/perm"])


@pytest.mark.parametrize("cfg", [(2, 16, 2, 0), (2, 64, 3, 3), (3, 8, 2, 1), (2, 256, 4, 4), (3, 32, 2, 2)])
def test_device_scatter_map_equals_host_analysis(cfg):
    """The scatter map of the original entries into the fronts (symbolic.cpp 5d on the host) is built by device
    kernels in a device analysis (factor.cu build_asm_map_device: count / scan / fill, one warp per elimination
    column): identical arrays to the host-only analysis of the same pattern and ordering."""
    import ctypes

    from paper_2009_08167_b200 import _lib

    s = P.build_system(*cfg)
    perm = np.ascontiguousarray(P.separator_ordering(s), dtype=np.int64)
    dev = Symbolic.on_device(s.device, perm)
    A = s.K.csr
    rp = np.ascontiguousarray(A.indptr, dtype=np.int64)
    ci = np.ascontiguousarray(A.indices, dtype=np.int32)
    L = _lib.lib()
    hh = ctypes.c_void_p()
    _lib.check(L.riga_symbolic_analyze(A.shape[0], _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(perm), ctypes.byref(hh)))
    try:
        out = []
        for handle in (dev.handle, hh):
            cnt = ctypes.c_int64()
            _lib.check(L.riga_symbolic_asm_map(handle, ctypes.byref(cnt), None, None, None))
            st = np.zeros(16, dtype=np.int64)
            _lib.check(L.riga_symbolic_stats(handle, _lib.ptr(st)))
            ptr = np.zeros(st[2] + 1, dtype=np.int64)
            slot = np.zeros(cnt.value, dtype=np.int32)
            loc = np.zeros(cnt.value, dtype=np.int32)
            _lib.check(L.riga_symbolic_asm_map(handle, ctypes.byref(cnt), _lib.ptr(ptr), _lib.ptr(slot), _lib.ptr(loc)))
            out.append((cnt.value, ptr, slot, loc))
        assert out[0][0] == out[1][0] == (A.nnz + A.shape[0]) // 2
        for a, b in zip(out[0][1:], out[1][1:]):
            assert np.array_equal(a, b)
    finally:
        L.riga_symbolic_destroy(hh)


@pytest.mark.parametrize("d,ne,p,lv", [(1, 16, 2, 0), (2, 8, 3, 1), (3, 4, 2, 1), (2, 16, 2, 0)])
def test_small_assembly_bit_identical(golden, d, ne, p, lv):
    g = golden["systems"][f"s{d}_{ne}_{p}_{lv}"]
    s = P.build_system(d, ne, p, lv)
    assert sha(s.K.csr.data) == g["K_data"] and sha(s.M.csr.data) == g["M_data"]
    assert sha(s.K.csr.indptr.astype(np.int64)) == g["indptr"]
    assert sha(s.K.csr.indices.astype(np.int32)) == g["indices"]


def test_spmv_matches_scipy():
    s = P.build_system(2, 64, 3, 3)
    rng = np.random.default_rng(3)
    for _ in range(3):
        v = rng.standard_normal(s.dof_count)
        y = P.mass_matvec(s.M, v)
        ref = s.M.csr @ v
        np.testing.assert_allclose(y, ref, rtol=1e-13, atol=1e-15 * np.abs(ref).max())
        yk = P.mass_matvec(s.K, v)
        np.testing.assert_allclose(yk, s.K.csr @ v, rtol=1e-12, atol=1e-13 * np.abs(yk).max())


def test_mass_matvec_values_and_counters():
    c = P.CostCounters()
    I3 = sp.csr_array(sp.eye_array(3))
    v = np.array([1.0, 2.0, 3.0])
    np.testing.assert_array_equal(P.mass_matvec(I3, v, c), v)
    assert c.nmv == 1 and c.matvec.flops == 2 * 3
    M = P.build_system(1, 16, 3).M
    rng = np.random.default_rng(1)
    for _ in range(5):
        w = rng.standard_normal(M.dimension)
        assert w @ P.mass_matvec(M, w) > 0
    with pytest.raises(ValueError):
        P.mass_matvec(M, np.ones(M.dimension + 1))


@pytest.mark.parametrize("name", ["cfg1", "cfg2_riga", "cfg2_iga", "cfg3_riga", "cfg4_riga"])
def test_inertia_bit_exact_at_every_uniform_shift(golden, name):
    c = golden["configs"][name]
    s = P.build_system(c["d"], c["ne"], c["p"], c["level"])
    sym = Symbolic.on_device(s.device, P.separator_ordering(s))
    assert sym.stats["fill_nnz"] == (golden["systems"][name].get("fill_nnz")
                                     or golden["systems"][name]["factors"][0]["fill_nnz"])
    for sigma, nu in zip(c["shifts"], c["nu"]):
        f = numeric_factor(sym, sigma)
        assert f.n_negative == nu, (sigma, f.n_negative, nu)


def test_factor_diagonal_inertia_and_zero_pivot():
    A = sp.csr_array(sp.diags_array([2.0, -3.0, 5.0]))
    assert P.factor_ldl(A, ordering="natural").inertia == (1, 0, 2)
    with pytest.raises(P.ZeroPivot):
        P.factor_ldl(sp.csr_array(sp.diags_array([1.0, 1e-20, 3.0])), ordering="natural")
    with pytest.raises(ValueError):
        P.factor_ldl(A, ordering="bogus")
    with pytest.raises(ValueError):
        P.factor_ldl(A, ordering=np.arange(2))


def test_factor_stiffness_positive_definite():
    s = P.build_system(1, 16, 2)
    f = P.factor_ldl(s.K, ordering=P.separator_ordering(s))
    assert f.inertia == (0, 0, s.dof_count)


def test_inertia_between_third_and_fourth():
    s = P.build_system(1, 16, 2)
    lam = dense_eig(s)
    sigma = 0.5 * (lam[2] + lam[3])
    f = P.factor_ldl(s.K.csr - sigma * s.M.csr, ordering="nd")
    assert f.n_negative == 3


@pytest.mark.parametrize("d,ne,p,lv", [(1, 16, 3, 0), (1, 32, 2, 2), (2, 8, 2, 0), (2, 8, 3, 1)])
def test_inertia_matches_dense_count(d, ne, p, lv):
    s = P.build_system(d, ne, p, lv)
    lam = dense_eig(s)
    perm = P.separator_ordering(s)
    rng = np.random.default_rng(5)
    for sigma in rng.uniform(lam[0] * 0.5, lam[-1] * 1.05, size=10):
        f = P.factor_ldl(s.K.csr - sigma * s.M.csr, ordering=perm)
        assert f.n_negative == int(np.sum(lam < sigma)), sigma


@pytest.mark.parametrize("args", [(2, 8, 3, 1), (3, 8, 2, 1), (2, 64, 3, 3), (3, 16, 2, 1)])
def test_reconstruction_residual(args):
    s = P.build_system(*args)
    A = s.K.csr - 37.5 * s.M.csr
    f = P.factor_ldl(A, ordering=P.separator_ordering(s))
    L = f.l_matrix()
    rng = np.random.default_rng(0)
    n = A.shape[0]
    perm = f.permutation
    for _ in range(10):
        w = rng.standard_normal(n)
        y = L @ (f.D * (L.T @ w[perm]))
        lhs = np.empty(n)
        lhs[perm] = y
        ref = A @ w
        assert np.linalg.norm(lhs - ref) / np.linalg.norm(ref) < 1e-10


def test_d_and_inertia_agree_with_oracle(golden):
    from oracle import rigaeig_port as O

    c = golden["configs"]["cfg2_riga"]
    s = P.build_system(c["d"], c["ne"], c["p"], c["level"])
    so = O.build_system(c["d"], c["ne"], c["p"], c["level"])
    perm = P.separator_ordering(s)
    sigma = c["shifts"][1]
    f = P.factor_ldl(s.K.csr - sigma * s.M.csr, ordering=perm)
    fo = O.factor_ldl(so.K - sigma * so.M, ordering=f.permutation)  # same elimination order
    assert f.inertia == fo.inertia
    np.testing.assert_allclose(f.D, fo.D, rtol=1e-9, atol=1e-12 * np.abs(fo.D).max())


def test_solve_identity_and_bad_shape():
    f = P.factor_ldl(sp.csr_array(sp.eye_array(6)), ordering="natural")
    b = np.arange(6.0)
    np.testing.assert_allclose(P.solve_fb(f, b), b)
    with pytest.raises(ValueError):
        P.solve_fb(f, np.ones(5))


def test_solve_random_spd():
    A = random_spd(50, seed=1)
    f = P.factor_ldl(A, ordering="nd")
    b = np.random.default_rng(2).standard_normal(50)
    x = P.solve_fb(f, b)
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) < 1e-12


def test_solve_many_children_per_supernode():
    """Arrowhead pencil in natural order: the last column's supernode has dozens of children, more than
    the update-vector slots of the forward sweep (solve.cu kUpdSlots), so the overflow pull map runs."""
    n = 60
    rng = np.random.default_rng(5)
    D = np.diag(4.0 + rng.random(n))
    D[n - 1, :] = 0.1 * rng.standard_normal(n)
    D[:, n - 1] = D[n - 1, :]
    D[n - 1, n - 1] = 10.0
    A = sp.csr_array(D)
    f = P.factor_ldl(A, ordering="natural")
    b = rng.standard_normal(n)
    x = P.solve_fb(f, b)
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) < 1e-13


def test_solve_constructed_rhs():
    s = P.build_system(1, 32, 3, 1)
    A = s.K.csr
    f = P.factor_ldl(A, ordering=P.separator_ordering(s))
    ones = np.ones(A.shape[0])
    np.testing.assert_allclose(P.solve_fb(f, A @ ones), ones, atol=1e-12)


@pytest.mark.parametrize("args,sigma", [((2, 8, 2, 1), 0.0), ((2, 64, 3, 3), 1000.0), ((3, 16, 2, 1), 500.0),
                                        ((2, 256, 4, 4), 25754.73284416981), ((2, 64, 3, 3), 1431.09)])
def test_solve_roundtrip_and_oracle(args, sigma):
    """Round trip A^{-1}(A v) = v (ref tests/test_sparsela.py:124-130); near an
    eigenvalue (last case, 2.7e-6 relative) the bound is the oracle's own
    error on the same matrix, since the problem is ill-conditioned there."""
    from oracle import rigaeig_port as O

    s = P.build_system(*args)
    A = s.K.csr - sigma * s.M.csr
    f = P.factor_ldl(A, ordering=P.separator_ordering(s))
    v = np.random.default_rng(9).standard_normal(A.shape[0])
    rhs = np.asarray(A @ v)
    u = P.solve_fb(f, rhs)
    err = np.linalg.norm(u - v) / np.linalg.norm(v)
    if s.dof_count < 20000:
        fo = O.factor_ldl(A, ordering=f.permutation)
        err_o = np.linalg.norm(O.solve_fb(fo, rhs) - v) / np.linalg.norm(v)
        assert err < max(1e-10, 10 * err_o), (err, err_o)
        b = np.random.default_rng(10).standard_normal(A.shape[0])
        xo = O.solve_fb(fo, b)
        x = P.solve_fb(f, b)
        assert np.linalg.norm(x - xo) / np.linalg.norm(xo) < max(1e-9, 100 * err_o)
    else:
        assert err < 1e-10


def test_flop_counter_reproducible():
    s = P.build_system(2, 8, 2, 1)
    perm = P.separator_ordering(s)
    c1, c2 = P.CostCounters(), P.CostCounters()
    f1 = P.factor_ldl(s.K, ordering=perm, counters=c1)
    f2 = P.factor_ldl(s.K, ordering=perm, counters=c2)
    assert f1.factor_flops == f2.factor_flops and f1.fill_nnz == f2.fill_nnz
    assert c1.fact.flops == c2.fact.flops
    b = np.ones(s.dof_count)
    P.solve_fb(f1, b, c1)
    P.solve_fb(f2, b, c2)
    assert c1.fb.flops == c2.fb.flops == 2 * f1.fill_nnz
    # deterministic device arithmetic: bitwise identical D and solves
    np.testing.assert_array_equal(f1.D, f2.D)
    np.testing.assert_array_equal(P.solve_fb(f1, b), P.solve_fb(f2, b))


def test_m_inner_and_norm():
    assert P.m_norm(np.zeros(4)) == 0.0
    v = np.array([3.0, 4.0])
    assert P.m_inner(v, v) == 25.0
    M = P.build_system(1, 8, 2).M
    w = np.random.default_rng(4).standard_normal(M.dimension)
    np.testing.assert_allclose(P.m_norm(w, M) ** 2, P.m_inner(w, w, M), rtol=1e-14)
    with pytest.raises(P.NegativeNorm):
        P.m_norm(v, -sp.csr_array(sp.eye_array(2)))


@pytest.mark.parametrize("name", ["cfg4_riga", "cfg4_iga"])
def test_factor_and_solve_are_deterministic(golden, name):
    """Large 3D fronts: two factorizations at the same shift give bit-identical D, inverse/G blocks and
    solves (no FP atomics; guards against cross-CTA races in the panel steps)."""
    import torch

    c = golden["configs"][name]
    s = P.build_system(c["d"], c["ne"], c["p"], c["level"])
    sym = Symbolic.on_device(s.device, P.separator_ordering(s))
    sigma = float(c["shifts"][len(c["shifts"]) // 2])
    b = torch.randn(s.dof_count, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    outs = []
    for _ in range(2):
        f = numeric_factor(sym, sigma)
        x = f.solve_device(b)
        torch.cuda.synchronize()
        outs.append((sha(f.D), sha(x.cpu().numpy()), f.n_negative))
    assert outs[0] == outs[1]


@pytest.mark.slow
def test_cfg5_inertia_matches_kronecker_counts(golden):
    """3D 64^3 p = 3 (fronts up to 7526): inertia at several uniform shifts equals the exact count of the
    Kronecker spectrum below the shift, and solves have residual ~ machine precision."""
    import torch

    from paper_2009_08167_b200 import _lib

    c = golden["configs"]["cfg5_riga"]
    s = P.build_system(c["d"], c["ne"], c["p"], c["level"])
    lam = P.kronecker_spectrum(s)
    sym = Symbolic.on_device(s.device, P.separator_ordering(s))
    shifts = P.uniform_shifts(c["lambda_e"], c["S"])
    b = torch.randn(s.dof_count, dtype=torch.float64, device="cuda")
    r = torch.empty_like(b)
    for k in (0, 1, c["S"] // 2, c["S"]):
        f = numeric_factor(sym, float(shifts[k]))
        assert f.n_negative == int(np.sum(lam < f.sigma)), k
        x = f.solve_device(b)
        _lib.check(_lib.lib().riga_spmv(s.device.handle, 2, f.sigma, _lib.ptr(x), _lib.ptr(r)))
        assert float(torch.linalg.norm(r - b) / torch.linalg.norm(b)) < 1e-8


@pytest.mark.gpu
@pytest.mark.parametrize("name,k", [("cfg4_iga", 3), ("cfg5_riga", 31)])
def test_solve_backward_error_at_hard_shifts(golden, name, k):
    """The chain supernodes' explicit inverses lose backward stability at high indefinite shifts (cfg5 slice
    31 midpoint: 1.1e-8 with the inverse alone); the factor-time probe flags them and the solve refines them
    locally, so ||(K - sigma M) x - b|| / ||b|| stays at substitution level (< 1e-10) everywhere."""
    import torch

    from paper_2009_08167_b200 import _lib

    c = golden["configs"][name]
    s = P.build_system(c["d"], c["ne"], c["p"], c["level"])
    sh = c["shifts"]
    sigma = 0.5 * (sh[k] + sh[k + 1])
    sym = Symbolic.on_device(s.device, P.separator_ordering(s))
    f = numeric_factor(sym, sigma)
    rng = np.random.default_rng(7)
    for _ in range(3):
        b = torch.as_tensor(rng.standard_normal(s.dof_count), device="cuda")
        x = f.solve_device(b)
        r = torch.empty_like(b)
        _lib.check(_lib.lib().riga_spmv(s.device.handle, 2, float(sigma), _lib.ptr(x), _lib.ptr(r)))
        assert float(torch.linalg.norm(r - b) / torch.linalg.norm(b)) < 1e-10


@pytest.mark.parametrize("name", ["cfg1", "cfg2_riga", "cfg2_iga", "cfg3_riga", "cfg4_riga", "cfg4_iga", "cfg5_riga"])
def test_quadrature_assembly_matches_kronecker(golden, name):
    """Device element quadrature ((p+1)^d Gauss points per element, BASELINE configs) against the
    bit-identical Kronecker pencil: same CSR pattern, values equal to roundoff (|dK| <= 1e-14 max|K|
    per row, likewise M), deterministic run to run."""
    c = golden["configs"][name]
    sk = P.build_system(c["d"], c["ne"], c["p"], c["level"])
    sq = P.build_system(c["d"], c["ne"], c["p"], c["level"], assembly="quadrature")
    rk, ck, Kk, Mk = sk.device.host_arrays()
    rq, cq, Kq, Mq = sq.device.host_arrays()
    assert np.array_equal(rk, rq) and np.array_equal(ck, cq)
    rows = np.repeat(np.arange(rk.size - 1), np.diff(rk))
    for A, B in ((Kq, Kk), (Mq, Mk)):
        rmax = np.maximum.reduceat(np.abs(B), rk[:-1])
        assert np.all(np.abs(A - B) <= 1e-14 * rmax[rows] + 1e-300)
    sq2 = P.build_system(c["d"], c["ne"], c["p"], c["level"], assembly="quadrature")
    assert np.array_equal(sq2.device.host_arrays()[2], Kq)


def test_quadrature_assembled_slice_matches_exact_spectrum(golden):
    c = golden["configs"]["cfg2_riga"]
    s = P.build_system(c["d"], c["ne"], c["p"], c["level"], assembly="quadrature")
    lam = P.kronecker_spectrum(s)
    r = P.solve_slice(s, (c["shifts"][0], c["shifts"][1]), seed=0, m=2 * c["slice_counts"][0])
    assert r.eigenvalues.size == c["slice_counts"][0]
    np.testing.assert_allclose(r.eigenvalues, lam[: r.eigenvalues.size], rtol=1e-10)
    assert float(r.residuals.max()) <= 1e-8
