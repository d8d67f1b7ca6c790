"""GPU parity of the eigensolver drop-in: the reference's own
tests/test_eigensolver.py cases through paper_2009_08167_b200, plus the
BASELINE configs against the golden reference runs (counts exact,
eigenvalues rtol 1e-10, north-star residual <= 1e-8)."""
import numpy as np
import pytest
import scipy.linalg

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2009_08167_b200")
import paper_2009_08167_b200.eigensolver as E  # noqa: E402

E.DEBUG_INVARIANTS = True


def dense_eig(system, vectors=False):
    K, M = system.K.toarray(), system.M.toarray()
    if vectors:
        return scipy.linalg.eigh(K, M, driver="gvd")
    return scipy.linalg.eigh(K, M, eigvals_only=True, driver="gvd")


def cluster_slices(values, rel=1e-8):
    out, i, vals = [], 0, np.asarray(values)
    while i < len(vals):
        j = i + 1
        while j < len(vals) and vals[j] - vals[j - 1] <= rel * max(abs(vals[j]), 1.0):
            j += 1
        out.append(slice(i, j))
        i = j
    return out


def subspace_angle(X, Y, M):
    s = np.linalg.svd(X.T @ (M @ Y), compute_uv=False)
    return float(np.arccos(min(s.min(), 1.0)))


def resid_ns(K, M, lam, x):
    kx, mx = K @ x, M @ x
    return np.linalg.norm(kx - lam * mx) / (abs(lam) * np.linalg.norm(mx))


def test_operator_apply_counters_and_mapping():
    s = P.build_system(1, 16, 2)
    lam, X = dense_eig(s, vectors=True)
    sigma = 0.5 * (lam[0] + lam[1])
    c = P.CostCounters()
    f = P.factor_ldl(s.K.csr - sigma * s.M.csr, ordering=P.separator_ordering(s), counters=c)
    out = P.operator_apply(f, s.M, X[:, 3], c)
    np.testing.assert_allclose(out, X[:, 3] / (lam[3] - sigma), rtol=1e-9)
    assert c.nfb == 1 and c.nmv == 1


def test_lanczos_two_by_two_oracle():
    H = np.array([[2.0, 1.0], [1.0, 2.0]])
    st = P.LanczosState(lambda v: H @ v, 2, max_dim=2, start=np.array([1.0, 0.0]))
    P.lanczos_extend(st, 2)
    assert st.T[0, 0] == pytest.approx(2.0)
    assert st.T[1, 0] == pytest.approx(1.0)
    assert st.T[1, 1] == pytest.approx(2.0)
    np.testing.assert_allclose(np.linalg.eigh(st.T[:2, :2])[0], [1.0, 3.0], atol=1e-14)


def test_lanczos_breakdown_on_eigenvector_start():
    H = np.diag([3.0, 1.0])
    st = P.LanczosState(lambda v: H @ v, 2, max_dim=2, start=np.array([1.0, 0.0]),
                        rng=np.random.default_rng(0))
    st.step()
    assert st.T[0, 0] == pytest.approx(3.0)
    assert st.coupling[:1].max() == 0.0
    st.step()
    assert st.k == 2


def test_lanczos_projection_matches_t():
    s = P.build_system(1, 32, 3)
    lam = dense_eig(s)
    sigma = 0.5 * (lam[4] + lam[5])
    f = P.factor_ldl(s.K.csr - sigma * s.M.csr, ordering=P.separator_ordering(s))
    op = E.DeviceShiftInvert(f, s.M)
    st = P.LanczosState(op, s.dof_count, mass=s.M, shift=sigma, max_dim=12,
                        rng=np.random.default_rng(3))
    P.lanczos_extend(st, 12)
    V = st.V[: st.k].cpu().numpy()
    HV = np.column_stack([P.operator_apply(f, s.M, V[j]) for j in range(st.k)])
    T_explicit = V @ (s.M.csr @ HV)
    np.testing.assert_allclose(T_explicit, st.T[: st.k, : st.k], atol=1e-8)
    assert (np.diag(st.T[: st.k, : st.k], -1) >= 0).all()


def test_rayleigh_ritz_shift_mapping():
    st = P.LanczosState(lambda v: 0.5 * v, 1, shift=10.0, max_dim=1, start=np.array([1.0]))
    P.lanczos_extend(st, 1)
    pairs = P.rayleigh_ritz(st)
    assert pairs[0].theta == pytest.approx(0.5)
    assert pairs[0].lam == pytest.approx(12.0)
    assert pairs[0].converged


def test_thick_restart_keep_zero_and_retains_basis():
    H = np.diag(np.arange(1.0, 9.0))
    st = P.LanczosState(lambda v: H @ v, 8, max_dim=5, rng=np.random.default_rng(1))
    P.lanczos_extend(st, 5)
    P.thick_restart(st, 0)
    assert st.k == 0 and st.tridiagonal
    P.lanczos_extend(st, 3)
    assert st.k == 3
    s = P.build_system(1, 32, 3)
    lam = dense_eig(s)
    sigma = 0.5 * (lam[2] + lam[3])
    f = P.factor_ldl(s.K.csr - sigma * s.M.csr, ordering=P.separator_ordering(s))
    st = P.LanczosState(E.DeviceShiftInvert(f, s.M), s.dof_count, mass=s.M, shift=sigma,
                        max_dim=14, rng=np.random.default_rng(5))
    P.lanczos_extend(st, 14)
    P.thick_restart(st, 4)
    assert st.k == 4
    P.lanczos_extend(st, 10)
    assert st.k == 10
    st.check_invariants()


def test_converged_pair_matches_oracle_and_residual():
    s = P.build_system(1, 16, 2)
    lam = dense_eig(s)
    res = P.solve_spectrum(s, count=5, seed=4)
    np.testing.assert_allclose(res.eigenvalues, lam[:5], rtol=1e-10)
    for i in range(5):
        x = res.vectors[:, i]
        kx = s.K.csr @ x
        r = np.linalg.norm(kx - res.eigenvalues[i] * (s.M.csr @ x)) / np.linalg.norm(kx)
        assert r < 1e-8 and res.residuals[i] < 1e-8


def test_restarted_equals_unrestarted():
    s = P.build_system(1, 32, 3)
    small = P.solve_spectrum(s, count=10, seed=6, m=20)
    large = P.solve_spectrum(s, count=10, seed=6, m=200)
    np.testing.assert_allclose(small.eigenvalues, large.eigenvalues, rtol=1e-9)


def test_slice_below_first_eigenvalue_is_empty():
    s = P.build_system(2, 8, 2)
    r = P.solve_slice(s, (0.05, 1.0), seed=0)
    assert r.expected_count == 0 and r.eigenvalues.size == 0


def test_slice_degenerate_pair_at_5pi2():
    s = P.build_system(2, 8, 2)
    lam5 = 5 * np.pi**2
    r = P.solve_slice(s, (lam5 - 5.0, lam5 + 5.0), seed=1)
    assert r.expected_count == 2 and r.eigenvalues.size == 2
    np.testing.assert_allclose(r.eigenvalues[0], r.eigenvalues[1], rtol=1e-9)
    X = r.vectors
    g = X @ (s.M.csr @ X.T)
    assert abs(g[0, 1]) < 1e-6
    np.testing.assert_allclose(np.diag(g), 1.0, atol=1e-8)


def test_adjacent_slices_union_matches_merged():
    s = P.build_system(1, 32, 3)
    lam = dense_eig(s)
    lo, mid, hi = 0.9 * lam[0], 1.02 * lam[6], 1.05 * lam[12]
    left = P.solve_slice(s, (lo, mid), seed=2)
    right = P.solve_slice(s, (mid, hi), seed=3)
    merged = P.solve_slice(s, (lo, hi), seed=4)
    union = np.sort(np.concatenate([left.eigenvalues, right.eigenvalues]))
    np.testing.assert_allclose(union, merged.eigenvalues, rtol=1e-9)


def test_interval_count_equals_inertia_difference():
    s = P.build_system(2, 8, 3, 1)
    lam = dense_eig(s)
    rng = np.random.default_rng(12)
    for _ in range(3):
        lo = rng.uniform(0.5 * lam[0], lam[-1])
        hi = lo + rng.uniform(0.5, 0.05 * lam[-1])
        res = P.solve_spectrum(s, interval=(lo, hi), seed=13)
        lo_u, hi_u = res.slices[0][0], res.slices[-1][1]
        assert res.eigenvalues.size == int(np.sum((lam > lo_u) & (lam <= hi_u)))


def test_global_m_orthonormality_and_subspace_angles():
    s = P.build_system(2, 8, 2)
    lam, Xo = dense_eig(s, vectors=True)
    res = P.solve_spectrum(s, count=s.dof_count, seed=9)
    X = res.vectors
    G = X.T @ (s.M.csr @ X)
    assert np.abs(G - np.diag(np.diag(G))).max() < 1e-6
    np.testing.assert_allclose(np.diag(G), 1.0, atol=1e-8)
    for sl in cluster_slices(lam):
        assert subspace_angle(res.vectors[:, sl], Xo[:, sl], s.M.csr) < 1e-6


def test_nfa_is_nsh_plus_retries_and_validation():
    for seed in (0, 1):
        s = P.build_system(2, 8, 3)
        c = P.solve_spectrum(s, count=30, seed=seed).counters
        assert c.nfa == c.nsh + c.retries
        assert c.nmv >= c.nfb
    s = P.build_system(1, 8, 2)
    with pytest.raises(ValueError):
        P.solve_spectrum(s)
    with pytest.raises(ValueError):
        P.solve_spectrum(s, count=3, interval=(0, 1))
    with pytest.raises(ValueError):
        P.solve_spectrum(s, count=s.dof_count + 1)
    with pytest.raises(ValueError):
        P.solve_spectrum(s, interval=(2.0, 1.0))


@pytest.mark.parametrize("name", ["cfg1", "cfg2_riga", "cfg2_iga"])
def test_baseline_slices_match_reference(golden, golden_arrays, name):
    c = golden["configs"][name]
    s = P.build_system(c["d"], c["ne"], c["p"], c["level"])
    K, M = s.K.csr, s.M.csr
    for k in range(c["S"]):
        g = golden["slices"][f"{name}/{k}"]
        r = P.solve_slice(s, (c["shifts"][k], c["shifts"][k + 1]), seed=k, m=g["m"])
        assert r.expected_count == g["expected"] == r.eigenvalues.size
        np.testing.assert_allclose(r.eigenvalues, golden_arrays[f"{name}/slice{k}/eig"], rtol=1e-10)
        worst = max(resid_ns(K, M, l, x) for l, x in zip(r.eigenvalues, r.vectors))
        assert worst <= 1e-8, worst


def test_uniform_slices_driver_cfg2(golden, golden_arrays):
    c = golden["configs"]["cfg2_riga"]
    s = P.build_system(c["d"], c["ne"], c["p"], c["level"])
    res = P.solve_uniform_slices(s, c["shifts"], seeds=range(c["S"]), streams=2)
    assert list(res.nu) == c["nu"]
    assert list(res.found) == c["slice_counts"]
    ref = np.concatenate([golden_arrays[f"cfg2_riga/slice{k}/eig"] for k in range(c["S"])])
    np.testing.assert_allclose(res.eigenvalues, np.sort(ref), rtol=1e-10)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["cfg3_riga", "cfg4_riga"])
def test_large_config_slice0_matches_reference(golden, golden_arrays, name):
    """Slice 0 of the 2D (N = 91,809) and 3D (N = 42,875) baseline configs against the reference's own
    solve_slice eigenvalues (tests/golden), counts exact, residuals <= 1e-8."""
    c = golden["configs"][name]
    g = golden["slices"][f"{name}/0"]
    s = P.build_system(c["d"], c["ne"], c["p"], c["level"])
    r = P.solve_slice(s, (g["lo"], g["hi"]), seed=g["seed"], m=g["m"])
    assert r.expected_count == g["expected"] == r.eigenvalues.size
    np.testing.assert_allclose(r.eigenvalues, golden_arrays[f"{name}/slice0/eig"], rtol=1e-10)
    K, M = s.K.csr, s.M.csr
    worst = max(resid_ns(K, M, l, x) for l, x in zip(r.eigenvalues, r.vectors))
    assert worst <= 1e-8, worst


@pytest.mark.slow
def test_uniform_slices_cfg4_match_kronecker_spectrum(golden):
    """All 8 slices of the 3D config (inverse + doubling path): inertia counts equal the Kronecker counts
    recorded from the reference, eigenvalues equal the exact discrete spectrum to 1e-10."""
    c = golden["configs"]["cfg4_riga"]
    s = P.build_system(c["d"], c["ne"], c["p"], c["level"])
    lam = P.kronecker_spectrum(s)
    shifts = P.uniform_shifts(c["lambda_e"], c["S"])
    res = P.solve_uniform_slices(s, shifts, streams=8)
    assert list(res.expected) == c["slice_counts"]
    assert list(res.found) == c["slice_counts"]
    np.testing.assert_allclose(res.eigenvalues, lam[: c["count"]], rtol=1e-10)


@pytest.mark.slow
def test_cfg5_slices_match_kronecker_spectrum(golden):
    """Two slices of the largest config (3D 64^3, p = 3, N = 357,911): counts and eigenvalues against the
    exact Kronecker spectrum."""
    c = golden["configs"]["cfg5_riga"]
    s = P.build_system(c["d"], c["ne"], c["p"], c["level"])
    lam = P.kronecker_spectrum(s)
    shifts = P.uniform_shifts(c["lambda_e"], c["S"])
    for k in (0, c["S"] - 1):
        lo, hi = float(shifts[k]), float(shifts[k + 1])
        ref = lam[(lam > lo) & (lam <= hi)]
        r = P.solve_slice(s, (lo, hi), seed=k, m=2 * ref.size)
        assert r.expected_count == ref.size == r.eigenvalues.size == c["slice_counts"][k]
        np.testing.assert_allclose(r.eigenvalues, ref, rtol=1e-10)


def test_uploaded_pencil_with_kron_factors_matches_device_assembly():
    """Host CSR upload + attach_kron (the e2e path of bench.py): Lanczos mass
    products run axis by axis on the uploaded pencil; the slice must agree
    with the device-assembled system's to roundoff and keep the counts."""
    from paper_2009_08167_b200 import device as D
    from paper_2009_08167_b200.assembly import DeviceSystem, DiscreteSystem, SymSparseMatrix

    s = P.build_system(2, 16, 3, 2)
    lam = dense_eig(s)
    hi = 0.5 * (lam[14] + lam[15])
    dsys = DeviceSystem.upload(D.current(), s.K.csr.copy(), s.M.csr.copy())
    dsys.attach_kron(s.k1d, s.m1d)
    s2 = DiscreteSystem(SymSparseMatrix(device=dsys, which=0), SymSparseMatrix(device=dsys, which=1),
                        s.spaces, s.dim, s.dof_count, s.k1d, s.m1d, dsys)
    r1 = P.solve_slice(s, (0.0, hi), seed=3, m=30)
    r2 = P.solve_slice(s2, (0.0, hi), seed=3, m=30)
    assert r1.expected_count == r2.expected_count == 15
    assert np.allclose(r2.eigenvalues, lam[:15], rtol=1e-10, atol=0)
    assert np.allclose(r1.eigenvalues, r2.eigenvalues, rtol=1e-11, atol=0)
    with pytest.raises(ValueError):
        dsys.attach_kron(s.k1d[:1], s.m1d[:1])  # sizes do not multiply to n


def test_delayed_cgs2_matches_two_pass_cgs2():
    """The device step runs the reference's two Gram-Schmidt passes with the
    second one delayed into the next step's sweeps (lanczos.cu, delayed
    CGS2).  Against the undelayed variant (RIGA_CGS=classic: two full passes
    per step, ref _orthogonalize :204-212), with locked rows and across a
    thick restart: the basis stays M-orthonormal to 1e-8 (ref invariants),
    the first steps' recurrence agrees to rounding, and the converged Ritz
    values agree to 1e-10 (entries of T after convergence are driven by
    rounding noise in any Lanczos, so they are not compared)."""
    import os

    from paper_2009_08167_b200.eigensolver import DeviceShiftInvert, _state_pool

    s = P.build_system(2, 16, 3, 2)
    lam = dense_eig(s)
    sigma = 0.5 * (lam[3] + lam[4])
    f = P.factor_ldl(s.K.csr - sigma * s.M.csr, ordering=P.separator_ordering(s))
    M = s.M.csr
    _, vec = dense_eig(s, vectors=True)

    def run(mode):
        os.environ["RIGA_CGS"] = mode
        _state_pool.clear()  # a pooled state keeps the mode it was created with
        try:
            st = P.LanczosState(DeviceShiftInvert(f, s.M), s.dof_count, mass=s.M, shift=sigma, max_dim=40,
                                rng=np.random.default_rng(7),
                                locked_pairs=[(vec[:, 0], M @ vec[:, 0]), (vec[:, 1], M @ vec[:, 1])])
            P.lanczos_extend(st, 30)
            st.check_invariants()
            T6 = st.T[:6, :6].copy()
            P.thick_restart(st, 6)
            P.lanczos_extend(st, 40)
            st.check_invariants()
            conv = sorted(rp.lam for rp in P.rayleigh_ritz(st) if rp.converged)
            return T6, np.array(conv)
        finally:
            os.environ.pop("RIGA_CGS", None)
            _state_pool.clear()

    (Ta, ca), (Tb, cb) = run("delayed"), run("classic")
    np.testing.assert_allclose(Ta, Tb, rtol=0, atol=1e-12 * np.abs(Tb).max())
    assert ca.size >= 4 and ca.size == cb.size
    np.testing.assert_allclose(ca, cb, rtol=1e-10)
    for x in ca:  # and they are eigenvalues of the pencil (locked ones excluded)
        assert np.min(np.abs(lam[2:] - x)) <= 1e-10 * abs(x)


@pytest.mark.parametrize("mode", ["count", "interval"])
def test_solve_spectrum_parallel_matches_sequential(golden, mode):
    """solve_spectrum on concurrent streams (speculative inertia pre-pass + every slice on its own stream)
    returns the sequential reference driver's spectrum: same count, eigenvalues to 1e-10 (and the exact
    spectrum), residuals within the gate, M-orthonormal vectors."""
    c = golden["configs"]["cfg2_riga"]
    s = P.build_system(c["d"], c["ne"], c["p"], c["level"])
    lam = P.kronecker_spectrum(s)
    # interval endpoints in spectral gaps (2D eigenvalues come in degenerate pairs)
    gap = lambda i: next(j for j in range(i, lam.size - 1) if lam[j + 1] - lam[j] > 1e-6 * lam[j + 1])  # noqa: E731
    i0, i1 = gap(9), gap(79)
    kw = dict(count=100) if mode == "count" else dict(interval=(0.5 * (lam[i0] + lam[i0 + 1]),
                                                                0.5 * (lam[i1] + lam[i1 + 1])))
    seq = P.solve_spectrum(s, seed=3, m=40, **kw)
    par = P.solve_spectrum(s, seed=3, m=40, parallel=True, streams=8, **kw)
    assert par.eigenvalues.size == seq.eigenvalues.size == (100 if mode == "count" else i1 - i0)
    np.testing.assert_allclose(par.eigenvalues, seq.eigenvalues, rtol=1e-10)
    ref = lam[:100] if mode == "count" else lam[i0 + 1: i1 + 1]
    np.testing.assert_allclose(par.eigenvalues, ref, rtol=1e-10)
    assert float(par.north_residuals.max()) <= 1e-8
    X = par.vectors
    G = X.T @ (s.M.csr @ X)
    assert np.abs(G - np.eye(G.shape[0])).max() < 1e-8
    assert all(c_ <= 4 * 20 for _, _, c_ in par.slices)  # the march's acceptance bound, target = m / 2
    assert par.counters.nfa >= par.counters.nsh > 0
