"""Multi-process (gloo, world_size 2, CPU) coverage of the slice-partition
host logic used by solve_uniform_slices on N GPUs: the all-gather of the
boundary inertias / eigenvalues and the LPT assignment every rank computes
independently (it must agree across ranks and cover every slice once)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2009_08167_b200.slicing import _allgather, lpt_assign


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        S = 16
        # boundary pass: rank r factors shifts k = r (mod world)
        nu_true = [int(5 * k + k * k // 3) for k in range(S + 1)]
        mine = {k: (float(k), nu_true[k], 1.0) for k in range(S + 1) if k % world == rank}
        merged = {}
        for part in _allgather(mine, world):
            merged.update(part)
        nu = [merged[k][1] for k in range(S + 1)]
        counts = list(np.diff(nu))
        assign = lpt_assign(counts, world)
        # eigenvalue gather: each rank reports its slices
        local = {k: np.arange(counts[k], dtype=float) + 100 * k for k in assign[rank]}
        gathered = _allgather((local, {}), world)
        found = {}
        for le, _ in gathered:
            for k, v in le.items():
                found[k] = int(v.size)
        out[rank] = (nu, assign, found)
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_partition_and_gather():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    nu0, a0, f0 = out[0]
    nu1, a1, f1 = out[1]
    assert nu0 == nu1  # both ranks see every boundary inertia
    assert a0 == a1  # identical LPT partition computed independently
    assert sorted(a0[0] + a0[1]) == list(range(16))  # each slice exactly once
    counts = list(np.diff(nu0))
    assert f0 == f1 and all(f0[k] == counts[k] for k in range(16))


def test_single_rank_gather_is_identity():
    assert _allgather({1: 2}, 1) == [{1: 2}]


# ---------------------------------------------------------------------------
# boundary de-duplication (ref _Pool.add eigensolver.py:407-420,
# _dedup_and_orthonormalize :670-712)
# ---------------------------------------------------------------------------
from paper_2009_08167_b200.slicing import boundary_dedup  # noqa: E402


def _mass(n, seed=0):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n))
    return A @ A.T / n + np.eye(n)


def _mnormal(x, M):
    return x / np.sqrt(x @ M @ x)


def _planted(M, rng):
    n = M.shape[0]
    x = _mnormal(rng.standard_normal(n), M)
    y = rng.standard_normal(n)
    y = _mnormal(y - (x @ M @ y) * x, M)  # M-orthogonal to x
    xdup = _mnormal(x + 1e-6 * rng.standard_normal(n), M)  # the same pair found by the next slice
    lam = 100.0
    return [
        (0, 3, lam - 2e-8, x, M @ x),          # slice 0 found it just below the shared shift
        (1, 0, lam + 3e-8, xdup, M @ xdup),    # slice 1 found the same eigenvector just above it
        (1, 1, lam + 5e-8, y, M @ y),          # a different eigenvector at (almost) the same lam
    ]


def test_boundary_dedup_drops_planted_duplicate_once():
    M = _mass(40)
    rng = np.random.default_rng(1)
    ent = _planted(M, rng)
    drop, upd = boundary_dedup(ent, scale=200.0)
    assert drop == {(1, 0)}  # the later copy goes, as in the reference's sequential pool
    # the survivors (x, y) are M-orthonormal already (||G - I|| <= 1e-10): no Loewdin update needed
    for (k, j), (xn, mxn) in upd.items():
        assert np.allclose(mxn, M @ xn)


def test_boundary_dedup_keeps_distinct_pairs_and_orthonormalises_cluster():
    M = _mass(30, seed=3)
    rng = np.random.default_rng(4)
    x = _mnormal(rng.standard_normal(30), M)
    y = rng.standard_normal(30)
    y = _mnormal(y - (x @ M @ y) * x + 1e-6 * x, M)  # slightly non-orthogonal partner, same cluster
    ent = [(2, 0, 50.0, x, M @ x), (3, 0, 50.0 + 1e-8, y, M @ y)]
    drop, upd = boundary_dedup(ent, scale=60.0)
    assert not drop
    assert set(upd) == {(2, 0), (3, 0)}
    X = np.stack([upd[(2, 0)][0], upd[(3, 0)][0]])
    assert np.abs(X @ M @ X.T - np.eye(2)).max() < 1e-12
    # far-apart eigenvalues never interact
    z = _mnormal(rng.standard_normal(30), M)
    drop2, upd2 = boundary_dedup([(0, 0, 10.0, z, M @ z), (1, 0, 20.0, z, M @ z)], scale=20.0)
    assert not drop2 and not upd2


def _dedup_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        M = _mass(40)
        ent = _planted(M, np.random.default_rng(1))
        mine = [e for e in ent if e[0] % world == rank]  # slice k lives on rank k mod 2
        gathered = _allgather(mine, world)
        allent = sorted((e for part in gathered for e in part), key=lambda e: (e[0], e[1]))
        drop, upd = boundary_dedup(allent, 200.0)
        out[rank] = (sorted(drop), sorted(upd))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_boundary_dedup_agrees():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_dedup_worker, args=(world, port, out), nprocs=world, join=True)
    assert out[0] == out[1]
    assert out[0][0] == [(1, 0)]
