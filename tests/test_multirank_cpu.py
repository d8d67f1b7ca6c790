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
