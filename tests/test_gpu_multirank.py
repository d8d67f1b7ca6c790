"""The multi-GPU slice partition end to end with two ranks: two processes share the one GPU of
the test box and talk over gloo (the only collectives are host all-gathers of inertias, eigenvalues and
boundary pairs, so no rank ever waits on another rank's kernels).  Each rank factors its share of the
boundary shifts, solves the slices LPT assigns it, and the gathered spectrum must equal the single-rank run's
(counts exact, eigenvalues within 1e-10) and the exact Kronecker spectrum."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2009_08167_b200")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import paper_2009_08167_b200 as P

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = P.build_system(cfg["d"], cfg["ne"], cfg["p"], cfg["level"])
        res = P.solve_uniform_slices(s, cfg["shifts"], seeds=range(cfg["S"]), streams=4, rank=rank, world=world)
        out[rank] = (list(res.local_slices), res.eigenvalues.tolist(), list(res.found), list(res.nu),
                     float(res.max_residual), {int(k): v.tolist() for k, v in res.local_eigenvalues.items()})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["cfg2_riga", "cfg3_riga"])
def test_two_ranks_match_single_rank(golden, name):
    import torch.multiprocessing as mp

    c = golden["configs"][name]
    cfg = {k: c[k] for k in ("d", "ne", "p", "level", "shifts", "S")}
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, cfg, out), nprocs=world, join=True)
    (s0, e0, f0, n0, r0, l0), (s1, e1, f1, n1, r1, l1) = out[0], out[1]
    assert sorted(s0 + s1) == list(range(c["S"]))  # every slice on exactly one rank
    assert e0 == e1 and f0 == f1 and n0 == n1  # every rank holds the gathered result
    assert n0 == c["nu"] and f0 == c["slice_counts"]
    assert max(r0, r1) <= 1e-8
    s = P.build_system(c["d"], c["ne"], c["p"], c["level"])
    single = P.solve_uniform_slices(s, c["shifts"], seeds=range(c["S"]), streams=4)
    np.testing.assert_allclose(np.array(e0), single.eigenvalues, rtol=1e-10, atol=0)
    lam = P.kronecker_spectrum(s)
    np.testing.assert_allclose(np.array(e0), lam[: c["count"]], rtol=1e-10, atol=0)
    # each rank's own slices are the ones it reports
    assert sorted(l0) == sorted(s0) and sorted(l1) == sorted(s1)
