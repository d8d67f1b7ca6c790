"""Isolated single-stream timing of each hot-path operation (CUDA events).

    python tools/profile_ops.py [--config cfg3] [--reps 50]

Prints per-op device time and achieved bandwidth / FLOP rate against the
algorithmic work of SURVEY §8d, one operation at a time (no concurrency).
"""
import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2009_08167_b200 as P  # noqa: E402
from paper_2009_08167_b200 import _lib  # noqa: E402
from paper_2009_08167_b200.configs import CONFIGS  # noqa: E402
from paper_2009_08167_b200.eigensolver import DeviceShiftInvert  # noqa: E402
from paper_2009_08167_b200.sparsela import Symbolic, numeric_factor  # noqa: E402


def timeit(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--k", type=int, default=250)
    a = ap.parse_args()
    c = CONFIGS[a.config]
    L = _lib.lib()
    t0 = time.perf_counter()
    s = P.build_system(c.d, c.ne, c.p, c.level)
    torch.cuda.synchronize()
    t_asm = time.perf_counter() - t0
    lam_e, cnt = P.choose_lambda_e(s, c.n0)
    shifts = P.uniform_shifts(lam_e, c.slices)
    perm = P.separator_ordering(s)
    t0 = time.perf_counter()
    sym = Symbolic.on_device(s.device, perm)
    t_sym = time.perf_counter() - t0
    st = sym.stats
    n, nnz = s.dof_count, s.K.nnz
    out = {"config": a.config, "N": n, "nnz": nnz, "symbolic": st, "assembly_s": t_asm, "symbolic_s": t_sym}
    sig = float(shifts[len(shifts) // 2])
    # factorization
    fms = []
    for _ in range(5):
        t0 = time.perf_counter()
        f = numeric_factor(sym, sig)
        fms.append((f.device_ms, (time.perf_counter() - t0) * 1e3))
    dev_ms = min(x[0] for x in fms)
    out["factor"] = {"device_ms": dev_ms, "wall_ms": min(x[1] for x in fms),
                     "tflops": st["factor_flops"] / dev_ms / 1e9,
                     "tflops_relaxed": st["relaxed_flops"] / dev_ms / 1e9}
    # solve
    b = torch.randn(n, dtype=torch.float64, device="cuda")
    x = torch.empty_like(b)
    ms = timeit(lambda: L.riga_factor_solve(f.handle, _lib.ptr(b), _lib.ptr(x)), a.reps)
    by = 16.0 * st["fill_nnz"] + 32.0 * n
    out["solve"] = {"ms": ms, "GBs": by / ms / 1e6, "bytes": by}
    # spmv
    ms = timeit(lambda: L.riga_spmv(s.device.handle, 1, 0.0, _lib.ptr(b), _lib.ptr(x)), a.reps)
    by = 12.0 * nnz + 4.0 * (n + 1) + 16.0 * n
    out["spmv"] = {"ms": ms, "GBs": by / ms / 1e6, "bytes": by}
    # lanczos: basis of k vectors, one extend step timing and CGS pass share
    k = min(a.k, n - 1)
    st_ = P.LanczosState(DeviceShiftInvert(f, s.M), n, mass=s.M, shift=sig, max_dim=k + 1,
                         rng=np.random.default_rng(0))
    P.lanczos_extend(st_, k)
    L.riga_prof_reset()
    L.riga_prof_enable(1)
    P.thick_restart(st_, 0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    P.lanczos_extend(st_, k)
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    L.riga_prof_enable(0)
    msv, work, sc = np.zeros(6), np.zeros(6), np.zeros(6, np.int64)
    L.riga_prof_read(_lib.ptr(msv), _lib.ptr(work), _lib.ptr(sc), 6)
    names = ["factor", "solve", "spmv", "cgs", "vec", "lift"]
    out["extend"] = {"steps": k, "wall_ms_per_step": wall * 1e3 / k,
                     "device_ms_per_step": e0.elapsed_time(e1) / k,
                     "by_cat_ms_per_step": {nm: msv[i] / k for i, nm in enumerate(names) if sc[i]},
                     "by_cat_GBs": {nm: work[i] / (msv[i] / 1e3) / 1e9 for i, nm in enumerate(names) if sc[i]}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
