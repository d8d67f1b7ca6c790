"""Generate per-slice golden fixtures for the large BASELINE configs by running the REFERENCE itself.

Run here (the container that has /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_slices.py [--workers 8]

Every slice (sigma_k, sigma_k+1] of the uniform shifts of cfg3 rIGA (16 slices), cfg4 rIGA and cfg4 IGA
(8 slices each) is solved with the reference's ``rigaeig.solve_slice(system, (lo, hi), seed=k, m=2 count_k)``
(ref eigensolver.py:636-660; the BASELINE protocol of SURVEY §8d), one process per slice with one BLAS
thread (the reference CLI's ProcessPool mode, ref cli.py:208-210).  Recorded per slice: eigenvalues
(npz), expected/found counts, the reference's counters, and the north-star residual
||K u - lam M u|| / (|lam| ||M u||) of each returned pair (max and count above 1e-8), so the GPU tests can
compare eigenvalues at rtol 1e-10 and show the reference's own residual misses.
For cfg4 IGA it also records the reference LDL^T inertia at every uniform shift (ref sparsela.py:212-262).

Outputs ``tests/golden/golden_slices.json`` and ``tests/golden/golden_slices.npz``.  Nothing under tests/
reads /root/reference at run time; only this script.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor, as_completed

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# name -> (d, ne, p, level)
CONFIGS = {"cfg3_riga": (2, 256, 4, 4), "cfg4_riga": (3, 32, 2, 2), "cfg4_iga": (3, 32, 2, 0)}


def _golden():
    with open(os.path.join(HERE, "golden.json")) as fh:
        return json.load(fh)


def _slice_job(name: str, k: int):
    import rigaeig as rg

    g = _golden()["configs"][name]
    d, ne, p, lv = CONFIGS[name]
    system = rg.build_system(d, ne, p, lv)
    lo, hi = g["shifts"][k], g["shifts"][k + 1]
    m = 2 * g["slice_counts"][k]
    t0 = time.perf_counter()
    res = rg.solve_slice(system, (lo, hi), seed=k, m=m)
    dt = time.perf_counter() - t0
    K, M = system.K.csr, system.M.csr
    rn = [float(np.linalg.norm(K @ x - l * (M @ x)) / (abs(l) * np.linalg.norm(M @ x)))
          for l, x in zip(res.eigenvalues, res.vectors)]
    rec = {"lo": res.lo, "hi": res.hi, "seed": k, "m": m, "expected": res.expected_count,
           "count": int(res.eigenvalues.size), "seconds": dt, "max_resid": max(rn) if rn else 0.0,
           "n_resid_above_1e8": int(sum(r > 1e-8 for r in rn)),
           "nfa": res.counters.nfa, "nfb": res.counters.nfb, "nmv": res.counters.nmv, "nit": res.counters.nit}
    return ("slice", name, k, rec, np.asarray(res.eigenvalues))


def _inertia_job(name: str, i: int):
    import rigaeig as rg

    g = _golden()["configs"][name]
    d, ne, p, lv = CONFIGS[name]
    system = rg.build_system(d, ne, p, lv)
    perm = rg.separator_ordering(system)
    s = g["shifts"][i]
    t0 = time.perf_counter()
    f = rg.factor_ldl(system.K.csr - s * system.M.csr, ordering=perm)
    return ("inertia", name, i, {"sigma": s, "inertia": [int(v) for v in f.inertia],
                                 "seconds": time.perf_counter() - t0}, None)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 8)
    args = ap.parse_args()
    import rigaeig as rg

    g = _golden()
    jobs = []
    # longest first (cfg4 IGA factors are the slowest), so the pool drains evenly
    for k in range(8):
        jobs.append((_slice_job, "cfg4_iga", k))
    for i in range(9):
        jobs.append((_inertia_job, "cfg4_iga", i))
    for k in range(16):
        jobs.append((_slice_job, "cfg3_riga", k))
    for k in range(8):
        jobs.append((_slice_job, "cfg4_riga", k))
    out = {"generator": "tests/golden/make_golden_slices.py", "reference": "rigaeig " + rg.__version__,
           "protocol": "solve_slice(system, (sigma_k, sigma_k+1], seed=k, m=2 count_k), 1 BLAS thread per process",
           "slices": {}, "inertia": {}}
    arrays = {}
    t0 = time.perf_counter()
    with ProcessPoolExecutor(max_workers=args.workers) as ex:
        futs = [ex.submit(fn, name, k) for fn, name, k in jobs]
        for fut in as_completed(futs):
            kind, name, k, rec, eig = fut.result()
            if kind == "slice":
                out["slices"][f"{name}/{k}"] = rec
                arrays[f"{name}/slice{k}/eig"] = eig
            else:
                out["inertia"].setdefault(name, {})[str(k)] = rec
            print(f"{time.perf_counter() - t0:8.1f}s {kind} {name} {k} {rec}", flush=True)
    for name in out["inertia"]:
        d = out["inertia"][name]
        out["inertia"][name] = [d[str(i)] for i in range(len(d))]
    with open(os.path.join(HERE, "golden_slices.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "golden_slices.npz"), **arrays)
    print("wrote", len(arrays), "arrays", flush=True)


if __name__ == "__main__":
    sys.exit(main())
