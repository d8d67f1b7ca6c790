"""Generate the golden fixtures by running the REFERENCE package itself.

Run here (the container that has /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--big]

It imports ``rigaeig`` (the reference, read-only) and records, for the
systems and shifts the parity tests use:

* structural facts: N, nnz, sha256 of K/M CSR arrays, the separator
  ordering (full for small systems, sha256 for large ones);
* LDL^T facts at fixed shifts: inertia, fill_nnz, factor_flops, sha256 of D
  (and D itself for small systems);
* f/b solves of seeded right-hand sides (small systems);
* solve_slice eigenvalues, counts and counters on seeded runs;
* the Kronecker (1D-pencil) spectrum lambda_e / per-slice counts of the
  five BASELINE configs (the identity ref tests/test_assembly.py:64-72 uses).

Outputs ``tests/golden/golden.json`` and ``tests/golden/golden_arrays.npz``.
Nothing under tests/ reads /root/reference at run time; only this script.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np
import scipy.linalg

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# (name, d, ne, p, level, N0, S)
CONFIGS = [
    ("cfg1", 2, 16, 2, 0, 20, 1),
    ("cfg2_riga", 2, 64, 3, 3, 100, 2),
    ("cfg2_iga", 2, 64, 3, 0, 100, 2),
    ("cfg3_riga", 2, 256, 4, 4, 2000, 16),
    ("cfg4_riga", 3, 32, 2, 2, 500, 8),
    ("cfg4_iga", 3, 32, 2, 0, 500, 8),
    ("cfg5_riga", 3, 64, 3, 2, 4000, 32),
]

SMALL = [(1, 16, 2, 0), (1, 32, 3, 1), (2, 8, 2, 0), (2, 8, 3, 1), (3, 4, 2, 1), (2, 16, 2, 0)]


def kron_spectrum(rg, d, ne, p, lv):
    sp1 = rg.make_spline_space(ne, p, lv)
    K1, M1 = rg.apply_dirichlet(*rg.assemble_1d(sp1))
    mu = scipy.linalg.eigh(K1.toarray(), M1.toarray(), eigvals_only=True, driver="gvd")
    lam = mu
    for _ in range(d - 1):
        lam = np.add.outer(lam, mu).ravel()
    return np.sort(lam)


def lam_e(lam, n0):
    i = n0 - 1
    while i + 1 < lam.size and lam[i + 1] - lam[i] <= 1e-8 * lam[i + 1]:
        i += 1
    return 0.5 * float(lam[i] + lam[i + 1]), i + 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also run cfg3/cfg4 factorizations and slices")
    args = ap.parse_args()
    import rigaeig as rg
    from rigaeig.sparsela import _etree_counts

    out = {"generator": "tests/golden/make_golden.py", "reference": "rigaeig " + rg.__version__,
           "systems": {}, "configs": {}, "slices": {}}
    arrays = {}

    def system_facts(key, system, shifts, keep_arrays):
        K, M = system.K.csr, system.M.csr
        perm = rg.separator_ordering(system)
        rec = {"N": int(system.dof_count), "nnz": int(K.nnz),
               "K_data": sha(K.data), "M_data": sha(M.data),
               "indptr": sha(K.indptr.astype(np.int64)), "indices": sha(K.indices.astype(np.int32)),
               "M_pattern_equal": bool(np.array_equal(K.indptr, M.indptr) and np.array_equal(K.indices, M.indices)),
               "perm": sha(perm.astype(np.int64)), "factors": []}
        if keep_arrays:
            arrays[f"{key}/perm"] = perm.astype(np.int64)
            arrays[f"{key}/K_data"] = K.data
            arrays[f"{key}/M_data"] = M.data
        for j, sigma in enumerate(shifts):
            t0 = time.perf_counter()
            f = rg.factor_ldl(K - sigma * M, ordering=perm)
            fr = {"sigma": float(sigma), "inertia": list(f.inertia), "fill_nnz": int(f.fill_nnz),
                  "factor_flops": int(f.factor_flops), "D": sha(f.D), "seconds": time.perf_counter() - t0}
            if keep_arrays:
                arrays[f"{key}/D{j}"] = f.D
                b = np.random.default_rng(100 + j).standard_normal(system.dof_count)
                arrays[f"{key}/b{j}"] = b
                arrays[f"{key}/x{j}"] = rg.solve_fb(f, b)
            rec["factors"].append(fr)
            print(key, fr, flush=True)
        out["systems"][key] = rec

    # small systems: full arrays
    for d, ne, p, lv in SMALL:
        system = rg.build_system(d, ne, p, lv)
        lam = np.sort(kron_spectrum(rg, d, ne, p, lv))
        shifts = [0.0, 0.5 * (lam[2] + lam[3]), 0.5 * (lam[-2] + lam[-1]) if lam.size > 1 else 2 * lam[0]]
        system_facts(f"s{d}_{ne}_{p}_{lv}", system, shifts, True)

    # BASELINE configs: Kronecker lambda_e and per-slice counts
    for name, d, ne, p, lv, n0, S in CONFIGS:
        lam = kron_spectrum(rg, d, ne, p, lv)
        le, cnt = lam_e(lam, n0)
        shifts = [k * le / S for k in range(S + 1)]
        nu = [int(np.sum(lam < s)) for s in shifts]
        rel = [float(np.min(np.abs(lam - s)) / max(s, 1e-300)) for s in shifts[1:]]
        out["configs"][name] = {"d": d, "ne": ne, "p": p, "level": lv, "N0": n0, "S": S,
                                "N": int(lam.size), "lambda_e": le, "count": cnt,
                                "shifts": shifts, "nu": nu,
                                "slice_counts": [nu[k + 1] - nu[k] for k in range(S)],
                                "min_rel_dist": min(rel)}
        arrays[f"{name}/lam_first"] = lam[: cnt + 8]
        print(name, le, cnt, flush=True)

    # cfg1 and cfg2 full reference runs (structure + every shift + every slice)
    for name in ("cfg1", "cfg2_riga", "cfg2_iga"):
        c = out["configs"][name]
        system = rg.build_system(c["d"], c["ne"], c["p"], c["level"])
        system_facts(name, system, c["shifts"], name == "cfg1")
        for k in range(c["S"]):
            lo, hi = c["shifts"][k], c["shifts"][k + 1]
            m = 2 * c["slice_counts"][k]
            t0 = time.perf_counter()
            res = rg.solve_slice(system, (lo, hi), seed=k, m=m)
            dt = time.perf_counter() - t0
            K, M = system.K.csr, system.M.csr
            resid = [float(np.linalg.norm(K @ x - l * (M @ x)) / (abs(l) * np.linalg.norm(M @ x)))
                     for l, x in zip(res.eigenvalues, res.vectors)]
            out["slices"][f"{name}/{k}"] = {
                "lo": res.lo, "hi": res.hi, "seed": k, "m": m, "expected": res.expected_count,
                "count": int(res.eigenvalues.size), "seconds": dt, "max_resid": max(resid) if resid else 0.0,
                "nfa": res.counters.nfa, "nfb": res.counters.nfb, "nmv": res.counters.nmv,
                "nit": res.counters.nit}
            arrays[f"{name}/slice{k}/eig"] = res.eigenvalues
            print(name, k, out["slices"][f"{name}/{k}"], flush=True)

    # symbolic-only facts for the big configs (etree counts, no numeric)
    for name in ("cfg3_riga", "cfg4_riga", "cfg4_iga", "cfg5_riga"):
        c = out["configs"][name]
        system = rg.build_system(c["d"], c["ne"], c["p"], c["level"])
        perm = rg.separator_ordering(system)
        import scipy.sparse as sp
        B = system.K.csr[perm][:, perm]
        U = sp.triu(B, format="csc")
        parent, lnz = _etree_counts(system.dof_count, U.indptr.astype(np.int64), U.indices.astype(np.int32))
        out["systems"][name] = {"N": int(system.dof_count), "nnz": int(system.K.csr.nnz),
                                "K_data": sha(system.K.csr.data), "M_data": sha(system.M.csr.data),
                                "perm": sha(perm.astype(np.int64)),
                                "fill_nnz": int(lnz.sum()) + int(system.dof_count),
                                "factor_flops": int(np.sum((lnz + 1) ** 2)), "factors": []}
        print(name, out["systems"][name], flush=True)
        if args.big and name in ("cfg3_riga", "cfg4_riga"):
            # inertia at every uniform shift (the oracle's own numeric LDL^T)
            for s in c["shifts"]:
                t0 = time.perf_counter()
                f = rg.factor_ldl(system.K.csr - s * system.M.csr, ordering=perm)
                out["systems"][name]["factors"].append(
                    {"sigma": s, "inertia": list(f.inertia), "D": sha(f.D),
                     "seconds": time.perf_counter() - t0})
                print(name, s, f.inertia, flush=True)
            # lowest slice, reference run
            lo, hi = c["shifts"][0], c["shifts"][1]
            m = 2 * c["slice_counts"][0]
            t0 = time.perf_counter()
            res = rg.solve_slice(system, (lo, hi), seed=0, m=m)
            out["slices"][f"{name}/0"] = {"lo": res.lo, "hi": res.hi, "seed": 0, "m": m,
                                          "expected": res.expected_count, "count": int(res.eigenvalues.size),
                                          "seconds": time.perf_counter() - t0,
                                          "nfa": res.counters.nfa, "nfb": res.counters.nfb,
                                          "nmv": res.counters.nmv, "nit": res.counters.nit}
            arrays[f"{name}/slice0/eig"] = res.eigenvalues
            print(name, "slice0", out["slices"][f"{name}/0"], flush=True)
        del system

    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "golden_arrays.npz"), **arrays)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    sys.exit(main())
