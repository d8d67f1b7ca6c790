"""Per-slice residual-gate diagnostics on one BASELINE config (GPU):
initial / final max north-star residual, refinement rounds, max eigenvalue error vs the exact Kronecker
spectrum and vs the reference's own solve_slice eigenvalues (tests/golden/golden_slices.npz).

    python tools/gate_probe.py cfg4_iga [streams]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_08167_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4_iga"
streams = int(sys.argv[2]) if len(sys.argv) > 2 else 8
g = json.load(open(os.path.join(ROOT, "tests/golden/golden.json")))["configs"][name]
ref = dict(np.load(os.path.join(ROOT, "tests/golden/golden_slices.npz")))
s = P.build_system(g["d"], g["ne"], g["p"], g["level"])
lam = P.kronecker_spectrum(s)
shifts = P.uniform_shifts(g["lambda_e"], g["S"])
t0 = time.perf_counter()
r = P.solve_uniform_slices(s, shifts, seeds=range(g["S"]), streams=streams)
dt = time.perf_counter() - t0
out = {"config": name, "seconds": dt, "max_residual": r.max_residual, "slices": []}
for k in range(g["S"]):
    lo, hi = float(r.shifts[k]), float(r.shifts[k + 1])
    ev = r.local_eigenvalues[k]
    ex = lam[(lam > lo) & (lam <= hi)]
    gi = r.gate_info[k]
    rec = {"k": k, "count": int(ev.size), "rounds": gi.rounds if gi else 0,
           "initial_max": gi.initial_max if gi else 0.0, "final_max": gi.final_max if gi else 0.0,
           "err_vs_kron": float(np.max(np.abs(ev - ex) / ex)) if ev.size else 0.0}
    key = f"{name}/slice{k}/eig"
    if key in ref:
        rec["err_vs_ref"] = float(np.max(np.abs(ev - ref[key]) / ref[key]))
        rec["ref_err_vs_kron"] = float(np.max(np.abs(ref[key] - ex) / ex))
    out["slices"].append(rec)
    print(rec, flush=True)
print(json.dumps({k: v for k, v in out.items() if k != "slices"}))
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"gate_{name}.json"), "w"), indent=1)
