"""solve_spectrum(count) on cfg3: concurrent-stream driver vs the sequential reference driver (GPU).

    python tools/spectrum_parallel.py [count] [m] [--no-seq]
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_08167_b200 as P  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 60
s = P.build_system(2, 256, 4, 4)
lam = P.kronecker_spectrum(s)
out = {"config": "cfg3", "count": count, "m": m}
for rep in range(2):  # second run warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = P.solve_spectrum(s, count=count, seed=0, m=m, parallel=True, streams=16)
    torch.cuda.synchronize()
    out["parallel_s"] = time.perf_counter() - t0
out["parallel_slices"] = len(r.slices)
out["phases"] = {k: round(v, 3) for k, v in r.counters.phase_s.items() if k.startswith("spectrum")}
out["parallel_err_vs_exact"] = float(np.max(np.abs(r.eigenvalues - lam[:count]) / lam[:count]))
out["parallel_max_residual"] = float(r.north_residuals.max())
out["eigenpairs_per_s"] = count / out["parallel_s"]
if "--no-seq" not in sys.argv:
    t0 = time.perf_counter()
    q = P.solve_spectrum(s, count=count, seed=0, m=m)
    torch.cuda.synchronize()
    out["sequential_s"] = time.perf_counter() - t0
    out["sequential_slices"] = len(q.slices)
    out["max_rel_diff_par_vs_seq"] = float(np.max(np.abs(r.eigenvalues - q.eigenvalues) / q.eigenvalues))
print(json.dumps(out))
