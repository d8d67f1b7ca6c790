"""One slice through solve_slice with the residual gate; prints the gate history (GPU).

    python tools/gate_slice.py cfg5_riga 31
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_08167_b200 as P  # noqa: E402
import paper_2009_08167_b200.eigensolver as E  # noqa: E402

name, k = sys.argv[1], int(sys.argv[2])
g = json.load(open(os.path.join(ROOT, "tests/golden/golden.json")))["configs"][name]
s = P.build_system(g["d"], g["ne"], g["p"], g["level"])
lam = P.kronecker_spectrum(s)
sh = P.uniform_shifts(g["lambda_e"], g["S"])
lo, hi = float(sh[k]), float(sh[k + 1])
ex = lam[(lam > lo) & (lam <= hi)]
infos = []
orig = E.residual_gate


def spy(*a, **kw):
    out = orig(*a, **kw)
    infos.append(out[4])
    return out


E.residual_gate = spy
t0 = time.perf_counter()
r = P.solve_slice(s, (lo, hi), seed=k, m=2 * ex.size, device=True, residual_gate=1e-8)
print(name, k, "count", r.eigenvalues.size, "expected", ex.size, "t", round(time.perf_counter() - t0, 2),
      "err_vs_kron", float(np.max(np.abs(r.eigenvalues - ex) / ex)), "gate", infos[-1], flush=True)
