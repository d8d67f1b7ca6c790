"""A short end-to-end engine run for compute-sanitizer (racecheck / synccheck / memcheck):
device assembly, symbolic + numeric LDL^T, solves, residual kernel, and a short Lanczos run
(delayed-CGS2 step graph, lift, lock, restart).

    compute-sanitizer --tool racecheck python tools/sanitize_case.py cfg2
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_08167_b200 as P  # noqa: E402
from paper_2009_08167_b200.configs import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
c = CONFIGS[name]
s = P.build_system(c.d, c.ne, c.p, c.level)
lam = P.kronecker_spectrum(s)
lo, hi = 0.0, 0.5 * float(lam[6] + lam[7])  # 7 eigenpairs: factor, solves, a few Lanczos cycles
r = P.solve_slice(s, (lo, hi), seed=1, m=16)
assert r.eigenvalues.size == 7, r.eigenvalues.size
np.testing.assert_allclose(r.eigenvalues, lam[:7], rtol=1e-10)
torch.cuda.synchronize()
print(name, "ok", r.eigenvalues.size, "max residual", float(r.residuals.max()))
