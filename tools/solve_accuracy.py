"""Backward error of the device LDL^T solve on a BASELINE pencil (GPU):
||(K - sigma M) x - b|| / ||b|| and the forward-error proxy of one refinement step, for random b.

    RIGA_CHAIN_INV=0 RIGA_SMALL_G=0 python tools/solve_accuracy.py cfg4_iga 3
(sigma = midpoint of uniform slice k)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_08167_b200 as P  # noqa: E402
from paper_2009_08167_b200 import _lib  # noqa: E402
from paper_2009_08167_b200.sparsela import Symbolic, numeric_factor  # noqa: E402

name, k = sys.argv[1], int(sys.argv[2])
g = json.load(open(os.path.join(ROOT, "tests/golden/golden.json")))["configs"][name]
s = P.build_system(g["d"], g["ne"], g["p"], g["level"])
sh = P.uniform_shifts(g["lambda_e"], g["S"])
sigma = 0.5 * (sh[k] + sh[k + 1])
sym = Symbolic.on_device(s.device, P.separator_ordering(s))
f = numeric_factor(sym, sigma)
rng = np.random.default_rng(0)
n = s.dof_count
worst, worst_x = 0.0, 0.0
for t in range(4):
    b = torch.as_tensor(rng.standard_normal(n), device="cuda")
    x = f.solve_device(b)
    r = torch.empty_like(b)
    _lib.check(_lib.lib().riga_spmv(s.device.handle, 2, float(sigma), _lib.ptr(x), _lib.ptr(r)))
    rr = r - b
    be = float(torch.linalg.norm(rr) / torch.linalg.norm(b))
    dx = f.solve_device(rr.contiguous())
    fe = float(torch.linalg.norm(dx) / torch.linalg.norm(x))
    worst, worst_x = max(worst, be), max(worst_x, fe)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(f.ctx.stream):
    x = f.solve_device(b)
    e0.record(f.ctx.stream)
    for _ in range(20):
        f.solve_device(b, out=x)
    e1.record(f.ctx.stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(json.dumps({"solve_ms": ms, "config": name, "slice": k, "sigma": sigma, "env": {e: os.environ.get(e) for e in
                  ("RIGA_CHAIN_INV", "RIGA_SMALL_G")}, "backward_err": worst, "forward_err_est": worst_x}))
