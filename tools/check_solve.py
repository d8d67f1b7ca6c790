"""Relative residual ||(K - sigma M) x - b|| / ||b|| of one device factor + solve.

    python tools/check_solve.py [--config cfg5] [--frac 0.0]
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_08167_b200 as P  # noqa: E402
from paper_2009_08167_b200 import _lib  # noqa: E402
from paper_2009_08167_b200.configs import CONFIGS  # noqa: E402
from paper_2009_08167_b200.sparsela import Symbolic, numeric_factor  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5")
ap.add_argument("--sigmas", default="0,0.01,0.5")
a = ap.parse_args()
c = CONFIGS[a.config]
s = P.build_system(c.d, c.ne, c.p, c.level)
lam = P.kronecker_spectrum(s)
lam_e, _ = P.choose_lambda_e(s, c.n0, lam)
sym = Symbolic.on_device(s.device, P.separator_ordering(s))
n = s.dof_count
b = torch.randn(n, dtype=torch.float64, device="cuda")
x = torch.empty_like(b)
r = torch.empty_like(b)
for fr in [float(t) for t in a.sigmas.split(",")]:
    sigma = fr * lam_e
    f = numeric_factor(sym, sigma)
    f.solve_device(b, x)
    _lib.check(_lib.lib().riga_spmv(s.device.handle, 2, f.sigma, _lib.ptr(x), _lib.ptr(r)))
    torch.cuda.synchronize()
    res = float(torch.linalg.norm(r - b) / torch.linalg.norm(b))
    print(f"{a.config} sigma={f.sigma:.6g} neg={f.n_negative} rel_residual={res:.3e}", flush=True)
