"""Factor once, then run `--solves` supernodal solves (for ncu launch lists)."""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_08167_b200 as P  # noqa: E402
from paper_2009_08167_b200.configs import CONFIGS  # noqa: E402
from paper_2009_08167_b200.sparsela import Symbolic, numeric_factor  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--solves", type=int, default=2)
a = ap.parse_args()
c = CONFIGS[a.config]
s = P.build_system(c.d, c.ne, c.p, c.level)
lam_e, _ = P.choose_lambda_e(s, c.n0)
sym = Symbolic.on_device(s.device, P.separator_ordering(s))
f = numeric_factor(sym, lam_e / 2)
b = torch.randn(s.dof_count, dtype=torch.float64, device="cuda")
x = torch.empty_like(b)
torch.cuda.synchronize()
for _ in range(a.solves):
    f.solve_device(b, x)
torch.cuda.synchronize()
print("ok", sym.stats["n_levels"])
