"""Solve of a cfg with the level-synchronous or the dataflow subtree kernels (RIGA_SUB_DATAFLOW); writes x."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_08167_b200 as P  # noqa
from paper_2009_08167_b200.configs import CONFIGS  # noqa
from paper_2009_08167_b200.sparsela import Symbolic, numeric_factor  # noqa
from paper_2009_08167_b200.slicing import solve_plan  # noqa
c = CONFIGS[sys.argv[1]]
s = P.build_system(c.d, c.ne, c.p, c.level)
lam_e, _ = P.choose_lambda_e(s, c.n0)
with solve_plan(int(sys.argv[3]) if len(sys.argv) > 3 else 6):
    sym = Symbolic.on_device(s.device, P.separator_ordering(s))
f = numeric_factor(sym, lam_e / 3)
b = torch.randn(s.dof_count, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
x = torch.empty_like(b)
f.solve_device(b, x)
torch.cuda.synchronize()
np.save(sys.argv[2], x.cpu().numpy())
print("ok", sys.argv[1])
