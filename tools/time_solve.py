"""Factor once at the middle of the spectrum range, then time isolated supernodal solves (CUDA events).

    python tools/time_solve.py cfg5 [reps]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_08167_b200 as P  # noqa: E402
from paper_2009_08167_b200 import _lib  # noqa: E402
from paper_2009_08167_b200.configs import CONFIGS  # noqa: E402
from paper_2009_08167_b200.sparsela import Symbolic, numeric_factor  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg5"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
s = P.build_system(c.d, c.ne, c.p, c.level)
lam_e, _ = P.choose_lambda_e(s, c.n0)
sym = Symbolic.on_device(s.device, P.separator_ordering(s))
f = numeric_factor(sym, lam_e / 2)
b = torch.randn(s.dof_count, dtype=torch.float64, device="cuda")
x = torch.empty_like(b)
for _ in range(3):
    f.solve_device(b, x)
torch.cuda.synchronize()
ms = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    f.solve_device(b, x)
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
r = torch.empty_like(b)
_lib.check(_lib.lib().riga_spmv(s.device.handle, 2, float(lam_e / 2), _lib.ptr(x), _lib.ptr(r)))
err = float(torch.linalg.norm(r - b) / torch.linalg.norm(b))
bytes_ = 16.0 * sym.stats["fill_nnz"] + 32.0 * s.dof_count
print(f"{c.name}: factor {f.device_ms:.2f} ms, solve median {np.median(ms):.3f} ms ({bytes_ / np.median(ms) / 1e6:.0f} GB/s algorithmic), "
      f"backward error {err:.2e}, levels {sym.stats['n_levels']}, max_ncol {sym.stats['max_ncol']}")
