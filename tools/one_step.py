"""Build a config, factor the middle shift, run `--steps` Lanczos steps
(the CUDA-graph step) and `--probes` standalone CGS2 passes over the
basis (for ncu launch lists / full captures of the step's kernels)."""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_08167_b200 as P  # noqa: E402
from paper_2009_08167_b200 import _lib  # noqa: E402
from paper_2009_08167_b200.configs import CONFIGS  # noqa: E402
from paper_2009_08167_b200.eigensolver import DeviceShiftInvert  # noqa: E402
from paper_2009_08167_b200.sparsela import Symbolic, numeric_factor  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--steps", type=int, default=250)
ap.add_argument("--probes", type=int, default=2)
ap.add_argument("--factor-only", action="store_true")
a = ap.parse_args()
c = CONFIGS[a.config]
s = P.build_system(c.d, c.ne, c.p, c.level)
lam_e, _ = P.choose_lambda_e(s, c.n0)
sh = P.uniform_shifts(lam_e, c.slices)
sym = Symbolic.on_device(s.device, P.separator_ordering(s))
f = numeric_factor(sym, float(sh[len(sh) // 2]))
print("factor ms", f.device_ms, "TF/s", f.factor_flops / f.device_ms / 1e9)
if not a.factor_only:
    st = P.LanczosState(DeviceShiftInvert(f, s.M), s.dof_count, mass=s.M, shift=f.sigma, max_dim=a.steps + 1,
                        rng=np.random.default_rng(0))
    P.lanczos_extend(st, a.steps)
    x = torch.randn(s.dof_count, dtype=torch.float64, device="cuda")
    rows = ctypes.c_int64()
    for _ in range(a.probes):
        _lib.check(_lib.lib().riga_lanczos_cgs_probe(st.handle, _lib.ptr(x), 2, ctypes.byref(rows)))
    torch.cuda.synchronize()
    print("ok k", st.k, "rows", rows.value)
