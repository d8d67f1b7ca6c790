"""Build an m-step Lanczos basis of the middle cfg3 slice, then run
`--probes` CGS2 probes against it (for ncu of the Gram-Schmidt kernels)."""
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
ap.add_argument("--m", type=int, default=250)
ap.add_argument("--probes", type=int, default=3)
ap.add_argument("--dcgs", action="store_true", help="the step's delayed-CGS2 sweeps instead of classic passes")
a = ap.parse_args()
c = CONFIGS[a.config]
s = P.build_system(c.d, c.ne, c.p, c.level)
lam_e, _ = P.choose_lambda_e(s, c.n0)
sh = P.uniform_shifts(lam_e, c.slices)
sym = Symbolic.on_device(s.device, P.separator_ordering(s))
f = numeric_factor(sym, float(sh[len(sh) // 2]))
st = P.LanczosState(DeviceShiftInvert(f, s.M), s.dof_count, mass=s.M, shift=f.sigma, max_dim=a.m + 1,
                    rng=np.random.default_rng(0))
P.lanczos_extend(st, a.m)
x = torch.randn(s.dof_count, dtype=torch.float64, device="cuda")
rows = ctypes.c_int64(0)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(a.probes):
    if a.dcgs:
        _lib.check(_lib.lib().riga_lanczos_dcgs_probe(st.handle, _lib.ptr(x), ctypes.byref(rows)))
    else:
        _lib.check(_lib.lib().riga_lanczos_cgs_probe(st.handle, _lib.ptr(x), 2, ctypes.byref(rows)))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
torch.cuda.synchronize()
print("rows", rows.value)
if os.environ.get("TIME_DCGS"):
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    ts = []
    for _ in range(20):
        flush.sum()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st.ctx.stream)
        _lib.check(_lib.lib().riga_lanczos_dcgs_probe(st.handle, _lib.ptr(x), ctypes.byref(rows)))
        e1.record(st.ctx.stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    by = 2.0 * rows.value * s.dof_count * 8 + 6.0 * s.dof_count * 8
    print(f"dcgs R={rows.value}: {ms * 1e3:.1f} us  {by / ms / 1e6:.0f} GB/s")
