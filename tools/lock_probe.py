"""Device time of the locking kernels (lift of c Ritz vectors, block
Gram-Schmidt against nl locked rows) at cfg3 sizes, isolated on one stream."""
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

c = CONFIGS["cfg3"]
s = P.build_system(c.d, c.ne, c.p, c.level)
lam_e, _ = P.choose_lambda_e(s, c.n0)
sh = P.uniform_shifts(lam_e, c.slices)
sym = Symbolic.on_device(s.device, P.separator_ordering(s))
f = numeric_factor(sym, float(sh[8]))
n = s.dof_count
st = P.LanczosState(DeviceShiftInvert(f, s.M), n, mass=s.M, shift=f.sigma, max_dim=251,
                    rng=np.random.default_rng(0))
P.lanczos_extend(st, 250)
L = _lib.lib()


def ev(fn, reps=5):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st.ctx.stream)
        fn()
        e1.record(st.ctx.stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


for cc in (8, 40, 100):
    W = np.random.default_rng(1).standard_normal((st.k, cc))
    t = ev(lambda: st.lift_many(W))
    print(f"lift k={st.k} c={cc}: {t:.3f} ms  ({2 * 2 * st.k * cc * n / t / 1e9:.2f} TF/s)")
# lock blocks against a growing locked set
X, MX = st.lift_many(np.random.default_rng(2).standard_normal((st.k, 40)))
nrm = np.zeros(40)
for nl in (0, 60, 120):
    while st.nlocked < nl:
        st.lock(X[st.nlocked % 40], MX[st.nlocked % 40])
    Xc, MXc = X.clone(), MX.clone()
    t = ev(lambda: _lib.check(L.riga_lanczos_lock_block(st.handle, _lib.ptr(Xc), _lib.ptr(MXc), 40, st.ld,
                                                         _lib.ptr(nrm))), reps=3)
    print(f"lock_block c=40 nlocked={st.nlocked}: {t:.3f} ms")
