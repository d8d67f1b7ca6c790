"""One numeric factorization of a config at its first uniform shift, the second
of two (the first warms up); under ncu use --profile-from-start off.

    python tools/one_factor.py cfg5
"""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_08167_b200 as P  # noqa: E402
from paper_2009_08167_b200.configs import CONFIGS  # noqa: E402
from paper_2009_08167_b200.sparsela import Symbolic, numeric_factor  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg5"]
s = P.build_system(c.d, c.ne, c.p, c.level)
lam_e, _ = P.choose_lambda_e(s, c.n0)
sh = P.uniform_shifts(lam_e, c.slices)
sym = Symbolic.on_device(s.device, P.separator_ordering(s))
sig = float(sh[1])
f = numeric_factor(sym, sig)
del f
torch.cuda.synchronize()
torch.cuda.profiler.start()
f = numeric_factor(sym, sig)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("factor ms", f.device_ms, "nneg", f.n_negative, "flops", sym.stats["factor_flops"])
