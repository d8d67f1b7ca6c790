"""sha256 of D and of the exported L values of a few factorizations (A/B of factorization kernels: RIGA_LIB)."""
import hashlib
import sys
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_08167_b200 as P  # noqa: E402
from paper_2009_08167_b200.sparsela import Symbolic, numeric_factor  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


for cfg, sig in [((2, 16, 2, 0), 50.0), ((2, 64, 3, 3), 700.0), ((2, 64, 3, 0), 700.0), ((3, 8, 2, 1), 100.0),
                 ((2, 256, 4, 4), 12000.0), ((3, 32, 2, 2), 600.0)]:
    s = P.build_system(*cfg)
    sym = Symbolic.on_device(s.device, P.separator_ordering(s))
    f = numeric_factor(sym, sig)
    print(cfg, sig, "nneg", f.n_negative, "D", sha(f.D), "L", sha(f._export()[2]), "ms", round(f.device_ms, 3))
