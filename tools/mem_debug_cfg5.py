import sys, os, gc, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2009_08167_b200 as P
from paper_2009_08167_b200 import device as D
from paper_2009_08167_b200.configs import CONFIGS
from paper_2009_08167_b200.sparsela import Symbolic, numeric_factor
GB = 1e9
def mem(tag):
    torch.cuda.synchronize()
    m = D.mem_info(0)
    f, t = torch.cuda.mem_get_info()
    print(f"{tag:28s} pool used {m['used']/GB:7.2f} high {m['used_high']/GB:7.2f} reserved {m['reserved']/GB:7.2f} | torch alloc {torch.cuda.memory_allocated()/GB:6.2f} reserved {torch.cuda.memory_reserved()/GB:6.2f} | device free {f/GB:7.2f} of {t/GB:7.2f}", flush=True)
c = CONFIGS["cfg5"]
mem("start")
s = P.build_system(c.d, c.ne, c.p, c.level)
mem("build_system")
perm = P.separator_ordering(s)
sym = Symbolic.on_device(s.device, perm)
mem("symbolic")
f = numeric_factor(sym, 0.0)
mem("factor 1")
g = numeric_factor(sym, 100.0)
mem("factor 2")
del f, g; gc.collect()
mem("del factors")
lam = P.kronecker_spectrum(s)
lam_e, _ = P.choose_lambda_e(s, c.n0, lam)
sh = P.uniform_shifts(lam_e, c.slices)
r = P.solve_slice(s, (float(sh[0]), float(sh[1])), seed=0, m=22)
mem("slice 0")
del r; gc.collect()
mem("del slice 0")
