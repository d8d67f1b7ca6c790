"""Which engine objects survive a solve_uniform_slices call, and who holds them."""
import gc
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_08167_b200 as P  # noqa: E402
from paper_2009_08167_b200 import eigensolver as E, sparsela as SL  # noqa: E402
from paper_2009_08167_b200.configs import CONFIGS  # noqa: E402

c = CONFIGS["cfg1"]
s = P.build_system(c.d, c.ne, c.p, c.level)
lam_e, _ = P.choose_lambda_e(s, c.n0)
sh = P.uniform_shifts(lam_e, 2)
r = P.solve_uniform_slices(s, sh, streams=2)
del r
gc.collect()
for cls in (SL.LDLFactorization, E.LanczosState):
    objs = [o for o in gc.get_objects() if isinstance(o, cls)]
    print(cls.__name__, "alive:", len(objs))
    for o in objs[:2]:
        for ref in gc.get_referrers(o):
            if ref is objs:
                continue
            d = type(ref).__name__
            keys = [k for k, v in ref.items() if v is o][:3] if isinstance(ref, dict) else ""
            print("   referrer", d, keys, str(ref)[:150].replace("\n", " "))
