"""Engine pool / torch memory across repeated solve_uniform_slices calls."""
import gc
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2009_08167_b200 as P  # noqa: E402
from paper_2009_08167_b200 import device as D  # noqa: E402
from paper_2009_08167_b200.configs import CONFIGS  # noqa: E402
from paper_2009_08167_b200.sparsela import Symbolic  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
collect = len(sys.argv) > 2 and sys.argv[2] == "gc"
s = P.build_system(c.d, c.ne, c.p, c.level)
lam_e, _ = P.choose_lambda_e(s, c.n0)
sh = P.uniform_shifts(lam_e, c.slices)
perm = P.separator_ordering(s)
sym = Symbolic.on_device(s.device, perm)
GB = 1e9
for it in range(5):
    r = P.solve_uniform_slices(s, sh, streams=16, pencil_symbolic=sym, perm=perm)
    del r
    if collect:
        gc.collect()
    torch.cuda.synchronize()
    m = D.mem_info(0, reset_high=True)
    print(it, "pool used %.2f GB (high %.2f) reserved %.2f GB (high %.2f)" % (
        m["used"] / GB, m["used_high"] / GB, m["reserved"] / GB, m["reserved_high"] / GB),
        "torch alloc %.2f reserved %.2f GB" % (torch.cuda.memory_allocated() / GB, torch.cuda.memory_reserved() / GB),
        "gc objs", len(gc.get_objects()), flush=True)
