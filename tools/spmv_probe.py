"""CSR SpMV (riga_spmv, M of the cfg3 pencil) with an L2 flush before each launch."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_08167_b200 as P  # noqa
from paper_2009_08167_b200 import _lib  # noqa
from paper_2009_08167_b200.configs import CONFIGS  # noqa
c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
s = P.build_system(c.d, c.ne, c.p, c.level)
n, nnz = s.dof_count, s.K.nnz
b = torch.randn(n, dtype=torch.float64, device="cuda"); y = torch.empty_like(b)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
st = s.device.ctx.stream
ts = []
for _ in range(20):
    (flush.sum() if os.environ.get('READFLUSH') else flush.zero_()); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    _lib.check(_lib.lib().riga_spmv(s.device.handle, 1, 0.0, _lib.ptr(b), _lib.ptr(y)))
    e1.record(st); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
by = 12.0 * nnz + 4.0 * (n + 1) + 16.0 * n
ms = float(np.median(ts))
print(c.name, os.environ.get("RIGA_SPMV_LANES", "auto"), os.environ.get("RIGA_SPMV_U", "autoU"), f"avg {nnz/n:.1f}", f"{ms*1e3:.1f} us  {by/ms/1e6:.0f} GB/s")
