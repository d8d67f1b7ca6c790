"""Host-side pieces of the e2e path (upload, ordering, symbolic + plans) timed."""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_08167_b200 as P  # noqa
from paper_2009_08167_b200 import device as D  # noqa
from paper_2009_08167_b200.assembly import DeviceSystem, DiscreteSystem, SymSparseMatrix  # noqa
from paper_2009_08167_b200.configs import CONFIGS  # noqa
from paper_2009_08167_b200.sparsela import Symbolic  # noqa
c = CONFIGS["cfg3"]
system = P.build_system(c.d, c.ne, c.p, c.level)
Kh, Mh = system.K.csr.copy(), system.M.csr.copy()
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dsys = DeviceSystem.upload(D.current(), Kh, Mh); dsys.attach_kron(system.k1d, system.m1d)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    sys2 = DiscreteSystem(SymSparseMatrix(device=dsys, which=0), SymSparseMatrix(device=dsys, which=1),
                          system.spaces, system.dim, system.dof_count, system.k1d, system.m1d, dsys)
    perm = P.separator_ordering(sys2); t2 = time.perf_counter()
    sym = Symbolic.on_device(dsys, perm); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.1f} ms  ordering {1e3*(t2-t1):.1f} ms  symbolic+plans+upload {1e3*(t3-t2):.1f} ms")
