"""Host-side pieces of the e2e path (upload, ordering, symbolic + plans) timed.

RIGA_SYM_TIME=1 adds the C-side split of the symbolic (download / analyze / plans / upload)."""
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
import scipy.sparse as sps  # noqa

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
system = P.build_system(c.d, c.ne, c.p, c.level)
K0, M0 = system.K.csr, system.M.csr


def pinned(a, dt):
    t = torch.empty(a.size, dtype=dt, pin_memory=True)
    t.numpy()[:] = a
    return t


rp_t = pinned(np.asarray(K0.indptr, np.int32), torch.int32)
ci_t = pinned(np.asarray(K0.indices, np.int32), torch.int32)
kv_t = pinned(np.asarray(K0.data, np.float64), torch.float64)
mv_t = pinned(np.asarray(M0.data, np.float64), torch.float64)
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Kh = sps.csr_array((kv_t.numpy(), ci_t.numpy(), rp_t.numpy()), shape=K0.shape)
    Mh = sps.csr_array((mv_t.numpy(), ci_t.numpy(), rp_t.numpy()), shape=M0.shape)
    Mh.indices, Mh.indptr = Kh.indices, Kh.indptr
    ta = time.perf_counter()
    dsys = DeviceSystem.upload(D.current(), Kh, Mh)
    tb = time.perf_counter()
    dsys.attach_kron(system.k1d, system.m1d)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    sys2 = DiscreteSystem(SymSparseMatrix(device=dsys, which=0), SymSparseMatrix(device=dsys, which=1),
                          system.spaces, system.dim, system.dof_count, system.k1d, system.m1d, dsys)
    perm = P.separator_ordering(sys2)
    t2 = time.perf_counter()
    sym = Symbolic.on_device(dsys, perm)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"csr {1e3*(ta-t0):.1f} upload {1e3*(tb-ta):.1f} kron {1e3*(t1-tb):.1f} ordering {1e3*(t2-t1):.1f} "
          f"symbolic+plans+upload {1e3*(t3-t2):.1f} ms", flush=True)
    del sym, sys2, dsys
