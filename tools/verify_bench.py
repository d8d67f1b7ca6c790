"""EV/EFL/EFE table of a whole cfg3 solve (2000 eigenpairs): device
error_table vs the same contractions on the host (the reference's
algorithm; its ErrorEvaluator is host numpy, ref verify.py:181-338)."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_08167_b200 as P  # noqa: E402
from paper_2009_08167_b200 import verify as V  # noqa: E402
from paper_2009_08167_b200.configs import CONFIGS  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
s = P.build_system(c.d, c.ne, c.p, c.level)
lam_e, cnt = P.choose_lambda_e(s, c.n0)
r = P.solve_uniform_slices(s, P.uniform_shifts(lam_e, c.slices), streams=16, vectors_to_host=False)
lams = np.concatenate([r.local_eigenvalues[k] for k in sorted(r.local_eigenvalues)])
X = torch.cat([r.local_vectors[k] for k in sorted(r.local_vectors)]).T  # columns = eigenvectors (device)
order = np.argsort(lams, kind="stable")
lams, X = lams[order], X[:, torch.as_tensor(order, device=X.device)]
out = {"config": c.name, "eigenpairs": int(lams.size)}
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    recs = V.error_table(lams, X, s)
    torch.cuda.synchronize()
    out["device_s"] = time.perf_counter() - t0
mask = [i for i, rr in enumerate(recs) if not np.isnan(rr.efl)]
out["unique_modes"] = len(mask)
out["max_ev"] = float(max(rr.ev for rr in recs))
out["max_efl"] = float(max(recs[i].efl for i in mask))
# host evaluation of the same EFLs (reference algorithm on the CPU)
ev = V.ErrorEvaluator(s, device="cpu")
modes = V.exact_spectrum(s.dim, count=lams.size)
Xh = X.cpu().numpy()
t0 = time.perf_counter()
n, uniq, C = V._aligned_batch(lams, Xh, modes, type("S", (), {"M": type("M", (), {"csr": s.M.csr})(), "dim": s.dim,
                                                               "dof_count": s.dof_count, "spaces": s.spaces})(), ev)
host = []
for q, i in enumerate(uniq):
    host.append(ev.l2_error_sq(C[q].numpy(), modes[i]))
out["host_s"] = time.perf_counter() - t0
out["host_vs_device_max_rel"] = float(max(abs(h - recs[i].efl) / recs[i].efl for h, i in zip(host, uniq)))
print(json.dumps(out))
