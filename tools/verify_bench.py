"""EV/EFL/EFE table of a whole cfg3 solve (2000 eigenpairs): device
error_table (engine kernels) vs the numpy restatement of the reference's
algorithm on the host (its ErrorEvaluator is host numpy, ref verify.py:181-338)."""
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
# host evaluation of the same EFLs: the numpy restatement of the reference algorithm (oracle/verify_port.py)
from oracle import rigaeig_port as O  # noqa: E402
from oracle import verify_port as VP  # noqa: E402

so = O.build_system(c.d, c.ne, c.p, c.level)
Xh = X.cpu().numpy()
t0 = time.perf_counter()
host = {i: f for i, _, _, f in VP.error_table(lams, Xh, so) if f is not None}
out["host_s"] = time.perf_counter() - t0
out["host_vs_device_max_rel"] = float(max(abs(host[i] - recs[i].efl) / recs[i].efl for i in mask))
print(json.dumps(out))
