"""Wall time of T concurrent cfg3 boundary factorizations (one host thread + context each), repeated: where the
boundary pass of a step goes."""
import os
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_08167_b200 as P  # noqa: E402
from paper_2009_08167_b200 import device as D  # noqa: E402
from paper_2009_08167_b200.configs import CONFIGS  # noqa: E402
from paper_2009_08167_b200.sparsela import Symbolic, numeric_factor  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
s = P.build_system(c.d, c.ne, c.p, c.level)
lam_e, _ = P.choose_lambda_e(s, c.n0)
sh = P.uniform_shifts(lam_e, c.slices)
sym = Symbolic.on_device(s.device, P.separator_ordering(s))
for T in (1, 4, 8, 17):
    ctxs = [D.Context() for _ in range(T)]
    jobs = list(range(len(sh)))
    for rep in range(3):
        q = list(jobs)
        lock = threading.Lock()
        dev_ms = []
        host_ms = []

        def work(i):
            with ctxs[i]:
                while True:
                    with lock:
                        if not q:
                            return
                        k = q.pop()
                    t0 = time.perf_counter()
                    f = numeric_factor(sym, float(sh[k]), ctxs[i])
                    ctxs[i].synchronize()
                    host_ms.append((time.perf_counter() - t0) * 1e3)
                    dev_ms.append(f.device_ms)
                    del f

        torch.cuda.synchronize()
        t0 = time.perf_counter()
        th = [threading.Thread(target=work, args=(i,)) for i in range(T)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
    print(f"T={T:2d}: {len(sh)} factorizations in {wall:6.1f} ms wall; per factorization device {sum(dev_ms) / len(dev_ms):5.1f} ms, "
          f"host call {sum(host_ms) / len(host_ms):5.1f} ms")
