"""Aggregate Lanczos-step throughput with T host threads x T streams.

    python tools/concurrency_probe.py [--config cfg3] [--steps 100]
"""
import argparse
import os
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2009_08167_b200 as P  # noqa: E402
from paper_2009_08167_b200 import device as D  # noqa: E402
from paper_2009_08167_b200.configs import CONFIGS  # noqa: E402
from paper_2009_08167_b200.eigensolver import DeviceShiftInvert  # noqa: E402
from paper_2009_08167_b200.sparsela import Symbolic, numeric_factor  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--what", default="extend", choices=["extend", "solve", "solveg"])
    ap.add_argument("--threads", default="1,2,4,8,16")
    ap.add_argument("--prelock", type=int, default=0, help="lock this many random rows first (R = k + locked)")
    ap.add_argument("--cycles", type=int, default=1, help="extend cycles per thread (thick restart keep 8 between)")
    a = ap.parse_args()
    c = CONFIGS[a.config]
    s = P.build_system(c.d, c.ne, c.p, c.level)
    lam_e, _ = P.choose_lambda_e(s, c.n0)
    sh = P.uniform_shifts(lam_e, c.slices)
    sym = Symbolic.on_device(s.device, P.separator_ordering(s))
    for T in [int(t) for t in a.threads.split(",")]:
        ctxs = [D.Context() for _ in range(T)]
        facts, states = [], []
        for i, ctx in enumerate(ctxs):
            with ctx:
                f = numeric_factor(sym, float(sh[i % c.slices]), ctx)
                st = P.LanczosState(DeviceShiftInvert(f, s.M), s.dof_count, mass=s.M, shift=f.sigma,
                                    max_dim=a.steps + 1, rng=np.random.default_rng(i), ctx=ctx)
                if a.prelock:
                    g = torch.Generator(device="cuda").manual_seed(i)
                    X = torch.randn(a.prelock, s.dof_count, dtype=torch.float64, device="cuda", generator=g)
                    X /= X.norm(dim=1, keepdim=True)
                    for q in range(a.prelock):
                        st.lock(X[q], X[q])
                facts.append(f)
                states.append(st)
        torch.cuda.synchronize()
        bar = threading.Barrier(T)
        graphs = [None] * T
        if a.what == "solveg":
            # a CUDA graph of 20 solves per stream: the device cost, not the host launches
            for i in range(T):
                with ctxs[i]:
                    b = torch.randn(s.dof_count, dtype=torch.float64, device="cuda")
                    x = torch.empty_like(b)
                    facts[i].solve_device(b, x)
                    ctxs[i].synchronize()
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=ctxs[i].stream, capture_error_mode="thread_local"):
                        for _ in range(20):
                            facts[i].solve_device(b, x)
                    graphs[i] = (g, b, x)
            torch.cuda.synchronize()

        def work(i):
            bar.wait()
            with ctxs[i]:
                if a.what == "extend":
                    for cyc in range(a.cycles):
                        if cyc:
                            P.thick_restart(states[i], 8)
                        P.lanczos_extend(states[i], a.steps)
                elif a.what == "solveg":
                    for _ in range(a.steps // 20):
                        graphs[i][0].replay()
                else:
                    b = torch.randn(s.dof_count, dtype=torch.float64, device="cuda")
                    x = torch.empty_like(b)
                    for _ in range(a.steps):
                        facts[i].solve_device(b, x)
                ctxs[i].synchronize()

        th = [threading.Thread(target=work, args=(i,)) for i in range(T)]
        prof = os.environ.get("PROBE_PROFILE_RANGE") == "1"
        if prof:
            torch.cuda.synchronize()
            torch.cuda.profiler.start()
        t0 = time.perf_counter()
        for t in th:
            t.start()
        for t in th:
            t.join()
        dt = time.perf_counter() - t0
        if prof:
            torch.cuda.synchronize()
            torch.cuda.profiler.stop()
        tot = T * (a.steps + (a.cycles - 1) * (a.steps - 8)) if a.what == "extend" else T * a.steps
        print(f"{a.what} threads={T:2d} cycles={a.cycles}: {tot / dt:8.1f} steps/s aggregate, "
              f"{dt * 1e3 / a.steps:7.3f} ms per step per thread", flush=True)
        del facts, states, ctxs
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
