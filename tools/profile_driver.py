"""Host-side profile of one slice solve (cProfile), to find driver overheads.

    python tools/profile_driver.py [--config cfg3] [--slice 8]
"""
import argparse
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2009_08167_b200 as P  # noqa: E402
from paper_2009_08167_b200.configs import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--slice", type=int, default=8)
    a = ap.parse_args()
    c = CONFIGS[a.config]
    s = P.build_system(c.d, c.ne, c.p, c.level)
    lam_e, cnt = P.choose_lambda_e(s, c.n0)
    sh = P.uniform_shifts(lam_e, c.slices)
    k = a.slice
    # warm
    P.solve_slice(s, (sh[0], sh[1] * 0.05 + sh[0] * 0.95), seed=0, m=20)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    r = P.solve_slice(s, (sh[k], sh[k + 1]), seed=k, m=2 * 130)
    torch.cuda.synchronize()
    pr.disable()
    dt = time.perf_counter() - t0
    print(f"slice {k}: {r.eigenvalues.size} eigenpairs in {dt:.3f} s; nfb {r.counters.nfb} nit {r.counters.nit}")
    pstats.Stats(pr).sort_stats("cumulative").print_stats(45)


if __name__ == "__main__":
    main()
