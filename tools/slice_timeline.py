"""Per-slice wall-clock timeline of one cfg3 solve_uniform_slices call."""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_08167_b200 as P  # noqa
from paper_2009_08167_b200.configs import CONFIGS  # noqa
from paper_2009_08167_b200.sparsela import Symbolic  # noqa
c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
streams = int(sys.argv[2]) if len(sys.argv) > 2 else 16
s = P.build_system(c.d, c.ne, c.p, c.level)
lam_e, cnt = P.choose_lambda_e(s, c.n0)
sh = P.uniform_shifts(lam_e, c.slices)
perm = P.separator_ordering(s)
from paper_2009_08167_b200.slicing import solve_plan, solve_sub_levels  # noqa: E402
with solve_plan(solve_sub_levels(min(streams, c.slices))):  # the plan the slice driver builds
    sym = Symbolic.on_device(s.device, perm)
import gc
if os.environ.get('NOGC'):
    gc.disable()
for it in range(int(sys.argv[3]) if len(sys.argv) > 3 else 2):
    t0 = time.perf_counter()
    c0 = os.times()
    r = P.solve_uniform_slices(s, sh, streams=streams, pencil_symbolic=sym, perm=perm)
    print("total", round(time.perf_counter() - t0, 3), "boundary", round(r.timings["boundary_s"], 3),
          "slices", round(r.timings["slices_s"], 3), "nfb", r.counters.nfb,
          "streams", r.timings.get("streams_used"), "kept", r.timings.get("kept_boundary_factors"),
          "cpu_s", round((os.times().user - c0.user) + (os.times().system - c0.system), 2))
    print("   phases", {k: round(v, 2) for k, v in r.counters.phase_s.items() if k != "cgs_rows"})
    sw = r.timings["slice_wall"]
    print("   ends:", " ".join(f"{k}:{v[1]:.2f}" for k, v in sorted(sw.items(), key=lambda kv: kv[1][1])))
print(json.dumps(r.timings["slice_wall"]))
print("nfb per slice", json.dumps(r.timings.get("slice_nfb")))
print("phase seconds summed over slices", {k: round(v, 3) for k, v in r.counters.phase_s.items()})
if r.counters.trace and len(r.counters.trace) < 100000:
    # slices per phase over time (50 ms bins, relative to the first event)
    tr = r.counters.trace
    t0 = min(e[1] for e in tr)
    t1 = max(e[2] for e in tr)
    names = sorted({n for n, *_ in tr})
    nb = int((t1 - t0) / 0.05) + 1
    occ = {n: np.zeros(nb) for n in names}
    rate = np.zeros(nb)
    for n, a, b, _, st in tr:
        if st and b > a:  # steps spread uniformly over the extend call
            for i in range(nb):
                lo, hi = t0 + 0.05 * i, t0 + 0.05 * (i + 1)
                ov = min(b, hi) - max(a, lo)
                if ov > 0:
                    rate[i] += st * ov / (b - a) / 0.05
    for n, a, b, _, _ in tr:
        for i in range(nb):
            lo, hi = t0 + 0.05 * i, t0 + 0.05 * (i + 1)
            ov = min(b, hi) - max(a, lo)
            if ov > 0:
                occ[n][i] += ov / 0.05
    print("bin_ms " + " ".join(f"{n[:7]:>7s}" for n in names) + "  steps/s")
    for i in range(nb):
        print(f"{50 * i:6d} " + " ".join(f"{occ[n][i]:7.2f}" for n in names) + f" {rate[i]:8.0f}")
