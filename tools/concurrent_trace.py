"""Device timeline of one concurrent solve_uniform_slices call (CUPTI via
torch.profiler): GPU-busy union, kernel time by name, mean kernel
concurrency, and per-stream busy time -- to see whether the 16-stream slice
phase is bound by device work or by host driving.

    python tools/concurrent_trace.py [cfg3] [streams]
"""
import collections
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2009_08167_b200 as P  # noqa: E402
from paper_2009_08167_b200.configs import CONFIGS  # noqa: E402
from paper_2009_08167_b200.sparsela import Symbolic  # noqa: E402


def main():
    c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
    streams = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    s = P.build_system(c.d, c.ne, c.p, c.level)
    lam_e, _ = P.choose_lambda_e(s, c.n0)
    sh = P.uniform_shifts(lam_e, c.slices)
    perm = P.separator_ordering(s)
    sym = Symbolic.on_device(s.device, perm)
    P.solve_uniform_slices(s, sh, streams=streams, pencil_symbolic=sym, perm=perm)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        r = P.solve_uniform_slices(s, sh, streams=streams, pencil_symbolic=sym, perm=perm)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    out = os.path.join(ROOT, "gpurun_out", "trace.json")
    prof.export_chrome_trace(out)
    ev = [e for e in json.load(open(out))["traceEvents"]
          if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    iv = sorted((e["ts"], e["ts"] + e["dur"]) for e in ev)
    busy, cur_s, cur_e = 0.0, None, None
    for a, b in iv:
        if cur_e is None or a > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = a, b
        else:
            cur_e = max(cur_e, b)
    if cur_e is not None:
        busy += cur_e - cur_s
    span = (iv[-1][1] - iv[0][0]) if iv else 0.0
    tot = sum(e["dur"] for e in ev)
    by = collections.Counter()
    cnt = collections.Counter()
    for e in ev:
        n = e["name"].split("(")[0].split("<")[0].replace("void ", "").replace("riga::", "")
        by[n] += e["dur"]
        cnt[n] += 1
    per_stream = collections.Counter()
    for e in ev:
        per_stream[e.get("args", {}).get("stream", -1)] += e["dur"]
    print(json.dumps({
        "wall_s": round(wall, 3), "timings": {k: v for k, v in r.timings.items() if k != "slice_wall"},
        "span_s": round(span / 1e6, 3), "gpu_busy_s": round(busy / 1e6, 3),
        "kernel_sum_s": round(tot / 1e6, 3), "mean_concurrency_when_busy": round(tot / max(busy, 1), 2),
        "n_events": len(ev),
        "by_kernel_ms": {k: [round(v / 1e3, 1), cnt[k]] for k, v in by.most_common(25)},
        "streams_busy_ms": sorted(round(v / 1e3, 1) for v in per_stream.values())[-20:],
    }, indent=1))
    os.remove(out)


if __name__ == "__main__":
    main()
