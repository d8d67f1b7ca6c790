"""Aggregate an ncu --csv launch list (gpu__time_duration.sum [+ DMMA pipe %]) by kernel name.

    python tools/agg_launches.py gpurun_out/factor_cfg5_r2.csv
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.defaultdict(dict)
names = {}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    per[r[ii]][r[mi]] = v
    names[r[ii]] = r[ki].split("(")[0].replace("void ", "")
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i, m in per.items():
    t = m.get("gpu__time_duration.sum", 0.0)
    a = agg[names[i]]
    a[0] += 1
    a[1] += t
    a[2] += t * m.get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0) / 100
    a[3] += m.get("sm__inst_executed_pipe_tensor_subpipe_dmma.sum", 0.0)
tot = sum(v[1] for v in agg.values())
print(f"total {tot / 1e6:.2f} ms over {sum(v[0] for v in agg.values())} launches")
print(f"{'kernel':44s} {'n':>6s} {'ms':>9s} {'share':>6s} {'dmma%':>6s} {'TF/s(dmma)':>10s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    # DMMA.8x8x4: 8*8*4 FMA = 512 flops per warp instruction
    tf = v[3] * 512 / (v[1] * 1e-9) / 1e12 if v[1] else 0.0
    print(f"{k[:44]:44s} {v[0]:6d} {v[1] / 1e6:9.3f} {100 * v[1] / tot:5.1f}% {100 * v[2] / max(v[1], 1e-9):6.1f} {tf:10.2f}")
