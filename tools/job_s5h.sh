#!/bin/bash
# session 5: ncu launch list of 250 cfg3 Lanczos steps (the 16-slice plan, subtree height 8), share per kernel of the
# last 20 steps (k ~ 230-250)
python - <<'PY' > gpurun_out/os5.log 2>&1 || exit 1
import paper_2009_08167_b200 as P
PY
RIGA_SUB_LEVELS=8 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5_step_launches_cfg3.csv python tools/one_step.py --steps 250 --probes 0 > gpurun_out/ncu_step.log 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open('gpurun_out/s5_step_launches_cfg3.csv')))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
L = [(r[ki].split("(")[0].replace("void ", "").replace("riga::", ""), float(r[vi].replace(",", "")) / 1e3) for r in rows[hi + 1:] if len(r) > vi]
# the step starts with k_perm_row; take the last 20 steps
starts = [i for i, (n, t) in enumerate(L) if n.startswith("k_perm_row")]
print("launches", len(L), "steps found", len(starts))
seg = L[starts[-21]:starts[-1]]
agg = collections.OrderedDict()
for n, t in seg:
    a = agg.setdefault(n, [0, 0.0]); a[0] += 1; a[1] += t
tot = sum(a[1] for a in agg.values())
print("last 20 steps: %.1f us per step, %d kernels per step" % (tot / 20, len(seg) / 20))
for n, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print("%-28s %4.1f per step %8.1f us per step %5.1f %%" % (n[:28], a[0] / 20, a[1] / 20, 100 * a[1] / tot))
PY
