#!/bin/bash
# per-kernel duration / DRAM bytes of the Gram-Schmidt kernels at m=250 (ncu, after a plain run)
python tools/one_cgs.py > gpurun_out/oc.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size --clock-control none -k regex:k_cgs --csv --log-file gpurun_out/cgs_metrics.csv python tools/one_cgs.py --probes 2 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/cgs_metrics.csv')))
hdr=None; data=[]
for r in rows:
    if r and r[0]=="ID": hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
by=collections.OrderedDict()
for d in data:
    by.setdefault(d["ID"],{"name":d["Kernel Name"].split("(")[0]})[d["Metric Name"]]=d["Metric Value"]
for v in list(by.values())[-4:]:
    t=float(v["gpu__time_duration.sum"]); b=float(v["dram__bytes_read.sum"])+float(v["dram__bytes_write.sum"])
    print("%-16s grid=%-6s t=%7.1fus dram=%7.1fMB  %6.0f GB/s occ=%s" % (v["name"], v["launch__grid_size"], t/1e3, b/1e6, b/t, v["sm__warps_active.avg.pct_of_peak_sustained_active"]))
PY
