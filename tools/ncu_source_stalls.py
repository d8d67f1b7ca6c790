"""Aggregate an `ncu --page source --csv` export by SASS opcode: stall samples, instruction counts, top stall reasons.

    ncu -i rep.ncu-rep --page source --csv > src.csv; python tools/ncu_source_stalls.py src.csv
"""
import csv,collections,sys
rows=list(csv.reader(open(sys.argv[1])))
h=rows[1]; ix={n:i for i,n in enumerate(h)}
data=[r for r in rows[2:] if len(r)>=len(h)-2]
def I(r,k):
    try: return int(r[ix[k]] or 0)
    except: return 0
tot=sum(I(r,"# Samples") for r in data); print("samples",tot, "instr", sum(I(r,"Instructions Executed") for r in data))
agg=collections.Counter(); cnt=collections.Counter(); st=collections.defaultdict(collections.Counter)
for r in data:
    t=r[ix["Source"]].split(); op=t[0] if t else ''
    if op.startswith('@') and len(t)>1: op=t[1]
    op=op.split('.')[0]; n=I(r,"# Samples"); agg[op]+=n; cnt[op]+=I(r,"Instructions Executed")
    for k in h:
        if k.startswith("stall_") and "Not Issued" not in k: st[op][k]+=I(r,k)
for op,n in agg.most_common(12): print(op,n,"%.1f%%"%(100*n/max(tot,1)),"inst",cnt[op],dict(st[op].most_common(3)))
