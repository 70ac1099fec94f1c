import csv, sys
from collections import OrderedDict
lines=open(sys.argv[1]).read().splitlines()
start=[i for i,l in enumerate(lines) if l.startswith('"ID"')][0]
rows=list(csv.reader(lines[start:]))
hdr=rows[0]; ki=hdr.index('Kernel Name'); vi=hdr.index('Metric Value')
agg=OrderedDict()
for r in rows[1:]:
    n=r[ki].split('(')[0].replace('(anonymous namespace)::','').replace('unnamed>::','')
    agg.setdefault(n,[]).append(float(r[vi].replace(',',''))/1e3)
tot=sum(sum(v) for v in agg.values())
for k,v in agg.items(): print(f"{k[:55]:55s} n={len(v):3d} mean_us={sum(v)/len(v):9.1f} share={sum(v)/tot:.3f}")
