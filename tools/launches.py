import csv, sys
from collections import defaultdict
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
hdr=rows[0]; iname=hdr.index('Kernel Name'); iv=hdr.index('Metric Value'); iu=hdr.index('Metric Unit')
agg=defaultdict(lambda:[0,0.0])
for r in rows[1:]:
    v=float(r[iv].replace(',','')); u=r[iu]
    us = v/1e3 if u=='nsecond' else (v if u=='usecond' else (v*1e3 if u=='msecond' else v))
    name=r[iname].split('(')[0][:70]
    agg[name][0]+=1; agg[name][1]+=us
tot=sum(v[1] for v in agg.values())
print('total us', round(tot,1))
for k,v in sorted(agg.items(), key=lambda x:-x[1][1]): print(f"{k:70s} {v[0]:5d} {v[1]:10.1f} {v[1]/v[0]:8.1f}")
