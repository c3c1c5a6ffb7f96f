import csv, sys
from collections import defaultdict
for f in sys.argv[1:]:
    rows=[r for r in csv.reader(open(f)) if len(r)>5]
    h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
    t=defaultdict(list)
    for r in rows[1:]: t[r[ki][:70]].append(float(r[vi].replace(',','')))
    for k,v in t.items(): print(f.split('/')[-1], k, len(v), round(sum(v[-3:])/len(v[-3:])/1000,1),'us')
