import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if r and r[0] == 'ID'][0]
hdr = rows[h]; data = rows[h + 1:]
ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value')
agg = defaultdict(list)
for r in data:
    if len(r) > vi:
        agg[r[ki][:70]].append(float(r[vi].replace(',', '')))
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:72s} n={len(v):4d} mean_us={sum(v)/len(v)/1e3:9.2f} share={100*sum(v)/tot:5.1f}%")
