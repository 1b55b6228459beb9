"""Summarise an ncu source page (SASS view, CSV) by instruction: top stall-sample
addresses and per-opcode totals.  usage: ncu -i X.ncu-rep --page source --csv > s.csv;
python tools/sass_hot.py s.csv [top]"""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
col = {k: i for i, k in enumerate(h)}
S = col["Warp Stall Sampling (All Samples)"]
E = col["Instructions Executed"]
stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = sum(float(r[S] or 0) for r in data)
toti = sum(float(r[E] or 0) for r in data)
print(f"total samples {tot:.0f}, warp instructions {toti:.0f}")
op = defaultdict(lambda: [0.0, 0.0])
for r in data:
    o = r[col["Source"]].split()[0] if r[col["Source"]].split() else "?"
    if o.startswith("@"):
        o = r[col["Source"]].split()[1]
    op[o.split(".")[0]][0] += float(r[S] or 0)
    op[o.split(".")[0]][1] += float(r[E] or 0)
print("opcode           samples%   instr%")
for k, v in sorted(op.items(), key=lambda kv: -kv[1][0])[:20]:
    print(f"{k:16s} {100*v[0]/tot:7.2f} {100*v[1]/toti:7.2f}")
print("\ntop instructions:")
for i, r in sorted(enumerate(data), key=lambda t: -float(t[1][S] or 0))[:top]:
    st = sorted(((float(r[col[k]] or 0), k[6:]) for k in stall_cols), reverse=True)[:3]
    print(f"{i:5d} {100*float(r[S] or 0)/tot:5.2f}% ex={r[E]:>9s} {r[col['Source']][:60]:60s} " +
          " ".join(f"{n}={v:.0f}" for v, n in st))
