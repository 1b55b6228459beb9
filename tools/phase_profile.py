"""Split an ncu SASS source page (CSV) of k_train_fused into the phases delimited by
the CS2R clock reads / barriers; per phase: warp-instructions and shared wavefronts per
CTA-iteration, stall mix.  usage: python tools/phase_profile.py s.csv CTAS ITERS"""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
norm = float(sys.argv[2]) * float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]; data = [r for r in rows[hi + 1:] if len(r) == len(h)]
c = {k: i for i, k in enumerate(h)}
E = c["Instructions Executed"]; S = c["Warp Stall Sampling (All Samples)"]; src = c["Source"]
W = c["L1 Wavefronts Shared"]
stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
ts = sum(float(r[S]) for r in data)
acc_e = acc_s = acc_w = 0.0; last = 0; st = Counter()
for i, r in enumerate(data):
    acc_e += float(r[E]); acc_s += float(r[S]); acc_w += float(r[W] or 0)
    for k in stall_cols: st[k[6:]] += float(r[c[k]] or 0)
    if ('CS2R' in r[src] and 'CLOCK' in r[src]) or 'BAR.SYNC' in r[src] or 'EXIT' in r[src]:
        if acc_s > 0.002 * ts:
            print(f"{last:5d}-{i:5d} instr {acc_e/norm:7.0f} wf {acc_w/norm:6.0f} samples {100*acc_s/ts:5.1f}% ",
                  " ".join(f"{k}={100*v/max(acc_s,1):.0f}" for k, v in st.most_common(4)))
        acc_e = acc_s = acc_w = 0.0; last = i; st = Counter()
