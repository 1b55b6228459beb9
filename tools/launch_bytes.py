"""Per-launch time and DRAM bytes from an ncu --csv launch list with gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum.  usage: python tools/launch_bytes.py list.csv"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
H = rows[h]
col = {k: i for i, k in enumerate(H)}
d = {}
for r in rows[h + 1:]:
    if len(r) != len(H):
        continue
    key = (int(r[col["ID"]]), r[col["Kernel Name"]].split("(")[0])
    d.setdefault(key, {})[r[col["Metric Name"]]] = float(r[col["Metric Value"]].replace(",", ""))
print(f"{'id':>3} {'kernel':58s} {'us':>9} {'MB read':>9} {'MB write':>9} {'GB/s':>7}")
for (i, name), m in sorted(d.items()):
    t = m["gpu__time_duration.sum"] * 1e-3
    rd, wr = m["dram__bytes_read.sum"] / 1e6, m["dram__bytes_write.sum"] / 1e6
    print(f"{i:3d} {name[-58:]:58s} {t:9.1f} {rd:9.1f} {wr:9.1f} {(rd + wr) / t * 1e3 if t else 0:7.0f}")
