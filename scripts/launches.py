"""Summarise an ncu --csv launch list: per-kernel duration and DRAM bytes (last N launches)."""
import csv
import sys
from collections import OrderedDict

path = sys.argv[1]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 16
rows = list(csv.reader(open(path)))
hdr = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hdr]
idx = {k: j for j, k in enumerate(h)}
d = OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) < len(h):
        continue
    key = (int(r[idx["ID"]]), r[idx["Kernel Name"]].split("(")[0][:48], r[idx["Grid Size"]])
    d.setdefault(key, {})[r[idx["Metric Name"]]] = float(r[idx["Metric Value"]].replace(",", ""))
keys = list(d)[-last:]
tot = sum(d[k].get("gpu__time_duration.sum", 0) for k in keys)
for k in keys:
    m = d[k]
    t = m.get("gpu__time_duration.sum", 0)
    rd = m.get("dram__bytes_read.sum", 0)
    wr = m.get("dram__bytes_write.sum", 0)
    bw = (rd + wr) / t if t else 0
    print(f"{k[1]:48s} {k[2]:>14s} {t/1e3:8.2f} us  {100*t/tot:5.1f}%  dram {(rd+wr)/1e6:8.2f} MB  {bw:6.0f} GB/s")
print(f"total {tot/1e3:.2f} us")
