"""Last step's kernels from an ncu --csv launch list: time and DRAM bytes.

    python tools/launch_table.py launches.csv [n_last]
"""
import csv
import sys
from collections import OrderedDict

lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
ui = h.index("Metric Unit")
d = OrderedDict()
for r in rows[1:]:
    d.setdefault(r[ii], {})["k"] = r[ki][:44]
    d[r[ii]][r[mi]] = (r[vi], r[ui])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
tot = 0.0
for x in list(d.values())[-n:]:
    t = x.get("gpu__time_duration.sum", ("0", ""))
    tv = float(t[0].replace(",", "")) / (1000.0 if t[1] in ("nsecond", "ns") else 1.0)
    tot += tv
    rd = x.get("dram__bytes_read.sum", ("", ""))
    wr = x.get("dram__bytes_write.sum", ("", ""))
    print(f"{x['k']:46s} {tv:9.2f} us  rd {rd[0]:>10s} {rd[1]:6s} wr {wr[0]:>10s} {wr[1]}")
print(f"sum {tot:.2f} us")
