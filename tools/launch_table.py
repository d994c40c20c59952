#!/usr/bin/env python
"""Print an ncu --csv launch list (gpu__time_duration [+ dram bytes]) as a table."""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
L = {}
for r in rows[hi + 1:]:
    d = dict(zip(h, r))
    L.setdefault(d["ID"], {"n": d["Kernel Name"], "g": d["Grid Size"]})[d["Metric Name"]] = d["Metric Value"]
tot = 0
for i, v in L.items():
    t = float(v["gpu__time_duration.sum"].replace(",", "")) / 1e3
    tot += t
    n = v["n"].replace("void ", "")
    m = re.search(r"instance (\d+)", n)
    dr = ""
    if "dram__bytes_read.sum" in v:
        dr = f"dram {(float(v['dram__bytes_read.sum'].replace(',', '')) + float(v['dram__bytes_write.sum'].replace(',', ''))) / 1e6:7.1f} MB"
    print(f"{i:>3} {t:8.1f}us grid {v['g']:>14} {dr} {n[:60]} {('inst ' + m.group(1)) if m else ''}")
print(f"total {tot:.1f} us over {len(L)} launches")
