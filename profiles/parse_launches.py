"""Summarise an ncu --csv launch list (gpu__time_duration + optional DRAM/inst metrics) per kernel."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    idi = h.index("ID")
    launches = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        key = (r[idi], r[ki])
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        if u == "usecond":
            v *= 1e3
        elif u == "msecond":
            v *= 1e6
        elif u == "Kbyte":
            v *= 1e3
        elif u == "Mbyte":
            v *= 1e6
        elif u == "Gbyte":
            v *= 1e9
        launches.setdefault(key, {})[r[mi]] = v
    return launches


def main(path, top=25):
    launches = load(path)
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    for (_, name), m in launches.items():
        a = agg[name[:70]]
        a["count"] += 1
        for k, v in m.items():
            a[k] += v
    total = sum(a.get("gpu__time_duration.sum", 0) for a in agg.values())
    print(f"{len(launches)} launches, {total/1e6:.3f} ms total")
    for name, a in sorted(agg.items(), key=lambda x: -x[1].get("gpu__time_duration.sum", 0))[:top]:
        t = a.get("gpu__time_duration.sum", 0)
        dr = a.get("dram__bytes_read.sum", 0) + a.get("dram__bytes_write.sum", 0)
        inst = a.get("smsp__inst_executed.sum", 0)
        print(f"{t/1e6:9.3f} ms {100*t/total:5.1f}% n={int(a['count']):4d} dram={dr/1e6:9.1f} MB "
              f"GB/s={dr/t if t else 0:8.1f} inst={inst/1e6:8.1f}M  {name}")


if __name__ == "__main__":
    main(sys.argv[1])
