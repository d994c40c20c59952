"""Print the key ncu --set full metrics of each captured launch (ncu -i rep --page details --csv)."""
import csv
import subprocess
import sys

KEEP = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
        "Registers Per Thread", "Theoretical Occupancy", "Issued Warp Per Scheduler", "No Eligible",
        "Active Warps Per Scheduler", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Executed Instructions", "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size",
        "Block Size", "Static Shared Memory Per Block", "Waves Per SM")


def main(rep, min_us=0.0):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ii, ki, ni, vi, ui = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    launches = {}
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        launches.setdefault((r[ii], r[ki]), {})[r[ni]] = (r[vi], r[ui])
    for (i, k), m in launches.items():
        d = m.get("Duration", ("0", "us"))
        dv = float(d[0].replace(",", "")) * (1e3 if d[1] == "ms" else (1e-3 if d[1] == "ns" else 1))
        if dv < min_us:
            continue
        print(f"== launch {i}: {k[:100]}")
        for name in KEEP:
            if name in m:
                print(f"   {name:40s} {m[name][0]} {m[name][1]}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 0.0)
