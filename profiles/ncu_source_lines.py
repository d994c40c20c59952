"""Aggregate ncu source-page samples / executed instructions per CUDA source line of one kernel.

usage: python profiles/ncu_source_lines.py REP KERNEL_SUBSTR [top]
"""
import csv
import subprocess
import sys


def main(rep, kname, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                          "-k", "regex:" + kname], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    h = rows[hi]
    si = h.index("Warp Stall Sampling (All Samples)")
    ei = h.index("Instructions Executed")
    stall_cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    agg = []
    cur = None
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        if r[0] and not r[0].isdigit():
            cur = None
            continue
        if r[0]:
            cur = [int(r[0]), r[1][:90], 0, 0, {}]
            agg.append(cur)
        elif cur is not None:
            try:
                cur[2] += int(r[si])
                cur[3] += int(r[ei])
                for i, c in stall_cols:
                    v = int(r[i])
                    if v:
                        cur[4][c] = cur[4].get(c, 0) + v
            except ValueError:
                pass
    tot = sum(a[2] for a in agg) or 1
    toti = sum(a[3] for a in agg) or 1
    print(f"samples {tot}, warp instructions {toti}")
    for ln, srcl, smp, ins, st in sorted(agg, key=lambda a: -a[2])[:top]:
        tops = ",".join(f"{k[6:]}={v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3])
        print(f"{ln:5d} {100*smp/tot:5.1f}% ins {100*ins/toti:5.1f}%  {srcl.strip()[:70]:70s} {tops}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
