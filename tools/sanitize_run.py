#!/usr/bin/env python
"""A compact workload for compute-sanitizer (memcheck / racecheck /
synccheck): every kernel family of the library on small inputs — window
slides through the small-batch graph and the regular pipeline (leaf tier,
lane tiers, CTA tier on hub groups, lazy and eager), the leaf-bucket front
end, the onesweep sort on multiple tiles, touched ranges, BFS, CC, PageRank,
SpMV, the device window in explicit mode — each checked against the
reference oracle so a silent corruption also fails the run."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from oracle.oracle import RefGraph, RefStream, RefWindow
    from paper_1709_05061_b200 import pmagraph as pg
    from paper_1709_05061_b200.abi import PMA_EAGER, graph_config

    ok = True
    for kind, nv, batches, mode in [("er", 1 << 12, [200, 700, 1500, 20000, 70000], 0),
                                    ("rmat", 1 << 12, [1500, 3000, 70000], PMA_EAGER)]:
        rs = RefStream.erdos_renyi(nv, 2.0 ** -3, 1).shuffle(2) if kind == "er" else RefStream.rmat(nv, 400000, 5)
        s, d, w, _ = rs.arrays()
        half = (len(s) + 1) // 2
        cfg = pg.GraphConfig(deletion_mode=mode)
        g = pg.DynamicGraph.from_edges(nv, s[:half], d[:half], None, cfg)
        r = RefGraph(nv, s[:half], d[:half], None, graph_config(deletion_mode=mode))
        win = RefWindow(rs)
        for b in batches:
            a, bb, ww, c, dd = win.slide(b)
            st = g.apply_batch(a, bb, None, c, dd)
            rst = r.apply_batch(a, bb, None, c, dd)
            same = all((x == y).all() for x, y in zip(g.pma().slots(), r.slots()))
            same &= st.slot_writes == rst.slot_writes and st.rounds == rst.rounds
            print(kind, b, "slots equal" if same else "SLOTS DIFFER", flush=True)
            ok &= same
        ok &= (pg.bfs(g, 1) == r.bfs(1)).all()
        ok &= (pg.connected_components(g) == r.cc()).all()
        pr = pg.pagerank(g)
        ok &= np.abs(pr.ranks - r.pagerank()[0]).max() <= 1e-6
        ok &= (pg.spmv(g, np.ones(nv)) == r.spmv(np.ones(nv))).all()
    k = np.random.default_rng(1).integers(0, 2 ** 63, 300_000, dtype=np.uint64)
    gk, _ = pg.sort_by_key(k, np.arange(len(k), dtype=np.uint32))
    ok &= (gk == np.sort(k, kind="stable")).all()
    st = pg.EdgeStream.erdos_renyi(1 << 10, 2.0 ** -4, 3)
    w = pg.SlidingWindow(st, 0)
    rng = pg.Mt19937_64(9)
    for _ in range(3):
        w.slide_explicit_random(500, rng)
    w.slide(300)
    print("sanitize workload", "OK" if ok else "MISMATCH", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
