#!/usr/bin/env python
"""Wall time of the C-ABI shard group's BFS / CC / PageRank at world 1 on the
C2 window (NCCL with one rank), next to the single-graph analytics."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import bench
    from paper_1709_05061_b200 import pmagraph as pg
    from paper_1709_05061_b200.abi import load_library
    from paper_1709_05061_b200.sharded import ShardGroup, nccl_unique_id
    load_library().gpma_warmup(0)
    stream = pg.EdgeStream.rmat(bench.NV, bench.NE, seed=1).shuffle(2)
    win = pg.SlidingWindow(stream, 0)
    info = win.info()
    init = info.initial_size
    e_src = bench._wrap_device(info.stream_src, init, torch.int32, 0)
    e_dst = bench._wrap_device(info.stream_dst, init, torch.int32, 0)
    G = ShardGroup(bench.NV, np.array([0, bench.NV], np.uint32), 0, 1, nccl_unique_id(), (e_src, e_dst, None))
    g = pg.DynamicGraph.from_edges_device(bench.NV, info.stream_src, info.stream_dst, None, init)
    ro = g.row_offsets()
    hub = int(np.argmax(np.diff(ro.astype(np.int64))))
    for name, f in [("group bfs", lambda: G.bfs(hub)), ("single bfs", lambda: pg.bfs(g, hub)),
                    ("group cc", G.connected_components), ("single cc", lambda: pg.connected_components(g))]:
        f()
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            t = time.perf_counter()
            f()
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t) * 1e3)
        print(f"{name}: wall ms {sorted(ts)[2]:.3f} (min {min(ts):.3f})", flush=True)


if __name__ == "__main__":
    main()
