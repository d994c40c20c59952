import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_1709_05061_b200 import pmagraph as pg
from paper_1709_05061_b200.abi import load_library
load_library().gpma_warmup(0)
stream = pg.EdgeStream.rmat(bench.NV, bench.NE, seed=1).shuffle(2)
win = pg.SlidingWindow(stream, 0); info = win.info()
g = pg.DynamicGraph.from_edges_device(bench.NV, info.stream_src, info.stream_dst, None, info.initial_size)
pr = pg.pagerank(g)
keep = []
for iters in [1, 2, 10, 1, 2, 10]:
    torch.cuda.synchronize(); t = time.perf_counter()
    r = pg.pagerank(g, warm_start=pr.ranks, epsilon=0.0, max_iters=iters)
    w = (time.perf_counter() - t) * 1e3
    keep.append(r)
    tm = g.last_timing()
    print(iters, f"wall {w:.3f} ms device(total) {tm.device_ms:.3f} iter-kernels {tm.rounds_ms:.3f}")
