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
res = []
for i in range(4):
    r = pg.pagerank(g, warm_start=pr.ranks, epsilon=0.0, max_iters=10)
    res.append(g.last_timing().rounds_ms / 10)
print("pr iter ms", [f"{x:.4f}" for x in res])
