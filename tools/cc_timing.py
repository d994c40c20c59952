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
res = []
for i in range(6):
    torch.cuda.synchronize(); t = time.perf_counter(); lab = pg.connected_components(g); w = time.perf_counter() - t
    res.append((w * 1e3, g.last_timing().device_ms))
print("cc wall/device ms", [f"{a:.3f}/{b:.3f}" for a, b in res[2:]])
