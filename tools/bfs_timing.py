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
ro = g.row_offsets(); hub = int(np.argmax(np.diff(ro.astype(np.int64))))
for r in [1360226, hub, 1360226, hub, 1360226]:
    torch.cuda.synchronize(); t = time.perf_counter(); d, n = pg.bfs(g, r, return_reached=True); w = time.perf_counter() - t
    tm = g.last_timing()
    print(r, n, f"wall {w*1e3:.2f} ms device {tm.device_ms:.2f} ms launches {tm.kernel_launches}", int(d[d != 0xFFFFFFFF].max()))
