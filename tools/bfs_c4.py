import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_1709_05061_b200 import pmagraph as pg
from paper_1709_05061_b200.abi import load_library
load_library().gpma_warmup(0)
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
stream = bench.make_stream(pg, cfg, 1)
win = pg.SlidingWindow(stream, 0); info = win.info()
g = pg.DynamicGraph.from_edges_device(cfg["nv"], info.stream_src, info.stream_dst, None, info.initial_size)
ro = g.row_offsets(); hub = int(np.argmax(np.diff(ro.astype(np.int64))))
a = b = None
for r in [hub, hub, hub]:
    torch.cuda.synchronize(); t = time.perf_counter(); a, b = pg.bfs(g, r, return_reached=True), a; w = time.perf_counter() - t
    print(r, a[1], f"wall {w*1e3:.2f} ms device {g.last_timing().device_ms:.2f} ms")
