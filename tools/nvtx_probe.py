import numpy as np, sys
sys.path.insert(0, ".")
from paper_1709_05061_b200 import pmagraph as pg
rng = np.random.default_rng(1)
nv = 1 << 12
s, d = rng.integers(0, nv, 50000), rng.integers(0, nv, 50000)
g = pg.DynamicGraph.from_edges(nv, s, d)
g.apply_batch(rng.integers(0, nv, 3000), rng.integers(0, nv, 3000), None, [], [])
pg.bfs(g, 1)
print("ok")
