"""Parity at the headline config's FULL size (C2: RMAT 2^21, 30.6M-edge
stream, 15.3M-edge window, batch 10^6) through size-independent properties —
the CPU reference needs minutes per batch at this size, so instead of a
slot-by-slot comparison (done at smaller sizes in test_graph_gpu.py /
test_golden_gpu.py) every invariant the reference guarantees is checked on
the device state after several slides:

* PMA layout: non-Empty keys strictly increasing in slot order, Empty slots
  all-zero (pma.hpp:31-33), counters equal to the state counts;
* content: the Valid non-guard keys are exactly the distinct edges of the
  window's arrival range (streaming.hpp:107-123: a slide inserts the next B
  arrivals and deletes the expired ones whose multiplicity reaches zero);
* row offsets: ro[u + 1] = guard slot of u + 1 (graph.hpp:167-190);
* BFS levels: root 0, every edge relaxed (dist[v] <= dist[u] + 1), every
  reached vertex has a parent one level up (analytics.hpp:22-48);
* CC labels: constant along edges, and each label is its component's
  minimum id (analytics.hpp:53-82);
* PageRank: the vector sums to 1 and one more power iteration moves it by
  less than epsilon (analytics.hpp:84-143)."""
import numpy as np
import pytest

from paper_1709_05061_b200 import pmagraph as pg

pytestmark = pytest.mark.gpu

NV, NE, B, SLIDES = 1 << 21, 30_600_000, 1_000_000, 4
GUARD = np.uint64(0xFFFFFFFF)


@pytest.fixture(scope="module")
def c2():
    stream = pg.EdgeStream.rmat(NV, NE, seed=1).shuffle(2)
    win = pg.SlidingWindow(stream, 0)
    win.reserve(SLIDES * B + 16)
    info = win.info()
    g = pg.DynamicGraph.from_edges_device(NV, info.stream_src, info.stream_dst, None, info.initial_size, device=0)
    half = info.initial_size
    slides = [win.slide(B) for _ in range(SLIDES)]
    info = win.info()
    for s in slides:
        g.apply_batch_device(info.stream_src + 4 * s.ins_offset, info.stream_dst + 4 * s.ins_offset, None, s.n_ins,
                             info.del_src + 4 * s.del_offset, info.del_dst + 4 * s.del_offset, s.n_del)
    src, dst = stream.arrays()
    lo, hi = SLIDES * B, half + SLIDES * B
    return g, src, dst, lo, hi


def test_layout_content_and_row_offsets(c2):
    g, src, dst, lo, hi = c2
    k, v, s = g.pma().slots()
    ne = s != 0
    assert np.all(np.diff(k[ne].astype(np.uint64)) > 0), "non-Empty keys must be strictly increasing"
    assert not k[~ne].any() and not v[~ne].any(), "Empty slots must be all-zero"
    p = g.pma()
    assert p.valid_count() == int((s == 1).sum()) and p.tombstone_count() == int((s == 2).sum())
    valid = k[s == 1]
    guards = (valid & GUARD) == GUARD
    edges = valid[~guards]
    want = np.unique((src[lo:hi].astype(np.uint64) << np.uint64(32)) | dst[lo:hi].astype(np.uint64))
    assert len(edges) == len(want) and (edges == want).all(), "window content differs"
    assert g.num_edges() == len(want)
    assert (valid[guards] >> np.uint64(32) == np.arange(NV, dtype=np.uint64)).all(), "one guard per vertex"
    ro = g.row_offsets()
    gslot = np.nonzero((s == 1) & ((k & GUARD) == GUARD))[0]
    assert ro[0] == 0 and (ro[1:] == gslot.astype(np.uint64) + 1).all()


def test_analytics_properties(c2):
    g, *_ = c2
    ro, col, val = g.csr_snapshot()
    deg = np.diff(ro.astype(np.int64))
    u = np.repeat(np.arange(NV, dtype=np.int64), deg)
    v = col.astype(np.int64)
    root = int(np.argmax(deg))  # the largest hub: a deep traversal
    dist = pg.bfs(g, root).astype(np.int64)
    inf = 0xFFFFFFFF
    assert dist[root] == 0
    reach = dist[u] != inf
    assert np.all(dist[v[reach]] <= dist[u[reach]] + 1), "an edge is not relaxed"
    par = np.full(NV, inf, np.int64)
    np.minimum.at(par, v[reach], dist[u[reach]])
    rv = np.nonzero((dist != inf) & (np.arange(NV) != root))[0]
    assert np.all(par[rv] == dist[rv] - 1), "a reached vertex without a parent one level up"
    lab = pg.connected_components(g).astype(np.int64)
    assert np.all(lab[u] == lab[v])
    order = np.argsort(lab, kind="stable")
    sl = lab[order]
    heads = np.concatenate([[True], sl[1:] != sl[:-1]])
    assert np.all(sl[heads] == order[heads]), "a label is not its component's minimum id"
    pr = pg.pagerank(g)
    x = pr.ranks
    assert pr.converged and abs(x.sum() - 1.0) < 1e-6
    od = deg.astype(np.float64)
    share = np.where(od > 0, 0.85 * x / np.maximum(od, 1), 0.0)
    y = np.full(NV, (1 - 0.85) / NV + 0.85 * x[od == 0].sum() / NV)
    np.add.at(y, v, share[u])
    assert np.abs(y - x).sum() < 1e-3, "not a fixed point within epsilon"
