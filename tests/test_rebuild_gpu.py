"""GPU parity of the rebuild-CSR baseline (RebuildCsrGraph, baselines.hpp:85-181)
against the UNMODIFIED reference class (oracle/_ref): after every batch the
CSR arrays (row offsets, columns, value bits) and the UpdateStats fields the
reference fills (batch_size, deletes_missed, slot_writes) are bit-exact."""
import numpy as np
import pytest

from oracle.oracle import RefRebuildCsr, RefStream, RefWindow
from paper_1709_05061_b200.pmagraph import DynamicGraph, RebuildCsrGraph

pytestmark = pytest.mark.gpu


def _same(g, r, ctx=""):
    a, b = g.csr_snapshot(), r.csr()
    assert (a[0] == b[0]).all(), f"row offsets {ctx}"
    assert (a[1] == b[1]).all(), f"columns {ctx}"
    assert (a[2].view(np.uint64) == b[2].view(np.uint64)).all(), f"values {ctx}"
    assert g.num_edges() == len(b[1])


def _same_stats(gs, rs, ctx=""):
    assert (gs.batch_size, gs.deletes_missed, gs.slot_writes) == (rs.batch_size, rs.deletes_missed,
                                                                  rs.slot_writes), ctx
    assert gs.rounds == rs.rounds and gs.segments_per_level == [] and rs.num_levels == 0, ctx


def test_worked_example():
    nv, s, d, w = 3, [0, 0, 1, 2, 2, 2], [0, 2, 2, 0, 1, 2], [1.0, 2.0, 3.0, 4.0, 5.0, 6.0]
    g = RebuildCsrGraph(nv, s, d, w)
    ro, col, val = g.csr_snapshot()
    assert list(ro) == [0, 2, 3, 6] and list(col) == [0, 2, 2, 0, 1, 2] and list(val) == [1, 2, 3, 4, 5, 6]
    st = g.apply_batch([1], [0], [7.0], [0, 2], [2, 9])
    assert (st.batch_size, st.deletes_missed, st.slot_writes) == (3, 1, 2 * 6 + 3 + 1)
    ro, col, val = g.csr_snapshot()
    assert list(ro) == [0, 1, 3, 6] and list(col) == [0, 0, 2, 0, 1, 2] and list(val) == [1, 7, 3, 4, 5, 6]


def test_out_of_range_rejected_and_empty():
    with pytest.raises(ValueError, match="RebuildCsrGraph: vertex id out of range"):
        RebuildCsrGraph(3, [0], [3])
    g = RebuildCsrGraph(4)
    assert g.num_edges() == 0 and list(g.csr_snapshot()[0]) == [0] * 5
    st = g.apply_batch([], [], None, [], [])
    assert (st.batch_size, st.deletes_missed, st.slot_writes) == (0, 0, 5)
    st = g.apply_batch([], [], None, [1, 7], [2, 0xFFFFFFFF])  # absent / out-of-range deletes are missed
    assert st.deletes_missed == 2 and g.num_edges() == 0


def test_duplicates_last_wins():
    rng = np.random.default_rng(11)
    for trial in range(8):
        nv = int(rng.integers(1, 200))
        ne = int(rng.integers(0, 5000))
        s, d = rng.integers(0, nv, ne), rng.integers(0, nv, ne)
        w = rng.integers(0, 50, ne).astype(float)
        g, r = RebuildCsrGraph(nv, s, d, w), RefRebuildCsr(nv, s, d, w)
        _same(g, r, f"build {trial}")
        for b in range(4):
            ni, nd = int(rng.integers(0, 3000)), int(rng.integers(0, 3000))
            args = (rng.integers(0, nv, ni), rng.integers(0, nv, ni), rng.integers(0, 50, ni).astype(float),
                    rng.integers(0, nv + 3, nd), rng.integers(0, nv + 3, nd))
            _same_stats(g.apply_batch(*args), r.apply_batch(*args), f"trial {trial} batch {b}")
            _same(g, r, f"trial {trial} batch {b}")


@pytest.mark.parametrize("kind,nv,param,batch", [("er", 4096, 2**-7, 512), ("rmat", 2**13, 60000, 1500),
                                                  ("rmat", 2**12, 30000, 7)])
def test_sliding_window_parity(kind, nv, param, batch):
    stream = RefStream.erdos_renyi(nv, param, 1) if kind == "er" else RefStream.rmat(nv, param, 1)
    stream.shuffle(2)
    s, d, w, _ = stream.arrays()
    half = (len(s) + 1) // 2
    g, r = RebuildCsrGraph(nv, s[:half], d[:half], w[:half]), RefRebuildCsr(nv, s[:half], d[:half], w[:half])
    _same(g, r, "init")
    win = RefWindow(stream)
    for slide in range(6):
        args = win.slide(batch)
        _same_stats(g.apply_batch(*args), r.apply_batch(*args), f"slide {slide}")
        _same(g, r, f"slide {slide}")


def test_same_graph_as_gpma():
    """The baseline and the PMA store hold the same graph after the same
    window slides (both follow graph.hpp's edge semantics)."""
    stream = RefStream.rmat(2**12, 40000, 3)
    stream.shuffle(4)
    s, d, w, _ = stream.arrays()
    half = (len(s) + 1) // 2
    g, p = RebuildCsrGraph(2**12, s[:half], d[:half], w[:half]), DynamicGraph.from_edges(2**12, s[:half], d[:half],
                                                                                        w[:half])
    win = RefWindow(stream)
    for _ in range(4):
        args = win.slide(2000)
        g.apply_batch(*args)
        p.apply_batch(*args)
        a, b = g.csr_snapshot(), p.csr_snapshot()
        assert all((x == y).all() for x, y in zip(a, b))


def test_device_entry_points():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(9)
    nv, ne = 1000, 20000
    s, d = rng.integers(0, nv, ne), rng.integers(0, nv, ne)
    r = RefRebuildCsr(nv, s, d)
    ts = torch.tensor(s.astype(np.int32), device="cuda")
    td = torch.tensor(d.astype(np.int32), device="cuda")
    g = RebuildCsrGraph.from_edges_device(nv, ts.data_ptr(), td.data_ptr(), None, ne)
    _same(g, r, "device build")
    a, b = rng.integers(0, nv, 3000), rng.integers(0, nv, 3000)
    c, e = s[:4000], d[:4000]
    ta, tb = (torch.tensor(x.astype(np.int32), device="cuda") for x in (a, b))
    tc, te = (torch.tensor(x.astype(np.int32), device="cuda") for x in (c, e))
    gs = g.apply_batch_device(ta.data_ptr(), tb.data_ptr(), None, 3000, tc.data_ptr(), te.data_ptr(), 4000)
    rs = r.apply_batch(a, b, None, c, e)
    _same_stats(gs, rs, "device batch")
    _same(g, r, "device batch")
