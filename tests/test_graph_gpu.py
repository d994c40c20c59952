"""GPU parity of DynamicGraph + analytics against the UNMODIFIED reference
(oracle/_ref): after every sliding-window batch the slot array, UpdateStats
and row offsets are bit-exact; BFS levels and CC labels are bit-exact; SpMV
is bit-exact (ordered accumulation, no FMA); PageRank within 1e-6 max-abs
per vertex (north_star tolerance) with equal iteration counts."""
import numpy as np
import pytest

from oracle.oracle import RefGraph, RefStream, RefWindow
from paper_1709_05061_b200.abi import PMA_EAGER, PMA_LAZY, graph_config
from paper_1709_05061_b200.pmagraph import (DynamicGraph, GraphConfig, bfs, connected_components, pagerank, spmv)
from tests.helpers import assert_same_slots, ref_parity

pytestmark = pytest.mark.gpu

PR_TOL = 1e-6  # north_star: PageRank within 1e-6 max abs error per vertex


def example():
    # test_graph.cpp:16-19 worked example (paper Fig. 6)
    return 3, [0, 0, 1, 2, 2, 2], [0, 2, 2, 0, 1, 2], [1.0, 2.0, 3.0, 4.0, 5.0, 6.0]


def test_worked_example_csr_and_analytics():
    nv, s, d, w = example()
    g = DynamicGraph.from_edges(nv, s, d, w)
    ro, col, val = g.csr_snapshot()
    assert list(ro) == [0, 2, 3, 6]
    assert list(col) == [0, 2, 2, 0, 1, 2]
    assert list(val) == [1, 2, 3, 4, 5, 6]
    assert list(bfs(g, 0)) == [0, 2, 1]                   # test_analytics.cpp:37-42
    assert list(connected_components(g)) == [0, 0, 0]     # :60-64
    assert list(spmv(g, [1.0, 1.0, 1.0])) == [3, 3, 15]   # :157-163
    with pytest.raises(ValueError):
        spmv(g, [1.0])


def test_pagerank_small_known_answers():
    g = DynamicGraph.from_edges(1, [], [])
    r = pagerank(g)
    assert r.converged and list(r.ranks) == [1.0]
    g2 = DynamicGraph.from_edges(2, [0, 1], [1, 0])
    r2 = pagerank(g2)
    assert r2.converged and abs(r2.ranks[0] - 0.5) < 1e-12 and abs(r2.ranks[1] - 0.5) < 1e-12


def test_out_of_range_ids_rejected():
    with pytest.raises(ValueError, match=r"edge \(0, 7\) outside vertex range 3"):
        DynamicGraph.from_edges(3, [0], [7])
    g = DynamicGraph.from_edges(3, [0], [1])
    with pytest.raises(ValueError, match="outside vertex range"):
        g.apply_batch([5], [0], [1.0], [], [])


def test_random_graphs_from_edges_match_reference():
    rng = np.random.default_rng(77)
    for trial in range(10):
        nv = int(rng.integers(1, 3000))
        ne = int(rng.integers(0, 20000))
        s = rng.integers(0, nv, ne)
        d = rng.integers(0, nv, ne)
        w = rng.integers(0, 100, ne).astype(float)
        g = DynamicGraph.from_edges(nv, s, d, w)
        r = RefGraph(nv, s, d, w)
        assert_same_slots(g.pma().slots(), r.slots(), f"trial {trial}")
        assert (g.row_offsets() == r.row_offsets()).all()
        a, b = g.csr_snapshot(), r.csr_snapshot()
        assert all((x == y).all() for x, y in zip(a, b))


def _window_stream(kind, nv, param, seed=1, shuffle=2):
    if kind == "er":
        st = RefStream.erdos_renyi(nv, param, seed)
    else:
        st = RefStream.rmat(nv, param, seed)
    if shuffle is not None:
        st.shuffle(shuffle)
    return st


@pytest.mark.parametrize("mode", [PMA_LAZY, PMA_EAGER])
# (batches of up to 16384 updates take the captured small-batch graph; its
# one-CTA sort runs 1, 2 or 4 items per thread: 512 -> 1024 updates, 700 ->
# ~1400, 1500 -> ~3000)
@pytest.mark.parametrize("kind,nv,param,batch", [("er", 4096, 2**-7, 512), ("rmat", 2**13, 60000, 1500),
                                                  ("rmat", 2**12, 30000, 7), ("er", 4096, 2**-7, 700)])
def test_sliding_window_parity(mode, kind, nv, param, batch):
    stream = _window_stream(kind, nv, param, shuffle=2 if kind == "er" else None)
    s, d, w, _ = stream.arrays()
    half = (len(s) + 1) // 2
    cfg = GraphConfig(deletion_mode=mode)
    g = DynamicGraph.from_edges(nv, s[:half], d[:half], w[:half], cfg)
    r = RefGraph(nv, s[:half], d[:half], w[:half], graph_config(deletion_mode=mode))
    assert_same_slots(g.pma().slots(), r.slots(), "init")
    win = RefWindow(stream)
    rng = np.random.default_rng(3)
    warm_g = warm_r = None
    for slide in range(6):
        a, b, ww, c, dd = win.slide(batch)
        gs = g.apply_batch(a, b, ww, c, dd)
        rs = r.apply_batch(a, b, ww, c, dd)
        ctx = f"slide {slide}"
        assert gs.parity() == ref_parity(r, rs), ctx
        assert_same_slots(g.pma().slots(), r.slots(), ctx)
        assert (g.row_offsets() == r.row_offsets()).all(), ctx
        root = int(rng.integers(0, nv))
        assert (bfs(g, root) == r.bfs(root)).all(), ctx
        assert (connected_components(g) == r.cc()).all(), ctx
        pg = pagerank(g, warm_start=warm_g)
        pr = r.pagerank(warm=warm_r)
        assert np.abs(pg.ranks - pr[0]).max() <= PR_TOL, ctx
        assert pg.iterations == pr[1] and pg.converged == pr[2], ctx
        warm_g, warm_r = pg.ranks, pr[0]
        x = rng.random(nv)
        assert (spmv(g, x) == r.spmv(x)).all(), ctx


def test_pagerank_fixed_iterations_tight():
    rng = np.random.default_rng(107)
    for _ in range(3):
        nv, ne = 500, 3000
        s, d = rng.integers(0, nv, ne), rng.integers(0, nv, ne)
        g = DynamicGraph.from_edges(nv, s, d)
        r = RefGraph(nv, s, d)
        pg = pagerank(g, epsilon=0.0, max_iters=25)
        pr = r.pagerank(epsilon=0.0, max_iters=25)
        assert pg.iterations == 25 and not pg.converged
        assert np.abs(pg.ranks - pr[0]).max() <= 1e-12


def test_guard_deletes_are_dropped_and_counted():
    nv, s, d, w = example()
    g = DynamicGraph.from_edges(nv, s, d, w)
    r = RefGraph(nv, s, d, w)
    args = ([1], [0], [7.0], [0, 2, 1], [0xFFFFFFFF, 1, 1])
    gs = g.apply_batch(*args)
    rs = r.apply_batch(*args)
    assert gs.parity() == ref_parity(r, rs)
    assert gs.deletes_missed == rs.deletes_missed
    assert_same_slots(g.pma().slots(), r.slots())


@pytest.mark.parametrize("mode", [PMA_LAZY, PMA_EAGER])
def test_out_of_layout_deletes_match_reference(mode):
    """Deletes whose ids lie outside [0, |V|) (not guards) stay in the batch as
    missed deletes and still shape the decisions (graph.hpp:141-147); the
    device front end's |V|-derived key layout cannot hold them, so the batch is
    redone on the generic key-reduction path — results must not change."""
    rng = np.random.default_rng(5)
    nv = 300
    s = rng.integers(0, nv, 2000)
    d = rng.integers(0, nv, 2000)
    g = DynamicGraph.from_edges(nv, s, d, None, GraphConfig(deletion_mode=mode))
    r = RefGraph(nv, s, d, None, graph_config(deletion_mode=mode))
    for t in range(6):
        ins_s = rng.integers(0, nv, 200)
        ins_d = rng.integers(0, nv, 200)
        del_s = np.concatenate([s[rng.integers(0, len(s), 150)], rng.integers(nv, 2**32 - 1, 20), [7, 7]])
        del_d = np.concatenate([d[rng.integers(0, len(d), 150)], rng.integers(0, 2**32 - 2, 20), [2**31, 2**31]])
        args = (ins_s, ins_d, None, del_s.astype(np.uint32), del_d.astype(np.uint32))
        gs = g.apply_batch(*args)
        rs = r.apply_batch(*args)
        assert gs.parity() == ref_parity(r, rs), t
        assert_same_slots(g.pma().slots(), r.slots())
        assert (g.row_offsets() == r.row_offsets()).all()


def test_bad_insert_reports_first_offender_and_leaves_graph_unchanged():
    nv, s, d, w = example()
    g = DynamicGraph.from_edges(nv, s, d, w)
    before = g.pma().slots()
    with pytest.raises(ValueError, match=r"edge \(5, 0\) outside vertex range 3"):
        g.apply_batch([0, 5, 9], [1, 0, 0], None, [0], [2])
    after = g.pma().slots()
    assert all((a == b).all() for a, b in zip(before, after))
    assert list(bfs(g, 0)) == [0, 2, 1]


@pytest.mark.parametrize("mode", [PMA_LAZY, PMA_EAGER])
def test_large_batches_parity(mode):
    """Batches of >= 2^16 updates take the leaf-bucket front end when the
    leaf count is within 4x the batch: slots, stats and row offsets stay
    bit-exact with the reference over several 150K-arrival slides."""
    nv = 2**16
    stream = _window_stream("rmat", nv, 900000, shuffle=2)
    s, d, w, _ = stream.arrays()
    half = (len(s) + 1) // 2
    cfg = GraphConfig(deletion_mode=mode)
    g = DynamicGraph.from_edges(nv, s[:half], d[:half], w[:half], cfg)
    r = RefGraph(nv, s[:half], d[:half], w[:half], graph_config(deletion_mode=mode))
    win = RefWindow(stream)
    for slide in range(3):
        a, b, ww, c, dd = win.slide(150000)
        gs = g.apply_batch(a, b, ww, c, dd)
        rs = r.apply_batch(a, b, ww, c, dd)
        assert gs.batch_size >= 2**16
        ctx = f"slide {slide}"
        assert gs.parity() == ref_parity(r, rs), ctx
        assert_same_slots(g.pma().slots(), r.slots(), ctx)
        assert (g.row_offsets() == r.row_offsets()).all(), ctx


def test_pinned_host_batches_read_in_place():
    """gpma_apply_batch reads page-locked endpoint arrays in place over PCIe
    (zero-copy) and stages pageable ones: both give the reference's result."""
    torch = pytest.importorskip("torch")
    stream = _window_stream("rmat", 2**12, 30000)
    s, d, w, _ = stream.arrays()
    half = (len(s) + 1) // 2
    g = DynamicGraph.from_edges(2**12, s[:half], d[:half], w[:half])
    r = RefGraph(2**12, s[:half], d[:half], w[:half])
    win = RefWindow(stream)

    def pin(x, off=0):
        t = torch.empty(len(x) + 3, dtype=torch.int32).pin_memory()
        v = t.numpy().view(np.uint32)[off:off + len(x)]  # off: 16-byte misaligned starts
        v[:] = x
        return v, t

    for slide in range(6):
        a, b, ww, c, dd = win.slide(1500 + slide)
        if slide % 2 == 0:
            o = slide // 2
            (a, _ta), (b, _tb), (c, _tc), (dd, _td) = pin(a, o), pin(b, o), pin(c, (o + 1) % 3), pin(dd, o)
        gs = g.apply_batch(a, b, ww, c, dd)
        rs = r.apply_batch(a, b, ww, c, dd)
        assert gs.parity() == ref_parity(r, rs), slide
        assert_same_slots(g.pma().slots(), r.slots(), f"slide {slide}")
    # a guard delete and an invalid insert arriving through mapped memory
    (a, _ta), (b, _tb) = pin(np.array([1], np.uint32)), pin(np.array([2**12 + 5], np.uint32))
    with pytest.raises(ValueError, match="outside vertex range"):
        g.apply_batch(a, b, None, [], [])
    assert_same_slots(g.pma().slots(), r.slots(), "after rejected batch")


@pytest.mark.parametrize("mode", [PMA_LAZY, PMA_EAGER])
@pytest.mark.parametrize("kind,nv,param,batch", [("er", 2**14, 2**-6, 100000), ("rmat", 2**16, 600000, 90000)])
def test_leaf_bucket_front_end_parity(mode, kind, nv, param, batch):
    """Batches >= 2^16 updates take the leaf-bucket front end (leaf found per
    update, counting sort by leaf, in-bucket rank): slot arrays, stats and row
    offsets must stay bit-exact with the reference."""
    stream = _window_stream(kind, nv, param)
    s, d, w, _ = stream.arrays()
    half = (len(s) + 1) // 2
    g = DynamicGraph.from_edges(nv, s[:half], d[:half], w[:half], GraphConfig(deletion_mode=mode))
    r = RefGraph(nv, s[:half], d[:half], w[:half], graph_config(deletion_mode=mode))
    win = RefWindow(stream)
    seen = set()
    for slide in range(3):
        a, b, ww, c, dd = win.slide(batch)
        gs = g.apply_batch(a, b, ww, c, dd)
        seen.add(int(g.last_timing().front_end))
        rs = r.apply_batch(a, b, ww, c, dd)
        assert gs.parity() == ref_parity(r, rs), slide
        assert_same_slots(g.pma().slots(), r.slots(), f"slide {slide}")
        assert (g.row_offsets() == r.row_offsets()).all()
    assert 1 in seen or 2 in seen, seen


def test_leaf_bucket_overflow_redo():
    """A burst of inserts between two neighbouring keys overflows one leaf
    bucket: the batch is redone through the radix sort (front_end 2) with the
    same result, and duplicate / cancelling updates inside buckets resolve as
    in the reference."""
    rng = np.random.default_rng(12)
    nv = 2**14
    s = rng.integers(0, nv, 50000)
    d = rng.integers(0, nv, 50000)
    g = DynamicGraph.from_edges(nv, s, d)
    r = RefGraph(nv, s, d)
    # 80k inserts: 3000 onto vertex 77 (one bucket), the rest random with duplicates
    a = np.concatenate([np.full(3000, 77), rng.integers(0, nv, 77000)])
    b = np.concatenate([np.arange(3000) % nv, rng.integers(0, nv, 77000)])
    a, b = np.concatenate([a, a[:5000]]), np.concatenate([b, b[:5000]])
    w = rng.integers(0, 9, len(a)).astype(float)
    c, dd = s[:20000], d[:20000]
    gs = g.apply_batch(a, b, w, c, dd)
    assert int(g.last_timing().front_end) == 2
    rs = r.apply_batch(a, b, w, c, dd)
    assert gs.parity() == ref_parity(r, rs)
    assert_same_slots(g.pma().slots(), r.slots(), "overflow redo")
    # the next batch stays on the radix sort (cool-down), still exact
    a2, b2 = rng.integers(0, nv, 70000), rng.integers(0, nv, 70000)
    gs = g.apply_batch(a2, b2, None, a[:9000], b[:9000])
    assert int(g.last_timing().front_end) == 0
    rs = r.apply_batch(a2, b2, None, a[:9000], b[:9000])
    assert gs.parity() == ref_parity(r, rs)
    assert_same_slots(g.pma().slots(), r.slots(), "after cool-down")


def test_read_api_matches_reference():
    """edge_list / degree / edge_weight / neighbors / guard_count
    (graph.hpp:94-126, 208-223) after a few window slides."""
    stream = _window_stream("rmat", 2**11, 20000)
    s, d, w, _ = stream.arrays()
    half = (len(s) + 1) // 2
    rng = np.random.default_rng(8)
    w = rng.integers(1, 50, len(s)).astype(float)
    g = DynamicGraph.from_edges(2**11, s[:half], d[:half], w[:half])
    r = RefGraph(2**11, s[:half], d[:half], w[:half])
    win = RefWindow(stream)
    for _ in range(3):
        args = win.slide(900)
        g.apply_batch(*args)
        r.apply_batch(*args)
    ro, col, val = r.csr_snapshot()
    es, ed, ew = g.edge_list()
    deg = np.diff(ro.astype(np.int64))
    assert (es == np.repeat(np.arange(2**11), deg)).all() and (ed == col).all() and (ew == val).all()
    assert g.guard_count() == 2**11
    for v in rng.integers(0, 2**11, 40):
        v = int(v)
        assert g.degree(v) == deg[v]
        nd, nw = g.neighbors(v)
        assert (nd == col[ro[v]:ro[v + 1]]).all() and (nw == val[ro[v]:ro[v + 1]]).all()
        if deg[v]:
            j = int(rng.integers(ro[v], ro[v + 1]))
            assert g.edge_weight(v, int(col[j])) == val[j]
    assert g.edge_weight(0, 2**11 - 1) is None or (0, 2**11 - 1) in set(zip(es.tolist(), ed.tolist()))
    with pytest.raises(IndexError):
        g.degree(2**11)


@pytest.mark.parametrize("mode", [PMA_LAZY, PMA_EAGER])
def test_leaf_bucket_edge_cases(mode):
    """The leaf-bucket front end (batch >= 2^16, few leaves) with duplicate
    and cancelling updates inside one leaf; guard deletes and deletes outside
    the key layout (both: the generic redo path, which drops guard deletes);
    a bad insert (rejected, graph unchanged) — all as the reference."""
    rng = np.random.default_rng(21)
    nv = 2**12
    s, d = rng.integers(0, nv, 30000), rng.integers(0, nv, 30000)
    g = DynamicGraph.from_edges(nv, s, d, None, GraphConfig(deletion_mode=mode))
    r = RefGraph(nv, s, d, None, graph_config(deletion_mode=mode))

    def both(args, ctx, fronts=(1, 2)):
        gs = g.apply_batch(*args)
        assert int(g.last_timing().front_end) in fronts, ctx
        rs = r.apply_batch(*args)
        assert gs.parity() == ref_parity(r, rs), ctx
        assert_same_slots(g.pma().slots(), r.slots(), ctx)
        assert (g.row_offsets() == r.row_offsets()).all(), ctx

    a, b = rng.integers(0, nv, 60000), rng.integers(0, nv, 60000)
    a[:300], b[:300] = 9, 33  # one key inserted 300 times
    c = np.concatenate([s[:9000], np.full(400, 9), rng.integers(0, nv, 500)]).astype(np.uint32)
    dd = np.concatenate([d[:9000], np.full(400, 33), np.full(500, 0xFFFFFFFF)]).astype(np.uint32)  # + guard deletes
    both((a, b, rng.integers(0, 9, 60000).astype(float), c, dd), "guards + duplicates", (0,))
    both((a[1000:], b[1000:], rng.integers(0, 9, 59000).astype(float), c[:9400], dd[:9400]), "duplicates")
    c2 = np.concatenate([s[9000:20000], [2**20, 5]]).astype(np.uint32)  # a delete outside the layout
    d2 = np.concatenate([d[9000:20000], [3, 2**30]]).astype(np.uint32)
    a2, b2 = rng.integers(0, nv, 60000), rng.integers(0, nv, 60000)
    both((a2, b2, None, c2, d2), "out-of-layout deletes", (0,))  # redone on the generic key path
    before = g.pma().slots()
    a3 = rng.integers(0, nv, 70000)
    a3[40000] = nv + 3
    with pytest.raises(ValueError, match=rf"edge \({nv + 3}, \d+\) outside vertex range {nv}"):
        g.apply_batch(a3, rng.integers(0, nv, 70000), None, [], [])
    assert all((x == y).all() for x, y in zip(before, g.pma().slots()))


@pytest.mark.parametrize("weighted", [True, False])
def test_leaf_bucket_pairs_front_end(weighted):
    """When key and arrival index do not fit one 64-bit word (|V| = 2^22,
    batch > 2^19) the leaf-bucket front end sorts (key, payload) pairs —
    or, unweighted, words carrying only the op: still bit-exact with the
    reference."""
    rng = np.random.default_rng(31)
    nv = 2**22
    s, d = rng.integers(0, nv, 600000), rng.integers(0, nv, 600000)
    g = DynamicGraph.from_edges(nv, s, d)
    r = RefGraph(nv, s, d)
    a, b = rng.integers(0, nv, 400000), rng.integers(0, nv, 400000)
    a[:200], b[:200] = 5, 6  # a duplicated key
    w = rng.integers(1, 9, 400000).astype(float) if weighted else None
    c = np.concatenate([s[:250000], np.full(100, 5)]).astype(np.uint32)
    dd = np.concatenate([d[:250000], np.full(100, 6)]).astype(np.uint32)
    gs = g.apply_batch(a, b, w, c, dd)
    assert int(g.last_timing().front_end) in (1, 2)
    rs = r.apply_batch(a, b, w, c, dd)
    assert gs.parity() == ref_parity(r, rs)
    assert_same_slots(g.pma().slots(), r.slots(), "pairs")
    assert (g.row_offsets() == r.row_offsets()).all()


@pytest.mark.parametrize("mode", [PMA_LAZY, PMA_EAGER])
def test_graph_edge_cases_match_reference(mode):
    """Empty batches, a batch deleting every edge (eager: the array shrinks),
    re-inserting them, deletes of absent edges only, and edges on the highest
    vertex id — stats, slots and row offsets as the reference."""
    rng = np.random.default_rng(41)
    nv = 2**12
    s = np.concatenate([rng.integers(0, nv, 6000), [nv - 1] * 5])
    d = np.concatenate([rng.integers(0, nv, 6000), [0, 1, nv - 1, 7, nv - 2]])
    g = DynamicGraph.from_edges(nv, s, d, None, GraphConfig(deletion_mode=mode))
    r = RefGraph(nv, s, d, None, graph_config(deletion_mode=mode))

    def both(args, ctx):
        gs = g.apply_batch(*args)
        rs = r.apply_batch(*args)
        assert gs.parity() == ref_parity(r, rs), ctx
        assert_same_slots(g.pma().slots(), r.slots(), ctx)
        assert (g.row_offsets() == r.row_offsets()).all(), ctx

    e = np.zeros(0, np.uint32)
    both((e, e, None, e, e), "empty batch")
    both((e, e, None, rng.integers(0, nv, 300).astype(np.uint32), rng.integers(0, nv, 300).astype(np.uint32)),
         "absent deletes")
    both((e, e, None, s.astype(np.uint32), d.astype(np.uint32)), "delete everything")
    assert g.num_edges() == 0
    both((s.astype(np.uint32), d.astype(np.uint32), None, e, e), "re-insert everything")
    both(([nv - 1], [nv - 1], [2.5], [nv - 1], [nv - 1]), "insert + delete of one key in one batch")
    assert (bfs(g, nv - 1) == r.bfs(nv - 1)).all()


@pytest.mark.parametrize("weighted", [True, False])
def test_radix_front_end_wide_keys(weighted):
    """|V| = 2^24 (49 key bits) with a 70K-update batch (17 index bits) and
    far more leaves than updates: the radix front end sorts (key, payload)
    pairs (weighted) or op-carrying words (unweighted) — bit-exact with the
    reference either way."""
    rng = np.random.default_rng(33)
    nv = 2**24
    s, d = rng.integers(0, nv, 200000), rng.integers(0, nv, 200000)
    g = DynamicGraph.from_edges(nv, s, d)
    r = RefGraph(nv, s, d)
    a, b = rng.integers(0, nv, 40000), rng.integers(0, nv, 40000)
    a[:50], b[:50] = 9, 9
    w = rng.integers(1, 9, 40000).astype(float) if weighted else None
    c = np.concatenate([s[:30000], np.full(30, 9)]).astype(np.uint32)
    dd = np.concatenate([d[:30000], np.full(30, 9)]).astype(np.uint32)
    gs = g.apply_batch(a, b, w, c, dd)
    assert int(g.last_timing().front_end) == 0
    rs = r.apply_batch(a, b, w, c, dd)
    assert gs.parity() == ref_parity(r, rs)
    assert_same_slots(g.pma().slots(), r.slots(), "wide keys")


@pytest.mark.parametrize("mode", [PMA_LAZY, PMA_EAGER])
def test_small_batch_sort_size_regimes(mode):
    """Batches of exactly n updates at every size regime of the captured
    small-batch graph's one-CTA sort (sort_block: P = 32 .. 4096 words, 1, 2
    or 4 items per thread, and the boundaries between them), each with
    duplicate inserts, insert + delete of one edge, deletes of present and
    absent edges; slots and stats bit-exact after every batch."""
    rng = np.random.default_rng(11)
    nv = 1 << 14
    stream = RefStream.rmat(nv, 200000, 9)
    s, d, w, _ = stream.arrays()
    half = (len(s) + 1) // 2
    cfg = GraphConfig(deletion_mode=mode)
    g = DynamicGraph.from_edges(nv, s[:half], d[:half], w[:half], cfg)
    r = RefGraph(nv, s[:half], d[:half], w[:half], graph_config(deletion_mode=mode))
    present_s, present_d = s[:half].astype(np.uint32), d[:half].astype(np.uint32)
    for n in (1, 2, 31, 32, 33, 100, 1023, 1024, 1025, 2047, 2048, 2049, 3000, 4095, 4096):
        nd = n // 3
        ni = n - nd
        a = rng.integers(0, nv, ni).astype(np.uint32)
        b = rng.integers(0, nv, ni).astype(np.uint32)
        if ni >= 4:  # duplicate insert, and an insert also deleted in the same batch
            a[1], b[1] = a[0], b[0]
        ww = rng.random(ni) + 0.5
        pick = rng.integers(0, len(present_s), nd)
        c, dd = present_s[pick].copy(), present_d[pick].copy()
        if nd >= 2:
            c[0], dd[0] = a[0], b[0]
            c[1], dd[1] = rng.integers(0, nv, 2).astype(np.uint32)  # (most likely) absent
        gs = g.apply_batch(a, b, ww, c, dd)
        rs = r.apply_batch(a, b, ww, c, dd)
        ctx = f"n={n}"
        assert gs.parity() == ref_parity(r, rs), ctx
        assert_same_slots(g.pma().slots(), r.slots(), ctx)
        assert (g.row_offsets() == r.row_offsets()).all(), ctx


@pytest.mark.parametrize("onecta,cluster", [("0", "1"), ("512", "1"), ("4096", "1"), ("0", "0")])
def test_small_batch_front_end_variants(onecta, cluster, monkeypatch):
    """The captured small-batch graph's front ends — one CTA (k_small_front)
    and chunks on separate SMs merged by rank, in a 16-CTA cluster
    (k_small_front_cluster) or a cooperative grid (k_small_front_grid) —
    forced per batch size by GPMA_SMALL_ONECTA / GPMA_SMALL_CLUSTER: the same words with the same
    duplicates spread over different chunks (repeated inserts, a key deleted
    twice, insert + delete of one key), guard deletes, deletes outside the
    layout (redone on the generic path) and the first of two bad inserts
    reported; slots, stats and row offsets bit-exact."""
    monkeypatch.setenv("GPMA_SMALL_ONECTA", onecta)
    monkeypatch.setenv("GPMA_SMALL_CLUSTER", cluster)
    rng = np.random.default_rng(int(onecta) + 5)
    nv = 1 << 14
    stream = RefStream.rmat(nv, 200000, 13)
    s, d, w, _ = stream.arrays()
    half = (len(s) + 1) // 2
    g = DynamicGraph.from_edges(nv, s[:half], d[:half], w[:half])
    r = RefGraph(nv, s[:half], d[:half], w[:half], graph_config())
    ps, pd = s[:half].astype(np.uint32), d[:half].astype(np.uint32)
    for n in (100, 700, 1025, 1500, 2500, 4096, 4097, 9000, 16384):
        nd = n // 3
        ni = n - nd
        a = rng.integers(0, nv, ni).astype(np.uint32)
        b = rng.integers(0, nv, ni).astype(np.uint32)
        for j in (1, ni // 2, ni - 1):  # one key inserted three times, in different chunks
            a[j], b[j] = a[0], b[0]
        pick = rng.integers(0, len(ps), nd)
        c, dd = ps[pick].copy(), pd[pick].copy()
        c[nd - 1], dd[nd - 1] = c[0], dd[0]  # a present key deleted twice
        c[nd // 2], dd[nd // 2] = a[0], b[0]  # the inserted key deleted too
        c[1], dd[1] = 7, 0xFFFFFFFF  # a guard delete
        ww = rng.random(ni) + 0.5
        gs = g.apply_batch(a, b, ww, c, dd)
        rs = r.apply_batch(a, b, ww, c, dd)
        ctx = f"n={n} onecta={onecta}"
        assert gs.parity() == ref_parity(r, rs), ctx
        assert_same_slots(g.pma().slots(), r.slots(), ctx)
        assert (g.row_offsets() == r.row_offsets()).all(), ctx
    # deletes outside the |V|-derived layout: the batch is redone on the generic path
    c2 = np.concatenate([ps[:1800], [2**20]]).astype(np.uint32)
    d2 = np.concatenate([pd[:1800], [3]]).astype(np.uint32)
    a2, b2 = rng.integers(0, nv, 900), rng.integers(0, nv, 900)
    gs = g.apply_batch(a2, b2, None, c2, d2)
    rs = r.apply_batch(a2, b2, None, c2, d2)
    assert gs.parity() == ref_parity(r, rs)
    assert_same_slots(g.pma().slots(), r.slots(), "out-of-layout deletes")
    # two bad inserts in different chunks: the first is reported, nothing changes
    before = g.pma().slots()
    for m, j in ((3000, 1700), (12000, 7000)):
        a3 = rng.integers(0, nv, m)
        a3[j], a3[m - 100] = nv + 3, nv + 9
        with pytest.raises(ValueError, match=rf"edge \({nv + 3}, \d+\) outside vertex range {nv}"):
            g.apply_batch(a3, rng.integers(0, nv, m), None, [], [])
    assert all((x == y).all() for x, y in zip(before, g.pma().slots()))


@pytest.mark.parametrize("mode", [PMA_LAZY, PMA_EAGER])
def test_mixed_batch_sizes_through_growth_and_shrink(mode):
    """Small (captured-graph) and large (host-loop) batches interleaved on one
    graph while it grows past several capacities and, in eager mode, shrinks
    back: every layout change re-captures the small-batch graph; slots, stats
    and row offsets bit-exact after every batch."""
    rng = np.random.default_rng(21)
    nv = 1 << 13
    s0 = rng.integers(0, nv, 2000).astype(np.uint32)
    d0 = rng.integers(0, nv, 2000).astype(np.uint32)
    cfg = GraphConfig(deletion_mode=mode)
    g = DynamicGraph.from_edges(nv, s0, d0, None, cfg)
    r = RefGraph(nv, s0, d0, None, graph_config(deletion_mode=mode))
    live_s, live_d = list(s0), list(d0)
    grows = shrinks = 0
    for step, n in enumerate([100, 30000, 7, 4096, 60000, 1, 3000, 120000, 50, 2048]):
        a = rng.integers(0, nv, n).astype(np.uint32)
        b = rng.integers(0, nv, n).astype(np.uint32)
        nd = min(len(live_s), n // 2)
        pick = rng.choice(len(live_s), nd, replace=False) if nd else np.zeros(0, np.int64)
        c = np.array([live_s[i] for i in pick], np.uint32)
        dd = np.array([live_d[i] for i in pick], np.uint32)
        gs = g.apply_batch(a, b, None, c, dd)
        rs = r.apply_batch(a, b, None, c, dd)
        ctx = f"step {step} n={n}"
        assert gs.parity() == ref_parity(r, rs), ctx
        assert_same_slots(g.pma().slots(), r.slots(), ctx)
        assert (g.row_offsets() == r.row_offsets()).all(), ctx
        grows += gs.grow_events
        shrinks += gs.shrink_events
        keep = np.ones(len(live_s), bool)
        keep[pick] = False
        live_s = [x for x, k in zip(live_s, keep) if k] + list(a)
        live_d = [x for x, k in zip(live_d, keep) if k] + list(b)
    # massive deletes at the end (eager mode shrinks the root)
    c = np.array(live_s, np.uint32)
    dd = np.array(live_d, np.uint32)
    e = np.zeros(0, np.uint32)
    gs = g.apply_batch(e, e, None, c, dd)
    rs = r.apply_batch(e, e, None, c, dd)
    assert gs.parity() == ref_parity(r, rs), "final deletes"
    assert_same_slots(g.pma().slots(), r.slots(), "final deletes")
    shrinks += gs.shrink_events
    assert grows >= 2, "the graph must grow through several capacities"
    if mode == PMA_EAGER:
        assert shrinks >= 1, "eager deletes must shrink the root"


@pytest.mark.parametrize("mode", [PMA_LAZY, PMA_EAGER])
def test_small_batches_custom_profile(mode):
    """A non-default DensityProfile (tighter leaf and root bounds) through the
    captured small-batch graph, whose commit nodes bake the per-level bounds
    in at capture: bit-exact against the reference with the same profile."""
    from paper_1709_05061_b200.pmagraph import DensityProfile
    rng = np.random.default_rng(8)
    nv = 1 << 12
    stream = RefStream.rmat(nv, 60000, 4)
    s, d, w, _ = stream.arrays()
    half = (len(s) + 1) // 2
    prof = DensityProfile(leaf_lower=0.2, leaf_upper=0.7, root_lower=0.3, root_upper=0.6)
    g = DynamicGraph.from_edges(nv, s[:half], d[:half], w[:half], GraphConfig(deletion_mode=mode, profile=prof))
    r = RefGraph(nv, s[:half], d[:half], w[:half], graph_config(deletion_mode=mode, profile=prof.c()))
    win = RefWindow(stream)
    for b in (10, 200, 1000, 1800, 3, 600):
        a, bb, ww, c, dd = win.slide(b)
        gs = g.apply_batch(a, bb, ww, c, dd)
        rs = r.apply_batch(a, bb, ww, c, dd)
        assert gs.parity() == ref_parity(r, rs), f"batch {b}"
        assert_same_slots(g.pma().slots(), r.slots(), f"batch {b}")
        assert (g.row_offsets() == r.row_offsets()).all(), f"batch {b}"


@pytest.mark.parametrize("mode", [PMA_LAZY, PMA_EAGER])
def test_round_disjointness_check(mode, monkeypatch):
    """GPMA_CHECK_ROUNDS=1 runs the reference's round-disjointness assert
    (segment_engine.hpp:400-405) on the device after every grouping: small
    (captured-graph) and large batches through several levels pass it and
    stay bit-exact with the reference."""
    monkeypatch.setenv("GPMA_CHECK_ROUNDS", "1")
    rng = np.random.default_rng(3)
    nv = 1 << 12
    stream = RefStream.rmat(nv, 300000, 17)
    s, d, w, _ = stream.arrays()
    half = (len(s) + 1) // 2
    cfg = GraphConfig(deletion_mode=mode)
    g = DynamicGraph.from_edges(nv, s[:half], d[:half], w[:half], cfg)
    r = RefGraph(nv, s[:half], d[:half], w[:half], graph_config(deletion_mode=mode))
    for n in (50, 900, 3000, 40000, 150000):
        a, b = rng.integers(0, nv, n).astype(np.uint32), rng.integers(0, nv, n).astype(np.uint32)
        pick = rng.integers(0, half, n // 2)
        c, dd = s[pick].astype(np.uint32), d[pick].astype(np.uint32)
        ww = rng.random(n)
        gs = g.apply_batch(a, b, ww, c, dd)
        rs = r.apply_batch(a, b, ww, c, dd)
        assert gs.parity() == ref_parity(r, rs), n
        assert_same_slots(g.pma().slots(), r.slots(), f"n={n}")
