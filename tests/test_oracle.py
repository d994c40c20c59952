"""CPU: pin the oracles.  The reference (oracle/_ref) and our C restatement
(oracle/_ref/libpmaport.so) are checked against the known answers the
reference's own tests hold (proj/tests/test_pma.cpp, test_segment_engine.cpp,
test_graph.cpp, test_analytics.cpp, support/fixtures.hpp) and against the
committed golden fixtures; then the restatement is cross-checked against the
reference on random traces."""
import numpy as np
import pytest

from oracle import oracle
from oracle.oracle import PortGraph, PortPMA, RefGraph, RefPMA, stats_dict
from paper_1709_05061_b200.abi import PMA_EAGER, PMA_LAZY, PMA_STRATEGY_LARGE, engine_config, graph_config
from tests import golden_replay as gr
from tests.helpers import fixture_arrays

pytestmark = pytest.mark.skipif(not oracle.have_ref(), reason="reference oracle not built")

IMPLS = [RefPMA, PortPMA]
GRAPHS = [RefGraph, PortGraph]


@pytest.mark.parametrize("P", IMPLS)
def test_fixture_five_insert_batch(P):
    # test_segment_engine.cpp:53-73
    p = P().load_slots(*fixture_arrays())
    keys = np.array([1, 4, 9, 35, 48], np.uint64)
    st = stats_dict(p.batch_update(keys, keys * 10, np.zeros(5, np.uint8)))
    assert st["rounds"] == 3 and st["segments_per_level"] == [1, 0, 2, 0] and st["grow_events"] == 0
    assert p.layout().valid_count == 23


@pytest.mark.parametrize("P", IMPLS)
def test_fixture_leaf_search_and_lazy_deletes(P):
    # test_pma.cpp:81-89, test_segment_engine.cpp:263-286
    p = P().load_slots(*fixture_arrays())
    assert list(p.binary_search_leaf([48, 35, 9, 1, 4, 1000])) == [5, 4, 1, 0, 0, 7]
    st = stats_dict(p.batch_update(np.array([30, 45, 999], np.uint64), np.zeros(3, np.uint64), np.ones(3, np.uint8)))
    assert (st["rounds"], st["tombstones_added"], st["deletes_missed"], st["num_touched_ranges"]) == (1, 2, 1, 0)


@pytest.mark.parametrize("P", IMPLS)
def test_even_placement_and_growth(P):
    # test_pma.cpp:228-247: 6 entries over 16 slots at {0,2,5,8,10,13}
    keys = np.array([100, 110, 120, 130, 140, 150], np.uint64)
    p = P().from_sorted(keys, keys, 0.5)
    k, v, s = p.slots()
    assert list(np.nonzero(s)[0]) == [0, 2, 5, 8, 10, 13]
    # test_segment_engine.cpp:250-261: root full at capacity 16 + 4 inserts -> one grow
    q = P().from_sorted(np.arange(12, dtype=np.uint64) * 7, np.arange(12, dtype=np.uint64), 0.9)
    assert q.layout().capacity == 16
    st = stats_dict(q.batch_update(np.array([3, 10, 17, 24], np.uint64), np.zeros(4, np.uint64), np.zeros(4, np.uint8)))
    assert st["grow_events"] == 1 and st["resized"] and q.layout().capacity == 32


@pytest.mark.parametrize("G", GRAPHS)
def test_worked_example_graph(G):
    # test_graph.cpp:51-58, test_analytics.cpp:37-42,60-64,157-163
    g = G(3, [0, 0, 1, 2, 2, 2], [0, 2, 2, 0, 1, 2], [1.0, 2.0, 3.0, 4.0, 5.0, 6.0])
    assert list(g.bfs(0)) == [0, 2, 1]
    assert list(g.cc()) == [0, 0, 0]
    assert list(g.spmv([1.0, 1.0, 1.0])) == [3, 3, 15]
    one = G(1, [], [])
    r, it, conv = one.pagerank()
    assert conv and list(r) == [1.0]
    pair = G(2, [0, 1], [1, 0])
    r, it, conv = pair.pagerank()
    assert conv and abs(r[0] - 0.5) < 1e-12 and abs(r[1] - 0.5) < 1e-12


def test_reference_csr_of_worked_example():
    g = RefGraph(3, [0, 0, 1, 2, 2, 2], [0, 2, 2, 0, 1, 2], [1.0, 2.0, 3.0, 4.0, 5.0, 6.0])
    ro, col, val = g.csr_snapshot()
    assert list(ro) == [0, 2, 3, 6] and list(col) == [0, 2, 2, 0, 1, 2] and list(val) == [1, 2, 3, 4, 5, 6]


def test_reference_rebuild_csr_baseline():
    """RebuildCsrGraph (baselines.hpp:85-181), the oracle of the GPU baseline:
    the worked example, one batch, and agreement with the PMA graph's CSR."""
    r = oracle.RefRebuildCsr(3, [0, 0, 1, 2, 2, 2], [0, 2, 2, 0, 1, 2], [1.0, 2.0, 3.0, 4.0, 5.0, 6.0])
    ro, col, val = r.csr()
    assert list(ro) == [0, 2, 3, 6] and list(col) == [0, 2, 2, 0, 1, 2] and list(val) == [1, 2, 3, 4, 5, 6]
    st = r.apply_batch([1], [0], [7.0], [0, 2], [2, 9])
    assert (st.batch_size, st.deletes_missed, st.slot_writes) == (3, 1, 16)
    ro, col, val = r.csr()
    assert list(ro) == [0, 1, 3, 6] and list(col) == [0, 0, 2, 0, 1, 2] and list(val) == [1, 7, 3, 4, 5, 6]
    with pytest.raises(oracle.OracleError, match="vertex id out of range"):
        oracle.RefRebuildCsr(3, [0], [3])
    rng = np.random.default_rng(4)
    s, d = rng.integers(0, 500, 4000), rng.integers(0, 500, 4000)
    r, g = oracle.RefRebuildCsr(500, s, d), RefGraph(500, s, d)
    for _ in range(3):
        a, b, c, e = (rng.integers(0, 500, 800) for _ in range(4))
        r.apply_batch(a, b, None, c, e)
        g.apply_batch(a, b, None, c, e)
        assert all((x == y).all() for x, y in zip(r.csr(), g.csr_snapshot()))


@pytest.mark.parametrize("name", ["window_er.npz", "window_rmat.npz"])
@pytest.mark.parametrize("G", GRAPHS)
def test_golden_windows(name, G):
    """Both oracles reproduce the committed golden sliding-window fixture."""
    z = gr.load(name)
    nv = int(z["nv"])
    s = z["stream_src"].astype(np.uint32)
    d = z["stream_dst"].astype(np.uint32)
    half = (len(s) + 1) // 2
    g = G(nv, s[:half], d[:half], None, graph_config(deletion_mode=int(z["mode"])))
    slots = g.slots() if G is RefGraph else g.pma().slots()
    assert gr.slot_hash(*slots) == str(z["init_hash"])
    warm = None
    for i, a, b, c, dd in gr.window_slides(z):
        st = stats_dict(g.apply_batch(a, b, None, c, dd))
        assert (gr.stats_vector(st) == z[f"s{i}_stats"]).all(), i
        assert st["segments_per_level"] == list(z[f"s{i}_spl"])
        slots = g.slots() if G is RefGraph else g.pma().slots()
        assert gr.slot_hash(*slots) == str(z[f"s{i}_hash"]), i
        assert (g.row_offsets() == z[f"s{i}_row_offsets"]).all()
        assert (g.bfs(int(z[f"s{i}_root"])) == z[f"s{i}_bfs"]).all()
        assert (g.cc() == z[f"s{i}_cc"]).all()
        ranks, iters, _ = g.pagerank(warm=warm)
        assert np.abs(ranks - z[f"s{i}_pr"]).max() <= 1e-12 and iters == int(z[f"s{i}_pr_iters"])
        warm = ranks
        assert (g.spmv(np.linspace(0.0, 1.0, nv)) == z[f"s{i}_spmv"]).all()


@pytest.mark.parametrize("P", IMPLS)
def test_golden_pma_trace(P):
    z = gr.load("pma_trace.npz")
    p = P().from_sorted(z["init_keys"], z["init_vals"], 0.5)
    assert gr.slot_hash(*p.slots()) == str(z["init_hash"])
    i = 0
    while f"b{i}_stats" in z:
        st = stats_dict(p.batch_update(z[f"b{i}_keys"], z[f"b{i}_vals"], z[f"b{i}_ops"],
                                       engine_config(deletion_mode=int(z[f"b{i}_mode"]))))
        assert (gr.stats_vector(st) == z[f"b{i}_stats"]).all(), i
        assert gr.slot_hash(*p.slots()) == str(z[f"b{i}_hash"]), i
        assert (p.binary_search_leaf(z[f"b{i}_probe"]) == z[f"b{i}_leaves"]).all()
        i += 1


def test_port_matches_reference_on_random_traces():
    rng = np.random.default_rng(1)
    for trial in range(60):
        mode = PMA_EAGER if trial % 2 else PMA_LAZY
        cfg = engine_config(deletion_mode=mode, force_strategy=PMA_STRATEGY_LARGE if trial % 5 == 0 else -1)
        universe = int(rng.integers(50, 100000))
        keys = np.unique(rng.integers(0, universe, int(rng.integers(0, 3000)), dtype=np.uint64))
        vals = rng.integers(0, 2**63, len(keys), dtype=np.uint64)
        fill = float(rng.uniform(0.1, 0.9))
        r, p = RefPMA().from_sorted(keys, vals, fill), PortPMA().from_sorted(keys, vals, fill)
        for b in range(5):
            n = int(rng.integers(0, 600))
            k = rng.integers(0, universe, n, dtype=np.uint64)
            v = rng.integers(0, 2**63, n, dtype=np.uint64)
            o = (rng.random(n) < rng.random()).astype(np.uint8)
            assert stats_dict(r.batch_update(k, v, o, cfg)) == stats_dict(p.batch_update(k, v, o, cfg))
            assert all((x == y).all() for x, y in zip(r.slots(), p.slots()))
            assert r.touched_ranges() == p.touched_ranges()
