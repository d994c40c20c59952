"""GPU: the product replays the committed golden fixtures (generated from the
unmodified reference, tests/golden/make_golden.py) — no oracle involved at
run time.  Slot arrays by sha256, every UpdateStats field, row offsets, BFS,
CC, SpMV bit-exact; PageRank within 1e-6 (north_star)."""
import numpy as np
import pytest

from paper_1709_05061_b200.pmagraph import (DynamicGraph, GraphConfig, PackedMemoryArray, SegmentEngineConfig,
                                            batch_update, bfs, connected_components, pagerank, spmv)
from tests import golden_replay as gr

pytestmark = pytest.mark.gpu


def stats_of(us):
    d = us.parity()
    d["num_touched_ranges"] = len(d.pop("touched_ranges"))
    return d


@pytest.mark.parametrize("name", ["window_er.npz", "window_rmat.npz"])
def test_golden_window(name):
    z = gr.load(name)
    nv = int(z["nv"])
    s = z["stream_src"].astype(np.uint32)
    d = z["stream_dst"].astype(np.uint32)
    half = (len(s) + 1) // 2
    g = DynamicGraph.from_edges(nv, s[:half], d[:half], None, GraphConfig(deletion_mode=int(z["mode"])))
    assert gr.slot_hash(*g.pma().slots()) == str(z["init_hash"])
    warm = None
    for i, a, b, c, dd in gr.window_slides(z):
        st = g.apply_batch(a, b, None, c, dd)
        assert (gr.stats_vector(stats_of(st)) == z[f"s{i}_stats"]).all(), i
        assert st.segments_per_level == list(z[f"s{i}_spl"])
        assert st.touched_ranges == [tuple(int(x) for x in r) for r in z[f"s{i}_touched"]]
        assert gr.slot_hash(*g.pma().slots()) == str(z[f"s{i}_hash"]), i
        assert (g.row_offsets() == z[f"s{i}_row_offsets"]).all()
        assert (bfs(g, int(z[f"s{i}_root"])) == z[f"s{i}_bfs"]).all()
        assert (connected_components(g) == z[f"s{i}_cc"]).all()
        pr = pagerank(g, warm_start=warm)
        assert np.abs(pr.ranks - z[f"s{i}_pr"]).max() <= 1e-6 and pr.iterations == int(z[f"s{i}_pr_iters"])
        warm = pr.ranks
        assert (spmv(g, np.linspace(0.0, 1.0, nv)) == z[f"s{i}_spmv"]).all()


def test_golden_pma_trace():
    z = gr.load("pma_trace.npz")
    p = PackedMemoryArray.from_sorted(z["init_keys"], z["init_vals"], 0.5)
    assert gr.slot_hash(*p.slots()) == str(z["init_hash"])
    i = 0
    while f"b{i}_stats" in z:
        st = batch_update(p, z[f"b{i}_keys"], z[f"b{i}_vals"], z[f"b{i}_ops"],
                          SegmentEngineConfig(deletion_mode=int(z[f"b{i}_mode"])))
        assert (gr.stats_vector(stats_of(st)) == z[f"b{i}_stats"]).all(), i
        assert gr.slot_hash(*p.slots()) == str(z[f"b{i}_hash"]), i
        assert (p.binary_search_leaf(z[f"b{i}_probe"]) == z[f"b{i}_leaves"]).all()
        i += 1
