"""Bit-exact parity at the BASELINE.json configs' STATED sizes.

tests/golden/config_<C>.json holds, per slide of the bench's own stream, what
the UNMODIFIED reference computed (tests/golden/make_config_fixtures.py runs
oracle/_ref: DynamicGraph::apply_batch over SlidingWindow::slide,
graph.hpp:130-162, streaming.hpp:107-123).  Here the same slides run on the
device path bench.py times (device generator + device window +
from_edges_device + apply_batch_device) and every slide must match:

* every UpdateStats field (batch_size, rounds, slot_writes,
  segments_per_level, grow/shrink events, deletes_missed, tombstones_added,
  resized) and the digest of touched_ranges in the reference's order;
* capacity, valid and tombstone counts;
* the per-chunk digest of the whole slot array (keys, values, states = gap
  positions; pma_slot_hash on the device = tests/golden/hashing.py on the
  reference's slots()) and of the row offsets;
* at the analytics checkpoints: BFS distances (digest + reached count) from
  the reference-protocol roots and the largest row, CC labels (digest), and
  PageRank iterations + ranks of 4096 sampled and the 64 top vertices within
  1e-6 (analytics.hpp:22-143).
"""
import json
import os

import numpy as np
import pytest

from paper_1709_05061_b200 import pmagraph as pg
from tests.golden.hashing import vec_hash

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CONFIGS = [c for c in ("C1", "C2", "C3", "C5", "C4") if os.path.exists(os.path.join(HERE, f"config_{c}.json"))]
STATS = ["batch_size", "rounds", "slot_writes", "grow_events", "shrink_events", "deletes_missed",
         "tombstones_added", "resized"]


def hexes(a):
    return [f"{int(x):016x}" for x in a]


def check_analytics(g, fx, want, ctx):
    for b in want["bfs"]:
        dist, reached = pg.bfs(g, b["root"], return_reached=True)
        assert reached == b["reached"], f"{ctx} bfs root {b['root']} reached"
        assert vec_hash(dist) == b["hash"], f"{ctx} bfs root {b['root']} distances"
    assert vec_hash(pg.connected_components(g)) == want["cc_hash"], f"{ctx} cc labels"
    pr = pg.pagerank(g)
    w = want["pagerank"]
    assert pr.iterations == w["iterations"] and pr.converged == w["converged"], f"{ctx} pagerank iterations"
    err = np.abs(pr.ranks[np.array(w["sample_ids"])] - np.array(w["sample"])).max()
    err_top = np.abs(pr.ranks[np.array(w["top_ids"])] - np.array(w["top"])).max()
    assert max(err, err_top) <= 1e-6, f"{ctx} pagerank max abs error {max(err, err_top)}"
    assert abs(pr.ranks.sum() - w["sum"]) <= 1e-6


@pytest.mark.parametrize("name", CONFIGS)
def test_config_bit_exact_per_slide(name):
    with open(os.path.join(HERE, f"config_{name}.json")) as f:
        fx = json.load(f)
    nv, B = fx["num_vertices"], fx["batch"]
    stream = (pg.EdgeStream.rmat(nv, int(fx["param"]), seed=1) if fx["generator"] == "rmat"
              else pg.EdgeStream.erdos_renyi(nv, fx["param"], seed=1))
    if fx["shuffle"] is not None:
        stream.shuffle(fx["shuffle"])
    assert len(stream) == fx["stream_edges"], "device generator differs from the reference's"
    win = pg.SlidingWindow(stream, 0)
    nsl = len(fx["slides"])
    win.reserve(nsl * B + 16)
    info = win.info()
    assert info.initial_size == fx["initial_size"]
    g = pg.DynamicGraph.from_edges_device(nv, info.stream_src, info.stream_dst, None, info.initial_size, device=0)
    p = g.pma()
    level = fx["chunk_log2"] - (p.leaf_size().bit_length() - 1)
    assert p.capacity() == fx["init"]["capacity"] and p.valid_count() == fx["init"]["valid_count"]
    assert hexes(p.slot_hash(level)) == fx["init"]["slot_hashes"], f"{name} initial slot array"
    assert vec_hash(g.row_offsets()) == fx["init"]["row_offsets_hash"]
    slides = [win.slide(B) for _ in range(nsl)]
    info = win.info()
    for i, (s, want) in enumerate(zip(slides, fx["slides"])):
        ctx = f"{name} slide {i}"
        assert (s.n_ins, s.n_del) == (want["n_ins"], want["n_del"]), f"{ctx} window batch"
        st = g.apply_batch_device(info.stream_src + 4 * s.ins_offset, info.stream_dst + 4 * s.ins_offset, None,
                                  s.n_ins, info.del_src + 4 * s.del_offset, info.del_dst + 4 * s.del_offset, s.n_del)
        got = {f: getattr(st, f) for f in STATS}
        tr = p.touched_ranges_array().reshape(-1)
        got["num_touched_ranges"] = len(tr) // 2
        assert got == want["stats"], ctx
        assert list(st.segments_per_level) == want["segments_per_level"], ctx
        assert vec_hash(tr) == want["touched_hash"], f"{ctx} touched ranges"
        assert (p.capacity(), p.valid_count(), p.tombstone_count()) == \
            (want["capacity"], want["valid_count"], want["tombstone_count"]), ctx
        lv = fx["chunk_log2"] - (p.leaf_size().bit_length() - 1)
        assert hexes(p.slot_hash(lv)) == want["slot_hashes"], f"{ctx} slot array"
        assert vec_hash(g.row_offsets()) == want["row_offsets_hash"], f"{ctx} row offsets"
        if "analytics" in want:
            check_analytics(g, fx, want["analytics"], ctx)
