"""Key-range sharded GPMA+  on one GPU: W shards in one process
(LocalComm — the same ShardedGraph code path as the NCCL deployment, the
collectives as loops).  Every global sliding-window batch is split into W
contiguous arrival shares, routed on the device (gpma_route_partition +
all-to-all) and applied per shard.  Checked after every batch, per shard,
bit-exact against a reference PackedMemoryArray built with from_sorted(shard
entries + shard guards, 0.5) and driven with batch_update(shard slice) — the
per-shard parity of SURVEY §8e — including every UpdateStats field and the
shard's row offsets; and globally against the single-graph reference:
BFS levels / CC labels / SpMV bit-exact, PageRank within 1e-6 with equal
iteration counts."""
import numpy as np
import pytest

from oracle.oracle import RefGraph, RefPMA, RefStream, RefWindow
from paper_1709_05061_b200 import sharding as sh
from paper_1709_05061_b200.abi import PMA_EAGER, PMA_LAZY, engine_config, graph_config
from paper_1709_05061_b200.pmagraph import GraphConfig
from paper_1709_05061_b200.sharded import LocalComm, ShardedGraph

pytestmark = pytest.mark.gpu

PR_TOL = 1e-6


def _dev(a, dtype):
    import torch
    arr = np.ascontiguousarray(a)
    if dtype == "u32":
        return torch.from_numpy(arr.astype(np.uint32).view(np.int32)).cuda()
    return torch.from_numpy(arr.astype(np.float64)).cuda()


def _ref_row_offsets(slots, lo, hi):
    k, _, s = slots
    ro = np.zeros(hi - lo + 1, np.uint64)
    g = np.nonzero((s == 1) & ((k & np.uint64(0xFFFFFFFF)) == np.uint64(0xFFFFFFFF)))[0]
    ro[(k[g] >> np.uint64(32)).astype(np.int64) - lo + 1] = g.astype(np.uint64) + np.uint64(1)
    return ro


@pytest.mark.parametrize("world,mode,kind,weighted,routing", [(2, PMA_LAZY, "rmat", False, "all_to_all"),
                                                              (3, PMA_EAGER, "rmat", True, "all_to_all"),
                                                              (4, PMA_LAZY, "er", True, "all_to_all"),
                                                              (2, PMA_EAGER, "rmat", True, "fused"),
                                                              (4, PMA_LAZY, "rmat", False, "fused")])
def test_sharded_window_parity(world, mode, kind, weighted, routing):
    """routing="fused": the owner partition writes straight into the owners'
    receive buffers (gpma_route_scatter_peer) instead of an all-to-all."""
    rng = np.random.default_rng(11)
    nv = 2**12
    stream = RefStream.rmat(nv, 40000, 5) if kind == "rmat" else RefStream.erdos_renyi(nv, 2**-8, 5)
    if kind == "er":
        stream.shuffle(2)
    s, d, w, _ = stream.arrays()
    half = (len(s) + 1) // 2
    w0 = rng.random(half) + 0.5 if weighted else None
    deg = np.bincount(s[:half], minlength=nv)
    bounds = sh.vertex_bounds(nv, world, deg)
    comm = LocalComm(world)
    edges = (_dev(s[:half], "u32"), _dev(d[:half], "u32"), _dev(w0, "f64") if weighted else None)
    G = ShardedGraph.from_edges_device(comm, nv, bounds, [edges] * world, GraphConfig(deletion_mode=mode),
                                       routing=routing)
    refs = []
    for r in range(world):
        lo, hi = int(bounds[r]), int(bounds[r + 1])
        keys, vals = sh.shard_entries(nv, s[:half], d[:half], w0, lo, hi)
        refs.append(RefPMA().from_sorted(keys, vals, 0.5))
        got = G.shard_slots(r)
        exp = refs[r].slots()
        assert all((x == y).all() for x, y in zip(got, exp)), f"init shard {r}"
    whole = RefGraph(nv, s[:half], d[:half], w0, graph_config(deletion_mode=mode))
    win = RefWindow(stream)
    warm_g = warm_r = None
    for slide in range(5):
        a, b, ww, c, dd = win.slide(1200)
        if weighted:
            ww = rng.random(len(a)) + 0.5
        if slide == 2:  # guard deletes and duplicate arrivals ride along
            c = np.concatenate([c, [int(bounds[1]) - 1, 3]]).astype(np.uint32)
            dd = np.concatenate([dd, [0xFFFFFFFF, 0xFFFFFFFF]]).astype(np.uint32)
            a = np.concatenate([a, a[:5]]).astype(np.uint32)
            b = np.concatenate([b, b[:5]]).astype(np.uint32)
            ww = np.concatenate([ww, ww[:5] + (1.0 if weighted else 0.0)])
        whole.apply_batch(a, b, ww, c, dd)
        ia = np.array_split(np.arange(len(a)), world)
        ic = np.array_split(np.arange(len(c)), world)
        slices = [(_dev(a[ia[r]], "u32"), _dev(b[ia[r]], "u32"), _dev(ww[ia[r]], "f64") if weighted else None,
                   _dev(c[ic[r]], "u32"), _dev(dd[ic[r]], "u32")) for r in range(world)]
        res = G.apply_batch(slices)
        for r in range(world):
            lo, hi = int(bounds[r]), int(bounds[r + 1])
            oi = sh.owner_of(a, bounds) == r
            od = sh.owner_of(c, bounds) == r
            keys, vals, ops, gdel = sh.shard_updates(a[oi], b[oi], ww[oi] if weighted else None, c[od], dd[od])
            rst = refs[r].batch_update(keys, vals, ops, engine_config(deletion_mode=mode))
            gst = res.stats[r]
            ctx = f"slide {slide} shard {r}"
            assert gst.batch_size == rst.batch_size, ctx
            assert gst.rounds == rst.rounds and gst.slot_writes == rst.slot_writes, ctx
            assert gst.deletes_missed == rst.deletes_missed + gdel, ctx
            assert gst.tombstones_added == rst.tombstones_added, ctx
            assert gst.segments_per_level == [rst.segments_per_level[i] for i in range(rst.num_levels)], ctx
            got = G.shard_slots(r)
            exp = refs[r].slots()
            assert all((x == y).all() for x, y in zip(got, exp)), ctx
            assert (G.shard_row_offsets(r) == _ref_row_offsets(exp, lo, hi)).all(), ctx
            assert res.routed[r] == int(oi.sum() + od.sum()), ctx
        root = int(rng.integers(0, nv))
        for dist in G.bfs(root):
            assert (dist.cpu().numpy().view(np.uint32) == whole.bfs(root)).all(), f"bfs slide {slide}"
        for lab in G.connected_components():
            assert (lab.cpu().numpy().view(np.uint32) == whole.cc()).all(), f"cc slide {slide}"
        x, it, conv = G.pagerank(warm_start=warm_g)
        pr = whole.pagerank(warm=warm_r)
        assert it == pr[1] and conv == pr[2], f"pagerank slide {slide}"
        for xi in x:
            assert np.abs(xi.cpu().numpy() - pr[0]).max() <= PR_TOL
        warm_g, warm_r = x[0].cpu().numpy(), pr[0]
        xv = rng.random(nv)
        for y in G.spmv(xv):
            assert (y.cpu().numpy() == whole.spmv(xv)).all(), f"spmv slide {slide}"


def test_route_partition_is_stable_and_exact():
    """gpma_route_partition == stable partition by owner (ids >= |V| go to
    the last rank), as EdgeKeys."""
    rng = np.random.default_rng(2)
    nv, world = 5000, 5
    bounds = np.array([0, 10, 1000, 1001, 4000, 5000], np.int64)
    comm = LocalComm(world)
    G = ShardedGraph.from_edges_device(comm, nv, bounds, [(_dev(np.zeros(0), "u32"), _dev(np.zeros(0), "u32"), None)]
                                       * world)
    for n in (0, 1, 3000, 70001):
        src = rng.integers(0, nv + 50, n).astype(np.uint32)
        src[::97] = (np.uint64(2 ** 31) + src[::97].astype(np.uint64)).astype(np.uint32)  # would alias via bit 63
        dst = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
        w = rng.random(n)
        ni = n // 3  # first third inserts, rest deletes (bit 63 on the wire)
        keys, ow, counts = G._route(0, _dev(src[:ni], "u32"), _dev(dst[:ni], "u32"), _dev(w[:ni], "f64"),
                                    _dev(src[ni:], "u32"), _dev(dst[ni:], "u32"))
        own = np.minimum(np.searchsorted(bounds, src.astype(np.int64), side="right") - 1, world - 1)
        order = np.argsort(own, kind="stable")
        isdel = np.arange(n) >= ni
        dbit = isdel.astype(np.uint64) << np.uint64(63)
        exp = (src.astype(np.uint64) << np.uint64(32)) | dst.astype(np.uint64) | dbit
        # a delete whose source is >= |V| travels as a key no graph holds (a
        # guard delete stays a guard delete): never an alias through bit 63
        absent = isdel & (src >= 2 ** 31)
        sentinel = np.where(dst == 0xFFFFFFFF, 0xFFFFFFFF,
                            np.minimum(dst.astype(np.uint64) | np.uint64(0x80000000), 0xFFFFFFFE)).astype(np.uint64)
        exp = np.where(absent, (np.uint64(0x7FFFFFFF) << np.uint64(32)) | sentinel | dbit, exp)[order]
        wexp = np.where(np.arange(n) < ni, w, 1.0)[order]
        bad = int(((src[:ni] >= nv) | (dst[:ni] >= nv)).sum())  # inserts outside the vertex range
        assert counts.cpu().tolist() == list(np.bincount(own, minlength=world)) + [bad]
        assert (keys.cpu().numpy().view(np.uint64) == exp).all()
        assert (ow.cpu().numpy() == wexp).all()


@pytest.mark.parametrize("routing", ["all_to_all", "fused"])
def test_sharded_bad_insert_rejected_everywhere(routing):
    """An insert naming a vertex >= |V| on ONE sender rejects the whole batch
    on every shard before any applies (check_ids, graph.hpp:133-137): no shard
    is left half-updated."""
    nv, world = 4096, 2
    rng = np.random.default_rng(3)
    s = rng.integers(0, nv, 5000).astype(np.uint32)
    d = rng.integers(0, nv, 5000).astype(np.uint32)
    bounds = np.array([0, nv // 2, nv], np.int64)
    G = ShardedGraph.from_edges_device(LocalComm(world), nv, bounds,
                                       [(_dev(s, "u32"), _dev(d, "u32"), None)] * world, routing=routing)
    before = [G.shard_slots(r) for r in range(world)]
    good = (_dev(np.array([1, 2], np.uint32), "u32"), _dev(np.array([3, 4], np.uint32), "u32"), None,
            _dev(np.array([], np.uint32), "u32"), _dev(np.array([], np.uint32), "u32"))
    bad = (_dev(np.array([nv - 1, 7], np.uint32), "u32"), _dev(np.array([5, nv + 3], np.uint32), "u32"), None,
           _dev(np.array([], np.uint32), "u32"), _dev(np.array([], np.uint32), "u32"))
    with pytest.raises(ValueError, match=f"edge \\(7, {nv + 3}\\) outside vertex range {nv}"):
        G.apply_batch([good, bad])
    for r in range(world):
        assert all((x == y).all() for x, y in zip(G.shard_slots(r), before[r])), f"shard {r} changed"


@pytest.mark.parametrize("routing", ["all_to_all", "fused"])
def test_sharded_delete_high_id_never_aliases(routing):
    """A delete whose source lies in [2^31, 2^32) must not remove the edge
    (src - 2^31, dst) through the wire's delete bit: it is counted missed,
    as the reference counts an absent delete (graph.hpp:140-145)."""
    nv, world = 4096, 2
    s = np.array([2050, 10, 3000], np.uint32)
    d = np.array([7, 11, 12], np.uint32)
    bounds = np.array([0, nv // 2, nv], np.int64)
    G = ShardedGraph.from_edges_device(LocalComm(world), nv, bounds,
                                       [(_dev(s, "u32"), _dev(d, "u32"), None)] * world, routing=routing)
    before = [G.shard_slots(r) for r in range(world)]
    empty = _dev(np.array([], np.uint32), "u32")
    dels = (empty, empty, None, _dev(np.array([2 ** 31 + 2050, 5000], np.uint32), "u32"),
            _dev(np.array([7, 1], np.uint32), "u32"))
    res = G.apply_batch([dels, (empty, empty, None, empty, empty)])
    assert sum(st.deletes_missed for st in res.stats) == 2
    for r in range(world):
        assert all((x == y).all() for x, y in zip(G.shard_slots(r), before[r])), f"shard {r} changed"
