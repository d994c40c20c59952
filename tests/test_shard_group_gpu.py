"""The C-ABI shard group (gpma_shard_group_*, csrc/shard_group.cu): the
library issues every collective itself over NCCL.  One GPU per gpurun, so the
group runs with world = 1 here (NCCL's self send/recv, reduce-scatter,
all-gather and all-reduce all execute); it must match the single-graph
reference bit-exactly (slots, UpdateStats, BFS, CC, SpMV) and PageRank
within 1e-6, and reject a batch with an out-of-range insert without applying
it.  The world >= 2 partition logic is the same as the LocalComm/gloo paths
(test_sharded_gpu.py, test_sharding_gloo.py)."""
import numpy as np
import pytest

from oracle.oracle import RefGraph, RefStream, RefWindow
from paper_1709_05061_b200.abi import PMA_EAGER, PMA_LAZY, graph_config
from paper_1709_05061_b200.pmagraph import GraphConfig
from paper_1709_05061_b200.sharded import ShardGroup, nccl_unique_id

pytestmark = pytest.mark.gpu


def _dev(a, dtype="u32"):
    import torch
    arr = np.ascontiguousarray(a)
    if dtype == "u32":
        return torch.from_numpy(arr.astype(np.uint32).view(np.int32)).cuda()
    return torch.from_numpy(arr.astype(np.float64)).cuda()


@pytest.mark.parametrize("mode,weighted", [(PMA_LAZY, False), (PMA_EAGER, True)])
def test_shard_group_world1_matches_reference(mode, weighted):
    rng = np.random.default_rng(7)
    nv = 1 << 12
    stream = RefStream.rmat(nv, 60000, 3)
    s, d, w, _ = stream.arrays()
    half = (len(s) + 1) // 2
    w0 = rng.random(half) + 0.5 if weighted else None
    G = ShardGroup(nv, [0, nv], 0, 1, nccl_unique_id(),
                   (_dev(s[:half]), _dev(d[:half]), _dev(w0, "f64") if weighted else None),
                   GraphConfig(deletion_mode=mode))
    ref = RefGraph(nv, s[:half], d[:half], w0, graph_config(deletion_mode=mode))
    win = RefWindow(stream)
    for b in (500, 3000, 20000):
        a, bb, ww, c, dd = win.slide(b)
        if weighted:
            ww = rng.random(len(a)) + 0.5
        st, routed, sent = G.apply_batch(_dev(a), _dev(bb), _dev(ww, "f64") if weighted else None, _dev(c), _dev(dd))
        rst = ref.apply_batch(a, bb, ww if weighted else None, c, dd)
        assert (st.batch_size, st.rounds, st.slot_writes, st.deletes_missed, st.tombstones_added) == \
            (rst.batch_size, rst.rounds, rst.slot_writes, rst.deletes_missed, rst.tombstones_added)
        assert routed == len(a) + len(c) and sent == 0
        assert all((x == y).all() for x, y in zip(G.shard_slots(), ref.slots()))
        assert (G.shard_row_offsets() == ref.row_offsets()).all()
        root = int(np.argmax(np.diff(ref.row_offsets().astype(np.int64))))
        dist, reached = G.bfs(root)
        rdist = ref.bfs(root)
        assert (dist == rdist).all() and reached == int((rdist != 0xFFFFFFFF).sum())
        assert (G.connected_components() == ref.cc()).all()
        x, it, conv = G.pagerank()
        rx, rit, rconv = ref.pagerank()
        assert it == rit and conv == rconv and np.abs(x - rx).max() <= 1e-6
        xv = rng.random(nv)
        assert (G.spmv(xv) == ref.spmv(xv)).all()


def test_shard_group_rejects_out_of_range_insert():
    nv = 1024
    s = np.arange(100, dtype=np.uint32)
    d = (s * 7 % nv).astype(np.uint32)
    G = ShardGroup(nv, [0, nv], 0, 1, nccl_unique_id(), (_dev(s), _dev(d), None))
    before = G.shard_slots()
    with pytest.raises(ValueError, match=f"edge \\(3, {nv + 1}\\) outside vertex range {nv}"):
        G.apply_batch(_dev(np.array([1, 3], np.uint32)), _dev(np.array([2, nv + 1], np.uint32)), None,
                      _dev(np.array([], np.uint32)), _dev(np.array([], np.uint32)))
    assert all((x == y).all() for x, y in zip(G.shard_slots(), before))


def test_shard_group_bfs_hub_rows():
    """Rows longer than the mark kernel's hub threshold (4096 slots) are
    marked by CTA parts (k_group_bfs_mark_hubs): a dense RMAT whose top rows
    exceed it, BFS from the hub and from an ordinary vertex vs the reference."""
    nv = 1 << 12
    stream = RefStream.rmat(nv, 400000, 5)
    s, d, _, _ = stream.arrays()
    half = (len(s) + 1) // 2
    G = ShardGroup(nv, [0, nv], 0, 1, nccl_unique_id(), (_dev(s[:half]), _dev(d[:half]), None), GraphConfig())
    ref = RefGraph(nv, s[:half], d[:half], None, graph_config())
    ro = ref.row_offsets().astype(np.int64)
    lens = np.diff(ro)
    assert lens.max() > 4096, "the graph must have a hub row above the threshold"
    for root in (int(np.argmax(lens)), int(np.argsort(lens)[len(lens) // 2])):
        dist, reached = G.bfs(root)
        rdist = ref.bfs(root)
        assert (dist == rdist).all() and reached == int((rdist != 0xFFFFFFFF).sum())
