"""CPU, world size 2 over gloo: source-range sharding of the GPMA+ update path
(paper_1709_05061_b200/sharding.py).  Each rank holds half of every global
batch; updates are routed by an all-to-all; each owner applies its slice to
its shard.  Checked: (1) routed slices == the global batch filtered by owner,
in global arrival order; (2) every shard's slot array is bit-exact against a
reference PackedMemoryArray built from the shard's entries + guards and
driven with the shard slice (the per-shard parity definition of SURVEY §8e);
(3) the union of the shards equals the single-graph reference's edge set."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import oracle

pytestmark = pytest.mark.skipif(not oracle.have_ref(), reason="reference oracle not built")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_q):
    import torch.distributed as dist

    from oracle.oracle import RefGraph, RefPMA, RefStream, RefWindow, stats_dict
    from paper_1709_05061_b200 import sharding as sh

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nv = 2**10
        stream = RefStream.rmat(nv, 20000, seed=3)
        s, d, w, _ = stream.arrays()
        half = (len(s) + 1) // 2
        deg = np.bincount(s[:half], minlength=nv)
        bounds = sh.vertex_bounds(nv, world, deg)
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        keys, vals = sh.shard_entries(nv, s[:half], d[:half], w[:half], lo, hi)
        shard = RefPMA().from_sorted(keys, vals, 0.5)
        whole = RefGraph(nv, s[:half], d[:half], w[:half])  # single-graph reference
        win = RefWindow(stream)
        for it in range(5):
            a, b, ww, c, dd = win.slide(1500)
            whole.apply_batch(a, b, ww, c, dd)
            # this rank's contiguous share of the global batch (arrival order)
            ia = np.array_split(np.arange(len(a)), world)[rank]
            ic = np.array_split(np.arange(len(c)), world)[rank]
            (rs, rd, rw), (xs, xd) = sh.route_batch(a[ia], b[ia], ww[ia], c[ic], dd[ic], bounds)
            # (1) routing == global batch filtered by owner, in order
            own_i = sh.owner_of(a, bounds) == rank
            own_d = sh.owner_of(c, bounds) == rank
            assert (rs == a[own_i]).all() and (rd == b[own_i]).all() and (rw == ww[own_i]).all()
            assert (xs == c[own_d]).all() and (xd == dd[own_d]).all()
            # (2) per-shard engine (the reference PMA) on the routed slice
            k, v, o, guard_deletes = sh.shard_updates(rs, rd, rw, xs, xd)
            shard.batch_update(k, v, o)
        sk, sv, ss = shard.slots()
        mine = sk[ss == 1]
        allk = mine[(mine & np.uint64(0xFFFFFFFF)) != np.uint64(0xFFFFFFFF)]
        gathered = [None] * world
        dist.all_gather_object(gathered, allk.tolist())
        if rank == 0:
            wk, wv, ws = whole.slots()
            ref_edges = wk[(ws == 1) & ((wk & np.uint64(0xFFFFFFFF)) != np.uint64(0xFFFFFFFF))]
            union = np.array(sorted(x for part in gathered for x in part), np.uint64)
            result_q.put(("ok", bool((union == ref_edges).all()) and len(union) == len(ref_edges)))
    except Exception as e:  # pragma: no cover - surfaced to the parent
        result_q.put(("error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_sharded_updates_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, q), nprocs=2, join=True, start_method="spawn")
    status, ok = q.get(timeout=60)
    assert status == "ok" and ok, ok


def test_vertex_bounds_balance_edges():
    from paper_1709_05061_b200 import sharding as sh
    deg = np.zeros(100, np.int64)
    deg[:10] = 100  # hubs at low ids
    b = sh.vertex_bounds(100, 4, deg)
    assert b[0] == 0 and b[-1] == 100 and (np.diff(b) >= 0).all()
    w = np.add.reduceat(deg + 1, b[:-1])
    assert w.max() <= 2 * w.mean()
    assert list(sh.vertex_bounds(10, 3)) == [0, 3, 6, 10]


def _comm_worker(rank, world, port, result_q):
    import torch
    import torch.distributed as dist

    from paper_1709_05061_b200.sharded import TorchComm

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = TorchComm()
        # all_to_all_v: owner-major send buffers with variable counts
        rng = np.random.default_rng(rank)
        cnt = [int(x) for x in rng.integers(0, 5, world)]
        buf = torch.tensor([1000 * rank + 10 * r + j for r in range(world) for j in range(cnt[r])], dtype=torch.int64)
        (out,), (rc,), _ = c.all_to_all_v([buf], [cnt])
        allc = [[int(x) for x in np.random.default_rng(s).integers(0, 5, world)] for s in range(world)]
        exp = [1000 * s + 10 * rank + j for s in range(world) for j in range(allc[s][rank])]
        ok = out.tolist() == exp and rc == [allc[s][rank] for s in range(world)]
        for op, f in (("sum", sum), ("max", max), ("min", min)):
            t = torch.tensor([rank, 7 - rank, 3], dtype=torch.int32)
            c.all_reduce([t], op)
            ok &= t.tolist() == [f(range(world)), f(7 - r for r in range(world)), f([3] * world)]
        (g,) = c.all_gather_v([torch.arange(rank + 2, dtype=torch.float64) + rank])
        ok &= g.tolist() == [float(x + r) for r in range(world) for x in range(r + 2)]
        result_q.put(("ok", ok))
    except Exception as e:  # pragma: no cover
        result_q.put(("error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_torch_comm_collectives_gloo(world):
    """The collectives ShardedGraph runs between its device steps
    (paper_1709_05061_b200/sharded.py TorchComm): variable all-to-all in
    sender-rank order, sum/max/min all-reduce, variable all-gather."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    mp.start_processes(_comm_worker, args=(world, port, q), nprocs=world, join=True, start_method="spawn")
    res = [q.get(timeout=60) for _ in range(world)]
    assert all(s == "ok" and ok for s, ok in res), res


def test_fused_routing_offsets_match_all_to_all_order():
    """sharded.fused_offsets: each owner's receive buffer, filled by every
    sender at its offsets, equals the all-to-all concatenation (sender order,
    arrival order within a sender)."""
    from paper_1709_05061_b200.sharded import fused_offsets
    rng = np.random.default_rng(3)
    for W in (1, 2, 3, 8):
        M = rng.integers(0, 50, (W, W))
        before, nrecv = fused_offsets(M)
        sends = [[np.arange(M[s][r]) + 1000 * s + 100000 * r for r in range(W)] for s in range(W)]
        for r in range(W):
            buf = np.full(int(nrecv[r]), -1)
            for s in range(W):
                buf[before[s][r]:before[s][r] + M[s][r]] = sends[s][r]
            expect = np.concatenate([sends[s][r] for s in range(W)]) if W else np.zeros(0)
            assert (buf == expect).all()
