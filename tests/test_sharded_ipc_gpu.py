"""Fused routing across PROCESSES (one shard per process, as under torchrun):
the receive buffers are exported as CUDA IPC handles and every sender's
partition kernel stores into its peers' buffers.  Two processes share the
one GPU here (gloo for the count / handle exchange and the barrier); the
shards they end with must equal the in-process all-to-all run's."""
import os
import pickle
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NV, WORLD = 2**12, 2


def _data():
    from oracle.oracle import RefStream, RefWindow
    stream = RefStream.rmat(NV, 40000, 5)
    s, d, w, _ = stream.arrays()
    half = (len(s) + 1) // 2
    win = RefWindow(stream)
    batches = [win.slide(1500) for _ in range(3)]
    return s[:half], d[:half], batches


def _bounds(s):
    from paper_1709_05061_b200 import sharding as sh
    return sh.vertex_bounds(NV, WORLD, np.bincount(s, minlength=NV))


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).astype(np.uint32).view(np.int32)).cuda()


def _worker(rank, port, out):
    import torch
    import torch.distributed as dist
    from paper_1709_05061_b200.sharded import ShardedGraph, TorchComm
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    torch.cuda.set_device(0)
    s, d, batches = _data()
    bounds = _bounds(s)
    G = ShardedGraph.from_edges_device(TorchComm(), NV, bounds, [(_dev(s), _dev(d), None)], devices=[0],
                                       routing="fused")
    for a, b, _, c, dd in batches:
        ia = np.array_split(np.arange(len(a)), WORLD)[rank]
        ic = np.array_split(np.arange(len(c)), WORLD)[rank]
        G.apply_batch([(_dev(a[ia]), _dev(b[ia]), None, _dev(c[ic]), _dev(dd[ic]))])
    with open(out, "wb") as f:
        pickle.dump(G.shard_slots(0), f)
    dist.barrier()
    del G
    dist.destroy_process_group()


def test_fused_routing_across_processes():
    import torch.multiprocessing as mp
    from paper_1709_05061_b200.sharded import LocalComm, ShardedGraph
    tmp = tempfile.mkdtemp()
    outs = [os.path.join(tmp, f"shard{r}.pkl") for r in range(WORLD)]
    port = 29000 + os.getpid() % 1000
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=_worker, args=(r, port, outs[r])) for r in range(WORLD)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(240)
        assert p.exitcode == 0
    s, d, batches = _data()
    bounds = _bounds(s)
    G = ShardedGraph.from_edges_device(LocalComm(WORLD), NV, bounds, [(_dev(s), _dev(d), None)] * WORLD)
    for a, b, _, c, dd in batches:
        ia = np.array_split(np.arange(len(a)), WORLD)
        ic = np.array_split(np.arange(len(c)), WORLD)
        G.apply_batch([(_dev(a[ia[r]]), _dev(b[ia[r]]), None, _dev(c[ic[r]]), _dev(dd[ic[r]]))
                       for r in range(WORLD)])
    for r in range(WORLD):
        with open(outs[r], "rb") as f:
            got = pickle.load(f)
        assert all((x == y).all() for x, y in zip(got, G.shard_slots(r))), f"shard {r}"
