#!/usr/bin/env python
"""Phase timing of the sharded step (route / all-to-all / apply) at N = 1 (NCCL, one rank)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    import bench
    from paper_1709_05061_b200 import pmagraph as pg
    from paper_1709_05061_b200.abi import load_library
    from paper_1709_05061_b200.sharded import ShardedGraph, TorchComm
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29544")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    load_library().gpma_warmup(0)
    B = 1_000_000
    stream = pg.EdgeStream.rmat(bench.NV, bench.NE, seed=1).shuffle(2)
    win = pg.SlidingWindow(stream, 0)
    win.reserve(12 * B)
    info = win.info()
    init = info.initial_size
    e_src = bench._wrap_device(info.stream_src, init, torch.int32, 0)
    e_dst = bench._wrap_device(info.stream_dst, init, torch.int32, 0)
    G = ShardedGraph.from_edges_device(TorchComm(), bench.NV, [0, bench.NV], [(e_src, e_dst, None)], devices=[0])
    slides = [win.slide(B) for _ in range(10)]
    info = win.info()
    W = bench._wrap_device
    ph = {"route": 0.0, "a2a": 0.0, "apply": 0.0}
    for k, sl in enumerate(slides):
        sl_t = (W(info.stream_src + 4 * sl.ins_offset, sl.n_ins, torch.int32, 0),
                W(info.stream_dst + 4 * sl.ins_offset, sl.n_ins, torch.int32, 0), None,
                W(info.del_src + 4 * sl.del_offset, sl.n_del, torch.int32, 0),
                W(info.del_dst + 4 * sl.del_offset, sl.n_del, torch.int32, 0))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        keys, ow, cnt = G._route(0, sl_t[0], sl_t[1], None, sl_t[3], sl_t[4])
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        rk, _, _ = G.comm.all_to_all_v([keys], [cnt])
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        st = __import__("paper_1709_05061_b200.abi", fromlist=["pma_stats"]).pma_stats()
        import ctypes as C
        G._check(0, G._lib.gpma_apply_batch_routed_device(G.h[0], C.c_void_p(rk[0].data_ptr()), None, rk[0].numel(),
                                                           C.byref(st)))
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        if k >= 3:
            ph["route"] += (t1 - t0) * 1e3 / 7
            ph["a2a"] += (t2 - t1) * 1e3 / 7
            ph["apply"] += (t3 - t2) * 1e3 / 7
    print({k: round(v, 3) for k, v in ph.items()})
    tm = G.last_timing()
    print("sort", tm.sort_ms, "search", tm.search_ms, "rounds", tm.rounds_ms, "refresh", tm.refresh_ms)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
