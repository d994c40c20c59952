#!/usr/bin/env python
"""Host time per device-resident slide on a graph rebuilt while an older one
is alive (the bench's second pass): per-call wall vs device span."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    from paper_1709_05061_b200 import pmagraph as pg
    from paper_1709_05061_b200.abi import load_library

    load_library().gpma_warmup(0)
    cfg = bench.CONFIGS["C2"]
    B = cfg["batch"]
    stream = bench.make_stream(pg, cfg, 1)
    win = pg.SlidingWindow(stream, 0)
    win.reserve(15 * B + 16)
    info = win.info()
    slides = [win.slide(B) for _ in range(15)]
    info = win.info()

    def make():
        g = pg.DynamicGraph.from_edges_device(cfg["nv"], info.stream_src, info.stream_dst, None, info.initial_size)
        g.reserve_batch(2 * B + 16)
        return g

    def run(tag, g, sl):
        walls, devs = [], []
        for s in sl:
            torch.cuda.synchronize()
            t = time.perf_counter()
            g.apply_batch_device(info.stream_src + 4 * s.ins_offset, info.stream_dst + 4 * s.ins_offset, None,
                                 s.n_ins, info.del_src + 4 * s.del_offset, info.del_dst + 4 * s.del_offset, s.n_del)
            walls.append((time.perf_counter() - t) * 1e3)
            devs.append(g.last_timing().device_ms)
        print(tag, "wall", [round(x, 3) for x in walls], "dev", [round(x, 3) for x in devs], flush=True)

    a = make()
    run("A 0-14", a, slides)
    b = make()
    run("B 0-9 (A alive)", b, slides[:10])
    del a
    c = make()
    run("C 0-9 (A freed, B alive)", c, slides[:10])
    del b, c
    d = make()
    run("D 0-9 (alone)", d, slides[:10])


if __name__ == "__main__":
    main()
