#!/usr/bin/env python
"""Where the host time between device-resident slides goes: the C2 main
loop timed by CUDA events with (a) nothing else, (b) last_timing() per step,
(c) the NVML clock sampler thread running, (d) both — plus the wall time of
each apply_batch_device call against its device span."""
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

    def run(tag, with_timing, sampler, n=12):
        g = pg.DynamicGraph.from_edges_device(cfg["nv"], info.stream_src, info.stream_dst, None, info.initial_size)
        g.reserve_batch(2 * B + 16)
        ext = torch.cuda.ExternalStream(g._lib.gpma_cuda_stream(g.h), device=torch.device("cuda", 0))
        for s in slides[:3]:
            bench_apply(g, info, s)
        torch.cuda.synchronize()
        cs = bench.ClockSampler(0) if sampler else None
        if cs:
            cs.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        walls, devs = [], []
        e0.record(ext)
        for s in slides[3:3 + n]:
            t = time.perf_counter()
            bench_apply(g, info, s)
            walls.append((time.perf_counter() - t) * 1e3)
            if with_timing:
                devs.append(g.last_timing().device_ms)
        e1.record(ext)
        torch.cuda.synchronize()
        if cs:
            cs.stop()
        ms = e0.elapsed_time(e1) / n
        print(f"{tag}: {ms:.3f} ms/step (events); wall per call median {sorted(walls)[n // 2]:.3f} max "
              f"{max(walls):.3f}; device span {(sum(devs) / len(devs)) if devs else float('nan'):.3f}", flush=True)

    def bench_apply(g, info, s):
        return g.apply_batch_device(info.stream_src + 4 * s.ins_offset, info.stream_dst + 4 * s.ins_offset, None,
                                    s.n_ins, info.del_src + 4 * s.del_offset, info.del_dst + 4 * s.del_offset,
                                    s.n_del)

    for rep in range(2):
        run("plain", False, False)
        run("last_timing", True, False)
        run("sampler", False, True)
        run("both", True, True)


if __name__ == "__main__":
    main()
