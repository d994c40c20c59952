#!/usr/bin/env python
"""Small-batch latency breakdown on the C2 window: per batch size, the wall
time of apply_batch_device (host clock around the synchronous call), the
device time between its first and last kernel, and the per-stage /
per-level device times and launch counts the library reports."""
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
    stream = pg.EdgeStream.rmat(bench.NV, bench.NE, seed=bench.GEN_SEED).shuffle(bench.SHUFFLE_SEED)
    for B in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "10,100,1000,10000").split(",")]:
        win = pg.SlidingWindow(stream, 0)
        n = 12
        win.reserve(n * B + 16)
        info = win.info()
        g = pg.DynamicGraph.from_edges_device(bench.NV, info.stream_src, info.stream_dst, None, info.initial_size)
        slides = [win.slide(B) for _ in range(n)]
        info = win.info()
        walls, tms = [], []
        for i, s in enumerate(slides):
            torch.cuda.synchronize()
            t = time.perf_counter()
            st = g.apply_batch_device(info.stream_src + 4 * s.ins_offset, info.stream_dst + 4 * s.ins_offset, None,
                                      s.n_ins, info.del_src + 4 * s.del_offset, info.del_dst + 4 * s.del_offset,
                                      s.n_del)
            w = time.perf_counter() - t
            if i >= 4:
                walls.append(w * 1e6)
                tms.append((g.last_timing(), st))
        tm, st = tms[-1]
        print(f"B={B}: wall us median {sorted(walls)[len(walls) // 2]:.1f} min {min(walls):.1f}; "
              f"device {tm.device_ms * 1e3:.1f} us sort {tm.sort_ms * 1e3:.1f} search {tm.search_ms * 1e3:.1f} "
              f"rounds {tm.rounds_ms * 1e3:.1f} refresh {tm.refresh_ms * 1e3:.1f}; launches {tm.kernel_launches}; "
              f"rounds {st.rounds}; levels "
              + " ".join(f"{tm.level_ms[i] * 1e3:.0f}/{tm.level_groups[i]}" for i in range(16) if tm.level_groups[i]),
              flush=True)
        del g, win


if __name__ == "__main__":
    main()
