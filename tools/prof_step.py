#!/usr/bin/env python
"""One C2 sliding-window step under the CUDA profiler API, for ncu.

Builds the bench's C2 window (RMAT 2^21 / 30.6M stream, 15.3M-edge window),
runs W warm-up slides, then brackets ONE apply_batch slide (batch B) with
cudaProfilerStart/Stop so `ncu --profile-from-start off` captures exactly one
step's kernels:

  ncu --profile-from-start off --metrics gpu__time_duration.sum ... python tools/prof_step.py
  ncu --profile-from-start off --set full -k regex:NAME python tools/prof_step.py
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1_000_000)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--analytics", action="store_true", help="profile BFS + CC + one warm PageRank instead")
    ap.add_argument("--bfs-root", type=int, default=-1, help="with --analytics: this BFS root (default: the largest hub)")
    ap.add_argument("--config", default="C2", help="bench.CONFIGS key (stream and |V|)")
    args = ap.parse_args()
    import torch

    import bench
    from paper_1709_05061_b200 import pmagraph as pg
    from paper_1709_05061_b200.abi import load_library

    load_library().gpma_warmup(0)
    cfg = bench.CONFIGS[args.config]
    stream = bench.make_stream(pg, cfg, bench.GEN_SEED)
    nv = cfg["nv"]
    win = pg.SlidingWindow(stream, 0)
    win.reserve((args.warmup + args.steps) * args.batch + 16)
    info = win.info()
    g = pg.DynamicGraph.from_edges_device(nv, info.stream_src, info.stream_dst, None, info.initial_size, device=0)
    slides = [win.slide(args.batch) for _ in range(args.warmup + args.steps)]
    info = win.info()

    def apply(s):
        return g.apply_batch_device(info.stream_src + 4 * s.ins_offset, info.stream_dst + 4 * s.ins_offset, None,
                                    s.n_ins, info.del_src + 4 * s.del_offset, info.del_dst + 4 * s.del_offset, s.n_del)

    for s in slides[:args.warmup]:
        apply(s)
    torch.cuda.synchronize()
    if args.analytics:
        import numpy as np
        ro = g.row_offsets()
        root = int(np.argmax(np.diff(ro.astype(np.int64)))) if args.bfs_root < 0 else args.bfs_root
        pr = pg.pagerank(g)
        pg.bfs(g, root)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        pg.bfs(g, root)
        pg.connected_components(g)
        pg.pagerank(g, warm_start=pr.ranks, epsilon=0.0, max_iters=2)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        print("analytics ok")
        return
    torch.cuda.profiler.start()
    for s in slides[args.warmup:]:
        st = apply(s)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("step ok:", st.batch_size, "updates,", st.rounds, "rounds")


if __name__ == "__main__":
    main()
