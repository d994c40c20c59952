#!/usr/bin/env python
"""bench.py — GPMA+ sliding-window update throughput on B200 (+ analytics).

Metric (BASELINE.json): "GPMA+ updates/sec vs batch size; BFS/PageRank/CC
time per sliding window".  A step is one slide of the C2 workload
(configs[1]): an RMAT 2^21 / 30.6M-edge stream (gen_rmat seed 1, shuffle
seed 2, generators.hpp:26-63 + streaming.hpp:58-67) whose first half seeds the
window; each slide inserts the next B arrivals and deletes the expired edges
whose multiplicity reaches zero (streaming.hpp:107-123).  updates = the
reference's UpdateStats::batch_size (inserts + non-guard deletes).

  value : updates/s with the slide batches already resident in HBM,
          CUDA events on the library's own stream around K steps.
  e2e   : the same K slides through the host C ABI (gpma_apply_batch) from
          pinned host buffers: H2D of inputs + D2H of the stats in the region.
  --impl reference : the unmodified reference (oracle/_ref) on the host cores
          (all hardware threads), same config/metric.

N > 1 (torchrun): every rank owns an independent source-vertex shard of the
same shape (its own stream seed), so there is no data-path collective;
value = all ranks' updates / max-over-ranks time ("scaling": "weak").
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GPMA+ updates/sec vs batch size; BFS/PageRank/CC time per sliding window"
UNIT = "updates/s"
NV = 1 << 21
NE = 30_600_000
GEN_SEED, SHUFFLE_SEED, ROOT_SEED = 1, 2, 7

# BASELINE.json configs.  The headline bench line is
# C2 (configs[1]); the others run with --config for evidence at their sizes.
CONFIGS = {
    "C1": dict(gen="er", nv=1 << 16, param=2.0 ** -12, shuffle=2, batch=1024,
               workload="C1 uniform random graph 2^16 vertices / 1M-edge stream, sliding window, batches of 1024"),
    "C2": dict(gen="rmat", nv=NV, param=NE, shuffle=2, batch=1_000_000,
               workload="C2 Pokec-shaped sliding window: RMAT 2^21 vertices / 30.6M-edge stream, 15.3M-edge "
                        "window, GPMA+ apply_batch per slide"),
    "C3": dict(gen="rmat", nv=1 << 22, param=34_400_000, shuffle=None, batch=344_000,
               workload="C3 Reddit-like skewed stream: RMAT 2^22 / 34.4M edges in generation order, batch 1% "
                        "(344,000), PageRank per window"),
    "C4": dict(gen="rmat", nv=1 << 24, param=1 << 28, shuffle=2, batch=2_684_354,
               workload="C4 Graph500 RMAT scale 24, edge factor 16 (268M-edge stream, 134M-edge window), batch 1% "
                        "(2,684,354), CC per window"),
    "C5": dict(gen="er", nv=1_000_000, param=2e-4, shuffle=2, batch=1_000_000,
               workload="C5 random graph 1M vertices / 200M-edge stream (100M-edge window), batch 10^6 "
                        "(~50% deletions)"),
}


def make_stream(pg, cfg, seed):
    st = (pg.EdgeStream.rmat(cfg["nv"], int(cfg["param"]), seed=seed) if cfg["gen"] == "rmat"
          else pg.EdgeStream.erdos_renyi(cfg["nv"], cfg["param"], seed=seed))
    if cfg["shuffle"] is not None:
        st.shuffle(cfg["shuffle"])
    return st
BYTES_PER_MERGE_SLOT = 34  # 17 B read + 17 B write per rewritten slot


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=None, help="default: the config's batch")
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--sweep", default="100,1000,5000,10000,100000,1000000")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-analytics", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no sweep/baseline/analytics)")
    ap.add_argument("--routing", default="group", choices=["group", "fused", "all_to_all"],
                    help="sharded update routing: the library's own NCCL collectives through the C ABI (group), "
                         "the partition kernel storing into the owners' receive buffers over peer memory (fused), "
                         "or an NCCL all-to-all via torch.distributed")
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="N > 1: weak = the config scaled by N (default for C1-C3), strong = the config itself "
                         "(default for C4, C5)")
    ap.add_argument("--sharded", action="store_true",
                    help="run the key-range sharded (multi-GPU) path even at N = 1 (NCCL with one rank)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons during the timed region, read in-process
    through NVML (the nvidia-smi data source) so no subprocess contends for
    the driver while the timed kernels run."""

    REASONS = {  # nvmlClocksEventReason* bits
        0x0000000000000004: "sw_power_cap",
        0x0000000000000008: "hw_slowdown",
        0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000080: "hw_power_brake_slowdown",
    }

    def __init__(self, index, period=0.05):
        self.index = index
        self.period = period
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        self.started = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nvml = None
            self.max_mhz = None

    def _sample(self):
        nv = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except Exception:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        self.samples.append((sm, r))

    def start(self):
        self.started = True
        if self._nvml is None:
            return
        self._sample()

        def run():
            while not self._stop.wait(self.period):
                try:
                    self._sample()
                except Exception:
                    pass

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if self._nvml is None or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        try:
            self._sample()
        except Exception:
            pass
        sm = [s for s, _ in self.samples]
        reasons = sorted({name for _, r in self.samples for bit, name in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples), "source": "nvml (in-process, 50 ms period)"}


# ------------------------------------------------------------------ ours --

PMA_STATS_BYTES = 632  # sizeof(pma_stats), read back by every apply_batch


def full_slides(info, B):
    """Number of FULL slides of B arrivals the stream holds after the initial
    window (SlidingWindow::slide takes min(batch, remaining()),
    streaming.hpp:111): the bench never times a partial or empty slide."""
    P = int(info.stream_size - info.initial_size) // B
    if P < 1:
        raise SystemExit(f"bench: the stream holds no full slide of batch {B}")
    return P


def run_passes(g, make_graph, slides, P, W, K, on_step, dev, world, clocks, segments=None, stream_of=None,
               on_segment=None):
    """Drive W untimed warm-up steps then K timed steps over `slides` (the
    first min(W + K, P) full slides of the window, in order).  When a pass has
    used every slide the stream holds, the graph is rebuilt from the initial
    window (untimed) and the next pass replays the same slides — so every
    timed step is a full slide on a window in the state the reference would
    have.  Timed segments are bracketed by barrier + synchronize and timed by
    CUDA events on the library's stream; returns (graph, summed ms, passes);
    `segments` (if given) receives each timed segment's steps / event ms /
    host wall ms; on_segment(g, "start" | "end") runs just outside each timed
    segment."""
    import torch
    from paper_1709_05061_b200.abi import load_library
    lib = load_library()
    n_sl = len(slides)
    segments = [] if segments is None else segments
    total = 0.0
    cur = step = 0
    passes = 1
    while step < W + K:
        if cur == n_sl:
            g = None
            g = make_graph()
            cur = 0
            passes += 1
        timed = step >= W
        n = min(n_sl - cur, (W + K if timed else W) - step)
        if not timed:
            for s in slides[cur:cur + n]:
                on_step(g, s, False)
        else:
            sp = stream_of(g) if stream_of else lib.gpma_cuda_stream(g.h)
            ext = torch.cuda.ExternalStream(sp, device=torch.device("cuda", dev))
            if on_segment is not None:
                on_segment(g, "start")
            if world > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize()
            if clocks is not None and not clocks.started:
                clocks.start()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(ext)
            for s in slides[cur:cur + n]:
                on_step(g, s, True)
            e1.record(ext)
            torch.cuda.synchronize()
            wall = (time.perf_counter() - t0) * 1e3
            if world > 1:
                torch.distributed.barrier()
            total += e0.elapsed_time(e1)
            segments.append({"steps": n, "ms": round(e0.elapsed_time(e1), 4), "wall_ms": round(wall, 4)})
            if on_segment is not None:
                on_segment(g, "end")
        step += n
        cur += n
    return g, total, passes


def reduce_max_sum(ms, n, world):
    """(max over ranks of ms, sum over ranks of n)."""
    if world == 1:
        return ms, float(n)
    import torch
    t = torch.tensor([ms], device="cuda")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    u = torch.tensor([float(n)], device="cuda")
    torch.distributed.all_reduce(u)
    return float(t.item()), float(u.item())


def ncu_traffic(config):
    """DRAM bytes (read + write) per launch of the dominant kernel from the
    committed ncu --set full capture of THIS config, or None when none was
    taken (profiles/ncu_summary.json, keyed by config)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            rec = json.load(f).get("configs", {}).get(config)
        return None if rec is None else rec.get("commit_kernel_dram_bytes_per_launch")
    except Exception:
        return None


def gpu_local_cpus(dev):
    """The CPUs on the GPU's NUMA node (NVML): page-locked batches allocated
    from there sit next to the GPU's PCIe root, which the zero-copy reads of
    the front end feel directly.  None when NVML cannot tell."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(dev)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        return cpus or None
    except Exception:
        return None


def run_ours(args):
    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    all_cpus = os.sched_getaffinity(0)
    near = gpu_local_cpus(local)
    if near:  # host work and page-locked buffers on the GPU's NUMA node
        os.sched_setaffinity(0, near)
    if world > 1 or args.sharded:
        import torch.distributed as dist
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return run_sharded(args, rank, world, local)
    from paper_1709_05061_b200 import pmagraph as pg

    dev = local
    from paper_1709_05061_b200.abi import load_library
    load_library().gpma_warmup(dev)  # load every kernel before any timed region
    cfg = CONFIGS[args.config]
    nvx = cfg["nv"]
    B = args.batch or cfg["batch"]
    K, W = args.steps, args.warmup
    t0 = time.time()
    stream = make_stream(pg, cfg, GEN_SEED + rank)
    gen_s = time.time() - t0
    win = pg.SlidingWindow(stream, dev)
    info = win.info()
    # Every step is a FULL slide of B arrivals (streaming.hpp:108-112 takes
    # min(batch, remaining)): the stream holds P full slides after the initial
    # window, so W + K steps run in passes of at most P slides, the graph
    # rebuilt from the initial window (untimed) between passes.
    P = full_slides(info, B)
    win.reserve(min(W + K, P) * B + 16)
    info = win.info()
    slides = [win.slide(B) for _ in range(min(W + K, P))]
    for s in slides:
        assert s.n_ins == B and not s.final_partial, "bench slide is not a full slide"
    info = win.info()

    def make_graph():
        gr = pg.DynamicGraph.from_edges_device(nvx, info.stream_src, info.stream_dst, None, info.initial_size,
                                               device=dev)
        gr.reserve_batch(2 * B + 16)  # a slide = B inserts + <= B deletes: no allocation in a step
        return gr

    t1 = time.time()
    g = make_graph()
    load_s = time.time() - t1
    cap = g.pma().capacity()
    lib = g._lib

    def apply_dev(graph, s):
        return graph.apply_batch_device(info.stream_src + 4 * s.ins_offset, info.stream_dst + 4 * s.ins_offset,
                                        None, s.n_ins, info.del_src + 4 * s.del_offset,
                                        info.del_dst + 4 * s.del_offset, s.n_del)

    clocks = ClockSampler(dev)
    # Each timed step's stats land in a struct allocated before the timed
    # region (decoded after it); the timing records of the timed steps are
    # summed by the library (gpma_timing_sum, read once per timed segment):
    # reading every batch's record would wait for its deferred refresh tail.
    raw = [pg.pma_stats() for _ in range(K)]
    per_step = []
    tsums = []

    def on_step(graph, s, timed):
        if timed:
            st_raw = raw[len(per_step)]
            graph.apply_batch_device(info.stream_src + 4 * s.ins_offset, info.stream_dst + 4 * s.ins_offset, None,
                                     s.n_ins, info.del_src + 4 * s.del_offset, info.del_dst + 4 * s.del_offset,
                                     s.n_del, stats_out=st_raw)
            per_step.append(st_raw)
        else:
            apply_dev(graph, s)

    def on_segment(graph, phase):
        t, n = graph.timing_sum(reset=True)
        if phase == "end":
            tsums.append((t, n))

    segs = []
    g, ms, passes = run_passes(g, make_graph, slides, P, W, K, on_step, dev, world, clocks, segs,
                               on_segment=on_segment)
    clk = clocks.stop()
    updates = 0
    seg_ms = 0.0
    merge_slots = 0
    commit_bytes = 0
    launches = 0
    rounds = 0
    stage = {"sort_ms": 0.0, "search_ms": 0.0, "rounds_ms": 0.0, "refresh_ms": 0.0}
    level_ms = [0.0] * 16
    level_bytes = [0] * 16
    level_groups = [0] * 16
    level_big = [0] * 16
    level_maxs = [0] * 16
    per_step = [pg.UpdateStats.from_c(st) for st in per_step]
    for st in per_step:
        updates += st.batch_size
        seg_ms += st.segment_phase_ns / 1e6
        rounds += st.rounds
    tsum_batches = 0
    device_ms_sum = 0.0
    for tm, nb in tsums:
        tsum_batches += nb
        device_ms_sum += tm.device_ms
        merge_slots += tm.merge_slots
        commit_bytes += tm.commit_bytes
        launches += tm.kernel_launches
        for k in stage:
            stage[k] += getattr(tm, k)
        for lv in range(16):
            level_ms[lv] += tm.level_ms[lv]
            level_bytes[lv] += tm.level_bytes[lv]
            level_groups[lv] += tm.level_groups[lv]
            level_big[lv] += tm.level_big[lv]
            level_maxs[lv] = max(level_maxs[lv], tm.level_max_slice[lv])
    assert tsum_batches == K, f"timing sum covers {tsum_batches} batches, expected {K}"
    ms_max, total_updates = reduce_max_sum(ms, updates, world)
    value = total_updates / (ms_max / 1e3)

    # ---- e2e through the host C ABI from pinned buffers (same slides) ----
    # the drop-in call as a C++ caller makes it: page-locked inputs in, the
    # UpdateStats out including touched_ranges (update_stats.hpp:29, fetched
    # by include/pmagraph/update_stats.hpp every batch)
    del g
    hs, hd = stream.arrays()
    host = []
    for s in slides:
        a = torch.from_numpy(hs[s.ins_offset:s.ins_offset + s.n_ins]).pin_memory()
        b = torch.from_numpy(hd[s.ins_offset:s.ins_offset + s.n_ins]).pin_memory()
        c = torch.empty(s.n_del, dtype=torch.int32).pin_memory()
        d = torch.empty(s.n_del, dtype=torch.int32).pin_memory()
        win.deletions_host(s.del_offset, s.n_del, c.numpy().view(np.uint32), d.numpy().view(np.uint32))
        host.append((a.numpy().view(np.uint32), b.numpy().view(np.uint32), c.numpy().view(np.uint32),
                     d.numpy().view(np.uint32), (a, b, c, d)))
    host_by_slide = {id(s): h for s, h in zip(slides, host)}
    e2e_steps = []
    io = {"h2d": 0, "d2h": 0}

    def on_e2e(graph, s, timed):
        a, b, c, d, _ = host_by_slide[id(s)]
        st = graph.apply_batch(a, b, None, c, d, with_touched="array")
        ntr = len(st.touched_ranges)
        st.touched_ranges = None  # the caller consumed them (the page-locked block goes back to the cache)
        if timed:
            e2e_steps.append((st, graph.last_timing()))
            io["h2d"] += a.nbytes + b.nbytes + c.nbytes + d.nbytes
            io["d2h"] += PMA_STATS_BYTES + 16 * ntr  # (begin, end) per touched range

    g2, e2e_ms, _ = run_passes(make_graph(), make_graph, slides, P, W, K, on_e2e, dev, world, None)
    e2e_stage = {"sort_ms": 0.0, "search_ms": 0.0, "rounds_ms": 0.0, "refresh_ms": 0.0}
    e2e_updates = 0
    for st, tm2 in e2e_steps:
        for k in e2e_stage:
            e2e_stage[k] += getattr(tm2, k)
        e2e_updates += st.batch_size
    h2d, d2h = io["h2d"], io["d2h"]
    # the link the inputs cross: a step's bytes of page-locked memory moved by
    # the copy engines and read in place by SM loads (best of 5 each)
    hbuf = torch.empty(h2d // K, dtype=torch.uint8).pin_memory()
    cp_gbps, zc_gbps = C.c_double(), C.c_double()
    lib.gpma_probe_h2d(dev, C.c_void_p(hbuf.data_ptr()), hbuf.numel(), 5, C.byref(cp_gbps), C.byref(zc_gbps))
    del hbuf
    e2e_ms, e2e_updates = reduce_max_sum(e2e_ms, e2e_updates, world)
    e2e = {"value": e2e_updates / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d // K,
           "d2h_bytes_per_step": d2h // K, "ms_per_step": e2e_ms / K,
           "stage_ms_per_step": {k: round(v / K, 4) for k, v in e2e_stage.items()},
           "link_GBps": {"memcpy": round(cp_gbps.value, 1), "zero_copy_read": round(zc_gbps.value, 1)},
           "inputs": "page-locked host arrays, read in place over PCIe by the front-end kernel",
           "outputs": "pma_stats + UpdateStats.touched_ranges (reference order) read back every step",
           "host_cpus": f"{len(near)} GPU-local of {len(all_cpus)}" if near else f"all {len(all_cpus)}"}
    g = g2
    ext = torch.cuda.ExternalStream(lib.gpma_cuda_stream(g.h), device=torch.device("cuda", dev))

    # ---- cross-check of the commit kernel's span with CUDA events ----
    # The timed steps above take the level-0 commit span from %globaltimer
    # stamps the commit kernels write (first CTA start -> last CTA end): event
    # records between a level's kernels would break their programmatic (PDL)
    # edges and slow the step.  A short extra pass with GPMA_LEVEL_EVENTS=1
    # (events on the library's stream around the commit kernels) checks it.
    chk = {"ms": 0.0, "bytes": 0, "steps": 0}

    def on_chk(graph, s, timed):
        graph.apply_batch_device(info.stream_src + 4 * s.ins_offset, info.stream_dst + 4 * s.ins_offset, None,
                                 s.n_ins, info.del_src + 4 * s.del_offset, info.del_dst + 4 * s.del_offset, s.n_del)
        if timed:
            tm = graph.last_timing()
            chk["ms"] += tm.level_ms[0]
            chk["bytes"] += tm.level_bytes[0]
            chk["steps"] += 1

    os.environ["GPMA_LEVEL_EVENTS"] = "1"
    try:
        gchk = make_graph()
    finally:
        os.environ.pop("GPMA_LEVEL_EVENTS", None)
    kchk = max(1, min(K, 5))
    gchk, _, _ = run_passes(gchk, make_graph, slides[:min(P, 1 + kchk)], min(P, 1 + kchk), 1, kchk, on_chk, dev,
                            world, None)
    del gchk

    # ---- roofline of the dominant kernel (warp-tier commit: decide+merge+scatter) ----
    peak, peak_kind = measured_peak()
    # algorithmic bytes of the commit kernels, counted per examined group by the
    # kernels themselves (alg_bytes in csrc/pma.cu): slice + state
    # and key reads of every examined segment, value reads + key/value/state
    # writes of merged segments, state writes of tombstone commits
    # The dominant kernel is the leaf-level commit (k_commit_leaf, with the
    # k_commit_cta launch that takes its hub groups): its level-0 bytes over
    # the level-0 commit span (CUDA events on the library's stream).  The
    # level >= 1 commits (a few hundred groups, latency-bound) are reported
    # beside it in all_levels.
    l0_ms = level_ms[0] / K
    kernel_desc = ("leaf-level commit: k_commit_leaf (decide + merge + even re-dispatch + fused "
                   "header/row-offset refresh) + k_commit_cta for its hub groups")
    if l0_ms == 0 and level_bytes[0] > 0:
        # small batches (C1) run as one captured graph with no per-level
        # events: the level-0 bytes over the graph's whole device span (its
        # %globaltimer stamps) — a lower bound on the commit kernel's rate
        l0_ms = stage["sort_ms"] / K
        kernel_desc = ("small-batch graph (one-CTA front end, warp leaf search, round 0, refresh): level-0 commit "
                       "bytes over the whole graph device span")
    achieved = (level_bytes[0] / K) / (l0_ms / 1e3) / 1e9 if l0_ms > 0 else None
    all_achieved = (commit_bytes / K) / ((seg_ms / K) / 1e3) / 1e9 if seg_ms > 0 else None
    traffic = ncu_traffic(args.config)
    ev_ms = chk["ms"] / chk["steps"] if chk["steps"] else 0.0
    ev_ach = (chk["bytes"] / chk["steps"]) / (ev_ms / 1e3) / 1e9 if ev_ms > 0 else None
    roofline = {"bound": "hbm", "kernel": kernel_desc,
                "timing": "level-0 commit span from %globaltimer stamps written by the commit kernels during the "
                          "timed steps (first CTA start -> last CTA end); events_check = the same span from CUDA "
                          "events on the library's stream in a separate short pass (GPMA_LEVEL_EVENTS=1)",
                "events_check": {"steps": chk["steps"], "kernel_ms_per_step": ev_ms, "achieved": ev_ach,
                                 "frac": (ev_ach / peak) if ev_ach else None},
                "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "algorithmic_bytes_per_step": level_bytes[0] // K, "kernel_ms_per_step": l0_ms,
                "launches_per_step": "one k_commit_leaf launch (+ one k_commit_cta launch when the level has hub groups) per step: ms and bytes are per step = per launch",
                "all_levels": {"algorithmic_bytes_per_step": commit_bytes // K, "ms_per_step": seg_ms / K,
                               "achieved": all_achieved, "frac": (all_achieved / peak) if all_achieved else None},
                "scatter_bytes_per_step": BYTES_PER_MERGE_SLOT * merge_slots // K,
                "commit_ms_per_step_all_levels": seg_ms / K, "step_ms": ms / K,
                "stage_ms_per_step": {k: v / K for k, v in stage.items()},
                "device_ms_mean": round(device_ms_sum / K, 4),
                "timed_segments": segs,
                "commit_ms_per_level": [round(x / K, 4) for x in level_ms if x > 0],
                "groups_per_level": [x / K for x in level_groups if x > 0],
                "hub_groups_per_level": [x / K for x, g in zip(level_big, level_groups) if g > 0],
                "max_hub_slice_per_level": [x for x, g in zip(level_maxs, level_groups) if g > 0]}

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
           "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "u64", "data": f"synthetic: {cfg['gen'].upper()} stream restated from generators.hpp (seed 1+rank"
                                   f"{', shuffle 2' if cfg['shuffle'] else ', generation order'})",
           "config": {"workload": cfg["workload"],
                      "batch": B, "num_vertices": nvx, "stream_edges": len(stream), "pma_capacity": cap,
                      "parallelism": f"dp{world} (independent source-range shards)",
                      "l2": f"inputs larger than L2 (PMA slot array {17 * cap / 1e9:.2f} GB per GPU vs 126 MB L2)",
                      "full_slides_per_pass": P, "passes": passes,
                      "deletion_mode": "lazy", "rounds_per_step": rounds / K},
           "e2e": e2e, "gpu_launches": launches, "roofline": roofline, "clocks": clk,
           "setup_s": {"generate": round(gen_s, 2), "from_edges": round(load_s, 3)}}

    if rank == 0 and not args.profile:
        if not args.no_analytics:
            out["analytics"] = analytics(pg, g, ext, nvx)
        out["sweep"] = sweep(pg, stream, dev, [int(x) for x in args.sweep.split(",") if x], nvx)
        if args.config == "C2":
            c_abi_sweep(out["sweep"], dev)
        if world == 1 and not args.no_cpu_baseline and args.config in ("C1", "C2"):
            os.sched_setaffinity(0, all_cpus)  # the reference baseline gets every host thread
            out["cpu_baseline"] = cpu_baseline(stream, slides, win, W, nvx)
    if world > 1:
        torch.distributed.barrier()
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_sharded(args, rank, world, local):
    """The key-range sharded deployment: one GPMA+ shard per GPU
    over an edge-balanced source range (fixed from the initial window).

    Workload: BASELINE config --config; --scaling weak (default; C2, C3, C1):
    the config's stream scaled by N (RMAT: 2^k N vertices, N x edges; ER: N x
    vertices at density / N), a step = one global slide of N x batch arrivals;
    --scaling strong (default for C4, C5): the config itself, a step = one
    slide of its batch.  Rank r ingests the r-th contiguous share of every
    slide's inserts and deletes; --routing group (default): the library routes
    and applies it with its own NCCL collectives (gpma_shard_group_*, C ABI);
    fused / all_to_all: the Python ShardedGraph over torch.distributed.  Every
    timed step is a full slide (passes with untimed rebuilds, as run_ours);
    value = all ranks' updates / the max-over-ranks time of the K steps."""
    import torch
    import torch.distributed as dist

    from paper_1709_05061_b200 import pmagraph as pg
    from paper_1709_05061_b200 import sharding as sh
    from paper_1709_05061_b200.abi import load_library
    from paper_1709_05061_b200.sharded import NcclComm, ShardedGraph, ShardGroup, TorchComm, nccl_unique_id

    dev = local
    load_library().gpma_warmup(dev)
    cfg = CONFIGS[args.config]
    scaling = args.scaling or ("strong" if args.config in ("C4", "C5") else "weak")
    K, W = args.steps, args.warmup
    base_b = args.batch or cfg["batch"]
    if scaling == "weak":
        nv = cfg["nv"] * world
        param = int(cfg["param"]) * world if cfg["gen"] == "rmat" else cfg["param"] / world
        B = base_b * world
    else:
        nv, param, B = cfg["nv"], cfg["param"], base_b
    t0 = time.time()
    stream = (pg.EdgeStream.rmat(nv, int(param), seed=GEN_SEED) if cfg["gen"] == "rmat"
              else pg.EdgeStream.erdos_renyi(nv, param, seed=GEN_SEED))
    if cfg["shuffle"] is not None:
        stream.shuffle(cfg["shuffle"])
    win = pg.SlidingWindow(stream, dev)
    info = win.info()
    P = full_slides(info, B)
    win.reserve(min(W + K, P) * B + 16)
    info = win.info()
    slides = [win.slide(B) for _ in range(min(W + K, P))]
    for s_ in slides:
        assert s_.n_ins == B and not s_.final_partial, "bench slide is not a full slide"
    info = win.info()
    gen_s = time.time() - t0
    init = info.initial_size
    e_src = _wrap_device(info.stream_src, init, torch.int32, dev)
    e_dst = _wrap_device(info.stream_dst, init, torch.int32, dev)
    deg = torch.bincount(e_src.long(), minlength=nv).cpu().numpy()
    bounds = sh.vertex_bounds(nv, world, deg)
    group = args.routing == "group"
    if group:
        idt = torch.zeros(128, dtype=torch.uint8, device=f"cuda:{dev}")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        ncomm = NcclComm(bytes(idt.cpu().numpy()), world, rank, dev)
    else:
        comm = TorchComm()

    def make_graph():
        if group:
            return ShardGroup(nv, bounds, rank, world, None, (e_src, e_dst, None), device=dev, comm=ncomm)
        return ShardedGraph.from_edges_device(comm, nv, bounds, [(e_src, e_dst, None)], devices=[dev],
                                              routing=args.routing)

    def share(n, r):
        q, m = divmod(n, world)
        lo = r * q + min(r, m)
        return lo, lo + q + (1 if r < m else 0)

    def my_slice(sl):
        a0, a1 = share(sl.n_ins, rank)
        d0, d1 = share(sl.n_del, rank)
        return (_wrap_device(info.stream_src + 4 * (sl.ins_offset + a0), a1 - a0, torch.int32, dev),
                _wrap_device(info.stream_dst + 4 * (sl.ins_offset + a0), a1 - a0, torch.int32, dev), None,
                _wrap_device(info.del_src + 4 * (sl.del_offset + d0), d1 - d0, torch.int32, dev),
                _wrap_device(info.del_dst + 4 * (sl.del_offset + d0), d1 - d0, torch.int32, dev))

    def apply(G, sl_tensors):
        if group:
            st, routed, sent = G.apply_batch(*sl_tensors)
            return st, routed, sent, G
        res = G.apply_batch([sl_tensors])
        return res.stats[0], res.routed[0], res.sent[0], G

    def stream_of(G):
        return G.cuda_stream() if group else G.cuda_stream(0)

    t1 = time.time()
    G = make_graph()
    load_s = time.time() - t1
    acc = {"updates": 0, "routed": 0, "sent": 0, "launches": 0, "seg_ms": 0.0, "commit_bytes": 0.0}

    def on_step(g, sl, timed):
        st, routed, sent, _ = apply(g, my_slice(sl))
        if timed:
            acc["updates"] += st.batch_size
            acc["routed"] += routed
            acc["sent"] += sent
            acc["seg_ms"] += st.segment_phase_ns / 1e6
            acc["launches"] += 4 if group else 6  # (the routing's own launches; the engine's come from the sum)

    def on_segment(g, phase):
        # the engine's timing records summed by the library over the segment
        tm = pg.pma_timing()
        nb = C.c_uint64()
        load_library().gpma_timing_sum(g.graph_handle() if group else g.h[0], C.byref(tm), C.byref(nb), 1)
        if phase == "end":
            acc["launches"] += tm.kernel_launches
            acc["commit_bytes"] += tm.commit_bytes

    clocks = ClockSampler(dev)
    segs = []
    G, ms, passes = run_passes(G, make_graph, slides, P, W, K, on_step, dev, world, clocks, segs, stream_of=stream_of,
                               on_segment=on_segment)
    clk = clocks.stop()
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    u = torch.tensor([float(acc["updates"]), float(acc["sent"])], device="cuda")
    dist.all_reduce(u)
    ms_max, total_updates, total_sent = float(t.item()), float(u[0].item()), float(u[1].item())
    value = total_updates / (ms_max / 1e3)

    # ---- e2e: the same slides from page-locked host buffers (each rank's share copied in the region)
    host = {}
    for sl in slides:
        a, b, _, c, d = my_slice(sl)
        host[id(sl)] = tuple(x.cpu().pin_memory() for x in (a, b, c, d))
    e2e_acc = {"n": 0, "h2d": 0}

    def on_e2e(g, sl, timed):
        a, b, c, d = (x.cuda(non_blocking=True) for x in host[id(sl)])
        st, _, _, _ = apply(g, (a, b, None, c, d))
        if timed:
            e2e_acc["n"] += st.batch_size
            e2e_acc["h2d"] += sum(x.numel() * 4 for x in host[id(sl)])

    del G
    G2, e2e_ms, _ = run_passes(make_graph(), make_graph, slides, P, W, K, on_e2e, dev, world, None,
                               stream_of=stream_of)
    t = torch.tensor([e2e_ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    uu = torch.tensor([float(e2e_acc["n"])], device="cuda")
    dist.all_reduce(uu)
    e2e = {"value": float(uu.item()) / (float(t.item()) / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": e2e_acc["h2d"] // K, "d2h_bytes_per_step": PMA_STATS_BYTES,
           "inputs": "each rank's share of the slide in page-locked host memory, copied in the timed region"}

    peak, peak_kind = measured_peak()
    achieved = (acc["commit_bytes"] / K) / ((acc["seg_ms"] / K) / 1e3) / 1e9 if acc["seg_ms"] > 0 else None
    routing_desc = {"group": "the library's own NCCL all-to-all (gpma_shard_group_apply_batch, C ABI)",
                    "fused": "fused partition+transfer over CUDA IPC peer memory (Python ShardedGraph)",
                    "all_to_all": "NCCL all-to-all via torch.distributed (Python ShardedGraph)"}[args.routing]
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
           "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
           "dtype": "u64",
           "data": f"synthetic: {cfg['gen'].upper()} stream restated from generators.hpp ({nv} vertices, seed 1"
                   f"{', shuffle 2' if cfg['shuffle'] else ''})",
           "config": {"workload": (f"{args.config} x{world} (weak: the stream scaled by {world}, a step = one global "
                                   f"slide of {world} x {base_b})" if scaling == "weak" else
                                   f"{args.config} (strong: one slide of {B} per step over {world} shards)")
                                  + f"; each rank ingests 1/{world} of every slide and routes it to the owners",
                      "batch": B, "batch_per_gpu": B // world, "num_vertices": nv, "stream_edges": len(stream),
                      "parallelism": f"key-range shards x{world}, routing: {routing_desc}",
                      "vertex_bounds": [int(x) for x in bounds], "full_slides_per_pass": P, "passes": passes,
                      "l2": "inputs larger than L2 (each shard's slot array > 126 MB)", "deletion_mode": "lazy"},
           "e2e": e2e, "gpu_launches": acc["launches"],
           "routing": {"updates_sent_to_other_ranks_per_step": total_sent / K,
                       "wire_bytes_per_step": 8 * total_sent / K,
                       "nvlink_roofline": {"bound": "nvlink", "bytes_per_step": 8 * total_sent / K,
                                           "achieved_GBps": (8 * total_sent / K) / (ms_max / K / 1e3) / 1e9,
                                           "peak_GBps": 900.0 * world,
                                           "note": "wire bytes over the whole step time (an upper-bound view: the "
                                                   "exchange is a small part of the step)"}},
           "roofline": {"bound": "hbm", "kernel": "commit tier kernels (rank 0)", "achieved": achieved, "peak": peak,
                        "peak_kind": peak_kind, "unit": "GB/s", "frac": (achieved / peak) if achieved else None,
                        "traffic": None, "algorithmic_bytes_per_step": acc["commit_bytes"] / K,
                        "kernel_ms_per_step": acc["seg_ms"] / K, "timed_segments": segs},
           "clocks": clk, "setup_s": {"generate": round(gen_s, 2), "from_edges": round(load_s, 3)}}
    if not args.no_analytics and not args.profile:
        out["analytics"] = sharded_analytics(G2, nv, rank, group)
    if rank == 0:
        print(json.dumps(out), flush=True)
    del G2
    if group:
        ncomm.close()
    dist.barrier()
    dist.destroy_process_group()


def _wrap_device(ptr, n, dtype, dev):
    """Zero-copy torch view of n elements of library-owned device memory."""
    import torch
    if n == 0:
        return torch.empty(0, dtype=dtype, device=f"cuda:{dev}")
    itemsize = torch.empty(0, dtype=dtype).element_size()

    class _CAI:
        __cuda_array_interface__ = {"shape": (n,), "typestr": {torch.int32: "<i4", torch.float64: "<f8",
                                                              torch.int64: "<i8"}[dtype],
                                    "data": (int(ptr), False), "version": 2, "strides": None}
    del itemsize
    return torch.as_tensor(_CAI(), device=f"cuda:{dev}")


def sharded_analytics(G, nv, rank, group=False):
    """Per-window analytics on the sharded graph (all ranks take part)."""
    import torch
    import torch.distributed as dist
    rng = np.random.default_rng(ROOT_SEED)
    out = {}
    roots = [int(x) for x in rng.integers(0, nv, 3)]
    if group:  # steady state of a window loop: one untimed call of each (buffers, NCCL paths)
        G.bfs(roots[0])
        G.connected_components()
        G.pagerank(max_iters=2)
    ms = []
    for r in roots:
        dist.barrier()
        t = time.perf_counter()
        if group:
            _, n = G.bfs(r)
        else:
            d = G.bfs(r)[0]
            n = int((d != -1).sum().item())
        torch.cuda.synchronize()
        ms.append(((time.perf_counter() - t) * 1e3, n))
    out["bfs_ms"] = [x[0] for x in ms]
    out["bfs_reached"] = [x[1] for x in ms]
    dist.barrier()
    t = time.perf_counter()
    G.connected_components()
    torch.cuda.synchronize()
    out["cc_ms"] = (time.perf_counter() - t) * 1e3
    if not group:
        out["cc_rounds"] = G.cc_rounds
    dist.barrier()
    t = time.perf_counter()
    _, it, _ = G.pagerank()
    torch.cuda.synchronize()
    out["pagerank_ms_cold"] = (time.perf_counter() - t) * 1e3
    out["pagerank_iters_cold"] = it
    return out


def analytics(pg, g, ext, nv):
    """Per-window analytic time on the live gapped graph (bench.hpp:226-313),
    plus the PageRank iteration against the HBM roofline (SURVEY §8d:
    9 C + 8 E + 36 |V| bytes per iteration)."""
    import torch
    roots = pg.draw_below_sequence(ROOT_SEED, nv, 5)
    # steady state of a window loop: one untimed call of each analytic first
    # (pinned result buffers of the caching host allocator, lazy module loads)
    # (two results alive at once, as in the timed loops below: the caching
    # host allocator then holds both page-locked blocks before timing starts)
    # (the timed PageRank block below holds three rank vectors at once: three
    # page-locked blocks in the cache, as a window loop reuses its buffers)
    _w = pg.pagerank(g, max_iters=2)
    _w2 = pg.pagerank(g, warm_start=_w.ranks, max_iters=2)
    _w3 = pg.pagerank(g, warm_start=_w.ranks, max_iters=2)
    _b1, _b2 = pg.bfs(g, 0), pg.bfs(g, 0)
    _c1, _c2 = pg.connected_components(g), pg.connected_components(g)
    del _w, _w2, _w3, _b1, _b2, _c1, _c2
    bfs_ms, reached = [], []
    for r in roots:
        torch.cuda.synchronize()
        t = time.perf_counter()
        _, n = pg.bfs(g, int(r), return_reached=True)
        bfs_ms.append((time.perf_counter() - t) * 1e3)
        reached.append(int(n))
    # roots among non-isolated vertices (SURVEY §8d BFS-root caveat)
    ro = g.row_offsets()
    deg = np.diff(ro.astype(np.int64))
    nz = np.nonzero(deg > 1)[0]
    rng = np.random.default_rng(ROOT_SEED)
    hub_ms = []
    for r in rng.choice(nz, 3):
        t = time.perf_counter()
        _, n = pg.bfs(g, int(r), return_reached=True)
        hub_ms.append(((time.perf_counter() - t) * 1e3, int(n)))
    t = time.perf_counter()
    pg.connected_components(g)
    cc_ms = (time.perf_counter() - t) * 1e3
    t = time.perf_counter()
    pr = pg.pagerank(g)
    pr_ms = (time.perf_counter() - t) * 1e3
    t = time.perf_counter()
    pr2 = pg.pagerank(g, warm_start=pr.ranks)
    pr2_ms = (time.perf_counter() - t) * 1e3
    t = time.perf_counter()
    pr3 = pg.pagerank(g, warm_start=pr.ranks, epsilon=0.0, max_iters=10)  # 10 fixed iterations: the roofline
    pr3_ms = (time.perf_counter() - t) * 1e3
    pr3_dev_ms = g.last_timing().device_ms
    it_ms = g.last_timing().rounds_ms / max(pr3.iterations, 1)
    cap = g.pma().capacity()
    ne = g.num_edges()
    it_bytes = 9 * cap + 8 * ne + 36 * nv
    peak, peak_kind = measured_peak()
    return {"bfs_ms_reference_roots": bfs_ms, "bfs_reached": reached,
            "bfs_ms_nonisolated_roots": [x[0] for x in hub_ms], "bfs_reached_nonisolated": [x[1] for x in hub_ms],
            "cc_ms": cc_ms, "pagerank_ms_cold": pr_ms, "pagerank_iters_cold": pr.iterations,
            "pagerank_ms_warm": pr2_ms, "pagerank_iters_warm": pr2.iterations,
            "pagerank_10_iters_ms": pr3_ms, "pagerank_10_iters_device_ms": pr3_dev_ms,
            "pagerank_wall_over_device": pr3_ms / pr3_dev_ms if pr3_dev_ms > 0 else None,
            "pagerank_iter_ms": it_ms,
            "pagerank_iter_roofline": {"bound": "hbm", "algorithmic_bytes": it_bytes,
                                       "achieved": it_bytes / (it_ms / 1e3) / 1e9 if it_ms > 0 else None,
                                       "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                                       "frac": it_bytes / (it_ms / 1e3) / 1e9 / peak if it_ms > 0 else None}}


def sweep(pg, stream, dev, batches, nv):
    """updates/s vs batch size (device-resident inputs, 2 warmup + 3 timed slides),
    GPMA+ and the rebuild-the-CSR-per-batch baseline on the same slides."""
    import torch
    res = {}
    for B in batches:
        win = pg.SlidingWindow(stream, dev)
        win.reserve(6 * B + 16)
        info = win.info()
        g = pg.DynamicGraph.from_edges_device(nv, info.stream_src, info.stream_dst, None, info.initial_size,
                                              device=dev)
        slides = [win.slide(B) for _ in range(5)]
        info = win.info()
        ext = torch.cuda.ExternalStream(g._lib.gpma_cuda_stream(g.h), device=torch.device("cuda", dev))

        def go(s):
            return g.apply_batch_device(info.stream_src + 4 * s.ins_offset, info.stream_dst + 4 * s.ins_offset,
                                        None, s.n_ins, info.del_src + 4 * s.del_offset,
                                        info.del_dst + 4 * s.del_offset, s.n_del)
        for s in slides[:2]:
            go(s)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        n = 0
        for s in slides[2:]:
            n += go(s).batch_size
        e1.record(ext)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        res[str(B)] = {"updates_per_s": n / (ms / 1e3), "us_per_batch": ms * 1e3 / 3}
        del g
        # the paper's comparison point on the same slides: the CSR rebuilt per
        # batch (RebuildCsrGraph, baselines.hpp:85-181) on the device
        r = pg.RebuildCsrGraph.from_edges_device(nv, info.stream_src, info.stream_dst, None, info.initial_size,
                                                 device=dev)
        rext = torch.cuda.ExternalStream(r._lib.gpma_rebuild_cuda_stream(r.h), device=torch.device("cuda", dev))

        def rgo(s):
            return r.apply_batch_device(info.stream_src + 4 * s.ins_offset, info.stream_dst + 4 * s.ins_offset,
                                        None, s.n_ins, info.del_src + 4 * s.del_offset,
                                        info.del_dst + 4 * s.del_offset, s.n_del)
        for s in slides[:2]:
            rgo(s)
        torch.cuda.synchronize()
        e0.record(rext)
        n = 0
        for s in slides[2:]:
            n += rgo(s).batch_size
        e1.record(rext)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        res[str(B)]["rebuild_csr_updates_per_s"] = n / (ms / 1e3)
        res[str(B)]["rebuild_csr_us_per_batch"] = ms * 1e3 / 3
        del r, win
    return res


def c_abi_sweep(res, dev):
    """The same C2 slides through the drop-in C ABI with no Python in the
    loop (tools/cpp/small_batch_latency: gpma_apply_batch_device on device
    inputs, host steady_clock around each synchronous call, median of 200
    slides after 8 untimed): the small-batch latency a C++ caller sees.  The
    Python `us_per_batch` beside it adds ctypes and the UpdateStats object."""
    import subprocess
    tool = os.path.join(ROOT, "tools", "cpp", "small_batch_latency")
    sizes = [b for b in map(int, res) if b <= 10000]
    if not sizes or not os.path.exists(tool):
        return
    env = dict(os.environ, CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", str(dev)))
    try:
        out = subprocess.run([tool, *map(str, sizes)], capture_output=True, text=True, timeout=600, env=env).stdout
    except (OSError, subprocess.TimeoutExpired):
        return
    for line in out.splitlines():
        # B=100: C ABI wall per batch median 38.2 us, p10 37.7, p90 38.9 (device 27.6 us, 196 updates)
        if not line.startswith("B=") or "median" not in line:
            continue
        b = line[2:line.index(":")]
        try:
            med = float(line.split("median ")[1].split(" us")[0])
            p10 = float(line.split("p10 ")[1].split(",")[0])
            p90 = float(line.split("p90 ")[1].split(" ")[0])
            devus = float(line.split("(device ")[1].split(" us")[0])
        except (IndexError, ValueError):
            continue
        if b in res:
            res[b]["c_abi_us_per_batch"] = {"median": med, "p10": p10, "p90": p90, "device_us": devus}


def cpu_baseline(stream, slides, win, W, nv):
    """The reference (oracle/_ref) on the host cores, bounded sample: its
    DynamicGraph over the same initial window, then 2 of the same slides
    through apply_batch with all hardware threads (steady_clock around the
    call)."""
    from oracle import oracle
    if not oracle.have_ref():
        return None
    s, d = stream.arrays()
    half = (len(s) + 1) // 2
    t = time.time()
    ref = oracle.RefGraph(nv, s[:half], d[:half])
    build_s = time.time() - t
    cores = oracle.hardware_concurrency()
    ms_total, n_total = 0.0, 0
    sample = slides[:2]
    for sl in sample:
        a, b = s[sl.ins_offset:sl.ins_offset + sl.n_ins], d[sl.ins_offset:sl.ins_offset + sl.n_ins]
        c, dd = win.deletions_host(sl.del_offset, sl.n_del)
        st, ms = ref.apply_batch_timed(a, b, None, c, dd, cores)
        ms_total += ms
        n_total += st.batch_size
    # the next slide with one worker (workers = hardware threads and 1)
    sl = slides[2]
    a, b = s[sl.ins_offset:sl.ins_offset + sl.n_ins], d[sl.ins_offset:sl.ins_offset + sl.n_ins]
    c, dd = win.deletions_host(sl.del_offset, sl.n_del)
    st1, ms1 = ref.apply_batch_timed(a, b, None, c, dd, 1)
    return {"value": n_total / (ms_total / 1e3), "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"2 full slides of batch {slides[0].n_ins} on the same window via reference apply_batch "
                      f"({cores} workers); reference from_edges setup {build_s:.1f}s excluded",
            "one_worker": {"value": st1.batch_size / (ms1 / 1e3), "unit": UNIT, "cores": 1,
                           "sample": "the third slide through apply_batch with workers = 1"}}


# ------------------------------------------------------------- reference --

def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle
    if not oracle.have_ref():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libpmagraph_ref.so not built"}))
        return
    cfg = CONFIGS[args.config]
    B = args.batch or cfg["batch"]
    K, W = args.steps, args.warmup
    cores = oracle.hardware_concurrency()
    nvx = cfg["nv"]
    st = (oracle.RefStream.rmat(nvx, int(cfg["param"]), seed=GEN_SEED) if cfg["gen"] == "rmat"
          else oracle.RefStream.erdos_renyi(nvx, cfg["param"], seed=GEN_SEED))
    if cfg["shuffle"] is not None:
        st.shuffle(cfg["shuffle"])
    s, d, w, _ = st.arrays()
    half = (len(s) + 1) // 2
    # the same full-slide passes as our arm (run_passes): P full slides per
    # pass, the reference graph rebuilt from the initial window between passes
    P = (len(s) - half) // B
    if P < 1:
        raise SystemExit(f"bench: the stream holds no full slide of batch {B}")
    win = oracle.RefWindow(st)
    slides = [win.slide(B) for _ in range(min(W + K, P))]
    assert all(len(x[0]) == B for x in slides), "reference slide is not a full slide"
    total_ms, total_n = 0.0, 0
    ref, cur = None, len(slides)
    for i in range(W + K):
        if cur == len(slides):
            ref = None
            ref = oracle.RefGraph(nvx, s[:half], d[:half], w[:half])
            cur = 0
        a, b, ww, c, dd = slides[cur]
        cur += 1
        stt, ms = ref.apply_batch_timed(a, b, ww, c, dd, cores)
        if i >= W:
            total_ms += ms
            total_n += stt.batch_size
    value = total_n / (total_ms / 1e3)
    if world > 1:  # our arm: C2 per GPU over `world` key-range shards (run_sharded)
        workload = (f"C2 per GPU, key-range sharded over {world} GPUs (the reference runs one C2-sized share of "
                    f"it on the host cores: a bounded sample of the {world} x C2 workload)")
        sample = (f"{K} slides of batch {B} (after {W} warmup) of one C2-sized share through the reference "
                  f"DynamicGraph::apply_batch with {cores} workers")
    else:
        workload = cfg["workload"]
        sample = (f"{K} slides of batch {B} (after {W} warmup) through the reference DynamicGraph::apply_batch "
                  f"with {cores} workers")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
           "warmup": W, "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "u64",
           "data": f"synthetic: reference generators ({cfg['gen']}, seed 1{', shuffle 2' if cfg['shuffle'] else ''})",
           "config": {"workload": workload, "batch": B, "num_vertices": nvx, "stream_edges": len(s)},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
