"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run in the build container (needs /root/reference to build the oracle):
    python tests/golden/make_golden.py
The fixtures are small (a few hundred KB) and committed; the GPU box and the
CPU tests read them without /root/reference.

Fixtures
  window_er.npz   : ER(4096, 2^-6) stream (seed 1, shuffle 2), lazy mode;
                    initial window + 4 slides of 700: per-slide batches, stats,
                    sha256 of the slot arrays, row offsets, BFS/CC, PageRank.
  window_rmat.npz : RMAT(2^12, 40000) unshuffled (skewed, hot keys), eager
                    mode, 4 slides of 1500 — escalation + eager rebalancing.
  pma_trace.npz   : generic PMA (64-bit keys) random batches in both modes.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from paper_1709_05061_b200.abi import PMA_EAGER, PMA_LAZY, engine_config, graph_config  # noqa: E402


def slot_hash(k, v, s) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(k, np.uint64).tobytes())
    h.update(np.ascontiguousarray(v, np.uint64).tobytes())
    h.update(np.ascontiguousarray(s, np.uint8).tobytes())
    return h.hexdigest()


def window_fixture(name, stream, nv, batch, slides, mode, roots_seed=7):
    s, d, w, _ = stream.arrays()
    half = (len(s) + 1) // 2
    g = oracle.RefGraph(nv, s[:half], d[:half], w[:half], graph_config(deletion_mode=mode))
    win = oracle.RefWindow(stream)
    out = {"nv": nv, "stream_src": s.astype(np.uint16), "stream_dst": d.astype(np.uint16), "batch": batch, "mode": mode,
           "init_hash": slot_hash(*g.slots())}
    roots = oracle.draw_below_sequence(roots_seed, nv, slides)
    warm = None
    for i in range(slides):
        a, b, ww, c, dd = win.slide(batch)
        st = oracle.stats_dict(g.apply_batch(a, b, ww, c, dd))
        out[f"s{i}_del_src"], out[f"s{i}_del_dst"] = c.astype(np.uint16), dd.astype(np.uint16)
        out[f"s{i}_n_ins"] = len(a)
        out[f"s{i}_stats"] = np.array([st["batch_size"], st["rounds"], st["slot_writes"], st["grow_events"],
                                       st["shrink_events"], st["deletes_missed"], st["tombstones_added"],
                                       st["num_touched_ranges"], int(st["resized"])], np.uint64)
        out[f"s{i}_spl"] = np.array(st["segments_per_level"], np.uint64)
        out[f"s{i}_touched"] = np.array(g.touched_ranges(), np.uint64).reshape(-1, 2)
        out[f"s{i}_hash"] = slot_hash(*g.slots())
        out[f"s{i}_row_offsets"] = g.row_offsets()
        out[f"s{i}_bfs"] = g.bfs(int(roots[i]))
        out[f"s{i}_root"] = int(roots[i])
        out[f"s{i}_cc"] = g.cc()
        ranks, iters, conv = g.pagerank(warm=warm)
        out[f"s{i}_pr"], out[f"s{i}_pr_iters"] = ranks, iters
        warm = ranks
        x = np.linspace(0.0, 1.0, nv)
        out[f"s{i}_spmv"] = g.spmv(x)
    np.savez_compressed(os.path.join(HERE, name), **out)
    print(name, {k: v for k, v in out.items() if k.endswith("_stats")})


def pma_trace_fixture(name):
    rng = np.random.default_rng(20261017)
    keys = np.unique(rng.integers(0, 2**40, 3000, dtype=np.uint64))
    vals = rng.integers(0, 2**63, len(keys), dtype=np.uint64)
    out = {"init_keys": keys, "init_vals": vals}
    p = oracle.RefPMA().from_sorted(keys, vals, 0.5)
    out["init_hash"] = slot_hash(*p.slots())
    for i in range(8):
        mode = PMA_EAGER if i % 2 else PMA_LAZY
        n = int(rng.integers(1, 2500))
        k = rng.integers(0, 2**40, n, dtype=np.uint64)
        hit = rng.random(n) < 0.4
        k[hit] = rng.choice(keys, int(hit.sum()))
        o = (rng.random(n) < 0.45).astype(np.uint8)
        v = rng.integers(0, 2**63, n, dtype=np.uint64)
        st = oracle.stats_dict(p.batch_update(k, v, o, engine_config(deletion_mode=mode)))
        out[f"b{i}_keys"], out[f"b{i}_vals"], out[f"b{i}_ops"], out[f"b{i}_mode"] = k, v, o, mode
        out[f"b{i}_stats"] = np.array([st["batch_size"], st["rounds"], st["slot_writes"], st["grow_events"],
                                       st["shrink_events"], st["deletes_missed"], st["tombstones_added"],
                                       st["num_touched_ranges"], int(st["resized"])], np.uint64)
        out[f"b{i}_spl"] = np.array(st["segments_per_level"], np.uint64)
        out[f"b{i}_hash"] = slot_hash(*p.slots())
        probe = rng.integers(0, 2**40, 256, dtype=np.uint64)
        out[f"b{i}_probe"], out[f"b{i}_leaves"] = probe, p.binary_search_leaf(probe)
    np.savez_compressed(os.path.join(HERE, name), **out)
    print(name, "ok")


def main():
    oracle.build()
    window_fixture("window_er.npz", oracle.RefStream.erdos_renyi(4096, 2.0 ** -6, 1).shuffle(2), 4096, 700, 4,
                   PMA_LAZY)
    window_fixture("window_rmat.npz", oracle.RefStream.rmat(2**12, 40000, 1), 2**12, 1500, 4, PMA_EAGER)
    pma_trace_fixture("pma_trace.npz")


if __name__ == "__main__":
    main()
