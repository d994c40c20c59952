"""Source-vertex-range sharding of the GPMA+ store across GPUs.

Keys are ``src << 32 | dst``, so a contiguous source-vertex range is a
contiguous key range: segments never cross shards and the rounds, density
decisions and rebalances are entirely shard-local.  The only exchange in the
update path is routing each batch's updates to the shard that owns their
source vertex:

  1. every rank holds a contiguous slice of the global batch (arrival order);
  2. ``bucket_updates`` splits its slice by owner, stably;
  3. ``exchange`` is one variable-size all-to-all (counts first), over NCCL on
     GPUs or gloo on CPU; received chunks are concatenated in sender-rank
     order, which preserves the global arrival order of every key, so
     "last insert wins" (segment_engine.hpp:346-363) resolves exactly as in
     the single-GPU engine;
  4. each owner applies its slice to its local shard (one GPMA+ per GPU).

A shard of the reference's DynamicGraph over [lo, hi) holds the edges whose
source lies in the range plus the guards of its vertices; per shard the slot
array is bit-exact against a reference PackedMemoryArray built with
``from_sorted(shard entries + shard guards, 0.5)`` and driven with
``batch_update(shard slice)`` (both public reference API).
"""
from __future__ import annotations

import numpy as np

GUARD_DST = 0xFFFFFFFF


def vertex_bounds(num_vertices: int, world: int, out_degree=None) -> np.ndarray:
    """Boundaries b[0]=0 < ... < b[world]=num_vertices of the per-rank source
    ranges.  With ``out_degree`` the ranges balance edges + guards (fixed for
    the run so parity is reproducible); otherwise equal vertex ranges, as in
    the paper."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if out_degree is None:
        return np.array([(num_vertices * r) // world for r in range(world + 1)], np.int64)
    w = np.asarray(out_degree, np.int64) + 1  # + the guard slot
    c = np.concatenate([[0], np.cumsum(w)])
    targets = (c[-1] * np.arange(1, world)) // world
    inner = np.searchsorted(c, targets, side="left")
    b = np.concatenate([[0], inner, [num_vertices]]).astype(np.int64)
    return np.maximum.accumulate(b)


def owner_of(src, bounds: np.ndarray) -> np.ndarray:
    """Rank owning each source vertex."""
    return np.searchsorted(bounds, np.asarray(src, np.int64), side="right") - 1


def bucket_updates(src, dst, weight, op, bounds: np.ndarray):
    """Split one rank's update slice by owner, preserving arrival order.
    Returns (order, counts): ``order`` permutes the slice so owner r's updates
    are contiguous (stable), ``counts[r]`` their number."""
    own = owner_of(src, bounds)
    world = len(bounds) - 1
    order = np.argsort(own, kind="stable")
    counts = np.bincount(own, minlength=world).astype(np.int64)
    return order, counts


def pack_updates(src, dst, weight, op) -> np.ndarray:
    """Updates as one int64 matrix [n, 4] (src, dst, weight bits, op) so a
    single all-to-all moves them (17 B/update of payload on the wire)."""
    n = len(src)
    m = np.empty((n, 4), np.int64)
    m[:, 0] = np.asarray(src, np.int64)
    m[:, 1] = np.asarray(dst, np.int64)
    m[:, 2] = np.asarray(weight if weight is not None else np.ones(n), np.float64).view(np.int64)
    m[:, 3] = np.asarray(op, np.int64)
    return m


def unpack_updates(m: np.ndarray):
    return (m[:, 0].astype(np.uint32), m[:, 1].astype(np.uint32), m[:, 2].copy().view(np.float64),
            m[:, 3].astype(np.uint8))


def exchange(packed: np.ndarray, counts: np.ndarray, group=None, device=None) -> np.ndarray:
    """Variable-size all-to-all of packed update rows (counts exchanged
    first).  Chunks arrive concatenated in sender-rank order."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = device if device is not None else torch.device("cpu")
    send_counts = torch.as_tensor(np.asarray(counts, np.int64), device=dev)
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts, group=group)
    rc = recv_counts.cpu().numpy()
    src_t = torch.as_tensor(np.ascontiguousarray(packed).reshape(-1), device=dev)
    out = torch.empty(int(rc.sum()) * 4, dtype=torch.int64, device=dev)
    dist.all_to_all_single(out, src_t, output_split_sizes=[int(x) * 4 for x in rc],
                           input_split_sizes=[int(x) * 4 for x in counts], group=group)
    assert len(rc) == world
    return out.cpu().numpy().reshape(-1, 4)


def route_batch(ins_src, ins_dst, ins_w, del_src, del_dst, bounds, group=None, device=None):
    """Route this rank's slice of a DynamicGraph::apply_batch (inserts then
    deletes, graph.hpp:133-147) to the owners.  Guard deletes stay with their
    owner too (the owner counts them as missed).  Returns the owner-local
    (inserts, deletes) in global arrival order."""
    n_ins = len(ins_src)
    src = np.concatenate([np.asarray(ins_src, np.int64), np.asarray(del_src, np.int64)])
    dst = np.concatenate([np.asarray(ins_dst, np.int64), np.asarray(del_dst, np.int64)])
    w = np.concatenate([np.asarray(ins_w if ins_w is not None else np.ones(n_ins), np.float64),
                        np.zeros(len(del_src))])
    op = np.concatenate([np.zeros(n_ins, np.int64), np.ones(len(del_src), np.int64)])
    order, counts = bucket_updates(src, dst, w, op, bounds)
    packed = pack_updates(src[order], dst[order], w[order], op[order])
    got = exchange(packed, counts, group, device)
    s, d, ww, o = unpack_updates(got)
    ins = o == 0
    return (s[ins], d[ins], ww[ins]), (s[~ins], d[~ins])


def shard_entries(num_vertices, src, dst, weight, lo, hi):
    """Sorted (keys, values) of the shard [lo, hi): its edges (duplicates
    collapse to the last weight, graph.hpp:78-84) plus one guard per owned
    vertex (graph.hpp:85-88)."""
    src = np.asarray(src, np.uint64)
    dst = np.asarray(dst, np.uint64)
    w = np.asarray(weight if weight is not None else np.ones(len(src)), np.float64)
    m = (src >= lo) & (src < hi)
    keys = (src[m] << np.uint64(32)) | dst[m]
    vals = w[m].view(np.uint64)
    order = np.argsort(keys, kind="stable")
    keys, vals = keys[order], vals[order]
    last = np.ones(len(keys), bool)
    if len(keys) > 1:
        last[:-1] = keys[1:] != keys[:-1]
    keys, vals = keys[last], vals[last]
    guards = (np.arange(lo, hi, dtype=np.uint64) << np.uint64(32)) | np.uint64(GUARD_DST)
    allk = np.concatenate([keys, guards])
    allv = np.concatenate([vals, np.zeros(len(guards), np.uint64)])
    o = np.argsort(allk, kind="stable")
    return allk[o], allv[o]


def shard_updates(ins_src, ins_dst, ins_w, del_src, del_dst):
    """A routed (owner-local) batch as PMA updates: keys, values, ops with
    guard deletes dropped and counted (graph.hpp:141-147)."""
    ins_src = np.asarray(ins_src, np.uint64)
    ins_dst = np.asarray(ins_dst, np.uint64)
    del_src = np.asarray(del_src, np.uint64)
    del_dst = np.asarray(del_dst, np.uint64)
    keep = del_dst != GUARD_DST
    keys = np.concatenate([(ins_src << np.uint64(32)) | ins_dst, (del_src[keep] << np.uint64(32)) | del_dst[keep]])
    vals = np.concatenate([np.asarray(ins_w if ins_w is not None else np.ones(len(ins_src)), np.float64).view(np.uint64),
                           np.zeros(int(keep.sum()), np.uint64)])
    ops = np.concatenate([np.zeros(len(ins_src), np.uint8), np.ones(int(keep.sum()), np.uint8)])
    return keys, vals, ops, int((~keep).sum())
