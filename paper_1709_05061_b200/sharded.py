"""Key-range sharded GPMA+ across GPUs — the device data path.

One GPMA+ per GPU holds the edges whose source lies in its range [lo, hi)
(keys are ``src << 32 | dst``, so a source range is a key range: segments never
cross shards, every round / density decision / rebalance is shard-local) plus
the guards of its vertices.  What crosses GPUs:

* update routing, once per batch: every rank holds a contiguous share of the
  global batch (its arrivals); ``gpma_route_partition`` stably partitions it by
  owner on the device into EdgeKey words, then one variable-size all-to-all
  (counts first) per op type moves them to the owners.  Chunks arrive in
  sender-rank order, so every key keeps its global arrival order and "last
  insert wins" (segment_engine.hpp:346-363) resolves as on one GPU;
* BFS: per level the owners mark the out-neighbours of their frontier in a
  |V|-byte flag array, one MAX all-reduce, owners admit their unreached
  flagged vertices (owner-computes, analytics.hpp:22-48);
* CC: min-label propagation over replicated labels, one MIN all-reduce per
  round + pointer jumping (analytics.hpp:53-82; fixpoint = component minima);
* PageRank: owners push over their edges, one SUM all-reduce of y per
  iteration, replicated finish (analytics.hpp:84-143);
* SpMV: owners compute their rows, one all-gather (analytics.hpp:147-158).

Collectives go through a ``Comm`` over a LIST of local shards:
``TorchComm`` = one shard per process, torch.distributed (NCCL on GPUs);
``LocalComm`` = every shard in this process (tests on one GPU: the same code
path, collectives as loops).  Every library call is synchronous on its own
stream; tensors produced by torch ops are synchronised before the library
reads them.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from .abi import load_library, pma_stats
from .pmagraph import GraphConfig, PackedMemoryArray, UpdateStats, _host_out, _raise

UNREACHED = 0xFFFFFFFF


def _torch():
    import torch
    return torch


def _vp(t):
    return C.c_void_p(t.data_ptr()) if t is not None and t.numel() else None


def _sync(t):
    torch = _torch()
    if t.is_cuda:
        torch.cuda.current_stream(t.device).synchronize()


# ------------------------------------------------------------------ comms

class LocalComm:
    """All shards in this process; collectives are reductions over the list."""

    stream_ordered = False

    def __init__(self, world: int):
        self.world = world
        self.ranks = list(range(world))

    def all_reduce(self, ts, op: str):
        torch = _torch()
        acc = ts[0].clone()
        for t in ts[1:]:
            t = t.to(acc.device)  # (shards on different devices reduce on the first one's)
            if op == "sum":
                acc += t
            elif op == "max":
                acc = torch.maximum(acc, t)
            elif op == "min":
                acc = torch.minimum(acc, t)
            else:
                raise ValueError(op)
        for t in ts:
            t.copy_(acc)  # (copy_ crosses devices)

    def all_to_all_v(self, sends, send_counts):
        """sends[i]: local rank i's buffer, owner-major; send_counts[i][r]:
        elements for rank r (list or device tensor).  Returns per local rank
        the received buffer (sender-rank order), its per-sender counts, and
        the send counts as lists."""
        torch = _torch()
        send_counts = [c.cpu().tolist() if isinstance(c, torch.Tensor) else list(c) for c in send_counts]
        offs = [np.concatenate([[0], np.cumsum(c)]) for c in send_counts]
        recvs, rcounts = [], []
        for r in range(self.world):
            parts = [sends[s][int(offs[s][r]):int(offs[s][r + 1])] for s in range(self.world)]
            recvs.append(torch.cat(parts) if parts else sends[r][:0])
            rcounts.append([int(send_counts[s][r]) for s in range(self.world)])
        return recvs, rcounts, send_counts

    def all_gather_v(self, pieces):
        torch = _torch()
        full = torch.cat(pieces)
        return [full.clone() for _ in pieces]


class TorchComm:
    """One shard per process over torch.distributed (NCCL between GPUs).
    stream_ordered: the library runs on torch's current stream, so device
    steps and collectives need no host synchronisation between them."""

    stream_ordered = True

    _OPS = {"sum": "SUM", "max": "MAX", "min": "MIN"}

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.ranks = [dist.get_rank(group)]

    def all_reduce(self, ts, op: str):
        (t,) = ts
        self.dist.all_reduce(t, op=getattr(self.dist.ReduceOp, self._OPS[op]), group=self.group)

    def all_to_all_v(self, sends, send_counts):
        """send_counts: per-rank counts as a list or as a device int64 tensor
        (then the count exchange stays on the stream and one D2H brings both
        the send and the receive counts)."""
        torch = _torch()
        (buf,), (cnt,) = sends, send_counts
        sc = cnt if isinstance(cnt, torch.Tensor) else torch.as_tensor(np.asarray(cnt, np.int64), device=buf.device)
        rc = torch.empty_like(sc)
        self.dist.all_to_all_single(rc, sc, group=self.group)
        both = torch.cat([sc, rc]).cpu().tolist()
        scl, rcl = both[:self.world], both[self.world:]
        out = torch.empty(sum(rcl), dtype=buf.dtype, device=buf.device)
        self.dist.all_to_all_single(out, buf[:sum(scl)], output_split_sizes=rcl, input_split_sizes=scl,
                                    group=self.group)
        return [out], [rcl], [scl]

    def all_gather_v(self, pieces):
        torch = _torch()
        (p,) = pieces
        n = torch.tensor([p.numel()], device=p.device)
        ns = [torch.empty_like(n) for _ in range(self.world)]
        self.dist.all_gather(ns, n, group=self.group)
        m = int(max(int(x) for x in ns))
        pad = torch.zeros(m, dtype=p.dtype, device=p.device)
        pad[:p.numel()] = p
        outs = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(outs, pad, group=self.group)
        return [torch.cat([o[:int(k)] for o, k in zip(outs, ns)])]


def fused_offsets(M):
    """Fused routing's placement from the count matrix M[sender][owner]:
    sender s writes its owner-r updates at [before[s][r], before[s][r] +
    M[s][r]) of r's receive buffer — the senders' segments tile [0, nrecv[r])
    in sender-rank order, exactly where an all-to-all would put them."""
    M = np.asarray(M, np.int64)
    return np.cumsum(M, axis=0) - M, M.sum(axis=0)


# ------------------------------------------------------------------ graph

@dataclass
class ShardStats:
    stats: list          # UpdateStats of every local shard
    routed: list         # updates each local shard received
    sent: list           # updates each local shard sent to other ranks


class ShardedGraph:
    """Key-range sharded DynamicGraph; `shards[i]` is local rank comm.ranks[i]."""

    def __init__(self, comm, num_vertices: int, bounds, handles, devices, routing: str = "all_to_all"):
        if routing not in ("all_to_all", "fused"):
            raise ValueError("routing: 'all_to_all' or 'fused'")
        self.routing = routing
        self._rx = None  # fused routing: receive buffers (see _ensure_rx)
        self.comm = comm
        self.nv = int(num_vertices)
        self.bounds = np.asarray(bounds, np.int64)
        self.h = handles
        self.devices = devices
        if isinstance(comm, LocalComm) and len(set(devices)) > 1:
            # its collectives combine the shards' tensors directly and the fused
            # scatter stores into the others' buffers: one device only
            raise ValueError("LocalComm shards must share one device (use TorchComm across GPUs)")
        self._lib = load_library()
        torch = _torch()
        self._dbounds = [torch.as_tensor(self.bounds.astype(np.uint32).view(np.int32), device=f"cuda:{d}")
                         for d in devices]
        self._ordered = getattr(comm, "stream_ordered", False)
        if self._ordered:  # library calls on torch's stream: ordered with the NCCL collectives
            for h, d in zip(self.h, devices):
                self._lib.gpma_set_stream(h, C.c_void_p(torch.cuda.current_stream(d).cuda_stream), 0)

    # ---- construction
    @classmethod
    def from_edges_device(cls, comm, num_vertices: int, bounds, edges, config: GraphConfig | None = None,
                          devices=None, routing: str = "all_to_all"):
        """edges[i] = (src, dst, weights|None) device tensors given to local
        rank i — typically the same global edge list: each shard keeps the
        edges of its own sources (gpma_shard_from_edges_device)."""
        lib = load_library()
        bounds = np.asarray(bounds, np.int64)
        devices = devices if devices is not None else [e[0].device.index for e in edges]
        cfg = (config or GraphConfig()).c()
        hs = []
        for i, r in enumerate(comm.ranks):
            s, d, w = edges[i]
            _sync(s)
            h = C.c_void_p()
            rc = lib.gpma_shard_from_edges_device(C.byref(cfg), devices[i], num_vertices, int(bounds[r]),
                                                  int(bounds[r + 1]), _vp(s), _vp(d), _vp(w), s.numel(), C.byref(h))
            if rc:
                _raise(rc, lib.gpma_last_error(None).decode())
            hs.append(h)
        return cls(comm, num_vertices, bounds, hs, devices, routing)

    def __del__(self):
        self._free_rx()
        for h in getattr(self, "h", []) or []:
            if h:
                self._lib.gpma_destroy(h)
        self.h = []

    def _check(self, i, rc):
        if rc:
            _raise(rc, self._lib.gpma_last_error(self.h[i]).decode())

    def _sy(self, t):
        if not self._ordered:
            _sync(t)

    def range(self, i):
        r = self.comm.ranks[i]
        return int(self.bounds[r]), int(self.bounds[r + 1])

    # ---- updates
    def _route(self, i, a, b, w, c=None, d=None):
        """Stable owner partition of local rank i's share (inserts a,b,w then
        deletes c,d) into EdgeKeys (bit 63 = delete) + weights + counts."""
        torch = _torch()
        ni = a.numel()
        nd = c.numel() if c is not None else 0
        n = ni + nd
        keys = torch.empty(max(n, 1), dtype=torch.int64, device=a.device)
        ow = torch.empty(max(n, 1), dtype=torch.float64, device=a.device) if w is not None else None
        counts = torch.empty(self.comm.world + 1, dtype=torch.int64, device=a.device)
        if not self._ordered:
            _sync(a)
        self._check(i, self._lib.gpma_route_batch_async(self.h[i], _vp(a), _vp(b), _vp(w), ni, _vp(c), _vp(d), nd,
                                                         _vp(self._dbounds[i]), self.comm.world, _vp(keys), _vp(ow),
                                                         _vp(counts)))
        if not self._ordered:  # the async route ran on the library's own stream
            torch.cuda.ExternalStream(self._lib.gpma_cuda_stream(self.h[i]), device=a.device).synchronize()
        return keys[:n], (ow[:n] if ow is not None else None), counts

    def _reject_bad_inserts(self, slices, bad):
        """bad[r] = inserts of sender r naming a vertex >= |V| (counted by the
        routing kernels).  The reference rejects such a batch before any
        mutation (check_ids, graph.hpp:133-137), so every rank raises here,
        before any shard applies — never a half-applied batch or a rank left
        waiting in the next collective."""
        if not any(int(x) for x in bad):
            return
        for i, sl in enumerate(slices):
            if int(bad[self.comm.ranks[i]]):
                a = sl[0].cpu().numpy().view(np.uint32)
                b = sl[1].cpu().numpy().view(np.uint32)
                j = int(np.nonzero((a >= self.nv) | (b >= self.nv))[0][0])
                raise ValueError(f"edge ({a[j]}, {b[j]}) outside vertex range {self.nv}")
        r = next(r for r, x in enumerate(bad) if int(x))
        raise ValueError(f"apply_batch rejected on every shard: rank {r} holds an insert outside vertex range "
                         f"{self.nv}")

    # ---- fused routing: partition + transfer in one kernel (peer memory)
    def _free_rx(self):
        rx = getattr(self, "_rx", None)
        if not rx:
            return
        for p in rx.get("opened", []):
            self._lib.gpma_ipc_close(C.c_void_p(p))
        for p in rx.get("owned", []):
            self._lib.gpma_ipc_free(C.c_void_p(p))
        self._rx = None

    def _ensure_rx(self, need: int, weighted: bool):
        """Receive buffers of `need` EdgeKeys (+ weights) on every rank; every
        rank derives `need` from the same count matrix, so re-allocations are
        collective.  In one process the buffers are plain device tensors; across
        processes each rank exports its buffers as CUDA IPC handles and maps
        its peers' (cudaIpcOpenMemHandle)."""
        torch = _torch()
        rx = self._rx
        if rx and rx["cap"] >= need and rx["weighted"] == weighted:
            return rx
        self._free_rx()
        cap = max(1024, int(need * 1.25))
        W, L = self.comm.world, len(self.h)
        rx = {"cap": cap, "weighted": weighted, "owned": [], "opened": []}
        if isinstance(self.comm, LocalComm):
            keys = [torch.empty(cap, dtype=torch.int64, device=f"cuda:{d}") for d in self.devices]
            ws = [torch.empty(cap, dtype=torch.float64, device=f"cuda:{d}") for d in self.devices] if weighted else None
            kptr = [t.data_ptr() for t in keys]
            wptr = [t.data_ptr() for t in ws] if weighted else None
            rx.update(keys=keys, ws=ws, kptr_all=[kptr] * L, wptr_all=[wptr] * L,
                      mine_k=kptr, mine_w=wptr if weighted else [0] * L)
        else:
            (dev,), me = self.devices, self.comm.ranks[0]
            mine = []
            for nbytes in ([cap * 8, cap * 8] if weighted else [cap * 8]):
                ptr, hnd = C.c_void_p(), (C.c_char * 64)()
                self._check(0, self._lib.gpma_ipc_alloc(dev, nbytes, C.byref(ptr), hnd))
                rx["owned"].append(ptr.value)
                mine.append((ptr.value, bytes(hnd)))
            allh = [None] * W
            self.comm.dist.all_gather_object(allh, [h for _, h in mine], group=self.comm.group)
            ptrs = []
            for r in range(W):
                row = []
                for j, hb in enumerate(allh[r]):
                    if r == me:
                        row.append(mine[j][0])
                    else:
                        q = C.c_void_p()
                        self._check(0, self._lib.gpma_ipc_open(dev, (C.c_char * 64).from_buffer_copy(hb), C.byref(q)))
                        rx["opened"].append(q.value)
                        row.append(q.value)
                ptrs.append(row)
            kptr = [row[0] for row in ptrs]
            wptr = [row[1] for row in ptrs] if weighted else None
            rx.update(kptr_all=[kptr], wptr_all=[wptr], mine_k=[mine[0][0]],
                      mine_w=[mine[1][0]] if weighted else [0])
        # per local sender: device arrays of the W destination pointers
        rx["kdev"] = [torch.tensor(kp, dtype=torch.int64, device=f"cuda:{d}")
                      for kp, d in zip(rx["kptr_all"], self.devices)]
        rx["wdev"] = [torch.tensor(wp, dtype=torch.int64, device=f"cuda:{d}") if wp else None
                      for wp, d in zip(rx["wptr_all"], self.devices)]
        self._rx = rx
        return rx

    def _apply_fused(self, slices) -> ShardStats:
        torch = _torch()
        L, W = len(self.h), self.comm.world
        weighted = slices[0][2] is not None
        counts = []
        for i in range(L):
            a, b, w, c, d = slices[i]
            cnt = torch.empty(W + 1, dtype=torch.int64, device=a.device)
            if not self._ordered:
                _sync(a)
            self._check(i, self._lib.gpma_route_count(self.h[i], _vp(a), _vp(b), a.numel(), _vp(c), _vp(d),
                                                       c.numel() if c is not None else 0, _vp(self._dbounds[i]), W,
                                                       _vp(cnt)))
            counts.append(cnt)
        if not self._ordered:
            for i in range(L):
                torch.cuda.ExternalStream(self._lib.gpma_cuda_stream(self.h[i]),
                                          device=counts[i].device).synchronize()
        # the count matrix M[sender][owner] on every rank
        if isinstance(self.comm, LocalComm):
            M = np.stack([c.cpu().numpy() for c in counts])
        else:
            (cnt,) = counts
            if self.comm.dist.get_backend(self.comm.group) == "gloo":
                cnt = cnt.cpu()  # gloo: host tensors
            parts = [torch.empty_like(cnt) for _ in range(W)]
            self.comm.dist.all_gather(parts, cnt, group=self.comm.group)
            M = torch.stack(parts).cpu().numpy()
        self._reject_bad_inserts(slices, M[:, W])  # M[s][W]: sender s's inserts outside the vertex range
        M = M[:, :W]
        before, nrecv = fused_offsets(M)
        rx = self._ensure_rx(int(nrecv.max()) if W else 0, weighted)
        for i in range(L):
            a, b, w, c, d = slices[i]
            me = self.comm.ranks[i]
            off = torch.as_tensor(before[me].astype(np.int64), device=a.device)
            self._check(i, self._lib.gpma_route_scatter_peer(self.h[i], _vp(a), _vp(b), _vp(w), a.numel(), _vp(c),
                                                              _vp(d), c.numel() if c is not None else 0,
                                                              _vp(self._dbounds[i]), W, _vp(rx["kdev"][i]),
                                                              _vp(rx["wdev"][i]), _vp(off)))
        # every sender's stores land before any owner reads its buffer: with
        # NCCL a one-element all-reduce on the stream is that barrier (it runs
        # on every rank after the rank's scatter kernel); otherwise host syncs
        nccl = (not isinstance(self.comm, LocalComm) and self._ordered
                and self.comm.dist.get_backend(self.comm.group) == "nccl")
        if nccl:
            self.comm.dist.all_reduce(torch.zeros(1, device=f"cuda:{self.devices[0]}"), group=self.comm.group)
        else:
            for i in range(L):
                if self._ordered:
                    torch.cuda.current_stream(self.devices[i]).synchronize()
                else:
                    torch.cuda.ExternalStream(self._lib.gpma_cuda_stream(self.h[i]),
                                              device=torch.device("cuda", self.devices[i])).synchronize()
            if not isinstance(self.comm, LocalComm):
                self.comm.dist.barrier(group=self.comm.group)
        out, routed, sent = [], [], []
        for i in range(L):
            me = self.comm.ranks[i]
            st = pma_stats()
            n = int(nrecv[me])
            self._check(i, self._lib.gpma_apply_batch_routed_device(
                self.h[i], C.c_void_p(rx["mine_k"][i]), C.c_void_p(rx["mine_w"][i]) if weighted else None, n,
                C.byref(st)))
            out.append(UpdateStats.from_c(st))
            routed.append(n)
            sent.append(int(M[me].sum() - M[me][me]))
        return ShardStats(out, routed, sent)

    def apply_batch(self, slices) -> ShardStats:
        """slices[i] = (ins_src, ins_dst, ins_w|None, del_src, del_dst):
        local rank i's share of the global batch (device tensors, u32 ids as
        int32; weights given on every rank or on none).  One owner partition
        (gpma_route_batch) and one all-to-all of 8-B EdgeKeys per batch, then
        each shard applies its routed batch (DynamicGraph::apply_batch,
        graph.hpp:130-162).  routing="fused": the owner partition writes
        straight into the owners' receive buffers instead (_apply_fused)."""
        if self.routing == "fused":
            return self._apply_fused(slices)
        L = len(self.h)
        ks, ws, cs, bads = [], [], [], []
        for i in range(L):
            a, b, w, c, d = slices[i]
            k, ww, cnt = self._route(i, a, b, w, c, d)
            ks.append(k)
            ws.append(ww)
            cs.append(cnt[:-1])
            bads.append(cnt[-1:])
        # one scalar all-reduce: every rank learns of a bad insert anywhere
        # before any shard applies (or the all-to-all runs)
        tot = [x.clone() for x in bads]
        self.comm.all_reduce(tot, "sum")
        if int(tot[0].item()):
            bad = [0] * self.comm.world
            for i in range(L):
                bad[self.comm.ranks[i]] = int(bads[i].item())
            if not any(bad):
                bad[next(r for r in range(self.comm.world) if r not in self.comm.ranks)] = 1
            self._reject_bad_inserts(slices, bad)
        rk, _, scl = self.comm.all_to_all_v(ks, cs)
        rw = self.comm.all_to_all_v(ws, scl)[0] if ws[0] is not None else [None] * L
        cs = scl
        out, routed, sent = [], [], []
        for i in range(L):
            st = pma_stats()
            if not self._ordered:
                _sync(rk[i])
            self._check(i, self._lib.gpma_apply_batch_routed_device(self.h[i], _vp(rk[i]), _vp(rw[i]), rk[i].numel(),
                                                                     C.byref(st)))
            out.append(UpdateStats.from_c(st))
            routed.append(rk[i].numel())
            me = self.comm.ranks[i]
            sent.append(sum(cs[i]) - cs[i][me])
        return ShardStats(out, routed, sent)

    # ---- analytics
    def bfs(self, root: int):
        """Level-synchronous BFS (analytics.hpp:22-48); dist[v] = level,
        UNREACHED = 0xFFFFFFFF.  Returns the full |V| vector per local rank."""
        torch = _torch()
        L = len(self.h)
        if not 0 <= root < self.nv:
            raise ValueError("bfs: root outside vertex range")
        dist, fr, nx, flags, nf = [], [], [], [], []
        for i in range(L):
            lo, hi = self.range(i)
            dev = f"cuda:{self.devices[i]}"
            dl = torch.full((max(hi - lo, 1),), -1, dtype=torch.int32, device=dev)
            f = torch.empty(max(hi - lo, 1), dtype=torch.int32, device=dev)
            n = 0
            if lo <= root < hi:
                dl[root - lo] = 0
                f[0] = root
                n = 1
            dist.append(dl)
            fr.append(f)
            nx.append(torch.empty_like(f))
            flags.append(torch.empty(self.nv, dtype=torch.uint8, device=dev))
            nf.append(n)
        depth = 0
        while True:
            for i in range(L):
                self._sy(fr[i])
                self._check(i, self._lib.gpma_shard_bfs_mark(self.h[i], _vp(fr[i]), nf[i], _vp(flags[i])))
            self.comm.all_reduce(flags, "max")
            depth += 1
            tot = []
            for i in range(L):
                self._sy(flags[i])
                c = C.c_uint32(0)
                self._check(i, self._lib.gpma_shard_bfs_update(self.h[i], _vp(flags[i]), _vp(dist[i]), depth,
                                                                _vp(nx[i]), C.byref(c)))
                nf[i] = c.value
                tot.append(torch.tensor([c.value], dtype=torch.int64, device=flags[i].device))
            self.comm.all_reduce(tot, "sum")
            fr, nx = nx, fr
            if int(tot[0].item()) == 0:
                break
        pieces = [dist[i][:self.range(i)[1] - self.range(i)[0]] for i in range(L)]
        return self.comm.all_gather_v(pieces)

    def connected_components(self):
        """Labels = minimum vertex id of each (undirected) component
        (analytics.hpp:53-82)."""
        torch = _torch()
        L = len(self.h)
        lab = [torch.arange(self.nv, dtype=torch.int32, device=f"cuda:{d}") for d in self.devices]
        rounds = 0
        while True:
            prev = [t.clone() for t in lab]
            for i in range(L):
                self._sy(lab[i])
                self._check(i, self._lib.gpma_shard_cc_hook(self.h[i], _vp(lab[i])))
            self.comm.all_reduce(lab, "min")
            ch = []
            for i in range(L):
                self._sy(lab[i])
                c = C.c_int(0)
                self._check(i, self._lib.gpma_cc_jump(self.h[i], _vp(lab[i]), self.nv, _vp(prev[i]), C.byref(c)))
                ch.append(torch.tensor([c.value], dtype=torch.int32, device=lab[i].device))
            self.comm.all_reduce(ch, "max")
            rounds += 1
            if int(ch[0].item()) == 0:
                break
        self.cc_rounds = rounds
        return lab

    def pagerank(self, damping: float = 0.85, epsilon: float = 1e-3, max_iters: int = 200, warm_start=None):
        """Power iteration (analytics.hpp:84-143); returns (ranks per local
        rank, iterations, converged) with the reference's stopping rule."""
        torch = _torch()
        L = len(self.h)
        n = self.nv
        if n == 0:
            raise ValueError("pagerank: empty vertex set")
        if warm_start is not None and len(warm_start) != n:
            raise ValueError("pagerank: warm start size mismatch")
        od, x, y = [], [], []
        for i in range(L):
            dev = f"cuda:{self.devices[i]}"
            o = torch.empty(n, dtype=torch.int32, device=dev)
            self._check(i, self._lib.gpma_shard_outdeg(self.h[i], _vp(o)))
            od.append(o)
            if warm_start is not None:
                xi = torch.as_tensor(np.asarray(warm_start, np.float64), device=dev).clone()
            else:
                xi = torch.full((n,), 1.0 / n, dtype=torch.float64, device=dev)
            x.append(xi)
            y.append(torch.empty(n, dtype=torch.float64, device=dev))
        self.comm.all_reduce(od, "sum")
        converged = False
        it = 0
        for it in range(1, max_iters + 1):
            for i in range(L):
                self._sy(x[i])
                self._sy(od[i])
                self._check(i, self._lib.gpma_shard_pr_push(self.h[i], _vp(x[i]), _vp(od[i]), damping, _vp(y[i])))
            self.comm.all_reduce(y, "sum")
            l1 = C.c_double(0)
            for i in range(L):
                self._sy(y[i])
                self._check(i, self._lib.gpma_pr_finish(self.h[i], _vp(x[i]), _vp(y[i]), n, _vp(od[i]), damping,
                                                        C.byref(l1)))
            x, y = y, x
            if l1.value < epsilon:
                converged = True
                break
        return x, (it if converged else max_iters), converged

    def spmv(self, x):
        """y = A x (analytics.hpp:147-158): owners compute their rows with the
        single-GPU ordered accumulation, one all-gather."""
        torch = _torch()
        L = len(self.h)
        pieces = []
        for i in range(L):
            lo, hi = self.range(i)
            dev = f"cuda:{self.devices[i]}"
            xi = x.to(dev) if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x, np.float64), device=dev)
            yl = torch.empty(max(hi - lo, 1), dtype=torch.float64, device=dev)
            self._sy(xi)
            self._check(i, self._lib.gpma_shard_spmv(self.h[i], _vp(xi), _vp(yl)))
            pieces.append(yl[:hi - lo])
        return self.comm.all_gather_v(pieces)

    # ---- inspection (tests)
    def shard_slots(self, i):
        from .pmagraph import PackedMemoryArray
        p = PackedMemoryArray(_handle=self._lib.gpma_pma(self.h[i]), _owner=self)
        return p.slots()

    def shard_row_offsets(self, i):
        lo, hi = self.range(i)
        out = np.zeros(hi - lo + 1, np.uint64)
        self._check(i, self._lib.gpma_row_offsets(self.h[i], out.ctypes.data_as(C.c_void_p)))
        return out

    def num_edges(self):
        return [int(self._lib.gpma_num_edges(h)) for h in self.h]

    def last_timing(self, i=0):
        from .abi import pma_timing
        t = pma_timing()
        self._check(i, self._lib.gpma_last_timing(self.h[i], C.byref(t)))
        return t

    def cuda_stream(self, i=0):
        return self._lib.gpma_cuda_stream(self.h[i])


# ------------------------------------------------------- C-ABI shard group

def nccl_unique_id() -> bytes:
    """ncclGetUniqueId (128 bytes) through the library (rank 0 creates it)."""
    lib = load_library()
    buf = (C.c_char * 128)()
    rc = lib.gpma_nccl_unique_id(buf)
    if rc:
        _raise(rc, lib.gpma_shard_group_last_error(None).decode())
    return bytes(buf)


class NcclComm:
    """An NCCL communicator created by the library (gpma_nccl_comm_create)
    from a unique id every rank holds; shard groups may share it."""

    def __init__(self, nccl_id: bytes, world: int, rank: int, device: int = 0):
        self._lib = load_library()
        self.h = C.c_void_p()
        idb = (C.c_char * 128).from_buffer_copy(nccl_id)
        rc = self._lib.gpma_nccl_comm_create(idb, world, rank, device, C.byref(self.h))
        if rc:
            self.h = None
            _raise(rc, self._lib.gpma_shard_group_last_error(None).decode())

    def close(self):
        if getattr(self, "h", None):
            self._lib.gpma_nccl_comm_destroy(self.h)
            self.h = None


class ShardGroup:
    """This rank's shard of the key-range sharded graph with every collective
    issued by the library over NCCL (gpma_shard_group_*, csrc/shard_group.cu):
    the host only hands over device arrays.  bounds: world + 1 vertex bounds;
    nccl_id: the same 128-byte ncclUniqueId on every rank."""

    def __init__(self, num_vertices: int, bounds, rank: int, world: int, nccl_id: bytes | None, edges,
                 config: GraphConfig | None = None, device: int = 0, comm: "NcclComm | None" = None):
        self._lib = load_library()
        self.nv, self.rank, self.world, self.device = int(num_vertices), rank, world, device
        self.bounds = np.ascontiguousarray(np.asarray(bounds, np.uint32))
        s, d, w = edges
        cfg = (config or GraphConfig()).c()
        idb = (C.c_char * 128).from_buffer_copy(nccl_id) if nccl_id is not None else None
        self._comm = comm  # keeps a shared communicator alive while the group lives
        self.h = C.c_void_p()
        rc = self._lib.gpma_shard_group_create(C.byref(cfg), device, self.nv, _vp_np(self.bounds), world, rank, idb,
                                               comm.h if comm is not None else None, _vp(s), _vp(d), _vp(w),
                                               s.numel(), C.byref(self.h))
        if rc:
            self.h = None
            _raise(rc, self._lib.gpma_shard_group_last_error(None).decode())
        self.lo, self.hi = int(self.bounds[rank]), int(self.bounds[rank + 1])

    def __del__(self):
        if getattr(self, "h", None):
            self._lib.gpma_shard_group_destroy(self.h)
            self.h = None

    def _check(self, rc):
        if rc:
            _raise(rc, self._lib.gpma_shard_group_last_error(self.h).decode())

    def graph_handle(self):
        return self._lib.gpma_shard_group_graph(self.h)

    def cuda_stream(self):
        return self._lib.gpma_cuda_stream(self.graph_handle())

    def apply_batch(self, a, b, w, c, d):
        """(UpdateStats of this shard, updates this shard applied, updates sent away)."""
        st = pma_stats()
        routed, sent = C.c_uint64(), C.c_uint64()
        self._check(self._lib.gpma_shard_group_apply_batch(self.h, _vp(a), _vp(b), _vp(w), a.numel(), _vp(c), _vp(d),
                                                           c.numel() if c is not None else 0, C.byref(st),
                                                           C.byref(routed), C.byref(sent)))
        return UpdateStats.from_c(st), routed.value, sent.value

    def bfs(self, root: int):
        dist = _host_out(self.nv, np.uint32)  # (page-locked: the gathered result lands by DMA)
        reached = C.c_uint64()
        self._check(self._lib.gpma_shard_group_bfs(self.h, C.c_uint32(root), _vp_np(dist), C.byref(reached)))
        return dist, reached.value

    def connected_components(self):
        lab = _host_out(self.nv, np.uint32)
        self._check(self._lib.gpma_shard_group_cc(self.h, _vp_np(lab)))
        return lab

    def pagerank(self, damping=0.85, epsilon=1e-3, max_iters=200, warm_start=None):
        if warm_start is not None and len(warm_start) != self.nv:
            raise ValueError("pagerank: warm start size mismatch")
        ranks = _host_out(self.nv, np.float64)
        it, conv = C.c_uint64(), C.c_int()
        warm = None if warm_start is None else np.ascontiguousarray(warm_start, np.float64)
        self._check(self._lib.gpma_shard_group_pagerank(self.h, C.c_double(damping), C.c_double(epsilon), max_iters,
                                                        _vp_np(warm) if warm is not None else None, _vp_np(ranks),
                                                        C.byref(it), C.byref(conv)))
        return ranks, it.value, bool(conv.value)

    def spmv(self, x):
        xx = np.ascontiguousarray(x, np.float64)
        if len(xx) != self.nv:
            raise ValueError("spmv: dimension mismatch")
        y = np.empty(self.nv, np.float64)
        self._check(self._lib.gpma_shard_group_spmv(self.h, _vp_np(xx), _vp_np(y)))
        return y

    def shard_slots(self):
        h = self._lib.gpma_pma(self.graph_handle())
        return PackedMemoryArray(_handle=h, _owner=self).slots()

    def shard_row_offsets(self):
        out = np.zeros(self.hi - self.lo + 1, np.uint64)
        self._check(self._lib.gpma_row_offsets(self.graph_handle(), out.ctypes.data_as(C.c_void_p)))
        return out


def _vp_np(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None
