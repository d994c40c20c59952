"""Python mirror of the reference ``pmagraph`` interface over libpmagraph_cuda.so.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/pmagraph/*.hpp) so parity tests read like the
reference's own tests:

  PackedMemoryArray  (pma.hpp:125-612)         batch_update (segment_engine.hpp:365)
  DynamicGraph       (graph.hpp:62-240)        bfs / connected_components /
  UpdateStats        (update_stats.hpp:13-35)  pagerank / spmv (analytics.hpp)

Error mapping: std::invalid_argument -> ValueError,
std::out_of_range -> IndexError, std::logic_error -> LogicError,
device failure -> RuntimeError.  Every call runs on the GPU through the C ABI;
there is no CPU fallback (the import fails loudly without the library).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from .abi import (GPMA_UNREACHED, PMA_EAGER, PMA_EINVAL, PMA_ELOGIC, PMA_ERANGE, PMA_LAZY, PMA_STRATEGY_AUTO,
                  default_profile, engine_config, graph_config, load_library, pma_engine_config, pma_layout_info,
                  pma_profile, pma_stats, pma_timing)

kUnreached = GPMA_UNREACHED
kMinCapacity = 16


class LogicError(RuntimeError):
    """std::logic_error"""


def _raise(code: int, msg: str):
    if code == PMA_EINVAL:
        raise ValueError(msg)
    if code == PMA_ERANGE:
        raise IndexError(msg)
    if code == PMA_ELOGIC:
        raise LogicError(msg)
    raise RuntimeError(msg)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class DensityProfile:
    """pma.hpp:52-78"""
    leaf_lower: float = 0.08
    leaf_upper: float = 0.92
    root_lower: float = 0.40
    root_upper: float = 0.80
    allow_shrink: bool = True

    def c(self) -> pma_profile:
        return pma_profile(self.leaf_lower, self.leaf_upper, self.root_lower, self.root_upper,
                           1 if self.allow_shrink else 0, 0)


@dataclass
class UpdateStats:
    """update_stats.hpp:13-35"""
    batch_size: int = 0
    rounds: int = 0
    slot_writes: int = 0
    wall_ns: int = 0
    segment_phase_ns: int = 0
    segments_per_level: list = field(default_factory=list)
    grow_events: int = 0
    shrink_events: int = 0
    deletes_missed: int = 0
    tombstones_added: int = 0
    touched_ranges: list = field(default_factory=list)
    resized: bool = False

    @classmethod
    def from_c(cls, s: pma_stats, touched=None) -> "UpdateStats":
        return cls(s.batch_size, s.rounds, s.slot_writes, s.wall_ns, s.segment_phase_ns,
                   s.segments_per_level[:s.num_levels], s.grow_events, s.shrink_events,
                   s.deletes_missed, s.tombstones_added, touched if touched is not None else [], bool(s.resized))

    def parity(self) -> dict:
        """Fields compared bit-exactly against the reference (timing excluded)."""
        return {k: getattr(self, k) for k in ("batch_size", "rounds", "slot_writes", "segments_per_level",
                                              "grow_events", "shrink_events", "deletes_missed",
                                              "tombstones_added", "touched_ranges", "resized")}

    @staticmethod
    def csv_header():
        return "batch_size,rounds,slot_writes,wall_ns"

    def csv_row(self):
        return f"{self.batch_size},{self.rounds},{self.slot_writes},{self.wall_ns}"

    @staticmethod
    def csv_header_device():
        """The reference's columns plus the device ones SURVEY §5 names."""
        return UpdateStats.csv_header() + ",gpus,bytes_moved,hbm_frac,nvlink_frac"

    def csv_row_device(self, timing, gpus: int = 1, hbm_peak_gbps: float = None, nvlink_bytes: int = 0,
                       nvlink_peak_gbps: float = 900.0):
        """`timing`: the same call's `pma_timing` (DynamicGraph.last_timing()).
        bytes_moved = its algorithmic commit bytes;
        hbm_frac = bytes_moved / device time / the HBM peak (MEASURED_PEAKS.json
        when present, else 6650 GB/s); nvlink_frac = the routed bytes of a
        sharded batch / device time / one GPU's NVLink peak per direction
        (0 on one GPU)."""
        if hbm_peak_gbps is None:
            hbm_peak_gbps = _hbm_peak()
        sec = float(timing.device_ms) * 1e-3
        moved = int(timing.commit_bytes)
        hbm = moved / sec / (hbm_peak_gbps * 1e9) if sec > 0 else 0.0
        nvl = nvlink_bytes / sec / (nvlink_peak_gbps * 1e9) if sec > 0 and nvlink_bytes else 0.0
        return f"{self.csv_row()},{gpus},{moved},{hbm:.4f},{nvl:.4f}"


def _hbm_peak() -> float:
    import json
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6650.0


@dataclass
class SegmentEngineConfig:
    """segment_engine.hpp:43-60 (workers accepted, ignored: the grid replaces the pool)."""
    deletion_mode: int = PMA_LAZY
    workers: int = 1
    small_max: int = 32
    medium_max: int = 1024
    force_strategy: int = PMA_STRATEGY_AUTO

    def c(self) -> pma_engine_config:
        return engine_config(self.deletion_mode, self.workers, self.small_max, self.medium_max, self.force_strategy)


class PackedMemoryArray:
    """Device-resident PMA (pma.hpp:125-612)."""

    def __init__(self, profile: DensityProfile | None = None, device: int = 0, _handle=None, _owner=None):
        self._lib = load_library()
        self._owner = _owner
        if _handle is not None:
            self.h = C.c_void_p(_handle)
            self._owned = False
            return
        self.h = C.c_void_p()
        prof = (profile or DensityProfile()).c()
        rc = self._lib.pma_create(C.byref(prof), device, C.byref(self.h))
        if rc:
            _raise(rc, self._lib.pma_last_error(None).decode())
        self._owned = True

    def __del__(self):
        if getattr(self, "_owned", False) and self.h:
            self._lib.pma_destroy(self.h)
            self.h = None

    def _check(self, rc):
        if rc:
            _raise(rc, self._lib.pma_last_error(self.h).decode())

    # -- construction --
    @classmethod
    def from_sorted(cls, keys, values, fill_target: float, profile: DensityProfile | None = None,
                    device: int = 0) -> "PackedMemoryArray":
        p = cls(profile, device)
        k, v = _u64(keys), _u64(values)
        p._check(p._lib.pma_from_sorted(p.h, _p(k), _p(v), len(k), C.c_double(fill_target)))
        return p

    @classmethod
    def from_slots(cls, keys, values, states, profile: DensityProfile | None = None,
                   device: int = 0) -> "PackedMemoryArray":
        """Exact restore of a slot array (generalises from_slot_layout, pma.hpp:191-207)."""
        p = cls(profile, device)
        p.load_slots(keys, values, states)
        return p

    @classmethod
    def from_slot_layout(cls, capacity, placements, profile: DensityProfile | None = None, device: int = 0):
        """pma.hpp:191-207: placements = [(slot, key, value), ...]."""
        k = np.zeros(capacity, np.uint64)
        v = np.zeros(capacity, np.uint64)
        s = np.zeros(capacity, np.uint8)
        for slot, key, value in placements:
            k[slot], v[slot], s[slot] = key, value, 1
        return cls.from_slots(k, v, s, profile, device)

    def load_slots(self, keys, values, states):
        k, v, s = _u64(keys), _u64(values), _u8(states)
        self._check(self._lib.pma_load_slots(self.h, len(s), _p(k), _p(v), _p(s)))

    # -- accessors --
    def _layout(self) -> pma_layout_info:
        li = pma_layout_info()
        self._check(self._lib.pma_get_layout(self.h, C.byref(li)))
        return li

    def capacity(self) -> int:
        return self._layout().capacity

    def leaf_size(self) -> int:
        return self._layout().leaf_size

    def height(self) -> int:
        return self._layout().height

    def valid_count(self) -> int:
        return self._layout().valid_count

    def tombstone_count(self) -> int:
        return self._layout().tombstone_count

    def slot_writes(self) -> int:
        return self._layout().slot_writes

    def reset_slot_writes(self):
        self._check(self._lib.pma_reset_slot_writes(self.h))

    def slots(self):
        """slots() (pma.hpp:214) as SoA numpy arrays (keys, values, states)."""
        cap = self.capacity()
        k = np.zeros(cap, np.uint64)
        v = np.zeros(cap, np.uint64)
        s = np.zeros(cap, np.uint8)
        self._check(self._lib.pma_download(self.h, _p(k), _p(v), _p(s)))
        return k, v, s

    def min_entries(self, level: int) -> int:
        mn = C.c_uint64()
        self._check(self._lib.pma_bounds(self.h, level, C.byref(mn), None, None, None))
        return mn.value

    def max_entries(self, level: int) -> int:
        mx = C.c_uint64()
        self._check(self._lib.pma_bounds(self.h, level, None, C.byref(mx), None, None))
        return mx.value

    def thresholds(self, level: int):
        rho, tau = C.c_double(), C.c_double()
        self._check(self._lib.pma_bounds(self.h, level, None, None, C.byref(rho), C.byref(tau)))
        return rho.value, tau.value

    def reserve_batch(self, max_updates: int):
        """Pre-size every per-batch buffer (pma_reserve_batch)."""
        self._check(self._lib.pma_reserve_batch(self.h, max_updates))

    def set_grid_segment(self, min_slots: int):
        """Segments of >= min_slots slots merge in the grid tier (pma_set_grid_segment)."""
        self._check(self._lib.pma_set_grid_segment(self.h, min_slots))

    def slot_hash(self, level: int):
        """Per-segment parity digest of slots() at `level` (pma_slot_hash)."""
        n = self.capacity() // (self.leaf_size() << level) if 0 <= level <= self.height() else 1
        out = np.zeros(max(n, 1), np.uint64)
        self._check(self._lib.pma_slot_hash(self.h, level, _p(out)))
        return out[:n]

    def binary_search_leaf(self, keys):
        scalar = np.isscalar(keys)
        k = _u64(np.atleast_1d(keys))
        out = np.zeros(len(k), np.uint64)
        self._check(self._lib.pma_binary_search_leaf(self.h, _p(k), len(k), _p(out)))
        return int(out[0]) if scalar else out

    def search(self, key):
        k = _u64([key])
        v = np.zeros(1, np.uint64)
        f = np.zeros(1, np.uint8)
        self._check(self._lib.pma_search(self.h, _p(k), 1, _p(v), _p(f)))
        return int(v[0]) if f[0] else None

    def search_many(self, keys):
        k = _u64(keys)
        v = np.zeros(len(k), np.uint64)
        f = np.zeros(len(k), np.uint8)
        self._check(self._lib.pma_search(self.h, _p(k), len(k), _p(v), _p(f)))
        return v, f.astype(bool)

    def count_valid_in(self, begin: int, end: int) -> int:
        c = C.c_uint64()
        self._check(self._lib.pma_count_valid_in(self.h, begin, end, C.byref(c)))
        return c.value

    def to_entries(self):
        k, v, s = self.slots()
        m = s == 1
        return k[m], v[m]

    # -- sequential ops (pma.hpp:294-386, 471-479) --
    def insert(self, key: int, value: int):
        self._check(self._lib.pma_insert(self.h, C.c_uint64(key), C.c_uint64(value)))

    def erase(self, key: int) -> bool:
        r = C.c_int()
        self._check(self._lib.pma_erase(self.h, C.c_uint64(key), C.byref(r)))
        return bool(r.value)

    def mark_tombstone(self, key: int) -> bool:
        r = C.c_int()
        self._check(self._lib.pma_mark_tombstone(self.h, C.c_uint64(key), C.byref(r)))
        return bool(r.value)

    def redispatch(self, level: int, seg_index: int, keys=(), values=()):
        k, v = _u64(keys), _u64(values if len(values) else np.zeros(len(keys), np.uint64))
        self._check(self._lib.pma_redispatch(self.h, level, seg_index, _p(k), _p(v), len(k)))

    def touched_ranges_array(self, n: int | None = None):
        """UpdateStats::touched_ranges of the last batch as an (n, 2) u64 array
        in the reference's order (n: the count from pma_stats, saves a call)."""
        if n is None:
            c = C.c_size_t(0)
            self._check(self._lib.pma_touched_ranges(self.h, None, 0, C.byref(c)))
            n = c.value
        out = _host_out(2 * max(n, 1), np.uint64)  # page-locked: the copy is one DMA
        c = C.c_size_t(0)
        self._check(self._lib.pma_touched_ranges(self.h, _p(out), n, C.byref(c)))
        return out[:2 * n].reshape(n, 2)

    def touched_ranges(self):
        a = self.touched_ranges_array()
        return [(int(x), int(y)) for x, y in a]

    def last_timing(self) -> pma_timing:
        t = pma_timing()
        self._check(self._lib.pma_last_timing(self.h, C.byref(t)))
        return t


def batch_update(pma: PackedMemoryArray, keys, values, ops, cfg: SegmentEngineConfig | None = None,
                 pool=None, with_touched: bool = True) -> UpdateStats:
    """batch_update (segment_engine.hpp:365-470): ops 0 = insert, 1 = delete.
    ``pool`` (WorkerPool*) is accepted and ignored."""
    k, v, o = _u64(keys), _u64(values), _u8(ops)
    st = pma_stats()
    c = (cfg or SegmentEngineConfig()).c()
    pma._check(pma._lib.pma_batch_update(pma.h, _p(k), _p(v), _p(o), len(k), C.byref(c), C.byref(st)))
    return UpdateStats.from_c(st, pma.touched_ranges() if with_touched else None)


@dataclass
class GraphConfig:
    """graph.hpp:54-60 (engine must be the segment engine)."""
    deletion_mode: int = PMA_LAZY
    workers: int = 1
    fill_target: float = 0.5
    profile: DensityProfile = field(default_factory=DensityProfile)

    def c(self):
        return graph_config(self.deletion_mode, self.workers, self.fill_target, self.profile.c())


@dataclass
class PageRankResult:
    ranks: np.ndarray
    iterations: int
    converged: bool


class DynamicGraph:
    """CSR-on-PMA graph (graph.hpp:62-240) on the device."""

    def __init__(self, handle, lib, nv):
        self.h = handle
        self._lib = lib
        self._nv = nv

    @classmethod
    def from_edges(cls, num_vertices: int, src, dst, weights=None, config: GraphConfig | None = None,
                   device: int = 0) -> "DynamicGraph":
        lib = load_library()
        s, d, w = _u32(src), _u32(dst), _f64(weights)
        h = C.c_void_p()
        cfg = (config or GraphConfig()).c()
        rc = lib.gpma_from_edges(C.byref(cfg), device, num_vertices, _p(s), _p(d), _p(w), len(s), C.byref(h))
        if rc:
            _raise(rc, lib.gpma_last_error(None).decode())
        return cls(h, lib, num_vertices)

    @classmethod
    def from_edges_device(cls, num_vertices: int, d_src: int, d_dst: int, d_w: int | None, n: int,
                          config: GraphConfig | None = None, device: int = 0) -> "DynamicGraph":
        """Edge arrays already in device memory (raw pointers, e.g. tensor.data_ptr())."""
        lib = load_library()
        h = C.c_void_p()
        cfg = (config or GraphConfig()).c()
        rc = lib.gpma_from_edges_device(C.byref(cfg), device, num_vertices, C.c_void_p(d_src), C.c_void_p(d_dst),
                                        C.c_void_p(d_w) if d_w else None, n, C.byref(h))
        if rc:
            _raise(rc, lib.gpma_last_error(None).decode())
        return cls(h, lib, num_vertices)

    def __del__(self):
        if getattr(self, "h", None):
            self._lib.gpma_destroy(self.h)
            self.h = None

    def _check(self, rc):
        if rc:
            _raise(rc, self._lib.gpma_last_error(self.h).decode())

    def num_vertices(self) -> int:
        return self._nv

    def num_edges(self) -> int:
        return int(self._lib.gpma_num_edges(self.h))

    def pma(self) -> PackedMemoryArray:
        return PackedMemoryArray(_handle=self._lib.gpma_pma(self.h), _owner=self)

    def apply_batch(self, ins_src, ins_dst, ins_w, del_src, del_dst, pool=None,
                    with_touched=True) -> UpdateStats:
        """with_touched: True = touched_ranges as a list of pairs (the
        reference's vector), "array" = an (n, 2) u64 array (same fetch, no
        Python list), False = not fetched."""
        a, b, w = _u32(ins_src), _u32(ins_dst), _f64(ins_w)
        c, d = _u32(del_src), _u32(del_dst)
        st = pma_stats()
        self._check(self._lib.gpma_apply_batch(self.h, _p(a), _p(b), _p(w), len(a), _p(c), _p(d), len(c),
                                               C.byref(st)))
        if with_touched == "array":
            return UpdateStats.from_c(st, self.pma().touched_ranges_array(st.num_touched_ranges))
        return UpdateStats.from_c(st, self.pma().touched_ranges() if with_touched else None)

    def apply_batch_device(self, d_is: int, d_id: int, d_iw: int | None, ni: int, d_ds: int, d_dd: int,
                           nd: int, stats_out: pma_stats | None = None) -> UpdateStats | None:
        """stats_out: fill this raw struct instead of building an UpdateStats
        (for loops that decode the stats later: UpdateStats.from_c)."""
        # (the small-batch latency path: argtypes convert the raw addresses,
        # one stats struct per graph is reused)
        st = stats_out
        if st is None:
            st = self.__dict__.get("_dev_st")
            if st is None:
                st = self._dev_st = pma_stats()
        rc = self._lib.gpma_apply_batch_device(self.h, d_is, d_id, d_iw or None, ni, d_ds, d_dd, nd, C.byref(st))
        if rc:
            self._check(rc)
        return None if stats_out is not None else UpdateStats.from_c(st)

    def reserve_batch(self, max_updates: int):
        """Pre-size every per-batch buffer of apply_batch (gpma_reserve_batch)."""
        self._check(self._lib.gpma_reserve_batch(self.h, max_updates))

    def row_offsets(self):
        out = np.zeros(self._nv + 1, np.uint64)
        self._check(self._lib.gpma_row_offsets(self.h, _p(out)))
        return out

    def rebuild_row_offsets(self):
        self._check(self._lib.gpma_rebuild_row_offsets(self.h))

    def csr_snapshot(self):
        ne = self.num_edges()
        ro = np.zeros(self._nv + 1, np.uint64)
        col = np.zeros(max(ne, 1), np.uint32)
        val = np.zeros(max(ne, 1), np.float64)
        self._check(self._lib.gpma_csr_snapshot(self.h, _p(ro), _p(col), _p(val)))
        return ro, col[:ne], val[:ne]

    def last_timing(self, out: pma_timing | None = None) -> pma_timing:
        t = pma_timing() if out is None else out
        self._check(self._lib.gpma_last_timing(self.h, C.byref(t)))
        return t

    def timing_sum(self, reset: bool = False):
        """(summed pma_timing of the batches since the last reset, batch count)
        — gpma_timing_sum; reset starts a new sum."""
        t = pma_timing()
        n = C.c_uint64()
        self._check(self._lib.gpma_timing_sum(self.h, C.byref(t), C.byref(n), 1 if reset else 0))
        return t, n.value

    # -- read API (graph.hpp:94-126, 208-223), derived from device snapshots --
    def edge_list(self):
        """graph.hpp:208-217: (src, dst, weight) of every edge in key order."""
        ro, col, val = self.csr_snapshot()
        src = np.repeat(np.arange(self._nv, dtype=np.uint32), np.diff(ro.astype(np.int64)))
        return src, col, val

    def degree(self, v: int) -> int:
        """graph.hpp:116-120: Valid non-guard slots of row v (its guard is the
        row's last Valid slot)."""
        if not 0 <= v < self._nv:
            raise IndexError("vertex out of range")
        ro = self.row_offsets()
        return self.pma().count_valid_in(int(ro[v]), int(ro[v + 1])) - 1

    def edge_weight(self, src: int, dst: int):
        """graph.hpp:122-126: the weight, or None when the edge is absent."""
        v = self.pma().search((int(src) << 32) | int(dst))
        return None if v is None else float(np.array([v], np.uint64).view(np.float64)[0])

    def neighbors(self, v: int):
        """for_each_neighbor (graph.hpp:105-114) as arrays: (dst, weight) of row v."""
        ro = self.row_offsets()
        k, val, s = self.pma().slots()
        a, b = int(ro[v]), int(ro[v + 1])
        k, val, s = k[a:b], val[a:b], s[a:b]
        m = (s == 1) & ((k & np.uint64(0xFFFFFFFF)) != np.uint64(0xFFFFFFFF))
        return (k[m] & np.uint64(0xFFFFFFFF)).astype(np.uint32), val[m].view(np.float64)

    def guard_count(self) -> int:
        """graph.hpp:219-223"""
        k, _, s = self.pma().slots()
        return int(((s == 1) & ((k & np.uint64(0xFFFFFFFF)) == np.uint64(0xFFFFFFFF))).sum())


class RebuildCsrGraph:
    """The rebuild-the-CSR-per-batch baseline (baselines.hpp:85-181) on the
    device: the comparison point GPMA+ is measured against in the paper."""

    def __init__(self, num_vertices: int, src=(), dst=(), weights=None, device: int = 0, _handle=None):
        self._lib = load_library()
        self._nv = num_vertices
        if _handle is not None:
            self.h = _handle
            return
        s, d, w = _u32(src), _u32(dst), _f64(weights)
        self.h = C.c_void_p()
        rc = self._lib.gpma_rebuild_create(device, num_vertices, _p(s), _p(d), _p(w), len(s), C.byref(self.h))
        if rc:
            self.h = None
            _raise(rc, self._lib.gpma_rebuild_last_error(None).decode())

    @classmethod
    def from_edges_device(cls, num_vertices: int, d_src: int, d_dst: int, d_w: int | None, n: int,
                          device: int = 0) -> "RebuildCsrGraph":
        lib = load_library()
        h = C.c_void_p()
        rc = lib.gpma_rebuild_create_device(device, num_vertices, C.c_void_p(d_src), C.c_void_p(d_dst),
                                            C.c_void_p(d_w) if d_w else None, n, C.byref(h))
        if rc:
            _raise(rc, lib.gpma_rebuild_last_error(None).decode())
        return cls(num_vertices, _handle=h)

    def __del__(self):
        if getattr(self, "h", None):
            self._lib.gpma_rebuild_destroy(self.h)
            self.h = None

    def _check(self, rc):
        if rc:
            _raise(rc, self._lib.gpma_rebuild_last_error(self.h).decode())

    def num_vertices(self) -> int:
        return self._nv

    def num_edges(self) -> int:
        return int(self._lib.gpma_rebuild_num_edges(self.h))

    def apply_batch(self, ins_src, ins_dst, ins_w, del_src, del_dst) -> UpdateStats:
        a, b, w = _u32(ins_src), _u32(ins_dst), _f64(ins_w)
        c, d = _u32(del_src), _u32(del_dst)
        st = pma_stats()
        self._check(self._lib.gpma_rebuild_apply_batch(self.h, _p(a), _p(b), _p(w), len(a), _p(c), _p(d), len(c),
                                                       C.byref(st)))
        return UpdateStats.from_c(st)

    def apply_batch_device(self, d_is: int, d_id: int, d_iw: int | None, ni: int, d_ds: int, d_dd: int,
                           nd: int) -> UpdateStats:
        st = pma_stats()
        vp = C.c_void_p
        self._check(self._lib.gpma_rebuild_apply_batch_device(self.h, vp(d_is), vp(d_id), vp(d_iw) if d_iw else None,
                                                              ni, vp(d_ds), vp(d_dd), nd, C.byref(st)))
        return UpdateStats.from_c(st)

    def csr_snapshot(self):
        ne = self.num_edges()
        ro = np.zeros(self._nv + 1, np.uint64)
        col = np.zeros(max(ne, 1), np.uint32)
        val = np.zeros(max(ne, 1), np.float64)
        self._check(self._lib.gpma_rebuild_csr(self.h, _p(ro), _p(col), _p(val)))
        return ro, col[:ne], val[:ne]

    csr = csr_snapshot


_TORCH_DT = {np.uint32: "int32", np.float64: "float64", np.uint64: "int64"}


def _host_out(n: int, dtype):
    """Result vector for a device->host copy: page-locked (CUDA's caching host
    allocator, block reused once the array is dropped) so the D2H runs at
    full PCIe rate instead of through pageable staging; numpy when torch is
    absent.  No zero fill: the library writes every element."""
    try:
        import torch
        t = torch.empty(max(n, 1), dtype=getattr(torch, _TORCH_DT[dtype]), pin_memory=True)
        return t.numpy().view(dtype)[:n]
    except Exception:  # pragma: no cover - CPU-only environments
        return np.empty(n, dtype)


def bfs(g: DynamicGraph, root: int, return_reached: bool = False):
    """analytics.hpp:22-48"""
    dist = _host_out(g.num_vertices(), np.uint32)
    reached = C.c_uint64()
    g._check(g._lib.gpma_bfs(g.h, C.c_uint32(root), _p(dist), C.byref(reached)))
    return (dist, reached.value) if return_reached else dist


def connected_components(g: DynamicGraph):
    """analytics.hpp:53-82"""
    lab = _host_out(g.num_vertices(), np.uint32)
    g._check(g._lib.gpma_cc(g.h, _p(lab)))
    return lab


def pagerank(g: DynamicGraph, damping: float = 0.85, epsilon: float = 1e-3, max_iters: int = 200,
             warm_start=None) -> PageRankResult:
    """analytics.hpp:90-143"""
    if warm_start is not None and len(warm_start) != g.num_vertices():
        raise ValueError("pagerank: warm start size mismatch")
    ranks = _host_out(g.num_vertices(), np.float64)
    it = C.c_uint64()
    conv = C.c_int()
    w = _f64(warm_start)
    g._check(g._lib.gpma_pagerank(g.h, C.c_double(damping), C.c_double(epsilon), max_iters, _p(w), _p(ranks),
                                  C.byref(it), C.byref(conv)))
    return PageRankResult(ranks, it.value, bool(conv.value))


def spmv(g: DynamicGraph, x):
    """analytics.hpp:147-158"""
    if len(x) != g.num_vertices():
        raise ValueError("spmv: dimension mismatch")
    xx = _f64(x)
    y = _host_out(g.num_vertices(), np.float64)
    g._check(g._lib.gpma_spmv(g.h, _p(xx), _p(y)))
    return y


class EdgeStream:
    """Synthetic stream (generators.hpp:26-89 + streaming.hpp:58-67) built by
    the library's own generators (identical mt19937_64 draws)."""

    def __init__(self, handle, lib):
        self.h = handle
        self._lib = lib

    @staticmethod
    def _chk(lib, rc):
        if rc:
            _raise(rc, lib.gpma_stream_last_error().decode())

    @classmethod
    def rmat(cls, num_vertices, num_edges, seed=1, a=0.57, b=0.19, c=0.19, d=0.05) -> "EdgeStream":
        lib = load_library()
        h = C.c_void_p()
        cls._chk(lib, lib.gpma_stream_rmat(num_vertices, num_edges, a, b, c, d, seed, C.byref(h)))
        return cls(h, lib)

    @classmethod
    def erdos_renyi(cls, num_vertices, density, seed=1) -> "EdgeStream":
        lib = load_library()
        h = C.c_void_p()
        cls._chk(lib, lib.gpma_stream_erdos_renyi(num_vertices, C.c_double(density), seed, C.byref(h)))
        return cls(h, lib)

    @classmethod
    def from_arrays(cls, num_vertices, src, dst) -> "EdgeStream":
        lib = load_library()
        s, d = _u32(src), _u32(dst)
        h = C.c_void_p()
        cls._chk(lib, lib.gpma_stream_from_arrays(num_vertices, _p(s), _p(d), len(s), C.byref(h)))
        return cls(h, lib)

    def shuffle(self, seed) -> "EdgeStream":
        """assign_random_timestamps (streaming.hpp:58-67)."""
        self._chk(self._lib, self._lib.gpma_stream_shuffle(self.h, seed))
        return self

    def __len__(self):
        return int(self._lib.gpma_stream_size(self.h))

    @property
    def num_vertices(self):
        return int(self._lib.gpma_stream_num_vertices(self.h))

    def arrays(self):
        n = len(self)
        s = np.zeros(n, np.uint32)
        d = np.zeros(n, np.uint32)
        self._chk(self._lib, self._lib.gpma_stream_edges(self.h, _p(s), _p(d)))
        return s, d

    def __del__(self):
        if getattr(self, "h", None):
            self._lib.gpma_stream_destroy(self.h)
            self.h = None


def draw_below_sequence(seed: int, bound: int, n: int):
    """draw_below (streaming.hpp:43-50) over mt19937_64(seed)."""
    lib = load_library()
    out = np.zeros(n, np.uint64)
    EdgeStream._chk(lib, lib.gpma_draw_below_sequence(seed, bound, n, _p(out)))
    return out


class Mt19937_64:
    """A caller-owned std::mt19937_64 (streaming.hpp:129 takes one by reference)."""

    def __init__(self, seed: int):
        self._lib = load_library()
        self.h = C.c_void_p()
        EdgeStream._chk(self._lib, self._lib.gpma_rng_create(C.c_uint64(seed), C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            self._lib.gpma_rng_destroy(self.h)
            self.h = None


class SlidingWindow:
    """Device sliding window (streaming.hpp:76-123): slides return device
    offsets into the stream (inserts) and the window's deletion arrays."""

    def __init__(self, stream: EdgeStream, device: int = 0):
        from .abi import gpma_slide_t, gpma_window_info_t  # noqa: F401
        self._lib = stream._lib
        self.stream = stream
        self.h = C.c_void_p()
        EdgeStream._chk(self._lib, self._lib.gpma_window_create(stream.h, device, C.byref(self.h)))

    def info(self):
        from .abi import gpma_window_info_t
        i = gpma_window_info_t()
        self._lib.gpma_window_info(self.h, C.byref(i))
        return i

    def reserve(self, max_deletions: int):
        EdgeStream._chk(self._lib, self._lib.gpma_window_reserve(self.h, max_deletions))

    def slide(self, batch: int):
        from .abi import gpma_slide_t
        s = gpma_slide_t()
        EdgeStream._chk(self._lib, self._lib.gpma_window_slide(self.h, batch, C.byref(s)))
        return s

    def slide_explicit_random(self, batch: int, rng: "Mt19937_64"):
        """streaming.hpp:129-158: expiries drawn by `rng` (its state advances)."""
        from .abi import gpma_slide_t
        s = gpma_slide_t()
        EdgeStream._chk(self._lib, self._lib.gpma_window_slide_explicit_random(self.h, batch, rng.h, C.byref(s)))
        return s

    def window_size(self) -> int:
        return int(self._lib.gpma_window_size(self.h))

    def remaining(self) -> int:
        i = self.info()
        return int(i.stream_size - i.cursor)

    def deletions_host(self, offset: int, n: int, src=None, dst=None):
        """Copy deletions [offset, offset+n) to host arrays (pinned if given)."""
        s = np.zeros(n, np.uint32) if src is None else src
        d = np.zeros(n, np.uint32) if dst is None else dst
        EdgeStream._chk(self._lib, self._lib.gpma_window_deletions_host(self.h, offset, n, _p(s), _p(d)))
        return s, d

    def __del__(self):
        if getattr(self, "h", None):
            self._lib.gpma_window_destroy(self.h)
            self.h = None


__all__ = ["EdgeStream", "SlidingWindow", "Mt19937_64", "draw_below_sequence", "PackedMemoryArray", "DynamicGraph", "DensityProfile", "UpdateStats", "SegmentEngineConfig",
           "GraphConfig", "PageRankResult", "batch_update", "bfs", "connected_components", "pagerank", "spmv",
           "LogicError", "kUnreached", "kMinCapacity", "PMA_LAZY", "PMA_EAGER"]


# -- data-parallel primitives (primitives.hpp:21-84) on the device ----------

def _prim_check(lib, rc):
    if rc:
        _raise(rc, lib.gpma_primitives_last_error().decode())


def sort_by_key(keys, payload=None, begin_bit: int = 0, end_bit: int = 64, device: int = 0):
    """sort_by_key / sort_pairs_by_key (primitives.hpp:21-60): stable sort of
    64-bit keys by bits [begin_bit, end_bit), a u32 payload moving with its
    key.  Returns sorted copies (keys, payload or None)."""
    lib = load_library()
    k = np.array(keys, dtype=np.uint64, copy=True)
    p = None if payload is None else np.array(payload, dtype=np.uint32, copy=True)
    if p is not None and len(p) != len(k):
        raise ValueError("sort_by_key: payload size mismatch")
    _prim_check(lib, lib.gpma_sort_by_key(device, _p(k), _p(p) if p is not None else None, len(k), begin_bit,
                                          end_bit))
    return k, p


def sort_by_key_device(d_keys: int, d_payload: int | None, n: int, begin_bit: int = 0, end_bit: int = 64,
                       device: int = 0):
    """The same on device arrays (sorted in place)."""
    lib = load_library()
    _prim_check(lib, lib.gpma_sort_by_key_device(device, C.c_void_p(d_keys),
                                                 C.c_void_p(d_payload) if d_payload else None, n, begin_bit,
                                                 end_bit))


def exclusive_scan_device(d_in: int, d_out: int, n: int, device: int = 0):
    """exclusive_scan (primitives.hpp:74-84) of n u32 device values."""
    lib = load_library()
    _prim_check(lib, lib.gpma_exclusive_scan_device(device, C.c_void_p(d_in), C.c_void_p(d_out), n))
