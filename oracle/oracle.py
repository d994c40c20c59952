"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY (the checker, never the product).

ctypes front-ends for
  * ``Ref*``  — the UNMODIFIED reference (oracle/_ref/libpmagraph_ref.so,
                built by oracle/Makefile from /root/reference/proj/include);
  * ``Port*`` — our plain-C restatement (oracle/_ref/libpmaport.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_1709_05061_b200.abi import (PMA_MAX_LEVELS, engine_config, gpma_graph_config, graph_config,
                                       pma_engine_config, pma_layout_info, pma_profile, pma_stats,
                                       stats_dict)

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libpmagraph_ref.so")
PORT_SO = os.path.join(HERE, "_ref", "libpmaport.so")
REF_INCLUDE = os.environ.get("PMAGRAPH_REF_INCLUDE", "/root/reference/proj/include")


def build(force: bool = False) -> None:
    """Build the checkers (make -C oracle).  The reference .so is only built
    where /root/reference exists; on the GPU box the prebuilt one is used."""
    if force or not os.path.exists(PORT_SO) or (os.path.isdir(REF_INCLUDE) and not os.path.exists(REF_SO)):
        subprocess.check_call(["make", "-C", HERE, f"REF_INCLUDE={REF_INCLUDE}"])


def have_ref() -> bool:
    return os.path.exists(REF_SO)


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


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


_ref = None
_port = None


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"reference oracle not built at {REF_SO}")
        _ref = C.CDLL(REF_SO)
        _ref.ref_last_error.restype = C.c_char_p
        for n in ("ref_stream_size", "ref_stream_num_vertices", "ref_window_size", "ref_window_remaining",
                  "ref_graph_num_edges", "ref_rebuild_num_edges"):
            getattr(_ref, n).restype = C.c_uint64
        _ref.ref_hardware_concurrency.restype = C.c_uint
    return _ref


def port_lib():
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            raise RuntimeError(f"port oracle not built at {PORT_SO}")
        _port = C.CDLL(PORT_SO)
        _port.port_last_error.restype = C.c_char_p
        _port.port_graph_pma.restype = C.c_void_p
    return _port


def _check(lib, rc, errfn):
    if rc != 0:
        raise OracleError(rc, getattr(lib, errfn)().decode())


# ---------------------------------------------------------------- PMA side --

class _PmaBase:
    """Shared numpy front-end; subclasses bind the prefix (ref_/port_)."""
    prefix = ""
    errfn = ""

    def _lib(self):
        raise NotImplementedError

    def _call(self, name, *args):
        lib = self._lib()
        _check(lib, getattr(lib, self.prefix + name)(*args), self.errfn)

    def from_sorted(self, keys, values, fill_target):
        k, v = _u64(keys), _u64(values)
        self._call("pma_from_sorted", self.h, _p(k), _p(v), C.c_size_t(len(k)), C.c_double(fill_target))
        return self

    def load_slots(self, keys, values, states):
        k, v, s = _u64(keys), _u64(values), _u8(states)
        self._call("pma_load_slots", self.h, C.c_size_t(len(s)), _p(k), _p(v), _p(s))
        return self

    def layout(self):
        li = pma_layout_info()
        self._call("pma_get_layout", self.h, C.byref(li))
        return li

    def slots(self):
        cap = self.layout().capacity
        k = np.zeros(cap, np.uint64)
        v = np.zeros(cap, np.uint64)
        s = np.zeros(cap, np.uint8)
        self._call("pma_download", self.h, _p(k), _p(v), _p(s))
        return k, v, s

    def batch_update(self, keys, values, ops, cfg: pma_engine_config | None = None):
        k, v, o = _u64(keys), _u64(values), _u8(ops)
        st = pma_stats()
        cfg = cfg or engine_config()
        self._call("pma_batch_update", self.h, _p(k), _p(v), _p(o), C.c_size_t(len(k)), C.byref(cfg),
                   C.byref(st))
        return st

    def touched_ranges(self):
        n = C.c_size_t(0)
        self._call("pma_touched_ranges", self.h, None, C.c_size_t(0), C.byref(n))
        out = np.zeros(2 * max(n.value, 1), np.uint64)
        self._call("pma_touched_ranges", self.h, _p(out), C.c_size_t(n.value), C.byref(n))
        return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(n.value)]

    def binary_search_leaf(self, keys):
        k = _u64(keys)
        out = np.zeros(len(k), np.uint64)
        self._call("pma_binary_search_leaf", self.h, _p(k), C.c_size_t(len(k)), _p(out))
        return out


class RefPMA(_PmaBase):
    prefix, errfn = "ref_", "ref_last_error"

    def _lib(self):
        return ref_lib()

    def __init__(self, profile: pma_profile | None = None):
        self.h = C.c_void_p()
        self._call("pma_create", C.byref(profile) if profile else None, C.byref(self.h))

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_pma_destroy(self.h)
            self.h = None

    def bounds(self, level):
        mn, mx, rho, tau = C.c_uint64(), C.c_uint64(), C.c_double(), C.c_double()
        self._call("pma_bounds", self.h, C.c_int(level), C.byref(mn), C.byref(mx), C.byref(rho), C.byref(tau))
        return mn.value, mx.value, rho.value, tau.value

    def insert(self, key, value):
        self._call("pma_insert", self.h, C.c_uint64(key), C.c_uint64(value))

    def erase(self, key):
        r = C.c_int()
        self._call("pma_erase", self.h, C.c_uint64(key), C.byref(r))
        return bool(r.value)

    def mark_tombstone(self, key):
        r = C.c_int()
        self._call("pma_mark_tombstone", self.h, C.c_uint64(key), C.byref(r))
        return bool(r.value)

    def redispatch(self, level, seg, keys, values):
        k, v = _u64(keys), _u64(values)
        self._call("pma_redispatch", self.h, C.c_int(level), C.c_size_t(seg), _p(k), _p(v), C.c_size_t(len(k)))

    def search(self, keys):
        k = _u64(keys)
        vals = np.zeros(len(k), np.uint64)
        found = np.zeros(len(k), np.uint8)
        self._call("pma_search", self.h, _p(k), C.c_size_t(len(k)), _p(vals), _p(found))
        return vals, found

    def count_valid_in(self, b, e):
        c = C.c_uint64()
        self._call("pma_count_valid_in", self.h, C.c_size_t(b), C.c_size_t(e), C.byref(c))
        return c.value

    def assign_leaves_sorted(self, keys):
        k = _u64(keys)
        out = np.zeros(len(k), np.uint64)
        self._call("pma_assign_leaves_sorted", self.h, _p(k), C.c_size_t(len(k)), _p(out))
        return out


class PortPMA(_PmaBase):
    prefix, errfn = "port_", "port_last_error"

    def _lib(self):
        return port_lib()

    def __init__(self, profile: pma_profile | None = None, handle=None):
        self.owned = handle is None
        if handle is None:
            self.h = C.c_void_p()
            self._call("pma_create", C.byref(profile) if profile else None, C.byref(self.h))
        else:
            self.h = C.c_void_p(handle)

    def __del__(self):
        if getattr(self, "owned", False) and getattr(self, "h", None) and _port is not None:
            _port.port_pma_destroy(self.h)
            self.h = None


# -------------------------------------------------------------- graph side --

class _GraphBase:
    prefix = ""
    errfn = ""

    def _lib(self):
        raise NotImplementedError

    def _call(self, name, *args):
        lib = self._lib()
        _check(lib, getattr(lib, self.prefix + name)(*args), self.errfn)

    def _create(self, nv, src, dst, w, cfg):
        self.nv = nv
        s, d, ww = _u32(src), _u32(dst), _f64(w)
        self.h = C.c_void_p()
        cfg = cfg or graph_config()
        self._call("graph_from_edges", C.byref(cfg), C.c_size_t(nv), _p(s), _p(d), _p(ww), C.c_size_t(len(s)),
                   C.byref(self.h))

    def apply_batch(self, ins_src, ins_dst, ins_w, del_src, del_dst):
        a, b, w = _u32(ins_src), _u32(ins_dst), _f64(ins_w)
        c, d = _u32(del_src), _u32(del_dst)
        st = pma_stats()
        self._call("graph_apply_batch", self.h, _p(a), _p(b), _p(w), C.c_size_t(len(a)), _p(c), _p(d),
                   C.c_size_t(len(c)), C.byref(st))
        return st

    def row_offsets(self):
        out = np.zeros(self.nv + 1, np.uint64)
        self._call("graph_row_offsets", self.h, _p(out))
        return out

    def bfs(self, root):
        dist = np.zeros(self.nv, np.uint32)
        if self.prefix == "ref_":
            self._call("bfs", self.h, C.c_uint32(root), _p(dist), None)
        else:
            self._call("bfs", self.h, C.c_uint32(root), _p(dist))
        return dist

    def cc(self):
        lab = np.zeros(self.nv, np.uint32)
        if self.prefix == "ref_":
            self._call("cc", self.h, _p(lab), None)
        else:
            self._call("cc", self.h, _p(lab))
        return lab

    def pagerank(self, damping=0.85, epsilon=1e-3, max_iters=200, warm=None):
        ranks = np.zeros(self.nv, np.float64)
        it = C.c_uint64()
        conv = C.c_int()
        w = _f64(warm)
        extra = (None,) if self.prefix == "ref_" else ()
        self._call("pagerank", self.h, C.c_double(damping), C.c_double(epsilon), C.c_size_t(max_iters), _p(w),
                   _p(ranks), C.byref(it), C.byref(conv), *extra)
        return ranks, it.value, bool(conv.value)

    def spmv(self, x):
        xx = _f64(x)
        y = np.zeros(self.nv, np.float64)
        self._call("spmv", self.h, _p(xx), _p(y))
        return y


class RefGraph(_GraphBase):
    prefix, errfn = "ref_", "ref_last_error"

    def _lib(self):
        return ref_lib()

    def __init__(self, nv, src, dst, w=None, cfg: gpma_graph_config | None = None):
        self._create(nv, src, dst, w, cfg)

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_graph_destroy(self.h)
            self.h = None

    def layout(self):
        li = pma_layout_info()
        self._call("graph_layout", self.h, C.byref(li))
        return li

    def slots(self):
        cap = self.layout().capacity
        k = np.zeros(cap, np.uint64)
        v = np.zeros(cap, np.uint64)
        s = np.zeros(cap, np.uint8)
        self._call("graph_download", self.h, _p(k), _p(v), _p(s))
        return k, v, s

    def touched_ranges(self):
        n = C.c_size_t(0)
        self._call("graph_touched_ranges", self.h, None, C.c_size_t(0), C.byref(n))
        out = np.zeros(2 * max(n.value, 1), np.uint64)
        self._call("graph_touched_ranges", self.h, _p(out), C.c_size_t(n.value), C.byref(n))
        return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(n.value)]

    def num_edges(self):
        return int(ref_lib().ref_graph_num_edges(self.h))

    def csr_snapshot(self):
        ne = self.num_edges()
        ro = np.zeros(self.nv + 1, np.uint64)
        col = np.zeros(max(ne, 1), np.uint32)
        val = np.zeros(max(ne, 1), np.float64)
        self._call("graph_csr_snapshot", self.h, _p(ro), _p(col), _p(val))
        return ro, col[:ne], val[:ne]

    def apply_batch_timed(self, ins_src, ins_dst, ins_w, del_src, del_dst, workers):
        a, b, w = _u32(ins_src), _u32(ins_dst), _f64(ins_w)
        c, d = _u32(del_src), _u32(del_dst)
        st = pma_stats()
        ms = C.c_double()
        self._call("graph_apply_batch_timed", self.h, _p(a), _p(b), _p(w), C.c_size_t(len(a)), _p(c), _p(d),
                   C.c_size_t(len(c)), C.c_uint(workers), C.byref(st), C.byref(ms))
        return st, ms.value

    def timed_bfs(self, root):
        dist = np.zeros(self.nv, np.uint32)
        ms = C.c_double()
        self._call("bfs", self.h, C.c_uint32(root), _p(dist), C.byref(ms))
        return dist, ms.value


class PortGraph(_GraphBase):
    prefix, errfn = "port_", "port_last_error"

    def _lib(self):
        return port_lib()

    def __init__(self, nv, src, dst, w=None, cfg: gpma_graph_config | None = None):
        self._create(nv, src, dst, w, cfg)

    def __del__(self):
        if getattr(self, "h", None) and _port is not None:
            _port.port_graph_destroy(self.h)
            self.h = None

    def pma(self):
        return PortPMA(handle=port_lib().port_graph_pma(self.h))


# ---------------------------------------------------------------- streams --

class RefStream:
    """EdgeStream from the reference generators (generators.hpp, streaming.hpp)."""

    def __init__(self, handle):
        self.h = handle

    @classmethod
    def rmat(cls, nv, ne, seed=1, a=0.57, b=0.19, c=0.19, d=0.05):
        h = C.c_void_p()
        _check(ref_lib(), ref_lib().ref_gen_rmat(C.c_size_t(nv), C.c_size_t(ne), C.c_double(a), C.c_double(b),
                                                 C.c_double(c), C.c_double(d), C.c_uint64(seed), C.byref(h)),
               "ref_last_error")
        return cls(h)

    @classmethod
    def erdos_renyi(cls, nv, p, seed=1):
        h = C.c_void_p()
        _check(ref_lib(), ref_lib().ref_gen_erdos_renyi(C.c_size_t(nv), C.c_double(p), C.c_uint64(seed),
                                                        C.byref(h)), "ref_last_error")
        return cls(h)

    @classmethod
    def from_arrays(cls, nv, src, dst, w=None):
        s, d, ww = _u32(src), _u32(dst), _f64(w)
        h = C.c_void_p()
        _check(ref_lib(), ref_lib().ref_stream_from_arrays(C.c_size_t(nv), _p(s), _p(d), _p(ww),
                                                           C.c_size_t(len(s)), C.byref(h)), "ref_last_error")
        return cls(h)

    def shuffle(self, seed):
        _check(ref_lib(), ref_lib().ref_stream_shuffle(self.h, C.c_uint64(seed)), "ref_last_error")
        return self

    def __len__(self):
        return int(ref_lib().ref_stream_size(self.h))

    @property
    def num_vertices(self):
        return int(ref_lib().ref_stream_num_vertices(self.h))

    def arrays(self):
        n = len(self)
        s = np.zeros(n, np.uint32)
        d = np.zeros(n, np.uint32)
        w = np.zeros(n, np.float64)
        ts = np.zeros(n, np.uint64)
        _check(ref_lib(), ref_lib().ref_stream_edges(self.h, _p(s), _p(d), _p(w), _p(ts)), "ref_last_error")
        return s, d, w, ts

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_stream_destroy(self.h)
            self.h = None


class RefWindow:
    """SlidingWindow (streaming.hpp:76-193) over a RefStream."""

    def __init__(self, stream: RefStream):
        self.stream = stream
        self.h = C.c_void_p()
        _check(ref_lib(), ref_lib().ref_window_create(stream.h, C.byref(self.h)), "ref_last_error")

    def slide(self, batch):
        ni, nd = C.c_uint64(), C.c_uint64()
        _check(ref_lib(), ref_lib().ref_window_slide(self.h, C.c_size_t(batch), C.byref(ni), C.byref(nd)),
               "ref_last_error")
        a = np.zeros(ni.value, np.uint32)
        b = np.zeros(ni.value, np.uint32)
        w = np.zeros(ni.value, np.float64)
        c = np.zeros(nd.value, np.uint32)
        d = np.zeros(nd.value, np.uint32)
        _check(ref_lib(), ref_lib().ref_window_last(self.h, _p(a), _p(b), _p(w), _p(c), _p(d)), "ref_last_error")
        return a, b, w, c, d

    def slide_explicit_random(self, batch, rng: "RefRng"):
        """streaming.hpp:129-158 (rng state advances across calls)"""
        ni, nd = C.c_uint64(), C.c_uint64()
        _check(ref_lib(), ref_lib().ref_window_slide_explicit_random(self.h, C.c_size_t(batch), rng.h, C.byref(ni),
                                                                     C.byref(nd)), "ref_last_error")
        return self._last(ni.value, nd.value)

    def _last(self, ni, nd):
        a, b, w = np.zeros(ni, np.uint32), np.zeros(ni, np.uint32), np.zeros(ni, np.float64)
        c, d = np.zeros(nd, np.uint32), np.zeros(nd, np.uint32)
        _check(ref_lib(), ref_lib().ref_window_last(self.h, _p(a), _p(b), _p(w), _p(c), _p(d)), "ref_last_error")
        return a, b, w, c, d

    def remaining(self):
        return int(ref_lib().ref_window_remaining(self.h))

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_window_destroy(self.h)
            self.h = None


class RefRng:
    """std::mt19937_64(seed) owned by the caller (streaming.hpp:129)."""

    def __init__(self, seed):
        self.h = C.c_void_p()
        _check(ref_lib(), ref_lib().ref_rng_create(C.c_uint64(seed), C.byref(self.h)), "ref_last_error")

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_rng_destroy(self.h)
            self.h = None


def draw_below_sequence(seed, bound, n):
    out = np.zeros(n, np.uint64)
    _check(ref_lib(), ref_lib().ref_draw_below_sequence(C.c_uint64(seed), C.c_uint64(bound), C.c_size_t(n),
                                                        _p(out)), "ref_last_error")
    return out


def hardware_concurrency():
    return int(ref_lib().ref_hardware_concurrency())


__all__ = ["RefPMA", "PortPMA", "RefGraph", "PortGraph", "RefStream", "RefWindow", "RefRng", "OracleError", "build",
           "have_ref", "stats_dict", "draw_below_sequence", "hardware_concurrency", "PMA_MAX_LEVELS"]


class RefRebuildCsr:
    """The reference RebuildCsrGraph (baselines.hpp:85-181) — test oracle of
    the GPU rebuild-CSR baseline."""

    def __init__(self, nv, src, dst, w=None):
        self.nv = nv
        s, d, ww = _u32(src), _u32(dst), _f64(w)
        self.h = C.c_void_p()
        _check(ref_lib(), ref_lib().ref_rebuild_create(C.c_size_t(nv), _p(s), _p(d), _p(ww), C.c_size_t(len(s)),
                                                      C.byref(self.h)), "ref_last_error")

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_rebuild_destroy(self.h)
            self.h = None

    def apply_batch(self, ins_src, ins_dst, ins_w, del_src, del_dst):
        a, b, w = _u32(ins_src), _u32(ins_dst), _f64(ins_w)
        c, d = _u32(del_src), _u32(del_dst)
        st = pma_stats()
        _check(ref_lib(), ref_lib().ref_rebuild_apply_batch(self.h, _p(a), _p(b), _p(w), C.c_size_t(len(a)), _p(c),
                                                           _p(d), C.c_size_t(len(c)), C.byref(st)), "ref_last_error")
        return st

    def csr(self):
        ne = int(ref_lib().ref_rebuild_num_edges(self.h))
        ro = np.zeros(self.nv + 1, np.uint64)
        col = np.zeros(max(ne, 1), np.uint32)
        val = np.zeros(max(ne, 1), np.float64)
        _check(ref_lib(), ref_lib().ref_rebuild_csr(self.h, _p(ro), _p(col), _p(val)), "ref_last_error")
        return ro, col[:ne], val[:ne]


class RefIO:
    """The reference's file formats (io.hpp:24-181) — test oracle of
    paper_1709_05061_b200.io (byte-identical files, identical parses)."""

    @staticmethod
    def format_double(v: float) -> str:
        buf = C.create_string_buffer(64)
        _check(ref_lib(), ref_lib().ref_io_format_double(C.c_double(v), buf, C.c_size_t(64)), "ref_last_error")
        return buf.value.decode()

    @staticmethod
    def write_pairs(path, keys, values, text=False):
        k, v = np.ascontiguousarray(keys, np.uint64), np.ascontiguousarray(values, np.uint64)
        _check(ref_lib(), ref_lib().ref_io_write_pairs(str(path).encode(), int(text), _p(k), _p(v),
                                                       C.c_size_t(len(k))), "ref_last_error")

    @staticmethod
    def read_pairs(path, text=False):
        n = C.c_uint64()
        _check(ref_lib(), ref_lib().ref_io_read_pairs(str(path).encode(), int(text), C.byref(n)), "ref_last_error")
        k = np.zeros(max(n.value, 1), np.uint64)
        v = np.zeros(max(n.value, 1), np.uint64)
        _check(ref_lib(), ref_lib().ref_io_pairs_copy(_p(k), _p(v)), "ref_last_error")
        return k[:n.value], v[:n.value]

    @staticmethod
    def write_stream(path, nv, src, dst, w, ts, text=False):
        s, d = _u32(src), _u32(dst)
        ww, t = _f64(w), np.ascontiguousarray(ts, np.uint64)
        _check(ref_lib(), ref_lib().ref_io_write_stream(str(path).encode(), int(text), C.c_size_t(nv), _p(s), _p(d),
                                                        _p(ww), _p(t), C.c_size_t(len(s))), "ref_last_error")

    @staticmethod
    def read_stream(path, mode=0):
        """mode 0 read_stream (format probe), 1 text, 2 binary -> (nv, src, dst, w, ts)"""
        nv, n = C.c_uint64(), C.c_uint64()
        _check(ref_lib(), ref_lib().ref_io_read_stream(str(path).encode(), mode, C.byref(nv), C.byref(n)),
               "ref_last_error")
        m = max(n.value, 1)
        s, d = np.zeros(m, np.uint32), np.zeros(m, np.uint32)
        w, t = np.zeros(m, np.float64), np.zeros(m, np.uint64)
        _check(ref_lib(), ref_lib().ref_io_stream_copy(_p(s), _p(d), _p(w), _p(t)), "ref_last_error")
        k = n.value
        return nv.value, s[:k], d[:k], w[:k], t[:k]

    @staticmethod
    def write_vector(path, v, text=False):
        a = np.ascontiguousarray(v)
        kind = {np.dtype(np.float64): 0, np.dtype(np.uint32): 1, np.dtype(np.uint64): 2}[a.dtype]
        _check(ref_lib(), ref_lib().ref_io_write_vector(str(path).encode(), int(text), kind, _p(a),
                                                        C.c_size_t(len(a))), "ref_last_error")
