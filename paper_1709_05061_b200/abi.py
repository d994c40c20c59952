"""ctypes mirror of include/pmagraph_cuda.h (the C ABI of libpmagraph_cuda.so).

Only struct layouts, constants and the library loader live here.  The
library is built in-tree (``paper_1709_05061_b200/libpmagraph_cuda.so``, see
``build.py``); importing the package on a machine without it fails loudly —
there is no CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os

PMA_OK, PMA_EINVAL, PMA_ERANGE, PMA_ELOGIC, PMA_ECUDA = 0, 1, 2, 3, 4
PMA_MAX_LEVELS = 64
PMA_LAZY, PMA_EAGER = 0, 1
PMA_STRATEGY_AUTO, PMA_STRATEGY_SMALL, PMA_STRATEGY_MEDIUM, PMA_STRATEGY_LARGE = -1, 0, 1, 2
GPMA_UNREACHED = 0xFFFFFFFF

HERE = os.path.dirname(os.path.abspath(__file__))
# GPMA_LIB: an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("GPMA_LIB") or os.path.join(HERE, "libpmagraph_cuda.so")


class pma_profile(C.Structure):
    _fields_ = [
        ("leaf_lower", C.c_double),
        ("leaf_upper", C.c_double),
        ("root_lower", C.c_double),
        ("root_upper", C.c_double),
        ("allow_shrink", C.c_int32),
        ("_pad", C.c_int32),
    ]


class pma_engine_config(C.Structure):
    _fields_ = [
        ("deletion_mode", C.c_int32),
        ("workers", C.c_uint32),
        ("small_max", C.c_uint64),
        ("medium_max", C.c_uint64),
        ("force_strategy", C.c_int32),
        ("_pad", C.c_int32),
    ]


class pma_stats(C.Structure):
    _fields_ = [
        ("batch_size", C.c_uint64),
        ("rounds", C.c_uint64),
        ("slot_writes", C.c_uint64),
        ("wall_ns", C.c_uint64),
        ("segment_phase_ns", C.c_uint64),
        ("grow_events", C.c_uint64),
        ("shrink_events", C.c_uint64),
        ("deletes_missed", C.c_uint64),
        ("tombstones_added", C.c_uint64),
        ("num_touched_ranges", C.c_uint64),
        ("resized", C.c_int32),
        ("num_levels", C.c_int32),
        ("segments_per_level", C.c_uint64 * PMA_MAX_LEVELS),
    ]


class pma_layout_info(C.Structure):
    _fields_ = [
        ("capacity", C.c_uint64),
        ("leaf_size", C.c_uint64),
        ("height", C.c_int32),
        ("_pad", C.c_int32),
        ("valid_count", C.c_uint64),
        ("tombstone_count", C.c_uint64),
        ("slot_writes", C.c_uint64),
    ]


class pma_timing(C.Structure):
    _fields_ = [
        ("device_ms", C.c_double),
        ("sort_ms", C.c_double),
        ("search_ms", C.c_double),
        ("rounds_ms", C.c_double),
        ("refresh_ms", C.c_double),
        ("kernel_launches", C.c_uint64),
        ("merge_slots", C.c_uint64),
        ("tombstone_flips", C.c_uint64),
        ("level_ms", C.c_double * 16),
        ("level_groups", C.c_uint64 * 16),
        ("level_big", C.c_uint64 * 16),
        ("level_max_slice", C.c_uint64 * 16),
        ("commit_bytes", C.c_uint64),
        ("level_bytes", C.c_uint64 * 16),
        ("front_end", C.c_uint64),
        ("grid_merges", C.c_uint64),
    ]


class gpma_graph_config(C.Structure):
    _fields_ = [
        ("engine", C.c_int32),
        ("deletion_mode", C.c_int32),
        ("workers", C.c_uint32),
        ("_pad", C.c_int32),
        ("fill_target", C.c_double),
        ("profile", pma_profile),
    ]


class gpma_window_info_t(C.Structure):
    _fields_ = [
        ("stream_src", C.c_void_p),
        ("stream_dst", C.c_void_p),
        ("del_src", C.c_void_p),
        ("del_dst", C.c_void_p),
        ("stream_size", C.c_uint64),
        ("initial_size", C.c_uint64),
        ("cursor", C.c_uint64),
        ("num_deletions", C.c_uint64),
    ]


class gpma_slide_t(C.Structure):
    _fields_ = [
        ("ins_offset", C.c_uint64),
        ("n_ins", C.c_uint64),
        ("del_offset", C.c_uint64),
        ("n_del", C.c_uint64),
        ("final_partial", C.c_int32),
        ("_pad", C.c_int32),
    ]


def default_profile() -> pma_profile:
    """DensityProfile defaults (pma.hpp:52-57)."""
    return pma_profile(0.08, 0.92, 0.40, 0.80, 1, 0)


def engine_config(deletion_mode: int = PMA_LAZY, workers: int = 1, small_max: int = 32,
                  medium_max: int = 1024, force_strategy: int = PMA_STRATEGY_AUTO) -> pma_engine_config:
    """SegmentEngineConfig defaults (segment_engine.hpp:43-60)."""
    return pma_engine_config(deletion_mode, workers, small_max, medium_max, force_strategy, 0)


def graph_config(deletion_mode: int = PMA_LAZY, workers: int = 1, fill_target: float = 0.5,
                 profile: pma_profile | None = None) -> gpma_graph_config:
    """GraphConfig defaults (graph.hpp:54-60)."""
    return gpma_graph_config(0, deletion_mode, workers, 0, fill_target, profile or default_profile())


def stats_dict(s: pma_stats) -> dict:
    """UpdateStats as a dict (timing fields excluded: they are not parity data)."""
    return {
        "batch_size": s.batch_size,
        "rounds": s.rounds,
        "slot_writes": s.slot_writes,
        "segments_per_level": [s.segments_per_level[i] for i in range(s.num_levels)],
        "grow_events": s.grow_events,
        "shrink_events": s.shrink_events,
        "deletes_missed": s.deletes_missed,
        "tombstones_added": s.tombstones_added,
        "num_touched_ranges": s.num_touched_ranges,
        "resized": bool(s.resized),
    }


_P = C.c_void_p
_U64P = C.POINTER(C.c_uint64)

# (name, restype, argtypes) of every exported symbol; also used by the CPU
# test that checks the built library exports exactly what the header declares.
SIGNATURES = [
    ("pma_create", C.c_int, [C.POINTER(pma_profile), C.c_int, C.POINTER(_P)]),
    ("pma_destroy", C.c_int, [_P]),
    ("pma_last_error", C.c_char_p, [_P]),
    ("pma_from_sorted", C.c_int, [_P, _P, _P, C.c_size_t, C.c_double]),
    ("pma_load_slots", C.c_int, [_P, C.c_size_t, _P, _P, _P]),
    ("pma_download", C.c_int, [_P, _P, _P, _P]),
    ("pma_get_layout", C.c_int, [_P, C.POINTER(pma_layout_info)]),
    ("pma_reset_slot_writes", C.c_int, [_P]),
    ("pma_bounds", C.c_int, [_P, C.c_int, _U64P, _U64P, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("pma_batch_update", C.c_int, [_P, _P, _P, _P, C.c_size_t, C.POINTER(pma_engine_config), C.POINTER(pma_stats)]),
    ("pma_batch_update_device", C.c_int, [_P, _P, _P, _P, C.c_size_t, C.POINTER(pma_engine_config), C.POINTER(pma_stats)]),
    ("pma_touched_ranges", C.c_int, [_P, _P, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("pma_slot_hash", C.c_int, [_P, C.c_int, _P]),
    ("pma_reserve_batch", C.c_int, [_P, C.c_size_t]),
    ("pma_set_grid_segment", C.c_int, [_P, C.c_uint64]),
    ("pma_try_insert_plus", C.c_int, [_P, C.c_int, C.c_size_t, _P, _P, _P, C.c_size_t, C.POINTER(pma_engine_config),
                                      C.POINTER(C.c_int), _U64P, _U64P]),
    ("pma_binary_search_leaf", C.c_int, [_P, _P, C.c_size_t, _P]),
    ("pma_search", C.c_int, [_P, _P, C.c_size_t, _P, _P]),
    ("pma_count_valid_in", C.c_int, [_P, C.c_size_t, C.c_size_t, _U64P]),
    ("pma_insert", C.c_int, [_P, C.c_uint64, C.c_uint64]),
    ("pma_erase", C.c_int, [_P, C.c_uint64, C.POINTER(C.c_int)]),
    ("pma_mark_tombstone", C.c_int, [_P, C.c_uint64, C.POINTER(C.c_int)]),
    ("pma_redispatch", C.c_int, [_P, C.c_int, C.c_size_t, _P, _P, C.c_size_t]),
    ("pma_last_timing", C.c_int, [_P, C.POINTER(pma_timing)]),
    ("gpma_from_edges", C.c_int, [C.POINTER(gpma_graph_config), C.c_int, C.c_size_t, _P, _P, _P, C.c_size_t, C.POINTER(_P)]),
    ("gpma_from_edges_device", C.c_int, [C.POINTER(gpma_graph_config), C.c_int, C.c_size_t, _P, _P, _P, C.c_size_t, C.POINTER(_P)]),
    ("gpma_destroy", C.c_int, [_P]),
    ("gpma_last_error", C.c_char_p, [_P]),
    ("gpma_pma", _P, [_P]),
    ("gpma_num_vertices", C.c_uint64, [_P]),
    ("gpma_num_edges", C.c_uint64, [_P]),
    ("gpma_apply_batch", C.c_int, [_P, _P, _P, _P, C.c_size_t, _P, _P, C.c_size_t, C.POINTER(pma_stats)]),
    ("gpma_apply_batch_device", C.c_int, [_P, _P, _P, _P, C.c_size_t, _P, _P, C.c_size_t, C.POINTER(pma_stats)]),
    ("gpma_reserve_batch", C.c_int, [_P, C.c_size_t]),
    ("gpma_row_offsets", C.c_int, [_P, _P]),
    ("gpma_rebuild_row_offsets", C.c_int, [_P]),
    ("gpma_csr_snapshot", C.c_int, [_P, _P, _P, _P]),
    ("gpma_bfs", C.c_int, [_P, C.c_uint32, _P, _U64P]),
    ("gpma_cc", C.c_int, [_P, _P]),
    ("gpma_pagerank", C.c_int, [_P, C.c_double, C.c_double, C.c_size_t, _P, _P, _U64P, C.POINTER(C.c_int)]),
    ("gpma_spmv", C.c_int, [_P, _P, _P]),
    ("gpma_last_timing", C.c_int, [_P, C.POINTER(pma_timing)]),
    ("gpma_timing_sum", C.c_int, [_P, C.POINTER(pma_timing), C.POINTER(C.c_uint64), C.c_int]),
    ("gpma_cuda_stream", _P, [_P]),
    ("pma_cuda_stream", _P, [_P]),
    ("gpma_shard_from_edges_device", C.c_int, [C.POINTER(gpma_graph_config), C.c_int, C.c_size_t, C.c_uint32, C.c_uint32, _P, _P, _P, C.c_size_t, C.POINTER(_P)]),
    ("gpma_shard_range", C.c_int, [_P, _U64P, _U64P]),
    ("gpma_route_batch", C.c_int, [_P, _P, _P, _P, C.c_size_t, _P, _P, C.c_size_t, _P, C.c_int, _P, _P, _U64P]),
    ("gpma_apply_batch_routed_device", C.c_int, [_P, _P, _P, C.c_size_t, C.POINTER(pma_stats)]),
    ("gpma_route_batch_async", C.c_int, [_P, _P, _P, _P, C.c_size_t, _P, _P, C.c_size_t, _P, C.c_int, _P, _P, _P]),
    ("gpma_set_stream", C.c_int, [_P, _P, C.c_int]),
    ("gpma_route_count", C.c_int, [_P, _P, _P, C.c_size_t, _P, _P, C.c_size_t, _P, C.c_int, _P]),
    ("gpma_route_scatter_peer", C.c_int, [_P, _P, _P, _P, C.c_size_t, _P, _P, C.c_size_t, _P, C.c_int, _P, _P, _P]),
    ("gpma_ipc_alloc", C.c_int, [C.c_int, C.c_size_t, C.POINTER(_P), _P]),
    ("gpma_ipc_open", C.c_int, [C.c_int, _P, C.POINTER(_P)]),
    ("gpma_ipc_close", C.c_int, [_P]),
    ("gpma_ipc_free", C.c_int, [_P]),
    ("gpma_shard_bfs_mark", C.c_int, [_P, _P, C.c_uint32, _P]),
    ("gpma_shard_bfs_update", C.c_int, [_P, _P, _P, C.c_uint32, _P, C.POINTER(C.c_uint32)]),
    ("gpma_shard_cc_hook", C.c_int, [_P, _P]),
    ("gpma_cc_jump", C.c_int, [_P, _P, C.c_size_t, _P, C.POINTER(C.c_int)]),
    ("gpma_shard_outdeg", C.c_int, [_P, _P]),
    ("gpma_shard_pr_push", C.c_int, [_P, _P, _P, C.c_double, _P]),
    ("gpma_pr_finish", C.c_int, [_P, _P, _P, C.c_size_t, _P, C.c_double, C.POINTER(C.c_double)]),
    ("gpma_shard_spmv", C.c_int, [_P, _P, _P]),
    ("gpma_nccl_unique_id", C.c_int, [_P]),
    ("gpma_nccl_comm_create", C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.POINTER(_P)]),
    ("gpma_nccl_comm_destroy", C.c_int, [_P]),
    ("gpma_shard_group_create", C.c_int, [C.POINTER(gpma_graph_config), C.c_int, C.c_size_t, _P, C.c_int, C.c_int,
                                          _P, _P, _P, _P, _P, C.c_size_t, C.POINTER(_P)]),
    ("gpma_shard_group_destroy", C.c_int, [_P]),
    ("gpma_shard_group_last_error", C.c_char_p, [_P]),
    ("gpma_shard_group_graph", _P, [_P]),
    ("gpma_shard_group_apply_batch", C.c_int, [_P, _P, _P, _P, C.c_size_t, _P, _P, C.c_size_t,
                                               C.POINTER(pma_stats), _U64P, _U64P]),
    ("gpma_shard_group_bfs", C.c_int, [_P, C.c_uint32, _P, _U64P]),
    ("gpma_shard_group_cc", C.c_int, [_P, _P]),
    ("gpma_shard_group_pagerank", C.c_int, [_P, C.c_double, C.c_double, C.c_size_t, _P, _P, _U64P,
                                            C.POINTER(C.c_int)]),
    ("gpma_shard_group_spmv", C.c_int, [_P, _P, _P]),
    ("gpma_warmup", C.c_int, [C.c_int]),
    ("gpma_probe_h2d", C.c_int, [C.c_int, _P, C.c_size_t, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("gpma_rebuild_create", C.c_int, [C.c_int, C.c_size_t, _P, _P, _P, C.c_size_t, C.POINTER(_P)]),
    ("gpma_rebuild_create_device", C.c_int, [C.c_int, C.c_size_t, _P, _P, _P, C.c_size_t, C.POINTER(_P)]),
    ("gpma_rebuild_destroy", C.c_int, [_P]),
    ("gpma_rebuild_last_error", C.c_char_p, [_P]),
    ("gpma_rebuild_apply_batch", C.c_int, [_P, _P, _P, _P, C.c_size_t, _P, _P, C.c_size_t, C.POINTER(pma_stats)]),
    ("gpma_rebuild_apply_batch_device", C.c_int, [_P, _P, _P, _P, C.c_size_t, _P, _P, C.c_size_t, C.POINTER(pma_stats)]),
    ("gpma_rebuild_csr", C.c_int, [_P, _P, _P, _P]),
    ("gpma_rebuild_num_edges", C.c_uint64, [_P]),
    ("gpma_rebuild_cuda_stream", _P, [_P]),
    ("gpma_sort_by_key", C.c_int, [C.c_int, _P, _P, C.c_size_t, C.c_int, C.c_int]),
    ("gpma_sort_by_key_device", C.c_int, [C.c_int, _P, _P, C.c_size_t, C.c_int, C.c_int]),
    ("gpma_exclusive_scan_device", C.c_int, [C.c_int, _P, _P, C.c_size_t]),
    ("gpma_primitives_last_error", C.c_char_p, []),
    # pmagraph_stream.h
    ("gpma_stream_last_error", C.c_char_p, []),
    ("gpma_stream_rmat", C.c_int, [C.c_size_t, C.c_size_t, C.c_double, C.c_double, C.c_double, C.c_double, C.c_uint64, C.POINTER(_P)]),
    ("gpma_stream_erdos_renyi", C.c_int, [C.c_size_t, C.c_double, C.c_uint64, C.POINTER(_P)]),
    ("gpma_stream_shuffle", C.c_int, [_P, C.c_uint64]),
    ("gpma_stream_from_arrays", C.c_int, [C.c_size_t, _P, _P, C.c_size_t, C.POINTER(_P)]),
    ("gpma_stream_size", C.c_uint64, [_P]),
    ("gpma_stream_num_vertices", C.c_uint64, [_P]),
    ("gpma_stream_edges", C.c_int, [_P, _P, _P]),
    ("gpma_stream_destroy", C.c_int, [_P]),
    ("gpma_draw_below_sequence", C.c_int, [C.c_uint64, C.c_uint64, C.c_size_t, _P]),
    ("gpma_window_create", C.c_int, [_P, C.c_int, C.POINTER(_P)]),
    ("gpma_window_destroy", C.c_int, [_P]),
    ("gpma_window_info", C.c_int, [_P, C.POINTER(gpma_window_info_t)]),
    ("gpma_window_reserve", C.c_int, [_P, C.c_size_t]),
    ("gpma_window_slide", C.c_int, [_P, C.c_size_t, C.POINTER(gpma_slide_t)]),
    ("gpma_window_deletions_host", C.c_int, [_P, C.c_size_t, C.c_size_t, _P, _P]),
    ("gpma_rng_create", C.c_int, [C.c_uint64, C.POINTER(_P)]),
    ("gpma_rng_destroy", C.c_int, [_P]),
    ("gpma_window_slide_explicit_random", C.c_int, [_P, C.c_size_t, _P, C.POINTER(gpma_slide_t)]),
    ("gpma_window_size", C.c_uint64, [_P]),
    ("gpma_window_last_expiries", C.c_int, [_P, _P, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("gpma_window_distinct_edges", C.c_int, [_P, _P, _P, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("gpma_rng_set_state", C.c_int, [_P, C.c_char_p]),
    ("gpma_rng_get_state", C.c_int, [_P, _P, C.c_size_t, C.POINTER(C.c_size_t)]),
]

_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load libpmagraph_cuda.so; raise (never fall back) when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"libpmagraph_cuda.so not built at {path}: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the product has no CPU fallback)")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
