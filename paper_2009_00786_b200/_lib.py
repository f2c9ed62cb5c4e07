"""ctypes binding of the C ABI in include/tsgpu.h (libtsgpu.so, in-tree).

There is no fallback: if the library is missing or cannot find a CUDA
device, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# TSG_LIB_PATH: an alternative build of the same library (A/B timing runs).
LIB_PATH = os.environ.get("TSG_LIB_PATH") or os.path.join(PKG, "libtsgpu.so")

TSG_OK, TSG_INVALID_ARGUMENT, TSG_RUNTIME, TSG_LOGIC, TSG_CUDA, TSG_NCCL, TSG_OOM = range(7)

# Symbols declared in include/tsgpu.h (checked by tests/test_abi.py).
EXPORTS = (
    "tsg_last_error", "tsg_version", "tsg_config_default", "tsg_config_validate", "tsg_open", "tsg_close",
    "tsg_index_build", "tsg_index_build_device", "tsg_index_free", "tsg_index_info", "tsg_search",
    "tsg_search_device", "tsg_approximate_search", "tsg_summarise", "tsg_word_stride", "tsg_index_export", "tsg_index_export_fine",
    "tsg_generate_random_walk", "tsg_launch_count", "tsg_profile_enable", "tsg_profile_read",
    "tsg_generate_series", "tsg_index_build_file", "tsg_search_measure",
    "tsg_comm_unique_id", "tsg_comm_init", "tsg_comm_info", "tsg_breakpoints", "tsg_index_thresholds",
    "tsg_index_validate", "tsg_index_debug_poke",
)

TSG_TRANSPORT_NONE, TSG_TRANSPORT_LOCAL, TSG_TRANSPORT_NCCL = 0, 1, 2

TSG_MEASURE_ED, TSG_MEASURE_DTW = 0, 1


class tsg_measure(C.Structure):
    _fields_ = [("kind", C.c_int32), ("window", C.c_int32)]


class tsg_comm_id(C.Structure):
    _fields_ = [("internal", C.c_uint8 * 128)]


class tsg_config(C.Structure):
    _fields_ = [
        ("n", C.c_uint64), ("w", C.c_int32), ("max_card_bits", C.c_int32), ("leaf_capacity", C.c_uint64),
        ("chunk_size", C.c_uint64), ("n_index_workers", C.c_uint32), ("n_search_workers", C.c_uint32),
        ("n_queues", C.c_uint32), ("queue_mode", C.c_int32), ("initial_buffer_part_size", C.c_uint64),
    ]


class tsg_build_stats(C.Structure):
    _fields_ = [
        ("build_ns", C.c_uint64), ("series", C.c_uint64), ("nodes", C.c_uint64), ("inner_nodes", C.c_uint64),
        ("leaves", C.c_uint64), ("empty_leaves", C.c_uint64), ("overflow_leaves", C.c_uint64),
        ("max_depth", C.c_uint64), ("root_children", C.c_uint64), ("pages", C.c_uint64), ("h2d_ns", C.c_uint64),
        ("summarise_ms", C.c_double), ("organise_ms", C.c_double), ("leaves_ms", C.c_double),
    ]


class tsg_search_stats(C.Structure):
    _fields_ = [
        ("lb_node_calcs", C.c_uint64), ("lb_entry_calcs", C.c_uint64), ("real_dist_calcs", C.c_uint64),
        ("bsf_updates", C.c_uint64), ("pruned_subtrees", C.c_uint64), ("queue_insertions", C.c_uint64),
    ]


class tsg_validation_report(C.Structure):
    _fields_ = [
        ("nodes", C.c_uint64), ("inner_nodes", C.c_uint64), ("leaves", C.c_uint64), ("empty_leaves", C.c_uint64),
        ("overflow_leaves", C.c_uint64), ("max_depth", C.c_uint64), ("total_entries", C.c_uint64),
        ("leaf_fill_histogram", C.c_uint64 * 11), ("violation_count", C.c_uint64), ("n_violations", C.c_uint32),
        ("reserved", C.c_uint32), ("violations", (C.c_char * 160) * 20), ("pages", C.c_uint64),
        ("checked_boxes", C.c_uint64),
    ]


class tsg_result(C.Structure):
    _fields_ = [("distance", C.c_double), ("position", C.c_uint32), ("box_calcs", C.c_uint32),
                ("stats", tsg_search_stats), ("fine_calcs", C.c_uint64)]


_lib = None


def lib() -> C.CDLL:
    """Load libtsgpu.so (built in-tree by paper_2009_00786_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2009_00786_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, u64, u32, i32 = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int
    sigs = {
        "tsg_last_error": (C.c_char_p, []),
        "tsg_version": (C.c_char_p, []),
        "tsg_config_default": (None, [C.POINTER(tsg_config)]),
        "tsg_config_validate": (i32, [C.POINTER(tsg_config)]),
        "tsg_open": (i32, [i32, C.POINTER(C.c_int), C.POINTER(vp)]),
        "tsg_close": (i32, [vp]),
        "tsg_index_build": (i32, [vp, vp, u64, u64, C.POINTER(tsg_config), u64, C.POINTER(vp),
                                  C.POINTER(tsg_build_stats)]),
        "tsg_index_build_device": (i32, [vp, vp, u64, u64, C.POINTER(tsg_config), u64, C.POINTER(vp),
                                         C.POINTER(tsg_build_stats)]),
        "tsg_index_build_file": (i32, [vp, C.c_char_p, u64, C.POINTER(tsg_config), u64, C.POINTER(vp),
                                       C.POINTER(tsg_build_stats)]),
        "tsg_index_free": (i32, [vp]),
        "tsg_search_measure": (i32, [vp, vp, i32, u32, C.POINTER(tsg_measure), i32, C.POINTER(tsg_result)]),
        "tsg_index_info": (i32, [vp, C.POINTER(u64), C.POINTER(u64), C.POINTER(tsg_config),
                                 C.POINTER(tsg_build_stats)]),
        "tsg_search": (i32, [vp, vp, u32, C.POINTER(tsg_result)]),
        "tsg_search_device": (i32, [vp, vp, u32, C.POINTER(tsg_result)]),
        "tsg_approximate_search": (i32, [vp, vp, C.POINTER(tsg_result)]),
        "tsg_summarise": (i32, [vp, u64, u64, i32, i32, vp, vp, vp]),
        "tsg_word_stride": (i32, [i32]),
        "tsg_index_export": (i32, [vp, vp, vp, vp, vp, vp, vp]),
        "tsg_index_export_fine": (i32, [vp, vp, vp]),
        "tsg_generate_random_walk": (i32, [vp, u64, u64, u64, u64, i32, vp]),
        "tsg_launch_count": (u64, []),
        "tsg_generate_series": (i32, [i32, vp, u64, u64, u64, u64, i32, C.c_double, u64, u64, vp]),
        "tsg_profile_enable": (i32, [vp, i32]),
        "tsg_profile_read": (i32, [vp, C.POINTER(C.c_double), C.POINTER(u64), i32]),
        "tsg_comm_unique_id": (i32, [C.POINTER(tsg_comm_id)]),
        "tsg_comm_init": (i32, [vp, i32, i32, C.POINTER(tsg_comm_id)]),
        "tsg_comm_info": (i32, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
        "tsg_breakpoints": (i32, [i32, vp]),
        "tsg_index_thresholds": (i32, [vp, vp]),
        "tsg_index_validate": (i32, [vp, C.POINTER(tsg_validation_report)]),
        "tsg_index_debug_poke": (i32, [vp, i32, u64, vp, u64]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


class TsgError(RuntimeError):
    """Device-path failure (CUDA / NCCL / OOM / runtime)."""


class InvalidArgument(ValueError):
    """What the reference throws as std::invalid_argument."""


class LogicError(RuntimeError):
    """What the reference throws as std::logic_error."""


def check(status: int) -> None:
    if status == TSG_OK:
        return
    msg = lib().tsg_last_error().decode()
    if status == TSG_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if status == TSG_LOGIC:
        raise LogicError(msg)
    if status == TSG_OOM:
        raise MemoryError(msg)
    raise TsgError(f"tsg status {status}: {msg}")
