"""ctypes binding of the in-tree C-ABI library (include/zcgraph.h).

There is deliberately no fallback: if libzcgraph_b200.so is missing or does
not load, every traversal raises.  ctypes releases the GIL for the duration
of each foreign call.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from ._build import LIB_PATH, PROBE_LIB_PATH

ZC_OK, ZC_EINVAL, ZC_ECUDA, ZC_ENOMEM, ZC_ESTATE = 0, -1, -2, -3, -4
ZC_NAIVE, ZC_MERGED, ZC_MERGED_ALIGNED, ZC_PACKED, ZC_COMPRESSED = 0, 1, 2, 3, 4
ZC_PLACE_ZEROCOPY, ZC_PLACE_UVM, ZC_PLACE_HBM, ZC_PLACE_ZEROCOPY_MANAGED = 0, 1, 2, 3
ZC_F_DIRECTED, ZC_F_REGISTER, ZC_F_UVM_PREFETCH, ZC_F_NO_VALIDATE = 1, 2, 4, 8
ABI_VERSION = 1

PLACEMENTS = {"zerocopy": ZC_PLACE_ZEROCOPY, "uvm": ZC_PLACE_UVM, "hbm": ZC_PLACE_HBM,
              "zerocopy-managed": ZC_PLACE_ZEROCOPY_MANAGED}

# every symbol include/zcgraph.h declares
EXPORTED = (
    "zc_last_error", "zc_abi_version", "zc_device_count", "zc_graph_create",
    "zc_graph_destroy", "zc_graph_host_lists", "zc_graph_info", "zc_bfs", "zc_sssp",
    "zc_cc", "zc_run_log", "zc_host_alloc", "zc_host_free", "zc_generate_rmat",
    "zc_generate_uniform", "zc_set_options", "zc_set_tuning", "zc_run_traffic",
    "zc_graph_build_log",
    "zc_run_profile", "zc_graph_evict", "zc_graph_prefetch", "zc_part_create",
    "zc_part_exchange_elem_bytes", "zc_part_begin", "zc_part_expand", "zc_part_apply",
    "zc_part_result", "zc_generate_rmat_part", "zc_pagerank", "zc_graph_multigraph",
    "zc_part_fused_init", "zc_part_fused_connect", "zc_part_fused_reset", "zc_part_fused_expand",
    "zc_graph_open_emgi", "zc_graph_build_pairs", "zc_graph_build_compressed",
    "zc_bfs_async", "zc_sssp_async", "zc_sync", "zc_graph_compressed_index",
    "zc_graph_build_in_lists", "zc_run_directions", "zc_run_link_bytes",
    "zc_part_build_in_lists", "zc_part_unvisited_in", "zc_part_frontier_bits", "zc_part_pull",
    "zc_sssp_nearfar", "zc_cc_afforest", "zc_part_bitmap_init", "zc_part_bitmap_connect",
    "zc_part_bitmap_expand", "zc_part_bitmap_apply",
)
# every symbol include/zcprobe.h declares (the measurement tool library)
PROBE_EXPORTED = ("zc_link_probe", "zc_read_probe", "zc_bulk_probe", "zc_vmm_host_probe",
                  "zc_pin_probe", "zc_gather_probe")
ZC_OPT_TRAFFIC_MODEL, ZC_OPT_HOST_LOOP = 1, 2


class GraphDesc(C.Structure):
    _fields_ = [
        ("num_vertices", C.c_uint64), ("num_edges", C.c_uint64),
        ("offsets", C.c_void_p), ("edges", C.c_void_p), ("weights", C.c_void_p),
        ("src_edge_bytes", C.c_uint32), ("src_weight_bytes", C.c_uint32),
        ("edge_elem_bytes", C.c_uint32), ("weight_elem_bytes", C.c_uint32),
        ("placement", C.c_int32), ("device", C.c_int32),
        ("flags", C.c_uint32), ("reserved", C.c_uint32),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("iterations", C.c_uint64), ("total_traversed_edges", C.c_uint64),
        ("max_frontier", C.c_uint64), ("kernel_ms", C.c_double), ("total_ms", C.c_double),
        ("d2h_ms", C.c_double), ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
        ("launches", C.c_uint64), ("expand_ms", C.c_double), ("exchange_bytes", C.c_uint64),
        ("reserved", C.c_uint64 * 5),
    ]


class PartInfo(C.Structure):
    _fields_ = [("global_vertices", C.c_uint64), ("stride", C.c_uint64),
                ("bounds", C.c_void_p), ("nparts", C.c_uint32), ("part", C.c_uint32)]


_lib = None
_lock = threading.Lock()


class NativeLibraryError(RuntimeError):
    pass


def _declare(lib: C.CDLL) -> None:
    P, u64, u32, i32, i64, dbl = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int32, C.c_int64, C.c_double
    sig = {
        "zc_last_error": (C.c_char_p, []),
        "zc_abi_version": (C.c_int, []),
        "zc_device_count": (C.c_int, [C.POINTER(C.c_int)]),
        "zc_graph_create": (C.c_int, [C.POINTER(GraphDesc), C.POINTER(P)]),
        "zc_graph_destroy": (None, [P]),
        "zc_graph_open_emgi": (C.c_int, [C.c_char_p, i32, i32, u32, C.POINTER(P)]),
        "zc_graph_host_lists": (C.c_int, [P, C.POINTER(P), C.POINTER(P), C.POINTER(P)]),
        "zc_graph_info": (C.c_int, [P, C.POINTER(u64), C.POINTER(u64), C.POINTER(u32),
                                    C.POINTER(u32), C.POINTER(i32), C.POINTER(u32)]),
        "zc_bfs": (C.c_int, [P, u64, C.c_int, P, C.POINTER(Stats)]),
        "zc_sssp": (C.c_int, [P, u64, C.c_int, P, C.POINTER(Stats)]),
        "zc_cc": (C.c_int, [P, C.c_int, P, C.POINTER(Stats)]),
        "zc_sssp_nearfar": (C.c_int, [P, u64, C.c_int, u64, P, C.POINTER(Stats)]),
        "zc_cc_afforest": (C.c_int, [P, C.c_int, P, C.POINTER(Stats)]),
        "zc_bfs_async": (C.c_int, [P, u64, C.c_int, P, C.POINTER(Stats)]),
        "zc_sssp_async": (C.c_int, [P, u64, C.c_int, P, C.POINTER(Stats)]),
        "zc_sync": (C.c_int, [P]),
        "zc_pagerank": (C.c_int, [P, C.c_int, dbl, u64, dbl, P, C.POINTER(Stats)]),
        "zc_graph_multigraph": (C.c_int, [P, C.POINTER(C.c_int)]),
        "zc_graph_build_pairs": (C.c_int, [P]),
        "zc_graph_build_compressed": (C.c_int, [P, C.POINTER(u64)]),
        "zc_graph_compressed_index": (C.c_int, [P, C.c_void_p]),
        "zc_graph_build_in_lists": (C.c_int, [P, C.POINTER(u64)]),
        "zc_run_directions": (C.c_int, [P, C.c_void_p, u64]),
        "zc_run_link_bytes": (C.c_int, [P, C.POINTER(u64)]),
        "zc_part_build_in_lists": (C.c_int, [P, C.POINTER(u64)]),
        "zc_part_unvisited_in": (C.c_int, [P, C.POINTER(u64)]),
        "zc_part_frontier_bits": (C.c_int, [P, C.c_void_p]),
        "zc_part_pull": (C.c_int, [P, C.c_void_p, C.POINTER(u64), C.POINTER(u64)]),
        "zc_run_log": (C.c_int, [P, P, P, u64]),
        "zc_set_options": (C.c_int, [P, u32]),
        "zc_graph_build_log": (C.c_int, [P, C.c_char_p, C.c_size_t]),
        "zc_set_tuning": (C.c_int, [P, C.c_char_p]),
        "zc_run_profile": (C.c_int, [P, P, u64]),
        "zc_graph_evict": (C.c_int, [P]),
        "zc_graph_prefetch": (C.c_int, [P, C.POINTER(C.c_float)]),
        "zc_run_traffic": (C.c_int, [P, P, u64]),
        "zc_host_alloc": (P, [C.c_size_t]),
        "zc_host_free": (None, [P]),
        "zc_generate_rmat": (C.c_int, [u32, u32, dbl, dbl, dbl, u64, C.c_int, i64, i64, i32,
                                       i32, C.POINTER(P)]),
        "zc_generate_uniform": (C.c_int, [u64, u32, u32, u64, i64, i64, i32, i32,
                                          C.POINTER(P)]),
        "zc_part_create": (C.c_int, [C.POINTER(GraphDesc), C.POINTER(PartInfo), C.POINTER(P)]),
        "zc_part_exchange_elem_bytes": (C.c_size_t, [C.c_int]),
        "zc_part_begin": (C.c_int, [P, C.c_int, u64, C.c_int, C.POINTER(u64), C.POINTER(u64)]),
        "zc_part_expand": (C.c_int, [P, P]),
        "zc_part_apply": (C.c_int, [P, P, C.POINTER(u64), C.POINTER(u64)]),
        "zc_part_result": (C.c_int, [P, P, C.POINTER(Stats)]),
        "zc_part_fused_init": (C.c_int, [P, C.c_int, P, C.POINTER(P)]),
        "zc_part_fused_connect": (C.c_int, [P, P, P]),
        "zc_part_fused_reset": (C.c_int, [P]),
        "zc_part_fused_expand": (C.c_int, [P]),
        "zc_part_bitmap_init": (C.c_int, [P, P, C.POINTER(P)]),
        "zc_part_bitmap_connect": (C.c_int, [P, P, P]),
        "zc_part_bitmap_expand": (C.c_int, [P]),
        "zc_part_bitmap_apply": (C.c_int, [P, C.POINTER(u64), C.POINTER(u64)]),
        "zc_generate_rmat_part": (C.c_int, [u32, u32, dbl, dbl, dbl, u64, C.c_int, i64, i64, u32, u32,
                                            i32, i32, P, C.POINTER(P)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib() -> C.CDLL:
    """Load (once) the in-tree library; raise loudly if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryError(
                    f"{LIB_PATH} is missing: build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)")
            try:
                handle = C.CDLL(LIB_PATH)
            except OSError as exc:
                raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
            _declare(handle)
            if handle.zc_abi_version() != ABI_VERSION:
                raise NativeLibraryError("zcgraph ABI version mismatch; rebuild the library")
            _lib = handle
    return _lib


_probe = None


def probe_lib() -> C.CDLL:
    """Load (once) the probe tool library (include/zcprobe.h)."""
    global _probe
    if _probe is not None:
        return _probe
    lib()  # the probes report errors through the product library's zc_last_error
    with _lock:
        if _probe is None:
            try:
                handle = C.CDLL(PROBE_LIB_PATH)
            except OSError as exc:
                raise NativeLibraryError(f"cannot load {PROBE_LIB_PATH}: {exc}") from exc
            P, u64, u32, i32, dbl = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int32, C.c_double
            sig = {
                "zc_link_probe": (C.c_int, [i32, u64, C.c_int, C.POINTER(dbl), C.POINTER(dbl),
                                            C.POINTER(dbl)]),
                "zc_read_probe": (C.c_int, [i32, u64, C.c_int, u32, C.c_int, C.c_int,
                                            C.POINTER(dbl)]),
                "zc_bulk_probe": (C.c_int, [i32, u64, u32, C.c_int, C.c_int, C.POINTER(dbl)]),
                "zc_pin_probe": (C.c_int, [u64, C.c_int, C.c_int, C.POINTER(dbl), C.POINTER(dbl)]),
                "zc_gather_probe": (C.c_int, [i32, u64, C.c_int, C.POINTER(dbl)]),
                "zc_vmm_host_probe": (C.c_int, [i32, u64, C.POINTER(u64)]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _probe = handle
    return _probe


def last_error() -> str:
    msg = lib().zc_last_error()
    return msg.decode() if msg else ""


def check(rc: int) -> None:
    """Map a ZC_* status to the reference's exception types."""
    if rc == ZC_OK:
        return
    msg = last_error()
    if rc == ZC_EINVAL:
        raise ValueError(msg)
    if rc == ZC_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"zcgraph error {rc}: {msg}")
