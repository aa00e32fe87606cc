"""ctypes binding of libgraphlb_b200.so (include/graphlb_b200.h).

The shared library is the only compute path of this package: there is no CPU
fallback.  If the library is missing, :func:`lib` raises ImportError; if no
CUDA device is visible, the device calls fail with RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libgraphlb_b200.so"

GLB_OK = 0
GLB_EINVAL = 1
GLB_ERANGE = 2
GLB_ECOO_CAPACITY = 3
GLB_ECUDA = 4
GLB_ENOMEM = 5
GLB_EOVERFLOW = 6
GLB_ENODEV = 7
GLB_EPARSE = 8

GLB_BS, GLB_EP, GLB_WD, GLB_NS, GLB_HP = range(5)
GLB_TAG_WD_FALLBACK = 5
GLB_BFS, GLB_SSSP = 0, 1
GLB_LOOP_HOST, GLB_LOOP_GRAPH = 0, 1

_i32, _i64, _f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
_p64 = ctypes.POINTER(ctypes.c_int64)


class RunParams(ctypes.Structure):
    _fields_ = [
        ("strategy", _i32), ("algo", _i32), ("source", _i64), ("bins", _i32),
        ("chunked", _i32), ("mdt", _i64), ("max_cells", _i64), ("block_size", _i32),
        ("hp_fallback", _i32), ("virtual_threads", _i64), ("dist_bits", _i32),
        ("loop_mode", _i32), ("record_timing", _i32), ("instrument", _i32),
    ]


class RunStats(ctypes.Structure):
    _fields_ = [
        ("status", _i32), ("dist_bits", _i32), ("iterations", _i64), ("launches", _i64),
        ("sub_iterations", _i64), ("relax_ops", _i64), ("push_ops", _i64),
        ("edges_examined", _i64), ("active_items", _i64), ("mdt", _i64),
        ("num_split_nodes", _i64), ("num_children", _i64), ("split_fraction", _f64),
        ("device_ms", _f64), ("kernel_ms", _f64), ("overhead_ms", _f64), ("setup_ms", _f64),
        ("n_records", _i64),
    ]


class Record(ctypes.Structure):
    _fields_ = [
        ("iteration", _i32), ("sub_iteration", _i32), ("tag", _i32), ("reserved", _i32),
        ("active_items", _i64), ("threads", _i64), ("work_total", _i64), ("work_max", _i64),
        ("work_sumsq", _f64), ("relax_ops", _i64), ("push_ops", _i64), ("kernel_ms", _f64),
        ("overhead_ms", _f64), ("thread_work_offset", _i64),
    ]


class PeerStats(ctypes.Structure):
    _fields_ = [
        ("bsp_iterations", _i64), ("sent_entries", _i64), ("recv_entries", _i64),
        ("entry_bytes", _i32), ("parts", _i32), ("rank", _i32), ("transport", _i32),
        ("exchange_ms", _f64), ("wait_ms", _f64),
    ]


GLB_PEER_HANDLE_BYTES = 64
GLB_PEER_IPC, GLB_PEER_LOCAL = 1, 2

# name -> (restype, argtypes); the exported surface of include/graphlb_b200.h
SIGNATURES = {
    "glb_last_error": (ctypes.c_char_p, []),
    "glb_version": (ctypes.c_char_p, []),
    "glb_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "glb_kernel_launches": (ctypes.c_uint64, []),
    "glb_release_cached_memory": (ctypes.c_int, [ctypes.c_int, _p64]),
    "glb_graph_create": (ctypes.c_int, [_p64, _p64, _p64, _i64, _i64, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_void_p)]),
    "glb_graph_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "glb_graph_create_rmat": (ctypes.c_int, [ctypes.c_int, _i64, ctypes.c_double, ctypes.c_double,
                                             ctypes.c_double, ctypes.POINTER(ctypes.c_uint64),
                                             ctypes.POINTER(ctypes.c_uint64), ctypes.c_int, _i64,
                                             ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "glb_graph_download": (ctypes.c_int, [ctypes.c_void_p, _p64, _p64, _p64]),
    "glb_graph_download_u32": (ctypes.c_int, [ctypes.c_void_p, _p64, ctypes.POINTER(ctypes.c_uint32),
                                              ctypes.POINTER(ctypes.c_uint32)]),
    "glb_graph_partition": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _p64]),
    "glb_graph_restrict": (ctypes.c_int, [ctypes.c_void_p, _i64, _i64]),
    "glb_shard_begin": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(RunParams), _p64, ctypes.c_int,
                                       ctypes.c_int]),
    "glb_shard_local": (ctypes.c_int, [ctypes.c_void_p, _p64, ctypes.c_void_p, _i64, _p64]),
    "glb_shard_apply": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, _i64]),
    "glb_shard_advance": (ctypes.c_int, [ctypes.c_void_p, _p64]),
    "glb_shard_finish": (ctypes.c_int, [ctypes.c_void_p, _p64, ctypes.POINTER(RunStats)]),
    "glb_peer_create": (ctypes.c_int, [ctypes.c_void_p, _p64, ctypes.c_int, ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_void_p)]),
    "glb_peer_handle": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "glb_peer_connect": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "glb_peer_connect_local": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int]),
    "glb_peer_run": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(RunParams), _p64,
                                    ctypes.POINTER(RunStats), ctypes.POINTER(PeerStats)]),
    "glb_peer_run_local": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int,
                                          ctypes.POINTER(RunParams), ctypes.POINTER(_p64),
                                          ctypes.POINTER(RunStats), ctypes.POINTER(PeerStats)]),
    "glb_peer_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "glb_graph_info": (ctypes.c_int, [ctypes.c_void_p, _p64, _p64,
                                      ctypes.POINTER(ctypes.c_int),
                                      ctypes.POINTER(ctypes.c_int)]),
    "glb_graph_stream": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    "glb_run": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(RunParams), _p64,
                               ctypes.POINTER(RunStats), ctypes.POINTER(Record), _i64]),
    "glb_run_records": (ctypes.c_int, [ctypes.c_void_p, _i64, ctypes.POINTER(Record), _i64,
                                       _p64]),
    "glb_run_thread_work": (ctypes.c_int, [ctypes.c_void_p, _i64, _i64,
                                           ctypes.POINTER(ctypes.c_uint32), _p64]),
    "glb_graph_load_csrg": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int,
                                           ctypes.POINTER(ctypes.c_void_p)]),
    "glb_read_text_graph": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, _p64, _p64,
                                           ctypes.POINTER(ctypes.c_int), ctypes.POINTER(_p64),
                                           ctypes.POINTER(_p64), ctypes.POINTER(_p64)]),
    "glb_free": (None, [ctypes.c_void_p]),
    "glb_measure_gather": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)]),
    "glb_degree_stats": (ctypes.c_int, [ctypes.c_void_p, _p64, _p64,
                                        ctypes.POINTER(ctypes.c_double)]),
    "glb_histogram": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _p64, _p64,
                                     ctypes.POINTER(ctypes.c_int32), _p64]),
    "glb_split_graph": (ctypes.c_int, [ctypes.c_void_p, _i64, _p64, _p64, _p64, _p64, _p64,
                                       _p64, _p64]),
    "glb_csr_to_coo": (ctypes.c_int, [ctypes.c_void_p, _i64, _p64]),
    "glb_validate": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, _i64, _p64, _p64, _p64]),
    "glb_inclusive_scan": (ctypes.c_int, [_p64, _i64, _p64, ctypes.c_int]),
    "glb_find_offsets": (ctypes.c_int, [_p64, _i64, _i64, _i64, _p64, _p64, ctypes.c_int]),
}

_lib = None
_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    """Load libgraphlb_b200.so (in-tree); raise ImportError when it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = Path(os.environ.get("GRAPHLB_B200_LIB", LIB_PATH))
        if not path.exists():
            raise ImportError(
                f"{path} is missing: build the CUDA library first "
                "(python -c 'import __graft_entry__ as g; g.build()')"
            )
        h = ctypes.CDLL(str(path))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


class DeviceError(RuntimeError):
    """A CUDA-side failure inside libgraphlb_b200.so."""


def check(status: int, what: str = "") -> None:
    """Map a C-ABI status to the reference's exception types."""
    if status == GLB_OK:
        return
    msg = lib().glb_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if status == GLB_EINVAL:
        raise ValueError(msg)
    if status == GLB_ERANGE:
        raise IndexError(msg)
    if status == GLB_EOVERFLOW:
        raise OverflowError(msg)
    if status == GLB_ENOMEM:
        raise MemoryError(msg)
    raise DeviceError(msg)


def ptr64(a: np.ndarray | None):
    """int64* of a C-contiguous int64 array (None -> NULL)."""
    if a is None:
        return None
    assert a.dtype == np.int64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_p64)


def device_count() -> int:
    c = ctypes.c_int(0)
    check(lib().glb_device_count(ctypes.byref(c)))
    return c.value


def default_device() -> int:
    return int(os.environ.get("GRAPHLB_DEVICE", "0"))
