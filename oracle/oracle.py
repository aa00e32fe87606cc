"""ctypes wrapper of oracle/build/liboracle.so -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module, always as the checker or the timed CPU reference, never as part
of the product path.  Each function cites the reference code it restates
(paths under /root/reference/pkg/src/graphlb/); golden vectors pinning it live
in tests/golden/.
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "build" / "liboracle.so"
INF = (1 << 63) - 1

_p64 = ctypes.POINTER(ctypes.c_int64)
_lib = None


def build(force: bool = False) -> Path:
    srcs = [HERE / "graphlb_oracle.c", HERE / "graphlb_oracle_big.c"]
    if force or not LIB_PATH.exists() or any(LIB_PATH.stat().st_mtime < p.stat().st_mtime for p in srcs):
        subprocess.run(["make", "-s", "-C", str(HERE)] + (["-B"] if force else []), check=True)
    return LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        i64, i32 = ctypes.c_int64, ctypes.c_int32
        L.oracle_bfs.argtypes = [i64, _p64, _p64, i64, _p64]
        L.oracle_dijkstra.argtypes = [i64, i64, _p64, _p64, _p64, i64, _p64]
        L.oracle_histogram.argtypes = [i64, _p64, i32, _p64, _p64, ctypes.POINTER(i32), _p64]
        L.oracle_split_graph.argtypes = [i64, i64, _p64, _p64, _p64, i64, _p64, _p64, _p64,
                                         _p64, _p64, _p64, _p64]
        L.oracle_find_offsets.argtypes = [_p64, i64, i64, i64, _p64, _p64]
        L.oracle_find_offsets.restype = None
        L.oracle_inclusive_scan.argtypes = [_p64, i64, _p64]
        L.oracle_coo_src.argtypes = [i64, _p64, _p64]
        L.oracle_coo_src.restype = None
        L.oracle_bs_run.argtypes = [i64, _p64, _p64, _p64, i64, ctypes.c_int, _p64, _p64, _p64]
        L.oracle_max_threads.argtypes = []
        u32p, u64p = ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint64)
        L.oracle_rmat_u32.argtypes = [ctypes.c_int, i64, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, u64p, u64p, ctypes.c_int, i64, ctypes.c_int,
                                      _p64, u32p, u32p]
        L.oracle_bfs_u32.argtypes = [i64, _p64, u32p, i64, _p64]
        L.oracle_bfs_levels_u32.argtypes = [i64, _p64, u32p, i64, ctypes.c_int, _p64]
        L.oracle_bs_run_u32.argtypes = [i64, _p64, u32p, u32p, i64, ctypes.c_int, ctypes.c_double,
                                        _p64, _p64, _p64, ctypes.POINTER(ctypes.c_int)]
        L.oracle_wd_run_u32.argtypes = L.oracle_bs_run_u32.argtypes
        _lib = L
    return _lib


def _p(a):
    if a is None:
        return None
    assert a.dtype == np.int64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_p64)


def _arr(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.int64)


def sequential_bfs(row, col, source: int) -> np.ndarray:
    """oracles.py:13-30"""
    row, col = _arr(row), _arr(col)
    n = row.shape[0] - 1
    out = np.empty(n, dtype=np.int64)
    if lib().oracle_bfs(n, _p(row), _p(col), source, _p(out)) != 0:
        raise ValueError(f"source {source} out of range for {n} nodes")
    return out


def dijkstra(row, col, weights, source: int) -> np.ndarray:
    """oracles.py:33-55 (weights None -> unit weights)"""
    row, col, weights = _arr(row), _arr(col), _arr(weights)
    n = row.shape[0] - 1
    out = np.empty(n, dtype=np.int64)
    rc = lib().oracle_dijkstra(n, col.shape[0], _p(row), _p(col), _p(weights), source, _p(out))
    if rc == -1:
        raise ValueError(f"source {source} out of range for {n} nodes")
    if rc == -3:
        raise ValueError("negative edge weight")
    return out


def oracle_distances(g, source: int, algo: str) -> np.ndarray:
    """Expected dist for a CsrGraph-like object: BFS ignores weights
    (strategies/common.py:78-82)."""
    if algo == "bfs":
        return sequential_bfs(g.row_offsets, g.col_indices, source)
    return dijkstra(g.row_offsets, g.col_indices, g.weights, source)


def histogram(row, bins: int):
    """degrees.py:45-76 -> (counts, max_degree, arg_max_bin, mdt)"""
    row = _arr(row)
    counts = np.zeros(bins, dtype=np.int64)
    mx, mdt = ctypes.c_int64(), ctypes.c_int64()
    arg = ctypes.c_int32()
    if lib().oracle_histogram(row.shape[0] - 1, _p(row), bins, _p(counts), ctypes.byref(mx),
                              ctypes.byref(arg), ctypes.byref(mdt)) != 0:
        raise ValueError("bins must be >= 1")
    return counts, mx.value, arg.value, mdt.value


def split_graph(row, col, weights, mdt: int):
    """splitting.py:58-99 -> (new_row, new_col, new_w, parent_of, children_start)"""
    row, col, weights = _arr(row), _arr(col), _arr(weights)
    n, m = row.shape[0] - 1, col.shape[0]
    nn, kids = ctypes.c_int64(), ctypes.c_int64()
    L = lib()
    if L.oracle_split_graph(n, m, _p(row), _p(col), _p(weights), mdt, ctypes.byref(nn),
                            ctypes.byref(kids), None, None, None, None, None) != 0:
        raise ValueError("mdt must be >= 1")
    new_row = np.empty(nn.value + 1, dtype=np.int64)
    new_col = np.empty(m, dtype=np.int64)
    new_w = np.empty(m, dtype=np.int64) if weights is not None else None
    parent = np.empty(kids.value, dtype=np.int64)
    cs = np.empty(n + 1, dtype=np.int64)
    L.oracle_split_graph(n, m, _p(row), _p(col), _p(weights), mdt, ctypes.byref(nn),
                         ctypes.byref(kids), _p(new_row), _p(new_col), _p(new_w), _p(parent),
                         _p(cs))
    return new_row, new_col, new_w, parent, cs


def find_offsets(prefix, ept: int, threads: int):
    """workload.py:45-72 -> (node_offsets, edge_offsets)"""
    prefix = _arr(prefix)
    node = np.empty(threads, dtype=np.int64)
    edge = np.empty(threads, dtype=np.int64)
    lib().oracle_find_offsets(_p(prefix), prefix.shape[0], ept, threads, _p(node), _p(edge))
    return node, edge


def inclusive_scan(values) -> np.ndarray:
    """scan.py:19-65; raises OverflowError like the reference"""
    v = _arr(values)
    out = np.empty(v.shape[0], dtype=np.int64)
    if lib().oracle_inclusive_scan(_p(v), v.shape[0], _p(out)):
        raise OverflowError("prefix sum exceeds the 64-bit counter range")
    return out


def coo_src(row) -> np.ndarray:
    """csr.py:168"""
    row = _arr(row)
    n = row.shape[0] - 1
    out = np.empty(int(row[-1]), dtype=np.int64)
    lib().oracle_coo_src(n, _p(row), _p(out))
    return out


def bs_run(row, col, weights, source: int, threads: int = 0):
    """node_based.py:19-82 ported to C with OpenMP -> (dist, iterations, relax_ops)"""
    row, col, weights = _arr(row), _arr(col), _arr(weights)
    n = row.shape[0] - 1
    out = np.empty(n, dtype=np.int64)
    it, ops = ctypes.c_int64(), ctypes.c_int64()
    if lib().oracle_bs_run(n, _p(row), _p(col), _p(weights), source, threads, _p(out),
                           ctypes.byref(it), ctypes.byref(ops)) != 0:
        raise ValueError("bad source")
    return out, it.value, ops.value


def max_threads() -> int:
    return lib().oracle_max_threads()


# ------------------------------------------------------------- large configs
# Narrow layout (int64 row offsets, uint32 columns / weights) for the C3 / C5
# sizes; graphlb_oracle_big.c.  A NarrowGraph is what these helpers take.
class NarrowGraph:
    """CSR in the narrow layout: row int64[n+1], col uint32[m], w uint32[m] or None."""

    def __init__(self, row, col, w=None):
        self.row_offsets = np.ascontiguousarray(row, dtype=np.int64)
        self.col_indices = np.ascontiguousarray(col, dtype=np.uint32)
        self.weights = None if w is None else np.ascontiguousarray(w, dtype=np.uint32)

    @property
    def num_nodes(self) -> int:
        return int(self.row_offsets.shape[0] - 1)

    @property
    def num_edges(self) -> int:
        return int(self.col_indices.shape[0])

    def outdegrees(self) -> np.ndarray:
        return np.diff(self.row_offsets)


def _u32(a):
    if a is None:
        return None
    assert a.dtype == np.uint32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def rmat_narrow(scale: int, edge_factor: int, params=(0.45, 0.15, 0.15, 0.25), seed: int = 0,
                weighted: bool = True, max_weight: int = 100, threads: int = 0) -> NarrowGraph:
    """generate_rmat (generators.py:23-58) + from_edges (csr.py:97-118), the
    numpy PCG64 stream restated in C on all cores, narrow layout."""
    a, b, c, _ = params
    st = np.random.default_rng(seed).bit_generator.state["state"]
    mask = (1 << 64) - 1
    sv = (ctypes.c_uint64 * 2)(st["state"] >> 64, st["state"] & mask)
    iv = (ctypes.c_uint64 * 2)(st["inc"] >> 64, st["inc"] & mask)
    n = 1 << scale
    m = edge_factor * n
    row = np.empty(n + 1, dtype=np.int64)
    col = np.empty(m, dtype=np.uint32)
    w = np.empty(m, dtype=np.uint32) if weighted else None
    rc = lib().oracle_rmat_u32(scale, edge_factor, a, a + b, a + b + c, sv, iv, 1 if weighted else 0,
                               max_weight, threads, _p(row), _u32(col), _u32(w))
    if rc != 0:
        raise MemoryError("oracle_rmat_u32: allocation failed")
    return NarrowGraph(row, col, w)


def bfs_narrow(g, source: int, parallel: bool = True, threads: int = 0) -> np.ndarray:
    """sequential_bfs levels (oracles.py:13-30): FIFO, or level-synchronous on
    all cores (same level sets)."""
    out = np.empty(g.num_nodes, dtype=np.int64)
    if parallel:
        rc = lib().oracle_bfs_levels_u32(g.num_nodes, _p(g.row_offsets), _u32(g.col_indices),
                                         source, threads, _p(out))
    else:
        rc = lib().oracle_bfs_u32(g.num_nodes, _p(g.row_offsets), _u32(g.col_indices), source,
                                  _p(out))
    if rc == -1:
        raise ValueError("bad source")
    if rc:
        raise MemoryError("oracle bfs: allocation failed")
    return out


def bs_run_narrow(g, source: int, weighted: bool, threads: int = 0, max_seconds: float = 0.0):
    """run_bs (node_based.py:19-82) port over the narrow layout -> (dist,
    iterations, relax_ops, completed).  max_seconds > 0 bounds the run (a
    CPU-baseline sample); the distances are then partial."""
    out = np.empty(g.num_nodes, dtype=np.int64)
    it, ops, done = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
    w = g.weights if weighted else None
    rc = lib().oracle_bs_run_u32(g.num_nodes, _p(g.row_offsets), _u32(g.col_indices), _u32(w),
                                 source, threads, max_seconds, _p(out), ctypes.byref(it),
                                 ctypes.byref(ops), ctypes.byref(done))
    if rc == -1:
        raise ValueError("bad source")
    if rc:
        raise MemoryError("oracle bs_run: allocation failed")
    return out, it.value, ops.value, bool(done.value)


def wd_run_narrow(g, source: int, weighted: bool, threads: int = 0, max_seconds: float = 0.0):
    """run_wd (workload.py:75-189) port over the narrow layout, equal edge
    slices per host thread; results as bs_run_narrow."""
    out = np.empty(g.num_nodes, dtype=np.int64)
    it, ops, done = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
    w = g.weights if weighted else None
    rc = lib().oracle_wd_run_u32(g.num_nodes, _p(g.row_offsets), _u32(g.col_indices), _u32(w),
                                 source, threads, max_seconds, _p(out), ctypes.byref(it),
                                 ctypes.byref(ops), ctypes.byref(done))
    if rc == -1:
        raise ValueError("bad source")
    if rc:
        raise MemoryError("oracle wd_run: allocation failed")
    return out, it.value, ops.value, bool(done.value)


def narrow_distances(g, source: int, algo: str, threads: int = 0) -> np.ndarray:
    """Expected distances at the large sizes: BFS levels (level-synchronous),
    SSSP by the run_bs port (its fixpoint is the unique shortest-path array)."""
    if algo == "bfs":
        return bfs_narrow(g, source, parallel=True, threads=threads)
    return bs_run_narrow(g, source, weighted=g.weights is not None, threads=threads)[0]
