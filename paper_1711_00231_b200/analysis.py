"""Degree analysis, scan and verification (drop-in for degrees.py, scan.py,
oracles.verify).

The degree statistics, histogram and scan run on the GPU through
libgraphlb_b200.so; only the scalar MDT formula and the argmax over B bin
counts are evaluated on the host.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .graph import CsrGraph
from .runtime import DistArray


@dataclass
class DegreeStats:
    max: int
    avg: float
    stddev: float


def degree_stats(g: CsrGraph, device: int | None = None) -> DegreeStats:
    """Max, mean and population standard deviation of the outdegrees
    (degrees.py:27-32), reduced on the device."""
    if g.num_nodes < 1:
        raise ValueError("degree statistics need at least one node")
    mx, sm, sq = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
    _lib.check(_lib.lib().glb_degree_stats(g.device_graph(device), ctypes.byref(mx),
                                           ctypes.byref(sm), ctypes.byref(sq)),
               "glb_degree_stats")
    n = g.num_nodes
    avg = sm.value / n
    var = max(sq.value / n - avg * avg, 0.0)
    return DegreeStats(int(mx.value), float(avg), float(np.sqrt(var)))


@dataclass
class DegreeHistogram:
    bin_count: int
    bin_width: float
    counts: np.ndarray
    max_degree: int
    arg_max_bin: int  # 1-based, ties to the lowest bin
    mdt: int | None = None


def build_histogram(g: CsrGraph, bins: int = 10, device: int | None = None) -> DegreeHistogram:
    """Outdegrees into ``bins`` equal-width right-closed bins over [0, max];
    degree 0 lands in bin 1 (degrees.py:45-69).  Binned in shared memory on
    the device."""
    if bins < 1:
        raise ValueError("bins must be >= 1")
    counts = np.zeros(bins, dtype=np.int64)
    mx, arg, mdt = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int64()
    if g.num_nodes == 0:
        return DegreeHistogram(bins, 0.0, counts, 0, 1)
    _lib.check(_lib.lib().glb_histogram(g.device_graph(device), bins, _lib.ptr64(counts),
                                        ctypes.byref(mx), ctypes.byref(arg), ctypes.byref(mdt)),
               "glb_histogram")
    return DegreeHistogram(bins, mx.value / bins, counts, int(mx.value), int(arg.value))


def compute_mdt(h: DegreeHistogram) -> int:
    """max(1, arg_max_bin * max_degree // bin_count) (degrees.py:72-76)."""
    h.mdt = int(max(1, (h.arg_max_bin * h.max_degree) // h.bin_count))
    return h.mdt


def inclusive_scan(values, workers: int = 1, device: int | None = None) -> list[int]:
    """Running sums on the device (single-pass look-back scan); raises
    OverflowError when a prefix leaves int64 (scan.py:19-65)."""
    a = np.ascontiguousarray(np.asarray(values, dtype=np.int64).reshape(-1))
    n = a.shape[0]
    if n == 0:
        return []
    out = np.empty(n, dtype=np.int64)
    dev = _lib.default_device() if device is None else device
    _lib.check(_lib.lib().glb_inclusive_scan(_lib.ptr64(a), n, _lib.ptr64(out), dev),
               "glb_inclusive_scan")
    return out.tolist()


@dataclass
class VerificationReport:
    matched: bool
    mismatch_count: int
    first_mismatch: tuple[int, int, int] | None = None  # (node, expected, actual)


def _cells(d) -> np.ndarray:
    if isinstance(d, DistArray):
        return d.array
    if hasattr(d, "values") and not isinstance(d, np.ndarray):
        return np.asarray(d.values, dtype=np.int64)
    return np.asarray(d, dtype=np.int64)


def verify(expected, actual) -> VerificationReport:
    """Exact elementwise comparison of distance arrays (oracles.py:69-82)."""
    e, a = _cells(expected), _cells(actual)
    if e.shape[0] != a.shape[0]:
        raise ValueError(f"length mismatch: expected {e.shape[0]}, actual {a.shape[0]}")
    bad = np.flatnonzero(e != a)
    if bad.shape[0] == 0:
        return VerificationReport(True, 0, None)
    i = int(bad[0])
    return VerificationReport(False, int(bad.shape[0]), (i, int(e[i]), int(a[i])))


def validate_distances(g: CsrGraph, source: int, algo: str, dist,
                       device: int | None = None) -> VerificationReport:
    """Device certificate of a BFS/SSSP distance array (glb_validate): no
    oracle run, yet exact -- d[source] = 0, no edge out of a reached node can
    lower its head, and every reached node is reachable from the source over
    tight edges.  Replaces the sequential_bfs / dijkstra + verify pair of
    run_benchmark(verify=True) (oracles.py:13-82, bench.py:186-196).
    ``first_mismatch`` is (node, None, actual) -- a certificate knows which
    node is wrong, not its true distance."""
    if algo not in ("bfs", "sssp"):
        raise ValueError(f"unknown relaxation kind {algo!r}")
    a = np.ascontiguousarray(_cells(dist), dtype=np.int64)
    if a.shape[0] != g.num_nodes:
        raise ValueError(f"length mismatch: graph has {g.num_nodes} nodes, dist {a.shape[0]}")
    if not 0 <= source < g.num_nodes:
        raise ValueError(f"source {source} out of range for {g.num_nodes} nodes")
    nb, fb = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(_lib.lib().glb_validate(g.device_graph(device), 0 if algo == "bfs" else 1, int(source),
                                       _lib.ptr64(a), ctypes.byref(nb), ctypes.byref(fb)),
               "glb_validate")
    if nb.value == 0:
        return VerificationReport(True, 0, None)
    return VerificationReport(False, int(nb.value), (int(fb.value), None, int(a[fb.value])))
