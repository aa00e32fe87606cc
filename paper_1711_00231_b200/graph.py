"""Graph containers and generators (drop-in for graphlb's csr.py / generators.py).

Host-side containers keep the reference's int64 numpy layout
(csr.py:16-21, 42-118) so existing callers keep working; the first run on a
device uploads the CSR into HBM once (``CsrGraph.device_graph``) through
``glb_graph_create``, which narrows columns and weights to 32 bits on the GPU.

Generators reproduce the reference's numpy ``default_rng`` streams draw for
draw (generators.py:23-130), so graphs are bit-identical to the reference's
for the same arguments -- the parity tests rely on that.
"""

from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib

# "4 GB" device with 4-byte ids: the EP feasibility cliff (csr.py:16-18)
COO_ID_BYTES = 4
DEFAULT_COO_BUDGET_BYTES = 4_000_000_000
DEFAULT_COO_BUDGET_CELLS = DEFAULT_COO_BUDGET_BYTES // COO_ID_BYTES

INDEX_DTYPE = np.int64

DEFAULT_RMAT_PARAMS = (0.45, 0.15, 0.15, 0.25)
DEFAULT_MAX_WEIGHT = 100


class CooCapacityError(MemoryError):
    """The 2E (3E weighted) coordinate layout exceeds the cell budget (csr.py:23-32)."""

    def __init__(self, required_cells: int, available_cells: int):
        super().__init__(
            f"coordinate layout needs {required_cells} cells "
            f"but the budget allows {available_cells}"
        )
        self.required_cells = required_cells
        self.available_cells = available_cells


def _index_array(values, name: str) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(values, dtype=INDEX_DTYPE))
    if a.ndim != 1:
        raise ValueError(f"{name} must be one-dimensional")
    return a


def _destroy_handles(handles: dict) -> None:
    for h in handles.values():
        try:
            _lib.lib().glb_graph_destroy(h)
        except Exception:  # interpreter shutdown
            pass
    handles.clear()


@dataclass
class CsrGraph:
    """Directed CSR graph, immutable after construction (csr.py:42-118).

    ``weights`` None means unweighted: SSSP then uses unit weights and BFS
    ignores weights either way (strategies/common.py:78-82).
    """

    num_nodes: int
    num_edges: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    weights: np.ndarray | None = None
    _handles: dict = field(default_factory=dict, init=False, repr=False, compare=False)

    def __post_init__(self):
        self.row_offsets = _index_array(self.row_offsets, "row_offsets")
        self.col_indices = _index_array(self.col_indices, "col_indices")
        if self.weights is not None:
            self.weights = _index_array(self.weights, "weights")
        self._check()
        for a in (self.row_offsets, self.col_indices, self.weights):
            if a is not None:
                a.setflags(write=False)
        weakref.finalize(self, _destroy_handles, self._handles)

    def _check(self) -> None:
        n, m = self.num_nodes, self.num_edges
        if n < 0 or m < 0:
            raise ValueError("node and edge counts must be nonnegative")
        if self.row_offsets.shape[0] != n + 1:
            raise ValueError(f"row_offsets must have length {n + 1}")
        if self.col_indices.shape[0] != m:
            raise ValueError(f"col_indices must have length {m}")
        if self.row_offsets[0] != 0 or self.row_offsets[n] != m:
            raise ValueError("row_offsets must start at 0 and end at num_edges")
        if n > 0 and bool((self.row_offsets[1:] < self.row_offsets[:-1]).any()):
            raise ValueError("row_offsets must be nondecreasing")
        if m > 0 and (self.col_indices.min() < 0 or self.col_indices.max() >= n):
            raise ValueError("col_indices contains a node id out of range")
        if self.weights is not None:
            if self.weights.shape[0] != m:
                raise ValueError(f"weights must have length {m}")
            if m > 0 and self.weights.min() < 0:
                raise ValueError("edge weights must be nonnegative")

    @property
    def is_weighted(self) -> bool:
        return self.weights is not None

    def outdegrees(self) -> np.ndarray:
        return np.diff(self.row_offsets)

    def outdegree(self, node: int) -> int:
        return int(self.row_offsets[node + 1] - self.row_offsets[node])

    # ---------------------------------------------------------- device side
    def device_graph(self, device: int | None = None):
        """Handle of this graph resident in HBM on ``device`` (uploaded once)."""
        dev = _lib.default_device() if device is None else int(device)
        h = self._handles.get(dev)
        if h is None:
            out = ctypes.c_void_p()
            _lib.check(
                _lib.lib().glb_graph_create(
                    _lib.ptr64(self.row_offsets), _lib.ptr64(self.col_indices),
                    _lib.ptr64(self.weights), self.num_nodes, self.num_edges, dev,
                    ctypes.byref(out),
                ),
                "glb_graph_create",
            )
            h = out.value
            self._handles[dev] = h
        return h

    def release_device(self) -> None:
        """Free the HBM copies (they are re-uploaded on the next run)."""
        _destroy_handles(self._handles)

    @classmethod
    def from_edges(cls, num_nodes: int, src, dst, weights=None) -> "CsrGraph":
        """CSR from parallel edge arrays, grouping by source with a stable sort so
        edges of one source keep their input order (csr.py:97-118)."""
        src = _index_array(src, "src")
        dst = _index_array(dst, "dst")
        if src.shape[0] != dst.shape[0]:
            raise ValueError("src and dst must have equal length")
        m = src.shape[0]
        if m > 0 and (src.min() < 0 or src.max() >= num_nodes):
            raise ValueError("source node id out of range")
        perm = np.argsort(src, kind="stable")
        row = np.zeros(num_nodes + 1, dtype=INDEX_DTYPE)
        np.cumsum(np.bincount(src, minlength=num_nodes), out=row[1:])
        w = None if weights is None else _index_array(weights, "weights")[perm]
        return cls(num_nodes, m, row, dst[perm], w)


@dataclass
class CooGraph:
    """Edge list (src, dst, wt) sorted by source (csr.py:121-152)."""

    src: np.ndarray
    dst: np.ndarray
    wt: np.ndarray | None
    num_nodes: int

    def __post_init__(self):
        self.src = _index_array(self.src, "src")
        self.dst = _index_array(self.dst, "dst")
        if self.wt is not None:
            self.wt = _index_array(self.wt, "wt")
        if self.src.shape[0] != self.dst.shape[0]:
            raise ValueError("src and dst must have equal length")
        if self.wt is not None and self.wt.shape[0] != self.src.shape[0]:
            raise ValueError("wt must match the edge count")
        if self.src.shape[0] > 1 and bool((self.src[1:] < self.src[:-1]).any()):
            raise ValueError("edges must be sorted by source")
        for a in (self.src, self.dst, self.wt):
            if a is not None:
                a.setflags(write=False)

    @property
    def num_edges(self) -> int:
        return int(self.src.shape[0])

    @property
    def num_cells(self) -> int:
        return (3 if self.wt is not None else 2) * self.num_edges


def coo_cells_required(num_edges: int, weighted: bool) -> int:
    return (3 if weighted else 2) * num_edges


def csr_to_coo(g: CsrGraph, max_cells: int = DEFAULT_COO_BUDGET_CELLS,
               device: int | None = None) -> CooGraph:
    """Expand CSR to COO; the per-edge source ids are produced on the GPU
    (segment fill, K12).  Raises CooCapacityError over the budget (csr.py:155-170)."""
    required = coo_cells_required(g.num_edges, g.is_weighted)
    if required > max_cells:
        raise CooCapacityError(required, max_cells)
    src = np.empty(g.num_edges, dtype=INDEX_DTYPE)
    if g.num_edges:
        st = _lib.lib().glb_csr_to_coo(g.device_graph(device), int(max_cells), _lib.ptr64(src))
        if st == _lib.GLB_ECOO_CAPACITY:
            raise CooCapacityError(required, max_cells)
        _lib.check(st, "glb_csr_to_coo")
    wt = None if g.weights is None else g.weights.copy()
    return CooGraph(src, g.col_indices.copy(), wt, g.num_nodes)


# =============================================================== generators
def _uniform_weights(rng: np.random.Generator, m: int, max_weight: int) -> np.ndarray:
    return rng.integers(1, max_weight + 1, size=m, dtype=INDEX_DTYPE)


class DeviceCsrGraph:
    """A CSR graph that lives only in HBM (no host arrays), e.g. a scale-27
    R-MAT built by ``generate_rmat(..., device=d, download=False)``.  Runs
    through every strategy like a CsrGraph; ``to_host()`` copies it back."""

    def __init__(self, handle, num_nodes: int, num_edges: int, weighted: bool, device: int):
        self.num_nodes = num_nodes
        self.num_edges = num_edges
        self._weighted = weighted
        self._device = device
        self._handles = {device: handle}
        weakref.finalize(self, _destroy_handles, self._handles)

    @property
    def is_weighted(self) -> bool:
        return self._weighted

    def device_graph(self, device: int | None = None):
        dev = self._device if device is None else int(device)
        if dev != self._device:
            raise ValueError(f"graph lives on device {self._device}, not {dev}")
        return self._handles[dev]

    def release_device(self) -> None:
        _destroy_handles(self._handles)

    def download_narrow(self):
        """(row int64[n+1], col uint32[m], weights uint32[m] or None): the
        device layout as is, half the host memory of ``to_host``."""
        row = np.empty(self.num_nodes + 1, dtype=INDEX_DTYPE)
        col = np.empty(self.num_edges, dtype=np.uint32)
        w = np.empty(self.num_edges, dtype=np.uint32) if self._weighted else None
        u32 = ctypes.POINTER(ctypes.c_uint32)
        _lib.check(_lib.lib().glb_graph_download_u32(
            self._handles[self._device], _lib.ptr64(row), col.ctypes.data_as(u32),
            None if w is None else w.ctypes.data_as(u32)), "glb_graph_download_u32")
        return row, col, w

    def to_host(self) -> CsrGraph:
        row = np.empty(self.num_nodes + 1, dtype=INDEX_DTYPE)
        col = np.empty(self.num_edges, dtype=INDEX_DTYPE)
        w = np.empty(self.num_edges, dtype=INDEX_DTYPE) if self._weighted else None
        _lib.check(_lib.lib().glb_graph_download(self._handles[self._device], _lib.ptr64(row),
                                                 _lib.ptr64(col), _lib.ptr64(w)),
                   "glb_graph_download")
        g = CsrGraph(self.num_nodes, self.num_edges, row, col, w)
        return g


def _rmat_device(scale, edge_factor, a, b, c, seed, weighted, max_weight, device, download):
    st = np.random.default_rng(seed).bit_generator.state["state"]
    mask = (1 << 64) - 1
    state = (ctypes.c_uint64 * 2)(st["state"] >> 64, st["state"] & mask)
    inc = (ctypes.c_uint64 * 2)(st["inc"] >> 64, st["inc"] & mask)
    h = ctypes.c_void_p()
    _lib.check(_lib.lib().glb_graph_create_rmat(scale, edge_factor, float(a), float(a + b),
                                                float(a + b + c), state, inc, 1 if weighted else 0,
                                                int(max_weight), int(device), ctypes.byref(h)),
               "glb_graph_create_rmat")
    dg = DeviceCsrGraph(h.value, 1 << scale, edge_factor << scale, weighted, int(device))
    if not download:
        return dg
    g = dg.to_host()
    g._handles[int(device)] = dg._handles.pop(int(device))  # keep the HBM copy
    return g


def generate_rmat(
    scale: int,
    edge_factor: int,
    params: tuple[float, float, float, float] = DEFAULT_RMAT_PARAMS,
    seed: int = 0,
    weighted: bool = True,
    max_weight: int = DEFAULT_MAX_WEIGHT,
    device: int | None = None,
    download: bool = True,
) -> CsrGraph:
    """R-MAT graph with 2**scale nodes and edge_factor * 2**scale edges.

    Same draw order as generators.py:23-58: ``scale`` blocks of m uniforms
    (one quadrant decision per level for every edge), then m weights.  With
    ``device`` set, the graph is generated directly in HBM by the CUDA
    library (same PCG64 stream, identical arrays) and, unless ``download`` is
    False, copied back so the result is a regular CsrGraph already resident
    on that device.
    """
    a, b, c, d = params
    if abs(a + b + c + d - 1.0) > 1e-9:
        raise ValueError(f"quadrant probabilities must sum to 1, got {a + b + c + d}")
    if min(a, b, c, d) < 0:
        raise ValueError("quadrant probabilities must be nonnegative")
    if scale < 1:
        raise ValueError("scale must be >= 1")
    if edge_factor < 0:
        raise ValueError("edge_factor must be nonnegative")
    if device is not None:
        return _rmat_device(scale, edge_factor, a, b, c, seed, weighted, max_weight, device,
                            download)
    n = 1 << scale
    m = edge_factor * n
    rng = np.random.default_rng(seed)
    t_row = a + b           # u >= a+b          -> lower half (row bit)
    t_c = a + b + c         # u >= a+b+c        -> quadrant d
    src = np.zeros(m, dtype=INDEX_DTYPE)
    dst = np.zeros(m, dtype=INDEX_DTYPE)
    u = np.empty(m, dtype=np.float64)
    lower = np.empty(m, dtype=bool)
    right = np.empty(m, dtype=bool)
    tmp = np.empty(m, dtype=bool)
    for _ in range(scale):
        rng.random(out=u)
        np.greater_equal(u, t_row, out=lower)
        # right column: quadrant b (a <= u < a+b) or quadrant d (u >= a+b+c)
        np.greater_equal(u, a, out=right)
        np.less(u, t_row, out=tmp)
        right &= tmp
        np.greater_equal(u, t_c, out=tmp)
        right |= tmp
        src <<= 1
        src |= lower
        dst <<= 1
        dst |= right
    wt = _uniform_weights(rng, m, max_weight) if weighted else None
    return CsrGraph.from_edges(n, src, dst, wt)


def generate_er(
    num_nodes: int,
    num_edges: int,
    seed: int = 0,
    weighted: bool = True,
    max_weight: int = DEFAULT_MAX_WEIGHT,
) -> CsrGraph:
    """Uniform random endpoints (generators.py:61-81)."""
    if num_nodes < 0 or num_edges < 0:
        raise ValueError("counts must be nonnegative")
    if num_edges > num_nodes * num_nodes:
        raise ValueError(f"requested {num_edges} edges exceed {num_nodes}^2 possible endpoints")
    if num_edges > 0 and num_nodes == 0:
        raise ValueError("cannot place edges in an empty graph")
    rng = np.random.default_rng(seed)
    if num_edges:
        src = rng.integers(0, num_nodes, size=num_edges, dtype=INDEX_DTYPE)
        dst = rng.integers(0, num_nodes, size=num_edges, dtype=INDEX_DTYPE)
    else:
        src = dst = np.zeros(0, dtype=INDEX_DTYPE)
    wt = _uniform_weights(rng, num_edges, max_weight) if weighted else None
    return CsrGraph.from_edges(num_nodes, src, dst, wt)


def _fixture_weights(count: int, weighted: bool, seed: int):
    if not weighted:
        return None
    return _uniform_weights(np.random.default_rng(seed), count, DEFAULT_MAX_WEIGHT)


def path_graph(n: int, weighted: bool = False, seed: int = 0) -> CsrGraph:
    """0 -> 1 -> ... -> n-1 (generators.py:84-91)."""
    if n < 1:
        raise ValueError("path needs at least one node")
    s = np.arange(n - 1, dtype=INDEX_DTYPE)
    return CsrGraph.from_edges(n, s, s + 1, _fixture_weights(n - 1, weighted, seed))


def star_graph(n: int, weighted: bool = False, seed: int = 0) -> CsrGraph:
    """Node 0 points at every other node (generators.py:94-101)."""
    if n < 1:
        raise ValueError("star needs at least one node")
    return CsrGraph.from_edges(n, np.zeros(n - 1, dtype=INDEX_DTYPE),
                               np.arange(1, n, dtype=INDEX_DTYPE),
                               _fixture_weights(n - 1, weighted, seed))


def ring_graph(n: int, weighted: bool = False, seed: int = 0) -> CsrGraph:
    """Directed cycle (generators.py:104-111)."""
    if n < 1:
        raise ValueError("ring needs at least one node")
    s = np.arange(n, dtype=INDEX_DTYPE)
    return CsrGraph.from_edges(n, s, (s + 1) % n, _fixture_weights(n, weighted, seed))


def graph_from_degrees(degrees, weighted: bool = False, seed: int = 0) -> CsrGraph:
    """Outdegree multiset realised with every edge pointing at node 0 (generators.py:114-130)."""
    deg = np.asarray(degrees, dtype=INDEX_DTYPE)
    if deg.shape[0] == 0:
        raise ValueError("need at least one node")
    if deg.min() < 0:
        raise ValueError("degrees must be nonnegative")
    row = np.zeros(deg.shape[0] + 1, dtype=INDEX_DTYPE)
    np.cumsum(deg, out=row[1:])
    m = int(row[-1])
    return CsrGraph(deg.shape[0], m, row, np.zeros(m, dtype=INDEX_DTYPE),
                    _fixture_weights(m, weighted, seed))


def grid_graph(k: int, weighted: bool = True, seed: int = 1,
               max_weight: int = 255) -> CsrGraph:
    """k x k 4-neighbour grid with arcs in both directions (config C3; not in
    the reference).  Node (r, c) has id r*k + c; each row lists its neighbours
    in ascending id order (up, left, right, down); weights are drawn in CSR
    order from default_rng(seed).integers(1, max_weight + 1)."""
    if k < 1:
        raise ValueError("grid side must be >= 1")
    n = k * k
    r, c = np.divmod(np.arange(n, dtype=INDEX_DTYPE), k)
    has = [r > 0, c > 0, c < k - 1, r < k - 1]
    off = [-k, -1, 1, k]
    deg = sum(h.astype(INDEX_DTYPE) for h in has)
    row = np.zeros(n + 1, dtype=INDEX_DTYPE)
    np.cumsum(deg, out=row[1:])
    m = int(row[-1])
    col = np.empty(m, dtype=INDEX_DTYPE)
    cursor = row[:-1].copy()
    ids = np.arange(n, dtype=INDEX_DTYPE)
    for h, o in zip(has, off):
        sel = ids[h]
        col[cursor[sel]] = sel + o
        cursor[sel] += 1
    wt = (np.random.default_rng(seed).integers(1, max_weight + 1, size=m, dtype=INDEX_DTYPE)
          if weighted else None)
    return CsrGraph(n, m, row, col, wt)
