"""The five task-distribution strategies on the GPU (drop-in for graphlb.strategies).

Every ``run_*`` keeps the reference signature and return type
(strategies/__init__.py:17-41, node_based.py:19, edge_based.py:31,
workload.py:162, splitting.py:102, hierarchical.py:27) and executes through
``glb_run`` in libgraphlb_b200.so: graph upload happens once per graph and
device, and the whole worklist loop, preprocessing (histogram, MDT, split,
COO) and relaxation run on the device.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .graph import DEFAULT_COO_BUDGET_CELLS, INDEX_DTYPE, CsrGraph
from .runtime import DistArray, KernelConfig, MetricsRecord

INFEASIBLE_MEMORY = "infeasible: memory"   # common.py:18
STATUS_OK = "ok"
STRATEGY_TAGS = ("BS", "EP", "WD", "NS", "HP")  # strategies/__init__.py:14
FALLBACK_TAG = "WD-fallback"               # hierarchical.py:24
IDLE = -1

_TAG_OF = {_lib.GLB_BS: "BS", _lib.GLB_EP: "EP", _lib.GLB_WD: "WD", _lib.GLB_NS: "NS",
           _lib.GLB_HP: "HP", _lib.GLB_TAG_WD_FALLBACK: FALLBACK_TAG}
_ID_OF = {"BS": _lib.GLB_BS, "EP": _lib.GLB_EP, "WD": _lib.GLB_WD, "NS": _lib.GLB_NS,
          "HP": _lib.GLB_HP}


@dataclass(frozen=True)
class RelaxOp:
    """candidate = dist + 1 (BFS) or dist + weight (SSSP) (common.py:23-42)."""

    kind: str

    def __post_init__(self):
        if self.kind not in ("bfs", "sssp"):
            raise ValueError(f"unknown relaxation kind {self.kind!r}")

    def candidate(self, source_value: int, edge_weight: int) -> int:
        return source_value + (1 if self.kind == "bfs" else edge_weight)

    @classmethod
    def bfs(cls) -> "RelaxOp":
        return cls("bfs")

    @classmethod
    def sssp(cls) -> "RelaxOp":
        return cls("sssp")


@dataclass
class StrategyRun:
    """Outcome of one strategy execution (common.py:45-65).

    ``device`` carries the device-side totals of glb_run_stats (device_ms,
    relax_ops, edges_examined, dist_bits, ...).
    """

    strategy: str
    dist: DistArray | None
    records: list[MetricsRecord] = field(default_factory=list)
    status: str = STATUS_OK
    setup_overhead: float = 0.0
    mdt: int | None = None
    split_fraction: float | None = None
    device: dict | None = None

    @property
    def feasible(self) -> bool:
        return self.status == STATUS_OK

    def total_kernel_time(self) -> float:
        return sum(r.kernel_wall_time for r in self.records)

    def total_overhead_time(self) -> float:
        return self.setup_overhead + sum(r.overhead_wall_time for r in self.records)


def check_source(g: CsrGraph, source: int) -> None:
    if not 0 <= source < g.num_nodes:
        raise ValueError(f"source {source} out of range for {g.num_nodes} nodes")


def _records(h, stats: _lib.RunStats, buf) -> list[MetricsRecord]:
    n = stats.n_records
    raw = list(buf[: min(n, len(buf))])
    while len(raw) < n:  # more launches than the first buffer held
        more = (_lib.Record * min(n - len(raw), 1 << 16))()
        got = ctypes.c_int64()
        _lib.check(_lib.lib().glb_run_records(h, len(raw), more, len(more), ctypes.byref(got)))
        raw.extend(more[: got.value])
    # exact per-thread work lists of an instrumented run: one download of the
    # run's list, each record a view of its slice
    ptw = None
    total = ctypes.c_int64()
    if any(r.thread_work_offset >= 0 for r in raw):
        _lib.check(_lib.lib().glb_run_thread_work(h, 0, 0, None, ctypes.byref(total)))
        if total.value:
            flat = np.empty(total.value, dtype=np.uint32)
            _lib.check(_lib.lib().glb_run_thread_work(
                h, 0, total.value, flat.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), None))
            ptw = flat.astype(np.int64)
    out = []
    for r in raw:
        lst = None
        if ptw is not None and r.thread_work_offset >= 0 and r.thread_work_offset + r.threads <= ptw.size:
            lst = ptw[r.thread_work_offset: r.thread_work_offset + r.threads]
        wmax, wsq = r.work_max, r.work_sumsq
        if lst is not None:  # HP's two kernels add into one list entry per thread
            wmax = int(lst.max(initial=0))
            wsq = float(np.dot(lst.astype(np.float64), lst.astype(np.float64)))
        out.append(MetricsRecord(
            iteration=r.iteration,
            strategy=_TAG_OF.get(r.tag, str(r.tag)),
            active_items=r.active_items,
            per_thread_work=lst,
            atomic_relax_ops=r.relax_ops,
            atomic_push_ops=r.push_ops,
            kernel_wall_time=r.kernel_ms / 1e3,
            overhead_wall_time=r.overhead_ms / 1e3,
            sub_iteration=None if r.sub_iteration < 0 else r.sub_iteration,
            n_threads=r.threads,
            total_work=r.work_total,
            max_work=wmax,
            work_sumsq=wsq,
        ))
    return out


def _device_run(tag: str, g: CsrGraph, source: int, op: RelaxOp, cfg: KernelConfig, *,
                bins: int = 10, mdt: int | None = None, chunked: bool = True,
                max_cells: int = DEFAULT_COO_BUDGET_CELLS, fallback: bool = True,
                want_records: bool = True) -> StrategyRun:
    check_source(g, source)
    if mdt is not None and mdt < 1:
        raise ValueError("mdt must be >= 1")
    if tag in ("NS", "HP") and mdt is None and bins < 1:
        raise ValueError("bins must be >= 1")
    h = g.device_graph(cfg.device)
    p = _lib.RunParams()
    p.strategy = _ID_OF[tag]
    p.algo = _lib.GLB_BFS if op.kind == "bfs" else _lib.GLB_SSSP
    p.source = source
    p.bins = bins
    p.chunked = 1 if chunked else 0
    p.mdt = 0 if mdt is None else int(mdt)
    p.max_cells = int(min(max_cells, (1 << 63) - 1))
    p.block_size = cfg.block_size
    p.hp_fallback = 1 if fallback else 0
    p.virtual_threads = cfg.virtual_threads or 0
    p.dist_bits = cfg.dist_bits
    p.loop_mode = _lib.GLB_LOOP_GRAPH if cfg.loop == "graph" else _lib.GLB_LOOP_HOST
    p.record_timing = 1 if cfg.record_timing else 0
    p.instrument = 1 if (cfg.instrument and want_records) else 0
    dist = np.empty(g.num_nodes, dtype=INDEX_DTYPE)
    stats = _lib.RunStats()
    cap = 4096 if want_records else 0
    buf = (_lib.Record * cap)() if cap else None
    _lib.check(_lib.lib().glb_run(h, ctypes.byref(p), _lib.ptr64(dist), ctypes.byref(stats),
                                  buf, cap), f"run_{tag.lower()}")
    info = {f: getattr(stats, f) for f, _ in _lib.RunStats._fields_}
    if stats.status == _lib.GLB_ECOO_CAPACITY:   # edge_based.py:41-46
        return StrategyRun(tag, None, status=INFEASIBLE_MEMORY, device=info)
    recs = _records(h, stats, buf) if want_records else []
    return StrategyRun(
        tag,
        DistArray.from_array(dist),
        recs,
        setup_overhead=stats.setup_ms / 1e3,
        mdt=stats.mdt if tag in ("NS", "HP") else None,
        split_fraction=stats.split_fraction if tag == "NS" else None,
        device=info,
    )


def run_bs(g: CsrGraph, source: int, op: RelaxOp, cfg: KernelConfig) -> StrategyRun:
    """Node-based distribution (node_based.py:19-82)."""
    return _device_run("BS", g, source, op, cfg)


def run_ep(g: CsrGraph, source: int, op: RelaxOp, cfg: KernelConfig, chunked: bool = True,
           max_cells: int = DEFAULT_COO_BUDGET_CELLS) -> StrategyRun:
    """Edge-based distribution over COO (edge_based.py:31-103)."""
    return _device_run("EP", g, source, op, cfg, chunked=chunked, max_cells=max_cells)


def run_wd(g: CsrGraph, source: int, op: RelaxOp, cfg: KernelConfig) -> StrategyRun:
    """Workload decomposition (workload.py:162-191)."""
    return _device_run("WD", g, source, op, cfg)


def run_ns(g: CsrGraph, source: int, op: RelaxOp, cfg: KernelConfig, bins: int = 10,
           mdt: int | None = None) -> StrategyRun:
    """Node splitting (splitting.py:102-186)."""
    return _device_run("NS", g, source, op, cfg, bins=bins, mdt=mdt)


def run_hp(g: CsrGraph, source: int, op: RelaxOp, cfg: KernelConfig, bins: int = 10,
           mdt: int | None = None, fallback: bool = True) -> StrategyRun:
    """Hierarchical processing (hierarchical.py:27-141)."""
    return _device_run("HP", g, source, op, cfg, bins=bins, mdt=mdt, fallback=fallback)


def run_strategy(tag: str, g: CsrGraph, source: int, op: RelaxOp, cfg: KernelConfig, *,
                 bins: int = 10, mdt: int | None = None, chunked: bool = True,
                 max_cells: int = DEFAULT_COO_BUDGET_CELLS) -> StrategyRun:
    """Run one strategy by tag, case-insensitive (strategies/__init__.py:17-41)."""
    t = tag.upper()
    if t == "BS":
        return run_bs(g, source, op, cfg)
    if t == "EP":
        return run_ep(g, source, op, cfg, chunked=chunked, max_cells=max_cells)
    if t == "WD":
        return run_wd(g, source, op, cfg)
    if t == "NS":
        return run_ns(g, source, op, cfg, bins=bins, mdt=mdt)
    if t == "HP":
        return run_hp(g, source, op, cfg, bins=bins, mdt=mdt)
    raise ValueError(f"unknown strategy tag {tag!r}")


# ============================================================ node splitting
@dataclass
class SplitGraph:
    """Split CSR + parent/child bookkeeping (splitting.py:26-55).  Children of
    original v are ids num_original + children_start[v] .. + children_start[v+1]."""

    graph: CsrGraph
    num_original: int
    parent_of: np.ndarray
    children_start: np.ndarray
    mdt: int

    @property
    def num_children(self) -> int:
        return int(self.parent_of.shape[0])

    @property
    def split_fraction(self) -> float:
        if self.num_original == 0:
            return 0.0
        return int(np.count_nonzero(np.diff(self.children_start))) / self.num_original

    def children_of(self, node: int) -> range:
        return range(self.num_original + int(self.children_start[node]),
                     self.num_original + int(self.children_start[node + 1]))


def split_graph(g: CsrGraph, mdt: int, device: int | None = None) -> SplitGraph:
    """Split every node of outdegree > mdt into ceil(deg/mdt) nodes on the GPU
    (splitting.py:58-99): child-count / edge scans, then segment copies."""
    if mdt < 1:
        raise ValueError("mdt must be >= 1")
    h = g.device_graph(device)
    L = _lib.lib()
    new_n, nkids = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(L.glb_split_graph(h, int(mdt), ctypes.byref(new_n), ctypes.byref(nkids),
                                 None, None, None, None, None), "glb_split_graph")
    rows = np.empty(new_n.value + 1, dtype=INDEX_DTYPE)
    cols = np.empty(g.num_edges, dtype=INDEX_DTYPE)
    wts = np.empty(g.num_edges, dtype=INDEX_DTYPE) if g.weights is not None else None
    parent = np.empty(nkids.value, dtype=INDEX_DTYPE)
    cstart = np.empty(g.num_nodes + 1, dtype=INDEX_DTYPE)
    _lib.check(L.glb_split_graph(h, int(mdt), ctypes.byref(new_n), ctypes.byref(nkids),
                                 _lib.ptr64(rows), _lib.ptr64(cols), _lib.ptr64(wts),
                                 _lib.ptr64(parent), _lib.ptr64(cstart)), "glb_split_graph")
    sg = CsrGraph(int(new_n.value), g.num_edges, rows, cols, wts)
    return SplitGraph(sg, g.num_nodes, parent, cstart, int(mdt))


# ===================================================== workload decomposition
@dataclass
class OffsetTable:
    """Per-thread (worklist index, edge offset); idle threads have -1 (workload.py:28-42)."""

    node_offsets: list[int]
    edge_offsets: list[int]

    def __len__(self) -> int:
        return len(self.node_offsets)

    def entry(self, tid: int) -> tuple[int, int]:
        return self.node_offsets[tid], self.edge_offsets[tid]


def _worklist_size(wl) -> int:
    if hasattr(wl, "size") and not isinstance(wl, np.ndarray):
        return int(wl.size)
    return len(wl)


def find_offsets(g: CsrGraph, wl, prefix, edges_per_thread: int, threads: int,
                 device: int | None = None) -> OffsetTable:
    """Thread t starts at active edge t*edges_per_thread, located by a binary
    search of the inclusive prefix on the device (workload.py:45-72)."""
    size = _worklist_size(wl)
    pre = np.ascontiguousarray(np.asarray(prefix, dtype=np.int64).reshape(-1))
    if pre.shape[0] != size:
        raise ValueError(f"prefix length {pre.shape[0]} does not match worklist size {size}")
    if edges_per_thread < 1:
        raise ValueError("edges_per_thread must be >= 1")
    node = np.empty(threads, dtype=np.int64)
    edge = np.empty(threads, dtype=np.int64)
    if threads > 0:
        dev = _lib.default_device() if device is None else device
        _lib.check(_lib.lib().glb_find_offsets(_lib.ptr64(pre), size, int(edges_per_thread),
                                               int(threads), _lib.ptr64(node), _lib.ptr64(edge),
                                               dev), "glb_find_offsets")
    return OffsetTable(node.tolist(), edge.tolist())
