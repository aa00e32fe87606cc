"""Launch configuration, distance cells and per-launch metrics.

Counterparts of graphlb's engine.py types, re-expressed for real device
launches: the virtual-thread emulation (launch_kernel, ThreadCtx, Python
locks) is replaced by CUDA kernels in libgraphlb_b200.so, and per-thread work
is summarised on the device (sum, sum of squares, max) instead of being
shipped back as a T-long list.
"""

from __future__ import annotations

from dataclasses import dataclass
from math import sqrt

import numpy as np

INF = (1 << 63) - 1            # engine.py:27
MAX_DEFAULT_THREADS = 1 << 14  # engine.py:28 (reference emulation cap; reported only)

LOOP_MODES = ("host", "graph")


class KernelLaunchError(RuntimeError):
    """A kernel failed (engine.py:31-36); thread_id is -1 for device failures."""

    def __init__(self, thread_id: int, cause: BaseException):
        super().__init__(f"kernel body failed on virtual thread {thread_id}: {cause!r}")
        self.thread_id = thread_id


@dataclass
class KernelConfig:
    """Launch configuration (engine.py:39-60) plus the device knobs.

    ``block_size`` keeps its reference role as the HP fallback threshold
    (hierarchical.py:49).  ``virtual_threads``/``workers``/``deterministic_replay``/
    ``schedule_seed`` only steered the CPU emulation; they are validated and
    kept for compatibility, the device sizes its own grids.  ``loop`` picks the
    device-driven CUDA graph ("graph", the default: one launch per traversal)
    or the host-driven loop ("host", one round trip per launch, CUDA-event
    time per launch).  ``dist_bits`` 0 picks the distance tier (24-bit cells
    for graphs whose 64-bit cells exceed twice the L2, else 32-bit), re-running
    at the next width on overflow; 24 / 32 / 64 pin one width.
    ``instrument`` records every launch's exact per-thread work list on the
    device (``MetricsRecord.per_thread_work``, as the reference's harness
    consumes it, bench.py:120-164); off, records carry the device's summed
    counters (sum, sum of squares, max) only.
    """

    virtual_threads: int | None = None
    block_size: int = 1024
    workers: int = 1
    deterministic_replay: bool = False
    schedule_seed: int | None = None
    device: int | None = None
    loop: str = "graph"
    dist_bits: int = 0
    record_timing: bool = True
    instrument: bool = True

    def __post_init__(self):
        if self.virtual_threads is not None and self.virtual_threads < 1:
            raise ValueError("virtual_threads must be >= 1")
        if self.block_size < 1:
            raise ValueError("block_size must be >= 1")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.loop not in LOOP_MODES:
            raise ValueError(f"loop must be one of {LOOP_MODES}")
        if self.dist_bits not in (0, 24, 32, 64):
            raise ValueError("dist_bits must be 0, 24, 32 or 64")


def resolve_threads(cfg: KernelConfig, active_items: int) -> int:
    """Reference thread-count rule (engine.py:63-70), kept for callers that
    size host-side tables such as find_offsets."""
    if cfg.virtual_threads is not None:
        return cfg.virtual_threads
    active_items = max(active_items, 1)
    blocks = -(-active_items // cfg.block_size)
    return min(MAX_DEFAULT_THREADS, blocks * cfg.block_size)


class DistArray:
    """Distance cells with the INF sentinel (engine.py:90-117).

    Backed by an int64 numpy array; ``values`` materialises the reference's
    list-of-int view on first use.
    """

    __slots__ = ("_a", "_list")

    def __init__(self, num_nodes: int, source: int | None = None):
        self._a = np.full(num_nodes, INF, dtype=np.int64)
        self._list = None
        if source is not None:
            if not 0 <= source < num_nodes:
                raise IndexError(f"source {source} out of range for {num_nodes} nodes")
            self._a[source] = 0

    @classmethod
    def from_array(cls, a: np.ndarray) -> "DistArray":
        d = cls.__new__(cls)
        d._a = np.ascontiguousarray(a, dtype=np.int64)
        d._list = None
        return d

    @property
    def array(self) -> np.ndarray:
        return self._a

    @property
    def values(self) -> list[int]:
        if self._list is None:
            self._list = self._a.tolist()
        return self._list

    def __len__(self) -> int:
        return int(self._a.shape[0])

    def __getitem__(self, node):
        return int(self._a[node]) if isinstance(node, (int, np.integer)) else self._a[node]

    def __eq__(self, other) -> bool:
        if isinstance(other, DistArray):
            return bool(np.array_equal(self._a, other._a))
        if isinstance(other, (list, tuple, np.ndarray)):
            o = np.asarray(other, dtype=np.int64)
            return o.shape == self._a.shape and bool(np.array_equal(self._a, o))
        if hasattr(other, "values"):
            return self.values == list(other.values)
        return NotImplemented

    __hash__ = None

    def to_list(self) -> list[int]:
        return list(self.values)

    def __repr__(self) -> str:
        return f"DistArray({self._a!r})"


@dataclass(eq=False)
class MetricsRecord:
    """Counters of one kernel invocation (engine.py:142-174).

    ``per_thread_work`` is the exact per-thread list of an instrumented run
    (an int64 numpy array, one entry per launched thread) or None; either way
    ``total_work``, ``max_work`` and ``work_sumsq`` hold the device's summed
    counters over ``n_threads`` threads and the accessors use them.  Wall
    times are seconds of device time on the library stream.
    """

    iteration: int
    strategy: str
    active_items: int
    per_thread_work: list[int] | None
    atomic_relax_ops: int
    atomic_push_ops: int
    kernel_wall_time: float
    overhead_wall_time: float = 0.0
    sub_iteration: int | None = None
    n_threads: int = 0
    total_work: int = 0
    max_work: int = 0
    work_sumsq: float = 0.0

    def _list(self):
        # a plain list given by the caller wins; device runs carry counters too
        w = self.per_thread_work
        if w is None or (self.n_threads and isinstance(w, np.ndarray)):
            return None
        return w

    @property
    def threads(self) -> int:
        w = self._list()
        return len(w) if w is not None else self.n_threads

    def work_total(self) -> int:
        w = self._list()
        return sum(w) if w is not None else self.total_work

    def work_max(self) -> int:
        w = self._list()
        if w is not None:
            return max(w) if len(w) else 0
        return self.max_work

    def work_avg(self) -> float:
        t = self.threads
        return self.work_total() / t if t else 0.0

    def work_stddev(self) -> float:
        t = self.threads
        if t == 0:
            return 0.0
        w = self._list()
        if w is not None:
            avg = self.work_total() / t
            return sqrt(sum((x - avg) ** 2 for x in w) / t)
        avg = self.total_work / t
        var = self.work_sumsq / t - avg * avg
        return sqrt(var) if var > 0 else 0.0
