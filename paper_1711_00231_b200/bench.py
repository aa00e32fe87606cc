"""Benchmark harness on the device (drop-in for graphlb/bench.py:1-226).

Runs the requested strategies on one graph through the CUDA path and folds
each run's invocation records into an ImbalanceSummary, with the same
dataclasses, columns and error behaviour as the reference harness:

* ``RunConfig`` (bench.py:37-71) gains ``device`` and ``loop``; ``threads``,
  ``workers`` and ``replay`` are validated and kept but, as in KernelConfig,
  steered only the CPU emulation;
* ``summarize_run`` (bench.py:117-160) pools the per-thread work of every
  invocation -- from the device's exact per-launch sum / sum of squares / max
  instead of a per-thread list, so the pooled count, mean, max and stddev are
  the reference's formulas over the same values;
* ``run_benchmark(verify=True)`` (bench.py:176-209) checks every feasible
  result with the device distance certificate (glb_validate: d[src] = 0, no
  relaxable edge, every reached node tight-reachable from the source) instead
  of running a sequential oracle on the host, and raises VerificationError on
  the first violation.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from pathlib import Path

from . import _lib
from .analysis import VerificationReport, validate_distances
from .graph import COO_ID_BYTES, DEFAULT_COO_BUDGET_BYTES, DEFAULT_RMAT_PARAMS, CsrGraph
from .graph import generate_er, generate_rmat
from .io import load_dimacs_gr, load_edge_list, read_csr_bin
from .runtime import KernelConfig
from .strategies import STRATEGY_TAGS, RelaxOp, StrategyRun, run_strategy


class VerificationError(RuntimeError):
    """A strategy's distances failed verification (bench.py:23-34)."""

    def __init__(self, strategy: str, report: VerificationReport):
        node, exp, act = report.first_mismatch
        want = "a certified distance" if exp is None else exp
        super().__init__(
            f"{strategy}: {report.mismatch_count} mismatching distance cells; "
            f"first at node {node}: expected {want}, got {act}"
        )
        self.strategy = strategy
        self.report = report


@dataclass
class RunConfig:
    """Declarative description of one benchmark run (bench.py:37-71)."""

    graph_path: str | None = None
    graph_format: str = "dimacs"  # dimacs | edgelist | bin
    weighted_edgelist: bool = True
    gen: str | None = None  # rmat | er
    scale: int = 14
    edge_factor: int = 8
    rmat_params: tuple[float, float, float, float] = DEFAULT_RMAT_PARAMS

    algo: str = "sssp"
    strategies: tuple[str, ...] = STRATEGY_TAGS
    source: int = 0
    threads: int | None = None
    workers: int = 1
    bins: int = 10
    mdt: int | None = None
    chunked: bool = True
    mem_budget_bytes: int = DEFAULT_COO_BUDGET_BYTES
    seed: int = 1
    verify: bool = False
    replay: bool = False
    graph_name: str = ""
    device: int | None = None
    loop: str = "host"

    def kernel_config(self) -> KernelConfig:
        return KernelConfig(
            virtual_threads=self.threads,
            workers=self.workers,
            deterministic_replay=self.replay,
            device=self.device,
            loop=self.loop,
        )


def load_graph(cfg: RunConfig) -> tuple[str, CsrGraph]:
    """Resolve the configured graph source to a (name, graph) pair (bench.py:74-96).
    Generators run on the device (bit-identical to numpy's stream)."""
    if cfg.graph_path is not None:
        path = Path(cfg.graph_path)
        if cfg.graph_format == "dimacs":
            g = load_dimacs_gr(path)
        elif cfg.graph_format == "edgelist":
            g = load_edge_list(path, weighted=cfg.weighted_edgelist)
        elif cfg.graph_format == "bin":
            g = read_csr_bin(path)
        else:
            raise ValueError(f"unknown graph format {cfg.graph_format!r}")
        return cfg.graph_name or path.name, g
    if cfg.gen == "rmat":
        dev = cfg.device if cfg.device is not None else (
            _lib.default_device() if _lib.device_count() > 0 else None)
        g = generate_rmat(cfg.scale, cfg.edge_factor, cfg.rmat_params, seed=cfg.seed, device=dev)
        return cfg.graph_name or f"rmat{cfg.scale}", g
    if cfg.gen == "er":
        n = 1 << cfg.scale
        g = generate_er(n, cfg.edge_factor * n, seed=cfg.seed)
        return cfg.graph_name or f"er{cfg.scale}", g
    raise ValueError("run config names neither a graph file nor a generator")


@dataclass
class ImbalanceSummary:
    """Per-strategy totals over all kernel invocations of a run (bench.py:99-114)."""

    strategy: str
    algo: str
    graph: str
    status: str
    iterations: int
    sub_iterations: int
    kernel_time: float
    overhead_time: float
    atomic_relax_ops: int
    atomic_push_ops: int
    total_active_items: int
    threads_max: int
    work_max: int
    work_avg: float
    work_stddev: float
    work_stddev_summed: float
    verified: bool | None = None
    mdt: int | None = None
    split_fraction: float | None = None


def summarize_run(run: StrategyRun, algo: str, graph_name: str,
                  verified: bool | None = None) -> ImbalanceSummary:
    """Fold a run's invocation records into one summary row (bench.py:117-160):
    work_max/avg/stddev pool every per-thread work value across invocations,
    work_stddev_summed adds up the per-invocation deviations."""
    count = total = wmax = 0
    sumsq = 0.0
    stddev_summed = 0.0
    for rec in run.records:
        if rec.per_thread_work is not None:
            count += len(rec.per_thread_work)
            total += sum(rec.per_thread_work)
            sumsq += float(sum(w * w for w in rec.per_thread_work))
        else:
            count += rec.threads
            total += rec.work_total()
            sumsq += rec.work_sumsq
        wmax = max(wmax, rec.work_max())
        stddev_summed += rec.work_stddev()
    avg = total / count if count else 0.0
    var = sumsq / count - avg * avg if count else 0.0
    return ImbalanceSummary(
        strategy=run.strategy,
        algo=algo,
        graph=graph_name,
        status=run.status,
        iterations=1 + max((r.iteration for r in run.records), default=-1),
        sub_iterations=sum(1 for r in run.records if r.sub_iteration is not None),
        kernel_time=run.total_kernel_time(),
        overhead_time=run.total_overhead_time(),
        atomic_relax_ops=sum(r.atomic_relax_ops for r in run.records),
        atomic_push_ops=sum(r.atomic_push_ops for r in run.records),
        total_active_items=sum(r.active_items for r in run.records),
        threads_max=max((r.threads for r in run.records), default=0),
        work_max=wmax,
        work_avg=avg,
        work_stddev=math.sqrt(max(0.0, var)),
        work_stddev_summed=stddev_summed,
        verified=verified,
        mdt=run.mdt,
        split_fraction=run.split_fraction,
    )


@dataclass
class RunResult:
    graph: str
    algo: str
    entries: list[tuple[ImbalanceSummary, StrategyRun]] = field(default_factory=list)

    @property
    def summaries(self) -> list[ImbalanceSummary]:
        return [s for s, _ in self.entries]

    @property
    def all_infeasible(self) -> bool:
        return bool(self.entries) and all(not run.feasible for _, run in self.entries)


def run_benchmark(cfg: RunConfig, graph: CsrGraph | None = None,
                  graph_name: str | None = None) -> RunResult:
    """Execute every requested strategy on the same graph (bench.py:176-209).
    Infeasible strategies are reported in their summary row; with ``verify``
    a result that fails the distance certificate raises VerificationError."""
    if graph is None:
        graph_name, graph = load_graph(cfg)
    elif graph_name is None:
        graph_name = cfg.graph_name or "graph"
    if not 0 <= cfg.source < graph.num_nodes:
        raise ValueError(f"source {cfg.source} out of range for {graph.num_nodes} nodes")
    if not cfg.strategies:
        raise ValueError("at least one strategy is required")
    op = RelaxOp(cfg.algo)
    kcfg = cfg.kernel_config()
    result = RunResult(graph_name, cfg.algo)
    for tag in cfg.strategies:
        run = run_strategy(tag, graph, cfg.source, op, kcfg, bins=cfg.bins, mdt=cfg.mdt,
                           chunked=cfg.chunked, max_cells=cfg.mem_budget_bytes // COO_ID_BYTES)
        verified = None
        if cfg.verify and run.feasible:
            report = validate_distances(graph, cfg.source, cfg.algo, run.dist, device=cfg.device)
            if not report.matched:
                raise VerificationError(run.strategy, report)
            verified = True
        result.entries.append((summarize_run(run, cfg.algo, graph_name, verified), run))
    return result


def paper_desk_suite(seed: int = 1) -> list[tuple[str, CsrGraph]]:
    """Default benchmark corpus (bench.py:212-218)."""
    return [
        ("rmat14", generate_rmat(14, 8, seed=seed)),
        ("rmat16", generate_rmat(16, 8, seed=seed)),
        ("er14", generate_er(1 << 14, 4 << 14, seed=seed)),
    ]
