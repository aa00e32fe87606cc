"""Invocation records of the drop-in feed the reference's own imbalance summary.

The reference folds a run's ``MetricsRecord``s into one row with
``summarize_run`` (graphlb/bench.py:120-164): it iterates every record's
``per_thread_work`` and calls ``work_stddev()``, ``total_kernel_time()`` ...
The drop-in must present the same surface, so a caller's harness runs
unchanged over it.

CPU tier:
* the records of tests/golden/report.json (synthetic invocations whose
  summaries the REFERENCE computed) rebuilt as this package's MetricsRecord /
  StrategyRun, summarised by ``summarize_like_reference`` below (a restatement
  of bench.py:120-164) -> equal to the reference's summaries;
* when /root/reference is present (this container, not the GPU box): the
  reference's summarize_run itself over the same objects.
GPU tier: device runs carry exact per-thread work lists (the instrumented
device counters), so the reference summary of a device run is consistent with
the device's summed counters.
"""

import dataclasses
import json
import math
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_1711_00231_b200 as pkg
from tests import graph_specs as gs

GOLD = json.loads((Path(__file__).parent / "golden" / "report.json").read_text())
REF_SRC = Path("/root/reference/pkg/src")


def summarize_like_reference(run, algo, graph_name, verified=None):
    """bench.py:120-164, restated field for field (test helper only)."""
    count = total = sumsq = wmax = 0
    stddev_summed = 0.0
    for rec in run.records:
        for w in rec.per_thread_work:
            count += 1
            total += w
            sumsq += w * w
            wmax = max(wmax, w)
        stddev_summed += rec.work_stddev()
    avg = total / count if count else 0.0
    var = sumsq / count - avg * avg if count else 0.0
    return dict(
        strategy=run.strategy, algo=algo, graph=graph_name, status=run.status,
        iterations=1 + max((r.iteration for r in run.records), default=-1),
        sub_iterations=sum(1 for r in run.records if r.sub_iteration is not None),
        kernel_time=run.total_kernel_time(), overhead_time=run.total_overhead_time(),
        atomic_relax_ops=sum(r.atomic_relax_ops for r in run.records),
        atomic_push_ops=sum(r.atomic_push_ops for r in run.records),
        total_active_items=sum(r.active_items for r in run.records),
        threads_max=max((r.threads for r in run.records), default=0),
        work_max=wmax, work_avg=avg, work_stddev=math.sqrt(max(0.0, var)),
        work_stddev_summed=stddev_summed, verified=verified, mdt=run.mdt,
        split_fraction=run.split_fraction)


def _runs():
    runs = []
    for tag, recs in GOLD["records"].items():
        out = [pkg.MetricsRecord(it, tag, act, list(w), rx, px, k, o, sub)
               for it, sub, act, w, rx, px, k, o in recs]
        runs.append(pkg.StrategyRun(tag, None, out, "ok" if recs else pkg.INFEASIBLE_MEMORY,
                                    0.002 if tag == "WD" else 0.0, 87 if tag == "HP" else None,
                                    None))
    return runs


def _close(got, want):
    for key, w in want.items():
        if isinstance(w, float):
            assert math.isclose(got[key], w, rel_tol=1e-12, abs_tol=1e-15), key
        else:
            assert got[key] == w, key


def test_records_summarise_like_the_reference():
    for run, want in zip(_runs(), GOLD["summaries"]):
        got = summarize_like_reference(run, "sssp", "synthetic", True if run.feasible else None)
        _close(got, want)


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference sources only exist in the build container")
def test_reference_summarize_run_accepts_the_drop_in():
    sys.path.insert(0, str(REF_SRC))
    try:
        from graphlb import bench as ref_bench
    finally:
        sys.path.remove(str(REF_SRC))
    for run, want in zip(_runs(), GOLD["summaries"]):
        s = ref_bench.summarize_run(run, "sssp", "synthetic", True if run.feasible else None)
        _close(dataclasses.asdict(s), want)


def test_summed_counters_agree_with_lists():
    """MetricsRecord built from device sums (no list) reports the same
    per-record statistics as the list it summarises."""
    for run in _runs():
        for r in run.records:
            w = r.per_thread_work
            s = pkg.MetricsRecord(r.iteration, r.strategy, r.active_items, None, r.atomic_relax_ops,
                                  r.atomic_push_ops, r.kernel_wall_time, r.overhead_wall_time,
                                  r.sub_iteration, n_threads=len(w), total_work=sum(w),
                                  max_work=max(w), work_sumsq=float(sum(x * x for x in w)))
            assert (s.threads, s.work_total(), s.work_max()) == (r.threads, r.work_total(), r.work_max())
            assert math.isclose(s.work_stddev(), r.work_stddev(), rel_tol=1e-12, abs_tol=1e-15)


# ---------------------------------------------------------------- GPU tier
@pytest.mark.gpu
def test_device_runs_carry_exact_per_thread_work():
    g = gs.build(pkg, gs.CORPUS["rmat10_skew"])
    for loop in ("host", "graph"):
        for tag in pkg.STRATEGY_TAGS:
            for algo in ("bfs", "sssp"):
                run = pkg.run_strategy(tag, g, 0, pkg.RelaxOp(algo), pkg.KernelConfig(loop=loop))
                for r in run.records:
                    w = np.asarray(r.per_thread_work, dtype=np.int64)
                    assert w.size == r.threads, (tag, algo, loop)
                    assert int(w.sum()) == r.total_work and int(w.max(initial=0)) == r.max_work
                s = summarize_like_reference(run, algo, "rmat10_skew")
                assert s["work_max"] == max(r.work_max() for r in run.records)
                assert s["atomic_relax_ops"] == run.device["relax_ops"]


@pytest.mark.gpu
def test_distance_certificate_rejects_wrong_arrays(golden):
    for gid in ("rmat10_s1", "quirks", "path17", "er1024"):
        g = gs.build(pkg, gs.CORPUS[gid])
        for algo in ("bfs", "sssp"):
            exp = golden["corpus"][f"{gid}|0|{algo}"].copy()
            ok = pkg.validate_distances(g, 0, algo, exp)
            assert ok.matched and ok.mismatch_count == 0
            reached = np.flatnonzero((exp != pkg.INF) & (np.arange(exp.size) != 0))
            unreached = np.flatnonzero(exp == pkg.INF)
            cases = []
            if reached.size:
                v = int(reached[reached.size // 2])
                for delta in (+1, -1):
                    d = exp.copy()
                    d[v] += delta
                    cases.append((d, v))
                d = exp.copy()
                d[v] = pkg.INF
                cases.append((d, v))
            if unreached.size:
                d = exp.copy()
                d[int(unreached[0])] = 3
                cases.append((d, int(unreached[0])))
            d = exp.copy()
            d[0] = 1
            cases.append((d, 0))
            for d, v in cases:
                r = pkg.validate_distances(g, 0, algo, d)
                assert not r.matched and r.mismatch_count >= 1, (gid, algo, v)
                assert r.first_mismatch[0] <= v or d[r.first_mismatch[0]] != exp[r.first_mismatch[0]]
    # a zero-weight cycle cannot certify itself: nodes 1 <-> 2 unreachable from 0
    g = pkg.CsrGraph.from_edges(3, [1, 2], [2, 1], [0, 0])
    r = pkg.validate_distances(g, 0, "sssp", [0, 5, 5])
    assert not r.matched and r.mismatch_count == 2 and r.first_mismatch == (1, None, 5)
    assert pkg.validate_distances(g, 0, "sssp", [0, pkg.INF, pkg.INF]).matched
