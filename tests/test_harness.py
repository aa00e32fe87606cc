"""The benchmark harness, report and CLI (bench.py, report.py, cli.py of the
reference) on top of the device path.

CPU tier: summaries and report text against the reference's own output for
the same invocation records (tests/golden/report.json, made by
tests/golden/make_report_golden.py), both for per-thread work lists and for
the device's summed counters; CLI argument errors.
GPU tier: degree-histogram CSVs against the reference's, run_benchmark with
the device distance certificate, the certificate's rejections, CLI runs.
"""

import dataclasses
import json
import math
from pathlib import Path

import numpy as np
import pytest

import paper_1711_00231_b200 as pkg
from paper_1711_00231_b200 import bench, cli, report
from tests import graph_specs as gs

GOLD = json.loads((Path(__file__).parent / "golden" / "report.json").read_text())


def _runs(summed: bool):
    runs = []
    for tag, recs in GOLD["records"].items():
        out = []
        for it, sub, act, w, rx, px, k, o in recs:
            if summed:
                out.append(pkg.MetricsRecord(it, tag, act, None, rx, px, k, o, sub, n_threads=len(w),
                                             total_work=sum(w), max_work=max(w),
                                             work_sumsq=float(sum(x * x for x in w))))
            else:
                out.append(pkg.MetricsRecord(it, tag, act, list(w), rx, px, k, o, sub))
        runs.append(pkg.StrategyRun(tag, None, out, "ok" if recs else pkg.INFEASIBLE_MEMORY,
                                    0.002 if tag == "WD" else 0.0, 87 if tag == "HP" else None,
                                    None))
    return runs


def _entries(summed: bool):
    return [(bench.summarize_run(r, "sssp", "synthetic", True if r.feasible else None), r)
            for r in _runs(summed)]


def test_summaries_and_reports_match_reference(tmp_path):
    entries = _entries(summed=False)
    assert [dataclasses.asdict(s) for s, _ in entries] == GOLD["summaries"]
    for fmt in ("csv", "json"):
        p = report.emit_report(entries, tmp_path / f"r.{fmt}", format=fmt)
        assert p.read_text() == GOLD[f"report_{fmt}"], fmt
    rows = report.read_report_csv(tmp_path / "r.csv")
    assert [r["strategy"] for r in rows] == ["WD", "WD", "HP", "HP", "HP", "WD", "HP", "EP"]
    assert rows[-1]["status"] == pkg.INFEASIBLE_MEMORY and rows[-3]["status"] == "summary"
    with pytest.raises(ValueError):
        report.emit_report(entries, tmp_path / "r.x", format="xml")


def test_summed_device_counters_summarise_like_thread_lists(tmp_path):
    """The device ships exact per-launch sum / sum of squares / max, not a
    per-thread list; the pooled statistics must come out the same."""
    for (s, _), ref in zip(_entries(summed=True), GOLD["summaries"]):
        got = dataclasses.asdict(s)
        for key, want in ref.items():
            if isinstance(want, float):
                assert math.isclose(got[key], want, rel_tol=1e-12, abs_tol=1e-15), key
            else:
                assert got[key] == want, key
    p = report.emit_report(_entries(summed=True), tmp_path / "s.csv")
    q = report.emit_report(_entries(summed=False), tmp_path / "l.csv")
    a, b = report.read_report_csv(p), report.read_report_csv(q)
    for ra, rb in zip(a, b):
        for key in ra:
            if isinstance(rb[key], float):
                assert math.isclose(ra[key], rb[key], rel_tol=1e-12, abs_tol=1e-15), key
            else:
                assert ra[key] == rb[key], key


def test_cli_rejects_bad_configuration(tmp_path, capsys):
    assert cli.main([]) == cli.EXIT_CONFIG                      # no graph source
    assert cli.main(["--gen", "rmat", "--strategy", "bs,xx"]) == cli.EXIT_CONFIG
    assert cli.main(["--gen", "rmat", "--rmat-params", "0.5,0.5"]) == cli.EXIT_CONFIG
    assert cli.main(["--gen", "rmat", "--plot"]) == cli.EXIT_CONFIG
    bad = tmp_path / "bad.gr"
    bad.write_text("a 1 2 3\np sp 2 1\n")
    assert cli.main(["--graph", str(bad)]) == cli.EXIT_CONFIG    # ParseError
    assert cli.main(["--graph", str(tmp_path / "missing.gr")]) == cli.EXIT_CONFIG
    err = capsys.readouterr().err
    assert "arc line before problem line" in err and "unknown strategy tag 'XX'" in err
    assert cli._parse_strategies("all") == pkg.STRATEGY_TAGS
    assert cli._parse_strategies(" wd , hp ") == ("WD", "HP")


# ---------------------------------------------------------------- GPU tier
@pytest.mark.gpu
def test_degree_histogram_csv_matches_reference(tmp_path):
    for key, want in GOLD["degree_hist"].items():
        gid, kind = key.split("|")
        g = gs.build(pkg, gs.CORPUS[gid])
        split = None
        if kind == "split":
            split = pkg.split_graph(g, pkg.compute_mdt(pkg.build_histogram(g, 10)))
        p = report.emit_degree_histogram(g, 10, tmp_path / "h.csv", split=split)
        assert p.read_text() == want, key


@pytest.mark.gpu
def test_run_benchmark_certifies_every_strategy(golden):
    for gid in ("rmat10_s1", "rmat10_skew", "degrees", "quirks", "grid24"):
        g = gs.build(pkg, gs.CORPUS[gid])
        for algo in ("bfs", "sssp"):
            cfg = bench.RunConfig(algo=algo, verify=True, loop="graph")
            res = bench.run_benchmark(cfg, graph=g, graph_name=gid)
            assert [s.strategy for s in res.summaries] == list(pkg.STRATEGY_TAGS)
            exp = golden["corpus"][f"{gid}|0|{algo}"]
            for s, run in res.entries:
                assert s.verified is True and s.status == "ok"
                assert np.array_equal(run.dist.array, exp), (gid, algo, s.strategy)
                assert s.atomic_relax_ops == sum(r.atomic_relax_ops for r in run.records)
                assert s.iterations >= 1 and s.work_max >= 1
    with pytest.raises(ValueError):
        bench.run_benchmark(bench.RunConfig(source=10**6), graph=g)


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


@pytest.mark.gpu
def test_cli_end_to_end(tmp_path, capsys):
    out = tmp_path / "r.csv"
    hist = tmp_path / "h.csv"
    rc = cli.main(["--gen", "rmat", "--scale", "10", "--algo", "sssp", "--verify", "--out", str(out),
                   "--degree-hist", str(hist), "--loop", "graph"])
    assert rc == cli.EXIT_OK
    rows = report.read_report_csv(out)
    assert {r["strategy"] for r in rows if r["status"] == "summary"} == set(pkg.STRATEGY_TAGS)
    assert hist.read_text().startswith("phase,degree_bin_low")
    text = capsys.readouterr().out
    assert "rmat10" in text and "kern_ms" in text
    # every strategy infeasible -> 4 (EP under a zero COO budget)
    assert cli.main(["--gen", "er", "--scale", "8", "--strategy", "ep", "--mem-budget", "0"]) == \
        cli.EXIT_INFEASIBLE
    # paper-desk suite, BFS, one strategy
    assert cli.main(["--suite", "paper-desk", "--algo", "bfs", "--strategy", "wd", "--verify"]) == 0
