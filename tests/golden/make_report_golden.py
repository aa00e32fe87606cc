"""Golden outputs of the REFERENCE's harness / report code (bench.py:117-160,
report.py:37-184), produced here where /root/reference exists:

    python tests/golden/make_report_golden.py

* summarize_run + emit_report (csv and json) over a fixed set of synthetic
  invocation records (per-thread work lists), so the drop-in's summaries and
  report text can be compared byte for byte;
* emit_degree_histogram (plain and pre/post split) on corpus graphs.
Writes tests/golden/report.json.
"""
import dataclasses
import json
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import graphlb  # noqa: E402
from graphlb import bench, report  # noqa: E402
from graphlb.strategies.common import StrategyRun  # noqa: E402

from tests import graph_specs as gs  # noqa: E402

OUT = Path(__file__).resolve().parent / "report.json"

# (strategy, iteration, sub, active, per-thread work, relax, push, kernel s, overhead s)
RECORDS = {
    "WD": [(0, None, 1, [3, 0, 5, 8], 16, 4, 0.00125, 0.0005),
           (1, None, 4, [7, 7, 6, 7, 0, 1], 28, 9, 0.0025, 0.00075)],
    "HP": [(0, None, 1, [9, 0], 9, 3, 0.001, 0.0),
           (1, 0, 3, [4, 4, 4], 12, 2, 0.0005, 0.0),
           (1, 1, 2, [2, 5], 7, 1, 0.00025, 0.0)],
    "EP": [],
}


def make_runs():
    runs = []
    for tag, recs in RECORDS.items():
        mr = [graphlb.MetricsRecord(it, tag if sub is None or tag != "HP" else "HP", act, list(w),
                                    rx, px, k, o, sub)
              for it, sub, act, w, rx, px, k, o in recs]
        status = "ok" if recs else "infeasible: memory"
        runs.append(StrategyRun(tag, None, mr, status, 0.002 if tag == "WD" else 0.0,
                                87 if tag == "HP" else None, None))
    return runs


def main():
    out = {"records": {k: [list(r[:3]) + [r[3]] + list(r[4:]) for r in v]
                       for k, v in RECORDS.items()}}
    runs = make_runs()
    entries = [(bench.summarize_run(r, "sssp", "synthetic", True if r.feasible else None), r)
               for r in runs]
    out["summaries"] = [dataclasses.asdict(s) for s, _ in entries]
    with tempfile.TemporaryDirectory() as td:
        for fmt in ("csv", "json"):
            p = Path(td) / f"r.{fmt}"
            report.emit_report(entries, p, format=fmt)
            out[f"report_{fmt}"] = p.read_text()
        hist = {}
        for gid in ("rmat10_s1", "rmat10_skew", "degrees", "er_empty", "path17"):
            g = gs.build(graphlb, gs.CORPUS[gid])
            p = Path(td) / "h.csv"
            report.emit_degree_histogram(g, 10, p)
            hist[f"{gid}|plain"] = p.read_text()
            mdt = graphlb.compute_mdt(graphlb.build_histogram(g, 10))
            sp = graphlb.split_graph(g, mdt)
            report.emit_degree_histogram(g, 10, p, split=sp)
            hist[f"{gid}|split"] = p.read_text()
        out["degree_hist"] = hist
    OUT.write_text(json.dumps(out, indent=1))
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
