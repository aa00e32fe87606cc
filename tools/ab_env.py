"""A/B environment knobs read per run (GLB_*), interleaved in one process.

    python tools/ab_env.py GLB_GRAPH_UNROLL=1 GLB_GRAPH_UNROLL=4 [--strategy WD] [--algo sssp]
"""
import argparse
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1711_00231_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("variants", nargs="+")
ap.add_argument("--strategy", default="WD")
ap.add_argument("--algo", default="sssp")
ap.add_argument("--scale", type=int, default=22)
ap.add_argument("--reps", type=int, default=9)
ap.add_argument("--grid", type=int, default=0, help="k x k grid (C3: 4096) instead of an R-MAT")
ap.add_argument("--skewed", action="store_true", help="C4's skewed R-MAT parameters")
a = ap.parse_args()
g = (pkg.grid_graph(a.grid, seed=1, max_weight=255) if a.grid else
     pkg.generate_rmat(a.scale, 16, params=(0.7, 0.15, 0.10, 0.05) if a.skewed else pkg.DEFAULT_RMAT_PARAMS,
                       seed=1, max_weight=255, device=0))
res = {v: [] for v in a.variants}
for rep in range(a.reps + 1):
    for v in a.variants:
        for kv in a.variants:
            os.environ.pop(kv.split("=")[0], None)
        if "=" in v:
            k, val = v.split("=", 1)
            os.environ[k] = val
        r = pkg.run_strategy(a.strategy, g, 0, pkg.RelaxOp(a.algo), pkg.KernelConfig(loop="graph"))
        if rep:
            res[v].append(r.device["device_ms"])
for v, xs in res.items():
    print(f"{v:28s} {a.strategy} {a.algo} median {statistics.median(xs):.3f} ms  min {min(xs):.3f}")
