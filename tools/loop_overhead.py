"""Per-iteration cost of the device loop with (almost) no work: BFS along a
path graph, one frontier node per iteration, grid kernels only
(GLB_NO_SMALL=1) vs the cluster small loop, host vs graph loop.

    python tools/loop_overhead.py [--n 4000]
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1711_00231_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4000)
a = ap.parse_args()
g = pkg.path_graph(a.n)
ENVS = [{}, {"GLB_NO_SMALL": "1"}, {"GLB_NO_SMALL": "1", "GLB_NO_FUSED_CTL": "1"},
        {"GLB_NO_SMALL": "1", "GLB_GRAPH_UNROLL": "1"}]
for env in ENVS:
    for k in ("GLB_NO_SMALL", "GLB_NO_FUSED_CTL", "GLB_GRAPH_UNROLL"):
        os.environ.pop(k, None)
    os.environ.update(env)
    for tag in ("BS", "WD", "HP"):
        for loop in ("graph", "host"):
            best = None
            for _ in range(3):
                r = pkg.run_strategy(tag, g, 0, pkg.RelaxOp("bfs"), pkg.KernelConfig(loop=loop))
                ms = r.device["device_ms"]
                best = ms if best is None or ms < best else best
            it = len(r.records)
            print(f"{str(env):55s} {tag} {loop:5s} {best:8.2f} ms  {it} iters  {best / it * 1e3:6.2f} us/iter")
