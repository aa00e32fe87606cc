"""Run one strategy a few times on a benchmark graph (for ncu / nsight captures).

    python tools/profile_run.py --strategy WD --algo sssp --scale 22 --runs 2 [--loop graph]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_1711_00231_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--strategy", default="WD")
ap.add_argument("--algo", default="sssp")
ap.add_argument("--scale", type=int, default=22)
ap.add_argument("--edge-factor", type=int, default=16)
ap.add_argument("--skewed", action="store_true")
ap.add_argument("--runs", type=int, default=2)
ap.add_argument("--loop", default="graph")
ap.add_argument("--records", action="store_true")
a = ap.parse_args()
params = (0.7, 0.15, 0.10, 0.05) if a.skewed else pkg.DEFAULT_RMAT_PARAMS
g = pkg.generate_rmat(a.scale, a.edge_factor, params=params, seed=1, max_weight=255)
cfg = pkg.KernelConfig(loop=a.loop)
for tag in a.strategy.split(","):
    for i in range(a.runs):
        t = time.perf_counter()
        r = pkg.run_strategy(tag, g, 0, pkg.RelaxOp(a.algo), cfg)
        print(tag, i, f"{(time.perf_counter()-t)*1e3:.2f} ms wall",
              f"{r.device['device_ms']:.3f} ms device", r.device["launches"], "launches", flush=True)
        if a.records and i == a.runs - 1:
            tot_k = tot_o = 0.0
            for rec in r.records:
                tot_k += rec.kernel_wall_time
                tot_o += rec.overhead_wall_time
                gb = (12 if a.algo == "sssp" else 8) * rec.work_total() + 20 * rec.active_items
                print(f"  it {rec.iteration:3d} sub {str(rec.sub_iteration):4s} {rec.strategy:11s} "
                      f"items {rec.active_items:9d} edges {rec.work_total():10d} "
                      f"k {rec.kernel_wall_time*1e6:8.1f}us o {rec.overhead_wall_time*1e6:7.1f}us "
                      f"{gb / max(rec.kernel_wall_time, 1e-9) / 1e9:7.1f} GB/s "
                      f"max {rec.work_max()} push {rec.atomic_push_ops}")
            print(f"  sum kernel {tot_k*1e3:.3f} ms overhead {tot_o*1e3:.3f} ms device {r.device['device_ms']:.3f} ms")
