"""Per-iteration records of one strategy on the C3 grid (or a smaller k).

    python tools/profile_grid.py --k 4096 --strategy WD --algo sssp [--loop host]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1711_00231_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--k", type=int, default=4096)
ap.add_argument("--strategy", default="WD")
ap.add_argument("--algo", default="sssp")
ap.add_argument("--loop", default="host")
a = ap.parse_args()
g = pkg.grid_graph(a.k, seed=1, max_weight=255)
cfg = pkg.KernelConfig(loop=a.loop)
pkg.run_strategy(a.strategy, g, 0, pkg.RelaxOp(a.algo), cfg)
r = pkg.run_strategy(a.strategy, g, 0, pkg.RelaxOp(a.algo), cfg)
recs = r.records
print(f"{a.strategy} {a.algo} k={a.k}: device {r.device['device_ms']:.2f} ms, {len(recs)} records, "
      f"launches {r.device['launches']}")
items = np.array([x.active_items for x in recs])
edges = np.array([x.work_total() for x in recs])
kt = np.array([x.kernel_wall_time for x in recs]) * 1e6
ot = np.array([x.overhead_wall_time for x in recs]) * 1e6
thr = np.array([x.threads for x in recs])
for lo, hi in ((0, 1e3), (1e3, 8192), (8192, 65536), (65536, 1e12)):
    sel = (items >= lo) & (items < hi)
    if sel.any():
        print(f"items [{lo:g},{hi:g}): {sel.sum():6d} iters, edges/iter {edges[sel].mean():10.0f}, "
              f"kernel {kt[sel].mean():7.1f} us, overhead {ot[sel].mean():6.1f} us, "
              f"sum kernel {kt[sel].sum()/1e3:8.2f} ms, small-loop iters {(thr[sel] == 8192).sum()}")
print(f"sum kernel {kt.sum()/1e3:.2f} ms, sum overhead {ot.sum()/1e3:.2f} ms")
