"""C3 (4096^2 grid) per-iteration breakdown: graph-loop device time vs the
host-loop records' kernel / scan times, and frontier-size histogram.

    python tools/c3_breakdown.py [--k 4096] [--strategies BS,WD] [--algo sssp]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1711_00231_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--k", type=int, default=4096)
ap.add_argument("--strategies", default="BS,WD,HP")
ap.add_argument("--algo", default="sssp")
a = ap.parse_args()
g = pkg.grid_graph(a.k, seed=1)
for tag in a.strategies.split(","):
    for loop in ("graph", "host"):
        r = pkg.run_strategy(tag, g, 0, pkg.RelaxOp(a.algo), pkg.KernelConfig(loop=loop))
        r = pkg.run_strategy(tag, g, 0, pkg.RelaxOp(a.algo), pkg.KernelConfig(loop=loop))
        recs = r.records
        k = np.array([x.kernel_wall_time for x in recs]) * 1e3
        o = np.array([x.overhead_wall_time for x in recs]) * 1e3
        act = np.array([x.active_items for x in recs])
        relax = np.array([x.atomic_relax_ops for x in recs])
        print(f"{tag} {loop}: device_ms {r.device['device_ms']:.2f} records {len(recs)} "
              f"sum kernel {k.sum():.2f} sum scan {o.sum():.2f}")
        if loop == "host":
            for lo, hi in ((0, 1024), (1024, 8192), (8192, 32768), (32768, 131072), (131072, 1 << 30)):
                m = (act >= lo) & (act < hi)
                if m.any():
                    print(f"   active [{lo},{hi}): {m.sum():5d} iters, kernel {k[m].sum():8.2f} ms "
                          f"({k[m].mean()*1e3:6.1f} us avg), scan {o[m].sum():7.2f}, "
                          f"relax {relax[m].sum()/1e6:8.1f}M")
