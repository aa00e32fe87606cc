"""Experiment: does a sorted worklist speed up the relax kernel on C3?

    GRAPHLB_B200_LIB=_exp/sort.so python tools/c3_sort_probe.py [--k 4096] [--tags BS,HP]
    python tools/c3_sort_probe.py --env GLB_BM_THR --thr 32768   # the id-ordered frontiers

The `_exp/sort.so` build (-DGLB_EXP_SORT) radix-sorts the in-list before every
host-loop relax step holding >= GLB_SORT_THR items; the sort itself is outside
the per-launch events, so the records show the relax kernel alone.  With
--env GLB_BM_THR the product's bitmap compaction is toggled instead (off =
GLB_BM_THR=0); its kernel is inside the relax step's events.
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1711_00231_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--k", type=int, default=4096)
ap.add_argument("--tags", default="BS")
ap.add_argument("--algo", default="sssp")
ap.add_argument("--thr", default="8192")
ap.add_argument("--env", default="GLB_SORT_THR")
a = ap.parse_args()
g = pkg.grid_graph(a.k, seed=1, max_weight=255)
ref = None
for tag in a.tags.split(","):
    for thr in ("", a.thr, "", a.thr):
        if thr:
            os.environ[a.env] = thr
        elif a.env == "GLB_SORT_THR":
            os.environ.pop(a.env, None)
        else:
            os.environ[a.env] = "0"
        r = pkg.run_strategy(tag, g, 0, pkg.RelaxOp(a.algo), pkg.KernelConfig(loop="host"))
        if ref is None:
            ref = r.dist
        ok = bool(np.array_equal(ref, r.dist))
        k = np.array([x.kernel_wall_time for x in r.records]) * 1e3
        act = np.array([x.active_items for x in r.records])
        print(f"{tag} sort_thr={thr or 'off'} equal={ok} iters={len(k)} kernel_ms={k.sum():.2f}")
        for lo, hi in ((0, 8192), (8192, 131072), (131072, 1 << 30)):
            m = (act >= lo) & (act < hi)
            if m.any():
                print(f"   active [{lo},{hi}): {m.sum():5d} iters, kernel {k[m].sum():8.2f} ms "
                      f"({k[m].mean()*1e3:6.1f} us avg)")
        sys.stdout.flush()
