"""C3 per-bucket relax-step time with and without id-ordered BS frontiers.

    python tools/c3_sort_probe.py --env GLB_BM_THR --thr 32768 [--k 4096] [--tags BS]

The bitmap compaction (k_bm_compact) is toggled by GLB_BM_THR (off = 0); its
kernel is inside the relax step's host-loop events.  The first experiment
(session 3, profiles/r02_c3_sorted_lists.txt) used a throw-away build that
radix-sorted the in-list outside the events (GLB_SORT_THR): relax kernel alone,
53 -> 29.6 us per >131K-node step.
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
ap.add_argument("--env", default="GLB_BM_THR")
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
