"""C5 (RMAT s27 on one B200): id-ordered (dense) WD scans vs list order.

    python tools/c5_dense_probe.py [--scale 27] [--reps 2]

GLB_WD_DENSE=1 scans frontiers holding >= N/8 nodes from the distance cells in
node-id order (packed cells; default in the 24-bit tier), GLB_WD_DENSE=0 takes
the worklist.  --bits 0 lets the library pick the tier (24 on C5).
Interleaved runs, device ms, results compared between the arms.
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1711_00231_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=27)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--tags", default="WD")
ap.add_argument("--bits", type=int, default=32, help="cell tier (0: the library's choice, 24 on C5)")
a = ap.parse_args()
g = pkg.generate_rmat(a.scale, 16, seed=1, max_weight=255, device=0, download=False)
for algo in ("bfs", "sssp"):
    for tag in a.tags.split(","):
        res = {}
        ref = None
        for rep in range(a.reps + 1):
            for arm in ("list", "dense"):
                os.environ["GLB_WD_DENSE"] = "1" if arm == "dense" else "0"
                r = pkg.run_strategy(tag, g, 0, pkg.RelaxOp(algo), pkg.KernelConfig(dist_bits=a.bits))
                d = np.asarray(r.dist.array)
                if ref is None:
                    ref = d
                assert np.array_equal(ref, d), (algo, tag, arm)
                if rep:
                    res.setdefault(arm, []).append(r.device["device_ms"])
                    relax = sum(x.atomic_relax_ops for x in r.records)
                    res.setdefault(arm + "_relax", []).append(relax)
        for arm in ("list", "dense"):
            print(f"{tag} {algo} {arm:5s} ms {sorted(res[arm])}  relax {res[arm + '_relax'][0]}", flush=True)
