"""C5 (RMAT s27, one B200): interleaved A/B of per-run GLB_* knobs.

    python tools/c5_env_probe.py GLB_NO_PDL=1 GLB_NO_PDL= GLB_BM_THR=0 --tags BS --algos bfs,sssp
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1711_00231_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("arms", nargs="+")
ap.add_argument("--scale", type=int, default=27)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--tags", default="BS")
ap.add_argument("--algos", default="bfs,sssp")
a = ap.parse_args()
g = pkg.generate_rmat(a.scale, 16, seed=1, max_weight=255, device=0, download=False)
keys = {arm.split("=", 1)[0] for arm in a.arms}
for algo in a.algos.split(","):
    for tag in a.tags.split(","):
        res, ref = {}, None
        for rep in range(a.reps + 1):
            for arm in a.arms:
                for k in keys:
                    os.environ.pop(k, None)
                k, _, v = arm.partition("=")
                if v:
                    os.environ[k] = v
                r = pkg.run_strategy(tag, g, 0, pkg.RelaxOp(algo), pkg.KernelConfig())
                d = np.asarray(r.dist.array)
                if ref is None:
                    ref = d
                assert np.array_equal(ref, d), (algo, tag, arm)
                if rep:
                    res.setdefault(arm, []).append(round(r.device["device_ms"], 2))
        for arm in a.arms:
            print(f"{tag} {algo} {arm:18s} ms {sorted(res[arm])}", flush=True)
