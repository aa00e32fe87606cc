"""A/B several builds of libgraphlb_b200.so on one graph in one process.

    python tools/ab_libs.py lib1.so lib2.so ... [--strategy WD,HP] [--algo sssp] [--reps 5]

Each library gets its own device graph; runs are interleaved round-robin so
clock drift hits every variant alike.  Prints the median device_ms per
(library, strategy).
"""
import argparse
import ctypes
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import paper_1711_00231_b200 as pkg  # noqa: E402
from paper_1711_00231_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--strategy", default="WD")
ap.add_argument("--algo", default="sssp")
ap.add_argument("--scale", type=int, default=22)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--loop", default="graph")
ap.add_argument("--skewed", action="store_true")
ap.add_argument("--dist-bits", type=int, default=0)
ap.add_argument("--grid", type=int, default=0, help="k x k grid (C3: 4096) instead of an R-MAT")
a = ap.parse_args()
params = (0.7, 0.15, 0.10, 0.05) if a.skewed else pkg.DEFAULT_RMAT_PARAMS
g = (pkg.grid_graph(a.grid, seed=1, max_weight=255) if a.grid else
     pkg.generate_rmat(a.scale, 16, params=params, seed=1, max_weight=255))
from oracle import oracle  # noqa: E402

exp = oracle.oracle_distances(g, 0, a.algo)

libs = []
bits_of = {}
for spec in a.libs:  # "lib.so" or "lib.so:24" (per-library dist_bits)
    path, _, b = spec.partition(":")
    path = spec if not b else path + ":" + b
    bits_of[path] = int(b) if b else a.dist_bits
    L = ctypes.CDLL(str(Path(path.partition(":")[0]).resolve()))
    for name, (res, args) in _lib.SIGNATURES.items():
        if not hasattr(L, name):  # older builds lack newer entry points
            continue
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    h = ctypes.c_void_p()
    st = L.glb_graph_create(_lib.ptr64(g.row_offsets), _lib.ptr64(g.col_indices),
                            _lib.ptr64(g.weights), g.num_nodes, g.num_edges, 0, ctypes.byref(h))
    assert st == 0, L.glb_last_error()
    libs.append((path, L, h))

tags = a.strategy.split(",")
res = {(p, t): [] for p, _, _ in libs for t in tags}
out = np.empty(g.num_nodes, dtype=np.int64)
for rep in range(a.reps + 1):
    for path, L, h in libs:
        for t in tags:
            p = _lib.RunParams()
            p.strategy = {"BS": 0, "EP": 1, "WD": 2, "NS": 3, "HP": 4}[t]
            p.algo = 0 if a.algo == "bfs" else 1
            p.bins, p.chunked, p.max_cells, p.block_size, p.hp_fallback = 10, 1, 1 << 40, 1024, 1
            p.loop_mode = 1 if a.loop == "graph" else 0
            p.record_timing = 1
            p.dist_bits = bits_of[path]
            stt = _lib.RunStats()
            rc = L.glb_run(h, ctypes.byref(p), _lib.ptr64(out) if rep == 0 else None,
                           ctypes.byref(stt), None, 0)
            assert rc == 0, L.glb_last_error()
            if rep == 0:
                assert np.array_equal(out, exp), (path, t)
            else:
                res[(path, t)].append(stt.device_ms)
for (path, t), v in res.items():
    print(f"{Path(path).name:28s} {t:3s} median {statistics.median(v):7.3f} ms  min {min(v):7.3f}  all {[round(x,2) for x in v]}")
