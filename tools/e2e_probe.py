"""Time the pieces of the e2e path (C-ABI create / run / destroy) on C2.

    python tools/e2e_probe.py [--loop host|graph] [--reps 4]
"""
import argparse
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1711_00231_b200 as pkg  # noqa: E402
from paper_1711_00231_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--loop", default="host")
ap.add_argument("--reps", type=int, default=4)
ap.add_argument("--strategy", default="WD")
a = ap.parse_args()
g = pkg.generate_rmat(22, 16, seed=1, max_weight=255, device=0)
L = _lib.lib()
out = np.empty(g.num_nodes, dtype=np.int64)
import bench  # noqa: E402

for i in range(a.reps):
    t0 = time.perf_counter()
    h = ctypes.c_void_p()
    _lib.check(L.glb_graph_create(_lib.ptr64(g.row_offsets), _lib.ptr64(g.col_indices),
                                  _lib.ptr64(g.weights), g.num_nodes, g.num_edges, 0, ctypes.byref(h)))
    t1 = time.perf_counter()
    p = bench.run_params(_lib, a.strategy, "sssp", a.loop)
    st = _lib.RunStats()
    _lib.check(L.glb_run(h, ctypes.byref(p), _lib.ptr64(out), ctypes.byref(st), None, 0))
    t2 = time.perf_counter()
    L.glb_graph_destroy(h)
    t3 = time.perf_counter()
    print(f"rep {i}: create {1e3*(t1-t0):7.2f} ms  run {1e3*(t2-t1):7.2f} ms (device {st.device_ms:.2f})"
          f"  destroy {1e3*(t3-t2):6.2f} ms  total {1e3*(t3-t0):7.2f} ms", flush=True)
print("host workers:", __import__("os").cpu_count())
