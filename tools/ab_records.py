"""Per-launch records of one strategy under two builds, side by side.

    python tools/ab_records.py a.so b.so [--strategy WD] [--algo sssp] [--scale 22]

Host loop with CUDA-event timing: each record's kernel_ms / overhead_ms
(scan) and relax counts, so a regression can be pinned to iterations.
"""
import argparse
import ctypes
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
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
g = pkg.generate_rmat(a.scale, 16, seed=1, max_weight=255)
rows = []
for path in a.libs:
    L = ctypes.CDLL(str(Path(path).resolve()))
    for name, (res, args) in _lib.SIGNATURES.items():
        if hasattr(L, name):
            getattr(L, name).restype = res
            getattr(L, name).argtypes = args
    h = ctypes.c_void_p()
    assert L.glb_graph_create(_lib.ptr64(g.row_offsets), _lib.ptr64(g.col_indices),
                              _lib.ptr64(g.weights), g.num_nodes, g.num_edges, 0,
                              ctypes.byref(h)) == 0
    best = None
    for rep in range(a.reps):
        p = _lib.RunParams()
        p.strategy = {"BS": 0, "EP": 1, "WD": 2, "NS": 3, "HP": 4}[a.strategy]
        p.algo = 0 if a.algo == "bfs" else 1
        p.bins, p.chunked, p.max_cells, p.block_size, p.hp_fallback = 10, 1, 1 << 40, 1024, 1
        p.loop_mode, p.record_timing = 0, 1
        st = _lib.RunStats()
        recs = (_lib.Record * 4096)()
        assert L.glb_run(h, ctypes.byref(p), None, ctypes.byref(st), recs, 4096) == 0
        n = min(st.n_records, 4096)
        r = [(recs[i].active_items, recs[i].relax_ops, recs[i].push_ops, recs[i].kernel_ms,
              recs[i].overhead_ms) for i in range(n)]
        if best is None or st.device_ms < best[0]:
            best = (st.device_ms, st.dist_bits, r)
    rows.append((Path(path).name, best))
for name, (ms, bits, r) in rows:
    print(f"{name}: device_ms {ms:.3f} dist_bits {bits} records {len(r)} "
          f"sum kernel {sum(x[3] for x in r):.3f} sum overhead {sum(x[4] for x in r):.3f}")
n = max(len(b[2]) for _, b in rows)
print("it | " + " | ".join(f"{nm[:10]:>10s} active relax push k_ms o_ms" for nm, _ in rows))
for i in range(n):
    parts = []
    for _, (ms, bits, r) in rows:
        if i < len(r):
            x = r[i]
            parts.append(f"{x[0]:9d} {x[1]:10d} {x[2]:9d} {x[3]:7.4f} {x[4]:7.4f}")
        else:
            parts.append(" " * 46)
    print(f"{i:3d} | " + " | ".join(parts))
