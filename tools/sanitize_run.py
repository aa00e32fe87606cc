"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every strategy x {bfs, sssp} x {host, graph loop} on small graphs with the
corpus quirks, plus the grid-kernel, fused/dense WD and id-ordered BS
frontier (compaction on every step) variants, each checked
against the oracle.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1711_00231_b200 as pkg  # noqa: E402
from oracle import oracle  # noqa: E402
from tests import graph_specs as gs  # noqa: E402

oracle.build()
QUICK = "--quick" in sys.argv  # racecheck-sized: fewer graphs and variants
if QUICK:
    graphs = [gs.build(pkg, gs.CORPUS[k]) for k in ("rmat10_skew", "quirks")]
    variants = [{}, {"GLB_NO_SMALL": "1"}, {"GLB_BM_THR": "1"}]
else:
    graphs = [gs.build(pkg, gs.CORPUS[k]) for k in ("rmat10_skew", "quirks", "grid24", "degrees", "er_empty")]
    graphs.append(pkg.generate_rmat(13, 8, seed=2, max_weight=255))
    variants = [{}, {"GLB_NO_SMALL": "1"}, {"GLB_NO_SMALL": "1", "GLB_WD_FUSED": "1"},
                {"GLB_NO_SMALL": "1", "GLB_WD_DENSE": "1"},
                {"GLB_BM_THR": "1"}, {"GLB_NO_SMALL": "1", "GLB_BM_THR": "1"}]
bad = 0
for var in variants:
    for k in ("GLB_NO_SMALL", "GLB_WD_FUSED", "GLB_WD_DENSE", "GLB_BM_THR"):
        os.environ.pop(k, None)
    os.environ.update(var)
    for g in graphs:
        for algo in ("bfs", "sssp"):
            exp = oracle.oracle_distances(g, 0, algo)
            for tag in pkg.STRATEGY_TAGS:
                for loop in ("host", "graph"):
                    r = pkg.run_strategy(tag, g, 0, pkg.RelaxOp(algo), pkg.KernelConfig(loop=loop))
                    if not np.array_equal(r.dist.array, exp):
                        bad += 1
                        print("MISMATCH", var, g.num_nodes, algo, tag, loop)
# 24-bit tier across renormalisations (> 256 generations), both loops, and
# the device distance certificate
for k in ("GLB_NO_SMALL", "GLB_WD_FUSED", "GLB_WD_DENSE", "GLB_BM_THR"):
    os.environ.pop(k, None)
long_path = pkg.path_graph(300 if QUICK else 700, weighted=True, seed=3)
for var in ({}, {"GLB_NO_SMALL": "1"}):
    os.environ.pop("GLB_NO_SMALL", None)
    os.environ.update(var)
    for algo in ("bfs", "sssp"):
        exp = oracle.oracle_distances(long_path, 0, algo)
        for tag in (("BS", "WD", "HP") if QUICK else pkg.STRATEGY_TAGS):
            for loop in ("host", "graph"):
                r = pkg.run_strategy(tag, long_path, 0, pkg.RelaxOp(algo),
                                     pkg.KernelConfig(loop=loop, dist_bits=24))
                if not np.array_equal(r.dist.array, exp):
                    bad += 1
                    print("MISMATCH 24-bit", var, algo, tag, loop)
for g in graphs[:3]:
    exp = oracle.oracle_distances(g, 0, "sssp")
    if not pkg.validate_distances(g, 0, "sssp", exp).matched:
        bad += 1
        print("CERTIFICATE rejected a correct array", g.num_nodes)
# round 2: HP / NS CTA bin (TMA-staged pieces, piece -> window table) on a
# hub-heavy graph, and the peer-memory sharded loop with virtual ranks
from paper_1711_00231_b200 import sharded  # noqa: E402

hub = pkg.generate_rmat(11 if QUICK else 13, 8, params=(0.7, 0.15, 0.10, 0.05), seed=1,
                        max_weight=255)
for algo in ("bfs", "sssp"):
    exp = oracle.oracle_distances(hub, 0, algo)
    for tag in ("HP", "NS", "WD"):
        for mdt in (None, 600):  # 600: windows above the 512-edge CTA-bin threshold
            r = pkg.run_strategy(tag, hub, 0, pkg.RelaxOp(algo), pkg.KernelConfig(loop="graph"),
                                 mdt=mdt)
            if not np.array_equal(r.dist.array, exp):
                bad += 1
                print("MISMATCH hub", algo, tag, mdt)
for parts in ((2,) if QUICK else (2, 3)):
    shards = [sharded.shard_graph(graphs[0], parts, r, 0) for r in range(parts)]
    for algo in ("bfs", "sssp"):
        exp = oracle.oracle_distances(graphs[0], 0, algo)
        for tag in sharded.SHARD_TAGS:
            d, _ = sharded.run_virtual_peer(tag, shards, 0, pkg.RelaxOp(algo))
            if not np.array_equal(d, exp):
                bad += 1
                print("MISMATCH peer", parts, algo, tag)
print("sanitize workload done, mismatches:", bad)
