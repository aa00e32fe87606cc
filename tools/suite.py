"""Every BASELINE.json single-GPU configuration x strategy x {bfs, sssp} on one
B200, each run checked bit-exactly against the pinned oracle.

    python tools/suite.py [--configs C1,C2,C3,C4] [--reps 3] [--out gpurun_out/suite.json]

C1: RMAT s16 ef16 (BFS node-based is the reference's CPU-runnable case)
C2: RMAT s22 ef16, weights 1..255
C3: 4096 x 4096 4-neighbour grid, weights 1..255 (high diameter: 8,191 BFS levels)
C4: skewed RMAT s22 ef16 (0.7, 0.15, 0.10, 0.05), hub degree 1.88M
All from source 0, seed 1, graph resident in HBM (device generator for the
R-MATs), CUDA-graph device loop.  GTEPS = E_r / device time per traversal,
E_r = sum of outdegrees of reached vertices.
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import paper_1711_00231_b200 as pkg  # noqa: E402
from oracle import oracle  # noqa: E402

TAGS = ("BS", "EP", "WD", "NS", "HP")


def build(cfg):
    if cfg == "C1":
        return pkg.generate_rmat(16, 16, seed=1, max_weight=255, device=0)
    if cfg == "C2":
        return pkg.generate_rmat(22, 16, seed=1, max_weight=255, device=0)
    if cfg == "C3":
        return pkg.grid_graph(4096, seed=1, max_weight=255)
    if cfg == "C4":
        return pkg.generate_rmat(22, 16, params=(0.7, 0.15, 0.10, 0.05), seed=1, max_weight=255,
                                 device=0)
    if cfg == "C5":  # scale 27 (2^31 edges) on ONE B200: HBM only, no host copy
        return pkg.generate_rmat(27, 16, seed=1, max_weight=255, device=0, download=False)
    raise ValueError(cfg)


def c5_reference(g, algo, tags, kc):
    """C5 has no host copy: BFS levels are checked against the C oracle on a
    one-off download when the host has the RAM; SSSP (and BFS otherwise) by
    agreement of all strategies with the first one."""
    import psutil

    deg = None
    if algo == "bfs" and psutil.virtual_memory().available > 48 << 30:
        h = g.to_host()
        exp = oracle.oracle_distances(h, 0, "bfs")
        deg = h.outdegrees()
        del h
        return exp, deg, "oracle"
    r = pkg.run_strategy(tags[0], g, 0, pkg.RelaxOp(algo), kc)
    return r.dist.array, None, f"agreement with {tags[0]}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4")
    ap.add_argument("--algos", default="bfs,sssp")
    ap.add_argument("--tags", default=",".join(TAGS))
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--loop", default="graph")
    ap.add_argument("--dist-bits", type=int, default=0)
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "suite.json"))
    a = ap.parse_args()
    oracle.build()
    rows = []
    for cfg in a.configs.split(","):
        t0 = time.time()
        g = build(cfg)
        gen_s = time.time() - t0
        deg = g.outdegrees() if hasattr(g, "outdegrees") else None
        for algo in a.algos.split(","):
            t0 = time.time()
            check = "oracle"
            if cfg == "C5":
                exp, d5, check = c5_reference(g, algo, a.tags.split(","),
                                              pkg.KernelConfig(loop=a.loop, dist_bits=a.dist_bits))
                if d5 is not None:
                    deg = d5
                if deg is None:
                    row = np.empty(g.num_nodes + 1, dtype=np.int64)
                    from paper_1711_00231_b200 import _lib
                    _lib.check(_lib.lib().glb_graph_download(g.device_graph(), _lib.ptr64(row),
                                                             None, None))
                    deg = np.diff(row)
            else:
                exp = oracle.oracle_distances(g, 0, algo)
            oracle_s = time.time() - t0
            reached = exp != pkg.INF
            e_r, n_r = int(deg[reached].sum()), int(reached.sum())
            for tag in a.tags.split(","):
                kc = pkg.KernelConfig(loop=a.loop, record_timing=True, dist_bits=a.dist_bits)
                r = pkg.run_strategy(tag, g, 0, pkg.RelaxOp(algo), kc)
                if not r.feasible:
                    rows.append(dict(config=cfg, algo=algo, strategy=tag, status=r.status))
                    continue
                ok = bool(np.array_equal(r.dist.array, exp))
                ms = []
                for _ in range(a.reps):
                    rr = pkg.run_strategy(tag, g, 0, pkg.RelaxOp(algo), kc)
                    ms.append(rr.device["device_ms"])
                t = float(np.median(ms))
                row = dict(config=cfg, algo=algo, strategy=tag, parity=ok, device_ms=round(t, 3),
                           gteps=round(e_r / (t / 1e3) / 1e9, 3), E_r=e_r, N_r=n_r,
                           relax_per_edge=round(rr.device["relax_ops"] / max(e_r, 1), 3),
                           launches=int(rr.device["launches"]),
                           iterations=int(rr.device["iterations"]),
                           max_thread_work=max((x.work_max() for x in rr.records), default=0),
                           mdt=rr.mdt, oracle_s=round(oracle_s, 2), gen_s=round(gen_s, 2),
                           check=check)
                rows.append(row)
                print(json.dumps(row), flush=True)
        g.release_device()
        del g
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps(rows, indent=1))
    # markdown table
    print("\n| cfg | algo | strategy | parity | ms | GTEPS | relax/E_r | launches | max thread work |")
    print("|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        if "device_ms" in r:
            print(f"| {r['config']} | {r['algo']} | {r['strategy']} | {'ok' if r['parity'] else 'FAIL'} | "
                  f"{r['device_ms']} | {r['gteps']} | {r['relax_per_edge']} | {r['launches']} | "
                  f"{r['max_thread_work']} |")
        else:
            print(f"| {r['config']} | {r['algo']} | {r['strategy']} | {r['status']} | | | | | |")


if __name__ == "__main__":
    main()
