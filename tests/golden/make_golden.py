"""Generate the golden vectors by importing the REFERENCE graphlb in place.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--big [C1 C2 C3 C4]]

Runs only in the build container (the GPU box has no /root/reference).  The
outputs are committed; tests/test_oracle_golden.py pins oracle/ against them
and the GPU parity tests compare the device results with them.

  generators.json  sha256 of (row, col, w) of reference generator outputs
  corpus.npz       reference oracle distances per (graph, source, algo); every
                   reference strategy (BS/EP/WD/NS/HP) is asserted to agree
  kats.json        SPEC.md known-answer vectors evaluated on the reference
  split.npz        reference split_graph arrays for corpus graphs
  scan.npz         reference inclusive_scan / find_offsets on random inputs
  big.json         (--big) digests of reference oracle distances at C1, C2
                   (RMAT s16 / s22), C3 (4096^2 grid) and C4 (skewed RMAT
                   s22), plus the graph digests, N_r / E_r
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

import graphlb as ref  # noqa: E402  (the reference, read-only)

from tests import graph_specs as gs  # noqa: E402

ALGOS = ("bfs", "sssp")


def oracle(g, src, algo):
    d = ref.sequential_bfs(g, src) if algo == "bfs" else ref.dijkstra(g, src)
    return np.array(d.values, dtype=np.int64)


def make_generators():
    out = {}
    for gid, spec in gs.CORPUS.items():
        if spec["kind"] == "grid":
            continue
        out[gid] = gs.digest(gs.build(ref, spec))
    extra = {
        "rmat4_ef8_s7": dict(kind="rmat", scale=4, edge_factor=8, seed=7),
        "rmat14_ef8_s1": dict(kind="rmat", scale=14, edge_factor=8, seed=1),
        "rmat14_skew": dict(kind="rmat", scale=14, edge_factor=16, seed=2, max_weight=255,
                            params=gs.SKEWED),
        "c1_rmat16": dict(kind="rmat", scale=16, edge_factor=16, seed=1, max_weight=255),
        "er14": dict(kind="er", num_nodes=1 << 14, num_edges=1 << 16, seed=3),
    }
    specs = {}
    for gid, spec in extra.items():
        out[gid] = gs.digest(gs.build(ref, spec))
        specs[gid] = spec
    (HERE / "generators.json").write_text(json.dumps({"digests": out, "extra_specs": specs},
                                                     indent=1, sort_keys=True))
    print("generators.json", len(out))


def make_corpus():
    arrays = {}
    cfg = ref.KernelConfig()
    for gid, spec in gs.CORPUS.items():
        g = gs.build(ref, spec)
        for src in gs.sources_for(g.num_nodes):
            for algo in ALGOS:
                exp = oracle(g, src, algo)
                arrays[f"{gid}|{src}|{algo}"] = exp
                if g.num_nodes <= 5000:
                    for tag in ("BS", "EP", "WD", "NS", "HP"):
                        r = ref.run_strategy(tag, g, src, ref.RelaxOp(algo), cfg)
                        if r.dist is None:
                            continue
                        got = np.array(r.dist.values, dtype=np.int64)
                        assert np.array_equal(got, exp), (gid, src, algo, tag)
        print("corpus", gid, g.num_nodes, g.num_edges, flush=True)
    np.savez_compressed(HERE / "corpus.npz", **arrays)


def make_kats():
    k = {}
    # find_offsets, Fig. 2
    g2 = ref.graph_from_degrees([5, 7])
    wl = ref.Worklist.from_items([0, 1])
    t = ref.find_offsets(g2, wl, [5, 12], 3, 4)
    k["find_offsets_fig2"] = {"prefix": [5, 12], "ept": 3, "threads": 4,
                              "node": t.node_offsets, "edge": t.edge_offsets}
    t = ref.find_offsets(g2, wl, [5, 12], 5, 8)
    k["find_offsets_idle"] = {"prefix": [5, 12], "ept": 5, "threads": 8,
                              "node": t.node_offsets, "edge": t.edge_offsets}
    # WD per-thread work on Fig. 2: node 0 -> {1, 2}; 1 has 5, 2 has 7 edges
    src = [0, 0] + [1] * 5 + [2] * 7
    dst = [1, 2] + [3] * 5 + [3] * 7
    fig = ref.CsrGraph.from_edges(4, src, dst)
    r = ref.run_wd(fig, 0, ref.RelaxOp("bfs"), ref.KernelConfig(virtual_threads=4))
    k["wd_fig2_work"] = [rec.per_thread_work for rec in r.records]
    # HP sub-iteration counts
    g100 = ref.CsrGraph.from_edges(2, [0] * 100, [1] * 100)
    r = ref.run_hp(g100, 0, ref.RelaxOp("bfs"), ref.KernelConfig(), mdt=5, fallback=False)
    k["hp_100_mdt5_subiters"] = sum(1 for rec in r.records if rec.iteration == 0)
    r = ref.run_hp(fig, 0, ref.RelaxOp("bfs"), ref.KernelConfig(), mdt=3, fallback=False)
    k["hp_fig4_subiters_per_iter"] = [sum(1 for rec in r.records if rec.iteration == i)
                                      for i in range(max(rec.iteration for rec in r.records) + 1)]
    r = ref.run_hp(fig, 0, ref.RelaxOp("bfs"), ref.KernelConfig(), mdt=3, fallback=True)
    k["hp_fig4_fallback_tags"] = [rec.strategy for rec in r.records]
    # split_graph
    for name, deg, mdt in (("split_7_4", [7], 4), ("split_9_2", [9], 2), ("split_mix_3", [0, 7, 2, 9, 3], 3)):
        sg = ref.split_graph(ref.graph_from_degrees(deg, weighted=True, seed=4), mdt)
        k[name] = {"degrees": deg, "mdt": mdt,
                   "new_degrees": np.diff(sg.graph.row_offsets).tolist(),
                   "row": sg.graph.row_offsets.tolist(), "col": sg.graph.col_indices.tolist(),
                   "w": sg.graph.weights.tolist(), "parent_of": sg.parent_of.tolist(),
                   "children_start": sg.children_start.tolist(),
                   "split_fraction": sg.split_fraction}
    # histogram / MDT
    h = ref.build_histogram(ref.graph_from_degrees([1, 1, 1, 9]), 3)
    k["hist_1119_b3"] = {"counts": h.counts.tolist(), "arg": h.arg_max_bin, "max": h.max_degree,
                         "mdt": ref.compute_mdt(h)}
    h = ref.build_histogram(ref.graph_from_degrees([1181] + [1] * 100), 10)
    k["mdt_rmat20_shape"] = {"counts": h.counts.tolist(), "arg": h.arg_max_bin, "mdt": ref.compute_mdt(h)}
    er23 = [10] + [3] * 50 + [1] * 10 + [0] * 3
    h = ref.build_histogram(ref.graph_from_degrees(er23), 10)
    k["mdt_er23_shape"] = {"degrees": er23, "counts": h.counts.tolist(), "arg": h.arg_max_bin,
                           "mdt": ref.compute_mdt(h)}
    h = ref.build_histogram(ref.graph_from_degrees([0, 0, 0]), 4)
    k["hist_all_zero"] = {"counts": h.counts.tolist(), "arg": h.arg_max_bin, "mdt": ref.compute_mdt(h)}
    ds = ref.degree_stats(ref.star_graph(5))
    k["degree_stats_star5"] = [ds.max, ds.avg, ds.stddev]
    # csr_to_coo
    coo = ref.csr_to_coo(ref.CsrGraph(2, 2, [0, 2, 2], [1, 0]))
    k["coo_small"] = {"src": coo.src.tolist(), "dst": coo.dst.tolist()}
    # generator counts
    g = ref.generate_rmat(4, 8, seed=7)
    k["rmat_4_8_7"] = [g.num_nodes, g.num_edges]
    # scan
    k["scan_5_7"] = ref.inclusive_scan([5, 7])
    try:
        ref.inclusive_scan([2**62, 2**62])
        k["scan_overflow_raises"] = False
    except OverflowError:
        k["scan_overflow_raises"] = True
    # COO feasibility cliff (SPEC.md acceptance 9, scaled down 10x)
    ger = ref.generate_er(2000, 60000, seed=9)
    r = ref.run_ep(ger, 0, ref.RelaxOp("sssp"), ref.KernelConfig(), max_cells=100_000)
    k["ep_cliff"] = {"status": r.status, "dist_is_none": r.dist is None}
    # NS / HP mdt + split fraction on a corpus graph
    g = gs.build(ref, gs.CORPUS["rmat10_s1"])
    r = ref.run_ns(g, 0, ref.RelaxOp("sssp"), ref.KernelConfig())
    k["ns_rmat10_s1"] = {"mdt": r.mdt, "split_fraction": r.split_fraction}
    r = ref.run_hp(g, 0, ref.RelaxOp("sssp"), ref.KernelConfig())
    k["hp_rmat10_s1"] = {"mdt": r.mdt}
    (HERE / "kats.json").write_text(json.dumps(k, indent=1, sort_keys=True))
    print("kats.json", len(k))


def make_split():
    arrays = {}
    for gid in ("rmat10_s1", "rmat10_skew", "degrees", "quirks", "er_empty"):
        g = gs.build(ref, gs.CORPUS[gid])
        h = ref.build_histogram(g, 10)
        for mdt in sorted({ref.compute_mdt(h), 1, 3}):
            sg = ref.split_graph(g, mdt)
            key = f"{gid}|{mdt}"
            arrays[key + "|row"] = sg.graph.row_offsets
            arrays[key + "|col"] = sg.graph.col_indices
            if sg.graph.weights is not None:
                arrays[key + "|w"] = sg.graph.weights
            arrays[key + "|parent"] = sg.parent_of
            arrays[key + "|cs"] = sg.children_start
        arrays[f"{gid}|hist10"] = np.concatenate([h.counts, [h.max_degree, h.arg_max_bin, ref.compute_mdt(h)]])
    np.savez_compressed(HERE / "split.npz", **arrays)
    print("split.npz", len(arrays))


def make_scan():
    rng = np.random.default_rng(11)
    arrays = {}
    for i, n in enumerate((1, 7, 4096, 4097, 12345, 100_000)):
        v = rng.integers(-1000, 100_000, size=n)
        arrays[f"scan{i}|in"] = v
        arrays[f"scan{i}|out"] = np.array(ref.inclusive_scan(v.tolist()), dtype=np.int64)
    for i, (size, threads) in enumerate(((1, 1), (5, 16), (300, 1024), (2000, 16384))):
        deg = rng.integers(0, 40, size=size)
        prefix = np.cumsum(deg)
        total = int(prefix[-1])
        ept = max(1, -(-total // threads))
        wl = ref.Worklist.from_items(list(range(size)))
        t = ref.find_offsets(None, wl, prefix.tolist(), ept, threads)
        arrays[f"fo{i}|prefix"] = prefix
        arrays[f"fo{i}|meta"] = np.array([ept, threads])
        arrays[f"fo{i}|node"] = np.array(t.node_offsets)
        arrays[f"fo{i}|edge"] = np.array(t.edge_offsets)
    np.savez_compressed(HERE / "scan.npz", **arrays)
    print("scan.npz", len(arrays))


BIG_SPECS = {
    "C1": dict(kind="rmat", scale=16, edge_factor=16, seed=1, max_weight=255),
    "C2": dict(kind="rmat", scale=22, edge_factor=16, seed=1, max_weight=255),
    # C3: the grid is not a reference generator; its arrays come from
    # paper_1711_00231_b200.grid_graph and the REFERENCE oracle runs on them
    "C3": dict(kind="grid", k=4096, seed=1, max_weight=255),
    "C4": dict(kind="rmat", scale=22, edge_factor=16, seed=1, max_weight=255,
               params=(0.7, 0.15, 0.10, 0.05)),
}


def _build_big(spec):
    if spec["kind"] == "grid":
        import paper_1711_00231_b200 as pkg

        h = pkg.grid_graph(spec["k"], seed=spec["seed"], max_weight=spec["max_weight"])
        return ref.CsrGraph(h.num_nodes, h.num_edges, h.row_offsets, h.col_indices, h.weights)
    return gs.build(ref, spec)


def make_big(names):
    path = HERE / "big.json"
    out = json.loads(path.read_text()) if path.exists() else {}
    for name in names:
        spec = BIG_SPECS[name]
        t0 = time.time()
        g = _build_big(spec)
        rec = {"spec": spec, "graph_digest": gs.digest(g), "n": g.num_nodes, "m": g.num_edges,
               "gen_s": time.time() - t0}
        deg = g.outdegrees()
        for algo in ALGOS:
            t0 = time.time()
            d = oracle(g, 0, algo)
            rec[f"{algo}_s"] = time.time() - t0
            reached = d != ref.INF
            rec[f"{algo}_digest"] = gs.dist_digest(d)
            rec["N_r"] = int(reached.sum())
            rec["E_r"] = int(deg[reached].sum())
            rec[f"{algo}_max_dist"] = int(d[reached].max())
        out[name] = rec
        print(name, rec, flush=True)
        del g
        path.write_text(json.dumps(out, indent=1, sort_keys=True))


if __name__ == "__main__":
    if "--big" in sys.argv:
        names = [a for a in sys.argv[1:] if a in BIG_SPECS] or list(BIG_SPECS)
        make_big(names)
    else:
        make_generators()
        make_kats()
        make_split()
        make_scan()
        make_corpus()
