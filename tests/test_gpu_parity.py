"""GPU parity: every strategy's device result against the reference's answers.

Bit-exact equality (levels and integer distances are integer data, no
tolerance): golden vectors from the reference (tests/golden/) and, at sizes
the reference cannot reach quickly, the pinned C oracle (oracle/).
"""

import math
import os

import numpy as np
import pytest

import paper_1711_00231_b200 as pkg
from paper_1711_00231_b200 import _lib
from tests import graph_specs as gs

pytestmark = pytest.mark.gpu

TAGS = ("BS", "EP", "WD", "NS", "HP")


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    _lib.lib()  # ImportError (test error) if the CUDA library was not built
    assert _lib.device_count() > 0, "no CUDA device visible to libgraphlb_b200.so"


# Execution variants of the same strategies: the CTA-cluster small-frontier
# loop (default; it takes every iteration of these small graphs), the
# grid-wide kernels alone (GLB_NO_SMALL), WD's fused item pushes and dense
# scans, and the graph-loop structure knobs.
VARIANTS = {"default": {}, "grid_kernels": {"GLB_NO_SMALL": "1"},
            "wd_fused": {"GLB_WD_FUSED": "1"},
            "grid_fused": {"GLB_NO_SMALL": "1", "GLB_WD_FUSED": "1"},
            "grid_dense": {"GLB_NO_SMALL": "1", "GLB_WD_DENSE": "1"},
            # id-order WD scans for every frontier size (24-bit tier included)
            "grid_dense_all": {"GLB_NO_SMALL": "1", "GLB_WD_DENSE": "2"},
            # graph-loop structure knobs: separate control kernel, one step per
            # WHILE iteration without programmatic dependent launch
            "grid_ctl_kernel": {"GLB_NO_SMALL": "1", "GLB_NO_FUSED_CTL": "1"},
            "grid_unroll1_nopdl": {"GLB_NO_SMALL": "1", "GLB_GRAPH_UNROLL": "1", "GLB_NO_PDL": "1"},
            # BS with warp push buffers (k_bs_warp)
            "grid_bs_warp": {"GLB_NO_SMALL": "1", "GLB_BS_WARP": "1"},
            # BS id-ordered frontiers on every step (k_bm_compact rebuilds each
            # list from its bitmap), alone and alternating with the cluster loop
            "grid_bm_every_step": {"GLB_NO_SMALL": "1", "GLB_BM_THR": "1"},
            "bm_every_step": {"GLB_BM_THR": "1"},
            "grid_bm_off": {"GLB_NO_SMALL": "1", "GLB_BM_THR": "0"},
            # cluster loop at the other size than the strategy's default (8 / 16 CTAs)
            "cluster8": {"GLB_SMALL_CTAS": "8"},
            "cluster16": {"GLB_SMALL_CTAS": "16"},
            # EP in the cluster loop with / without carried source levels (default: low-degree graphs only)
            "ep_no_carry": {"GLB_EP_CARRY": "0"},
            "ep_carry": {"GLB_EP_CARRY": "1"}}


@pytest.mark.parametrize("variant", list(VARIANTS))
@pytest.mark.parametrize("loop", ["host", "graph"])
def test_corpus_all_strategies_match_reference(golden, loop, variant, monkeypatch):
    for k, v in VARIANTS[variant].items():
        monkeypatch.setenv(k, v)
    cfg = pkg.KernelConfig(loop=loop)
    for gid, spec in gs.CORPUS.items():
        g = gs.build(pkg, spec)
        for src in gs.sources_for(g.num_nodes):
            for algo in ("bfs", "sssp"):
                exp = golden["corpus"][f"{gid}|{src}|{algo}"]
                for tag in TAGS:
                    r = pkg.run_strategy(tag, g, src, pkg.RelaxOp(algo), cfg)
                    assert r.feasible
                    got = r.dist.array
                    bad = np.flatnonzero(got != exp)
                    assert bad.size == 0, (gid, src, algo, tag, bad[:5], got[bad[:5]], exp[bad[:5]])


def test_dist_bits_64_and_small_blocks(golden):
    for gid in ("rmat10_s1", "rmat10_skew", "degrees", "quirks"):
        g = gs.build(pkg, gs.CORPUS[gid])
        for algo in ("bfs", "sssp"):
            exp = golden["corpus"][f"{gid}|0|{algo}"]
            for tag in TAGS:
                for cfg in (pkg.KernelConfig(dist_bits=64), pkg.KernelConfig(block_size=4),
                            pkg.KernelConfig(block_size=100000)):
                    r = pkg.run_strategy(tag, g, 0, pkg.RelaxOp(algo), cfg)
                    assert np.array_equal(r.dist.array, exp), (gid, algo, tag, cfg)
            for mdt in (1, 2, 7, 1000):
                for tag in ("NS", "HP"):
                    r = pkg.run_strategy(tag, g, 0, pkg.RelaxOp(algo), pkg.KernelConfig(), mdt=mdt)
                    assert np.array_equal(r.dist.array, exp) and r.mdt == mdt
            r = pkg.run_hp(g, 0, pkg.RelaxOp(algo), pkg.KernelConfig(), fallback=False)
            assert np.array_equal(r.dist.array, exp)


def test_u32_overflow_promotes_to_u64(oracle):
    # path with weights 2^31: distances pass 2^32 -> automatic 64-bit re-run
    n = 6
    w = np.full(n - 1, 1 << 31, dtype=np.int64)
    g = pkg.CsrGraph.from_edges(n, np.arange(n - 1), np.arange(1, n), w)
    exp = oracle.dijkstra(g.row_offsets, g.col_indices, g.weights, 0)
    for tag in TAGS:
        r = pkg.run_strategy(tag, g, 0, pkg.RelaxOp("sssp"), pkg.KernelConfig())
        assert np.array_equal(r.dist.array, exp), tag
        assert r.device["dist_bits"] == 64
        with pytest.raises(OverflowError):
            pkg.run_strategy(tag, g, 0, pkg.RelaxOp("sssp"), pkg.KernelConfig(dist_bits=32))


def test_24bit_cells_boundary_and_promotion(oracle):
    """dist_bits 24: 24-bit distances in one u32 cell per node (the automatic
    first tier only for graphs whose u64 cells exceed twice the L2).  The
    largest representable distance is 2^24 - 2; one more is an OverflowError
    at 24 bits and a 32-bit run under dist_bits 0."""
    top = (1 << 24) - 2
    for last, fits in ((top - 0x7FFFFF, True), (top + 1 - 0x7FFFFF, False)):
        g = pkg.CsrGraph.from_edges(3, [0, 1], [1, 2], [0x7FFFFF, last])
        exp = oracle.dijkstra(g.row_offsets, g.col_indices, g.weights, 0)
        for tag in TAGS:
            r = pkg.run_strategy(tag, g, 0, pkg.RelaxOp("sssp"), pkg.KernelConfig())
            assert np.array_equal(r.dist.array, exp) and r.device["dist_bits"] == 32, tag
            for loop in ("host", "graph"):
                cfg = pkg.KernelConfig(dist_bits=24, loop=loop)
                if fits:
                    r = pkg.run_strategy(tag, g, 0, pkg.RelaxOp("sssp"), cfg)
                    assert np.array_equal(r.dist.array, exp) and r.device["dist_bits"] == 24, tag
                else:
                    with pytest.raises(OverflowError):
                        pkg.run_strategy(tag, g, 0, pkg.RelaxOp("sssp"), cfg)


@pytest.mark.parametrize("variant", ["default", "grid_kernels", "grid_fused", "grid_dense_all"])
@pytest.mark.parametrize("loop", ["host", "graph"])
def test_24bit_generation_tags_renormalise(oracle, loop, variant, monkeypatch):
    """More than 256 generations: the 8-bit push tags of the 24-bit tier wrap
    and are renormalised every 128 generations (k_renorm); results must equal
    the 32- and 64-bit tiers' and the oracle's.  grid_dense_all scans every WD
    frontier from the cells' tags, across the renormalisations too (the step
    right after one takes its list instead)."""
    for k, v in VARIANTS[variant].items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(7)
    n = 700  # a path with shortcuts: ~600 generations, ragged frontiers
    src = np.concatenate([np.arange(n - 1), rng.integers(0, n, 60)])
    dst = np.concatenate([np.arange(1, n), rng.integers(0, n, 60)])
    w = rng.integers(1, 50, size=src.size)
    w[n - 1:] = 5000
    g = pkg.CsrGraph.from_edges(n, src, dst, w)
    grid = pkg.grid_graph(24, seed=3)
    for gr in (g, grid):
        for algo in ("bfs", "sssp"):
            exp = oracle.oracle_distances(gr, 0, algo)
            for tag in TAGS:
                for bits in (24, 32):
                    r = pkg.run_strategy(tag, gr, 0, pkg.RelaxOp(algo),
                                         pkg.KernelConfig(loop=loop, dist_bits=bits), mdt=None)
                    assert np.array_equal(r.dist.array, exp), (gr.num_nodes, algo, tag, bits)
                    assert r.device["dist_bits"] == bits


def test_random_graphs_with_quirks(oracle):
    rng = np.random.default_rng(123)
    for trial in range(25):
        n = int(rng.integers(1, 200))
        m = int(rng.integers(0, 6 * n))
        src = rng.integers(0, n, size=m)
        # a few hubs, self-loops and parallel edges, zero weights
        if m:
            src[: m // 4] = rng.integers(0, max(1, n // 10), size=m // 4)
        dst = rng.integers(0, n, size=m)
        w = rng.integers(0, 9, size=m) if trial % 3 else None
        g = pkg.CsrGraph.from_edges(n, src, dst, w)
        s = int(rng.integers(0, n))
        for algo in ("bfs", "sssp"):
            exp = oracle.oracle_distances(g, s, algo)
            for tag in TAGS:
                for mdt in (None, 1, 3):
                    if mdt is not None and tag not in ("NS", "HP"):
                        continue
                    r = pkg.run_strategy(tag, g, s, pkg.RelaxOp(algo), pkg.KernelConfig(), mdt=mdt)
                    assert np.array_equal(r.dist.array, exp), (trial, algo, tag, mdt)


def test_split_graph_device_matches_reference(golden):
    sp = golden["split"]
    for gid in ("rmat10_s1", "rmat10_skew", "degrees", "quirks", "er_empty"):
        g = gs.build(pkg, gs.CORPUS[gid])
        h = pkg.build_histogram(g, 10)
        ref_h = sp[f"{gid}|hist10"]
        assert np.array_equal(h.counts, ref_h[:10])
        assert [h.max_degree, h.arg_max_bin, pkg.compute_mdt(h)] == ref_h[10:].tolist()
        for key in [k for k in sp if k.startswith(gid + "|") and k.endswith("|row")]:
            mdt = int(key.split("|")[1])
            s = pkg.split_graph(g, mdt)
            base = f"{gid}|{mdt}"
            assert np.array_equal(s.graph.row_offsets, sp[base + "|row"]), base
            assert np.array_equal(s.graph.col_indices, sp[base + "|col"]), base
            if g.weights is not None:
                assert np.array_equal(s.graph.weights, sp[base + "|w"]), base
            assert np.array_equal(s.parent_of, sp[base + "|parent"]), base
            assert np.array_equal(s.children_start, sp[base + "|cs"]), base
    for name in ("split_7_4", "split_9_2", "split_mix_3"):
        k = golden["kats"][name]
        g = pkg.graph_from_degrees(k["degrees"], weighted=True, seed=4)
        s = pkg.split_graph(g, k["mdt"])
        assert np.diff(s.graph.row_offsets).tolist() == k["new_degrees"]
        assert s.graph.col_indices.tolist() == k["col"] and s.graph.weights.tolist() == k["w"]
        assert s.parent_of.tolist() == k["parent_of"]
        assert s.children_start.tolist() == k["children_start"]
        assert s.split_fraction == k["split_fraction"]


def test_histogram_mdt_kats(golden):
    k = golden["kats"]
    h = pkg.build_histogram(pkg.graph_from_degrees([1, 1, 1, 9]), 3)
    assert h.counts.tolist() == k["hist_1119_b3"]["counts"] and h.arg_max_bin == 1
    assert pkg.compute_mdt(pkg.build_histogram(pkg.graph_from_degrees([1181] + [1] * 100), 10)) == 118
    assert pkg.compute_mdt(pkg.build_histogram(pkg.graph_from_degrees(k["mdt_er23_shape"]["degrees"]), 10)) == 3
    h = pkg.build_histogram(pkg.graph_from_degrees([0, 0, 0]), 4)
    assert h.counts.tolist() == k["hist_all_zero"]["counts"] and pkg.compute_mdt(h) == 1
    ds = pkg.degree_stats(pkg.star_graph(5))
    assert [ds.max, ds.avg] == k["degree_stats_star5"][:2]
    assert math.isclose(ds.stddev, k["degree_stats_star5"][2], rel_tol=1e-12)
    r = pkg.run_ns(gs.build(pkg, gs.CORPUS["rmat10_s1"]), 0, pkg.RelaxOp("sssp"), pkg.KernelConfig())
    assert r.mdt == k["ns_rmat10_s1"]["mdt"] and r.split_fraction == k["ns_rmat10_s1"]["split_fraction"]
    r = pkg.run_hp(gs.build(pkg, gs.CORPUS["rmat10_s1"]), 0, pkg.RelaxOp("sssp"), pkg.KernelConfig())
    assert r.mdt == k["hp_rmat10_s1"]["mdt"]


def test_scan_and_find_offsets_on_device(golden):
    sc = golden["scan"]
    for key in [k for k in sc if k.endswith("|in")]:
        assert np.array_equal(np.array(pkg.inclusive_scan(sc[key])), sc[key[:-3] + "|out"])
    for key in [k for k in sc if k.endswith("|prefix")]:
        base = key[: -len("|prefix")]
        ept, threads = sc[base + "|meta"].tolist()
        prefix = sc[key]
        t = pkg.find_offsets(None, list(range(len(prefix))), prefix, ept, threads)
        assert t.node_offsets == sc[base + "|node"].tolist()
        assert t.edge_offsets == sc[base + "|edge"].tolist()
    k = golden["kats"]
    t = pkg.find_offsets(None, [0, 1], [5, 12], 3, 4)
    assert t.node_offsets == k["find_offsets_fig2"]["node"]
    assert t.edge_offsets == k["find_offsets_fig2"]["edge"]
    t = pkg.find_offsets(None, [0, 1], [5, 12], 5, 8)
    assert t.node_offsets == k["find_offsets_idle"]["node"]
    assert pkg.inclusive_scan([5, 7]) == k["scan_5_7"]
    with pytest.raises(OverflowError):
        pkg.inclusive_scan([2**62, 2**62])
    with pytest.raises(ValueError):
        pkg.find_offsets(None, [0, 1, 2], [5, 12], 3, 4)


def test_coo_and_ep_feasibility(golden):
    coo = pkg.csr_to_coo(pkg.CsrGraph(2, 2, [0, 2, 2], [1, 0]))
    assert coo.src.tolist() == golden["kats"]["coo_small"]["src"]
    g = gs.build(pkg, gs.CORPUS["rmat12_s4"])
    coo = pkg.csr_to_coo(g)
    assert np.array_equal(coo.src, np.repeat(np.arange(g.num_nodes), g.outdegrees()))
    with pytest.raises(pkg.CooCapacityError):
        pkg.csr_to_coo(g, max_cells=10)
    ger = pkg.generate_er(2000, 60000, seed=9)
    r = pkg.run_ep(ger, 0, pkg.RelaxOp("sssp"), pkg.KernelConfig(), max_cells=100_000)
    assert r.status == golden["kats"]["ep_cliff"]["status"] == pkg.INFEASIBLE_MEMORY
    assert r.dist is None
    for tag in ("BS", "WD", "NS", "HP"):
        assert pkg.run_strategy(tag, ger, 0, pkg.RelaxOp("sssp"), pkg.KernelConfig(),
                                max_cells=100_000).feasible


def test_hp_subiteration_structure(golden):
    k = golden["kats"]
    g100 = pkg.CsrGraph.from_edges(2, [0] * 100, [1] * 100)
    r = pkg.run_hp(g100, 0, pkg.RelaxOp("bfs"), pkg.KernelConfig(), mdt=5, fallback=False)
    assert sum(1 for rec in r.records if rec.iteration == 0) == k["hp_100_mdt5_subiters"] == 20
    fig = pkg.CsrGraph.from_edges(4, [0, 0] + [1] * 5 + [2] * 7, [1, 2] + [3] * 12)
    r = pkg.run_hp(fig, 0, pkg.RelaxOp("bfs"), pkg.KernelConfig(), mdt=3, fallback=False)
    per = [sum(1 for rec in r.records if rec.iteration == i) for i in range(max(x.iteration for x in r.records) + 1)]
    assert per == k["hp_fig4_subiters_per_iter"]
    r = pkg.run_hp(fig, 0, pkg.RelaxOp("bfs"), pkg.KernelConfig(), mdt=3, fallback=True)
    assert [rec.strategy for rec in r.records] == k["hp_fig4_fallback_tags"]


def test_records_and_counters():
    g = pkg.generate_rmat(14, 8, seed=1, max_weight=255)
    run = {t: pkg.run_strategy(t, g, 0, pkg.RelaxOp("bfs"), pkg.KernelConfig()) for t in TAGS}
    levels = int(run["BS"].dist.array[run["BS"].dist.array != pkg.INF].max())
    assert len(run["BS"].records) == levels + 1          # one launch per BFS level
    deg = g.outdegrees()
    reached = run["BS"].dist.array != pkg.INF
    e_r = int(deg[reached].sum())
    for t in ("BS", "WD"):                                 # BFS examines every reached edge once
        assert sum(r.work_total() for r in run[t].records) == e_r, t
    # chunked EP reserves once per destination range (SPEC acceptance 7)
    ch = pkg.run_ep(g, 0, pkg.RelaxOp("sssp"), pkg.KernelConfig(), chunked=True)
    un = pkg.run_ep(g, 0, pkg.RelaxOp("sssp"), pkg.KernelConfig(), chunked=False)
    assert ch.dist == un.dist
    assert sum(r.atomic_push_ops for r in ch.records) < sum(r.atomic_push_ops for r in un.records)
    # imbalance ordering on skewed RMAT (SPEC acceptance 8, device counters)
    sd = {t: sum(r.work_stddev() for r in pkg.run_strategy(t, g, 0, pkg.RelaxOp("sssp"),
                                                            pkg.KernelConfig()).records) for t in TAGS}
    assert sd["EP"] < sd["BS"] and sd["WD"] < sd["BS"] and sd["NS"] < sd["BS"], sd


@pytest.mark.parametrize("variant", ["grid_kernels", "wd_fused", "grid_dense", "grid_dense_all",
                                     "grid_bs_warp", "grid_bm_every_step"])
def test_random_graphs_execution_variants(oracle, variant, monkeypatch):
    for k, v in VARIANTS[variant].items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(321)
    for trial in range(10):
        n = int(rng.integers(1, 3000))
        m = int(rng.integers(0, 8 * n))
        src = rng.integers(0, n, size=m)
        if m:
            src[: m // 3] = rng.integers(0, max(1, n // 50), size=m // 3)  # hubs
        dst = rng.integers(0, n, size=m)
        w = rng.integers(0, 300, size=m) if trial % 2 else None
        g = pkg.CsrGraph.from_edges(n, src, dst, w)
        s = int(rng.integers(0, n))
        for algo in ("bfs", "sssp"):
            exp = oracle.oracle_distances(g, s, algo)
            for tag in TAGS:
                for loop in ("host", "graph"):
                    r = pkg.run_strategy(tag, g, s, pkg.RelaxOp(algo), pkg.KernelConfig(loop=loop))
                    assert np.array_equal(r.dist.array, exp), (variant, trial, algo, tag, loop)


@pytest.fixture(scope="module")
def c1_graph():
    return pkg.generate_rmat(16, 16, seed=1, max_weight=255)


def test_c1_all_strategies(c1_graph, oracle, golden):
    g = c1_graph
    for algo in ("bfs", "sssp"):
        exp = oracle.oracle_distances(g, 0, algo)
        if golden["big"]:
            assert gs.dist_digest(exp) == golden["big"]["C1"][f"{algo}_digest"]
        for tag in TAGS:
            for loop in ("host", "graph"):
                r = pkg.run_strategy(tag, g, 0, pkg.RelaxOp(algo), pkg.KernelConfig(loop=loop))
                assert np.array_equal(r.dist.array, exp), (algo, tag, loop)
        os.environ["GLB_WD_FUSED"] = "1"
        try:
            r = pkg.run_strategy("WD", g, 0, pkg.RelaxOp(algo), pkg.KernelConfig(loop="graph"))
            assert np.array_equal(r.dist.array, exp), (algo, "WD fused")
        finally:
            del os.environ["GLB_WD_FUSED"]


@pytest.mark.slow
def test_c2_rmat22_all_strategies(oracle, golden):
    g = pkg.generate_rmat(22, 16, seed=1, max_weight=255)
    big = golden["big"]
    if big:
        assert gs.digest(g) == big["C2"]["graph_digest"]
    for algo in ("bfs", "sssp"):
        exp = oracle.oracle_distances(g, 0, algo)
        if big:
            assert gs.dist_digest(exp) == big["C2"][f"{algo}_digest"]
        for tag in TAGS:
            r = pkg.run_strategy(tag, g, 0, pkg.RelaxOp(algo), pkg.KernelConfig(loop="graph"))
            assert np.array_equal(r.dist.array, exp), (algo, tag)
    g.release_device()


def test_device_rmat_generator_matches_numpy(golden):
    # bit-identical to the reference generator (and to the numpy path)
    d = golden["generators"]
    specs = dict(d["extra_specs"])
    specs.update({k: v for k, v in gs.CORPUS.items() if v["kind"] == "rmat"})
    for gid, spec in specs.items():
        if spec["kind"] != "rmat":
            continue
        kw = dict(seed=spec["seed"], weighted=spec.get("weighted", True))
        if "max_weight" in spec:
            kw["max_weight"] = spec["max_weight"]
        if "params" in spec:
            kw["params"] = tuple(spec["params"])
        g = pkg.generate_rmat(spec["scale"], spec["edge_factor"], device=0, **kw)
        assert gs.digest(g) == d["digests"][gid], gid
    # odd weights exercise the Lemire rejection threshold (2^32 mod W != 1)
    for w in (3, 7, 1000, 65535):
        a = pkg.generate_rmat(11, 8, seed=5, max_weight=w)
        b = pkg.generate_rmat(11, 8, seed=5, max_weight=w, device=0)
        assert gs.digest(a) == gs.digest(b), w
    dg = pkg.generate_rmat(12, 8, seed=3, device=0, download=False)
    r = pkg.run_wd(dg, 0, pkg.RelaxOp("sssp"), pkg.KernelConfig())
    h = pkg.generate_rmat(12, 8, seed=3)
    assert np.array_equal(r.dist.array, pkg.run_wd(h, 0, pkg.RelaxOp("sssp"), pkg.KernelConfig()).dist.array)


def test_sharded_virtual_ranks_match_reference(golden):
    from paper_1711_00231_b200 import sharded

    for gid in ("rmat10_s1", "rmat10_skew", "grid24", "quirks", "rmat12_s4", "degrees"):
        g = gs.build(pkg, gs.CORPUS[gid])
        for parts in (2, 3, 4):
            shards = [sharded.shard_graph(g, parts, r, 0) for r in range(parts)]
            for algo in ("bfs", "sssp"):
                exp = golden["corpus"][f"{gid}|0|{algo}"]
                for tag in sharded.SHARD_TAGS:
                    d, it = sharded.run_virtual(tag, shards, 0, pkg.RelaxOp(algo))
                    assert np.array_equal(d, exp), (gid, parts, algo, tag)
    # device-generated shards of an R-MAT vs the single-device run
    shards = [sharded.shard_rmat(14, 8, 4, r, 0, seed=3) for r in range(4)]
    h = pkg.generate_rmat(14, 8, seed=3, max_weight=255)
    for algo in ("bfs", "sssp"):
        exp = pkg.run_wd(h, 0, pkg.RelaxOp(algo), pkg.KernelConfig()).dist.array
        for tag in sharded.SHARD_TAGS:
            d, _ = sharded.run_virtual(tag, shards, 0, pkg.RelaxOp(algo))
            assert np.array_equal(d, exp), (algo, tag)


@pytest.mark.parametrize("ctas", ["", "8", "16"])
def test_high_diameter_grid_all_strategies(oracle, ctas, monkeypatch):
    """C3's shape at k=256 (511 BFS levels, ~530 SSSP iterations): long runs of
    small frontiers through the cluster loop (default, 8- and 16-CTA
    clusters), alternating with grid steps."""
    if ctas:
        monkeypatch.setenv("GLB_SMALL_CTAS", ctas)
    g = pkg.grid_graph(256, seed=1, max_weight=255)
    for algo in ("bfs", "sssp"):
        exp = oracle.oracle_distances(g, 0, algo)
        for tag in TAGS:
            for loop in ("host", "graph"):
                r = pkg.run_strategy(tag, g, 0, pkg.RelaxOp(algo), pkg.KernelConfig(loop=loop))
                assert np.array_equal(r.dist.array, exp), (algo, tag, loop)
            r = pkg.run_strategy(tag, g, 1000, pkg.RelaxOp(algo), pkg.KernelConfig(loop="graph"))
            assert np.array_equal(r.dist.array, oracle.oracle_distances(g, 1000, algo)), (algo, tag)


@pytest.mark.parametrize("thr", ["1", "300", "4096"])
def test_grid_bs_id_ordered_frontiers(oracle, thr, monkeypatch):
    """BS / NS on the grid with id-ordered frontiers at low thresholds: lists
    the cluster loop hands back (no bits, taken in push order) alternate with
    compacted grid steps; the device checks every compacted list has the
    worklist's length (a mismatch raises).  NS also mirrors onto split
    children (mdt 3 splits the degree-4 nodes)."""
    monkeypatch.setenv("GLB_BM_THR", thr)
    g = pkg.grid_graph(256, seed=1, max_weight=255)
    for algo in ("bfs", "sssp"):
        exp = oracle.oracle_distances(g, 0, algo)
        for tag, mdt in (("BS", None), ("NS", None), ("NS", 3)):
            for loop in ("host", "graph"):
                r = pkg.run_strategy(tag, g, 0, pkg.RelaxOp(algo), pkg.KernelConfig(loop=loop), mdt=mdt)
                assert np.array_equal(r.dist.array, exp), (thr, algo, tag, mdt, loop)
                assert r.records[-1].active_items >= 1
