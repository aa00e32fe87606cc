"""Pin the CPU oracle (oracle/graphlb_oracle.c) against golden vectors made by
the reference itself (tests/golden/make_golden.py)."""

import numpy as np
import pytest

import paper_1711_00231_b200 as pkg
from tests import graph_specs as gs


def test_oracle_distances_match_reference_corpus(oracle, golden):
    seen = 0
    for gid, spec in gs.CORPUS.items():
        g = gs.build(pkg, spec)
        for src in gs.sources_for(g.num_nodes):
            for algo in ("bfs", "sssp"):
                exp = golden["corpus"][f"{gid}|{src}|{algo}"]
                got = oracle.oracle_distances(g, src, algo)
                assert np.array_equal(got, exp), (gid, src, algo)
                seen += 1
    assert seen >= 60


def test_oracle_bs_port_matches_reference_corpus(oracle, golden):
    for gid, spec in gs.CORPUS.items():
        g = gs.build(pkg, spec)
        for src in gs.sources_for(g.num_nodes):
            for algo in ("bfs", "sssp"):
                w = g.weights if algo == "sssp" else None
                for threads in (1, 4):
                    d, it, ops = oracle.bs_run(g.row_offsets, g.col_indices, w, src, threads)
                    assert np.array_equal(d, golden["corpus"][f"{gid}|{src}|{algo}"]), (gid, src, algo)


def test_oracle_split_matches_reference(oracle, golden):
    sp = golden["split"]
    for gid in ("rmat10_s1", "rmat10_skew", "degrees", "quirks", "er_empty"):
        g = gs.build(pkg, gs.CORPUS[gid])
        counts, mx, arg, mdt = oracle.histogram(g.row_offsets, 10)
        ref_h = sp[f"{gid}|hist10"]
        assert np.array_equal(counts, ref_h[:10]) and [mx, arg, mdt] == ref_h[10:].tolist()
        for key in [k for k in sp if k.startswith(gid + "|") and k.endswith("|row")]:
            mdt = int(key.split("|")[1])
            row, col, w, parent, cs = oracle.split_graph(g.row_offsets, g.col_indices, g.weights, mdt)
            base = f"{gid}|{mdt}"
            assert np.array_equal(row, sp[base + "|row"])
            assert np.array_equal(col, sp[base + "|col"])
            if w is not None:
                assert np.array_equal(w, sp[base + "|w"])
            assert np.array_equal(parent, sp[base + "|parent"])
            assert np.array_equal(cs, sp[base + "|cs"])


def test_oracle_split_kats(oracle, golden):
    for name in ("split_7_4", "split_9_2", "split_mix_3"):
        k = golden["kats"][name]
        g = pkg.graph_from_degrees(k["degrees"], weighted=True, seed=4)
        row, col, w, parent, cs = oracle.split_graph(g.row_offsets, g.col_indices, g.weights, k["mdt"])
        assert np.diff(row).tolist() == k["new_degrees"]
        assert row.tolist() == k["row"] and col.tolist() == k["col"] and w.tolist() == k["w"]
        assert parent.tolist() == k["parent_of"] and cs.tolist() == k["children_start"]


def test_oracle_histogram_kats(oracle, golden):
    k = golden["kats"]
    g = pkg.graph_from_degrees([1, 1, 1, 9])
    counts, mx, arg, mdt = oracle.histogram(g.row_offsets, 3)
    assert counts.tolist() == k["hist_1119_b3"]["counts"] == [3, 0, 1]
    assert arg == k["hist_1119_b3"]["arg"] == 1
    g = pkg.graph_from_degrees([1181] + [1] * 100)
    assert oracle.histogram(g.row_offsets, 10)[3] == k["mdt_rmat20_shape"]["mdt"] == 118
    g = pkg.graph_from_degrees(k["mdt_er23_shape"]["degrees"])
    assert oracle.histogram(g.row_offsets, 10)[3] == k["mdt_er23_shape"]["mdt"] == 3
    g = pkg.graph_from_degrees([0, 0, 0])
    c, mx, arg, mdt = oracle.histogram(g.row_offsets, 4)
    assert c.tolist() == k["hist_all_zero"]["counts"] and mdt == k["hist_all_zero"]["mdt"]


def test_oracle_scan_and_offsets(oracle, golden):
    sc = golden["scan"]
    for key in [k for k in sc if k.endswith("|in")]:
        base = key[:-3]
        assert np.array_equal(oracle.inclusive_scan(sc[key]), sc[base + "|out"])
    for key in [k for k in sc if k.endswith("|prefix")]:
        base = key[: -len("|prefix")]
        ept, threads = sc[base + "|meta"].tolist()
        node, edge = oracle.find_offsets(sc[key], ept, threads)
        assert np.array_equal(node, sc[base + "|node"]) and np.array_equal(edge, sc[base + "|edge"])
    k = golden["kats"]["find_offsets_fig2"]
    node, edge = oracle.find_offsets(k["prefix"], k["ept"], k["threads"])
    assert node.tolist() == k["node"] == [0, 0, 1, 1] and edge.tolist() == k["edge"] == [0, 3, 1, 4]
    assert oracle.inclusive_scan([5, 7]).tolist() == golden["kats"]["scan_5_7"]
    with pytest.raises(OverflowError):
        oracle.inclusive_scan([2**62, 2**62])
    assert golden["kats"]["scan_overflow_raises"]


def test_oracle_coo(oracle, golden):
    assert oracle.coo_src([0, 2, 2]).tolist() == golden["kats"]["coo_small"]["src"]


# ------------------------------------------------ narrow-layout oracle (C3-C5)
def _narrow(oracle, g):
    return oracle.NarrowGraph(g.row_offsets, g.col_indices.astype(np.uint32),
                              None if g.weights is None else g.weights.astype(np.uint32))


def test_oracle_rmat_generator_matches_reference_digests(oracle, golden):
    """The C restatement of generate_rmat + from_edges (numpy PCG64 stream,
    Lemire-bounded weights, stable grouping by source) reproduces the
    reference's graphs byte for byte."""
    d = golden["generators"]
    specs = dict(d["extra_specs"])
    specs.update({k: v for k, v in gs.CORPUS.items() if v["kind"] == "rmat"})
    for gid, spec in specs.items():
        if spec["kind"] != "rmat":
            continue
        g = oracle.rmat_narrow(spec["scale"], spec["edge_factor"],
                               tuple(spec.get("params", pkg.DEFAULT_RMAT_PARAMS)), spec["seed"],
                               spec.get("weighted", True), spec.get("max_weight", 100), threads=3)
        assert gs.digest(g) == d["digests"][gid], gid
    for w in (1, 3, 7, 1000, 65535):  # rejection thresholds; W=1 draws nothing
        a = pkg.generate_rmat(11, 8, seed=5, max_weight=w)
        assert gs.digest(oracle.rmat_narrow(11, 8, seed=5, max_weight=w)) == gs.digest(a), w


def test_oracle_narrow_traversals_match_reference_corpus(oracle, golden):
    for gid, spec in gs.CORPUS.items():
        g = gs.build(pkg, spec)
        ng = _narrow(oracle, g)
        for src in gs.sources_for(g.num_nodes):
            for algo in ("bfs", "sssp"):
                exp = golden["corpus"][f"{gid}|{src}|{algo}"]
                if algo == "bfs":
                    assert np.array_equal(oracle.bfs_narrow(ng, src, parallel=False), exp), gid
                    assert np.array_equal(oracle.bfs_narrow(ng, src, threads=4), exp), gid
                else:
                    d, _, _, done = oracle.bs_run_narrow(ng, src, ng.weights is not None, threads=4)
                    assert done and np.array_equal(d, exp), gid
                # the run_wd port (the reference arm of bench.py): both kinds
                w = algo == "sssp" and ng.weights is not None
                for th in (1, 3):
                    d, _, _, done = oracle.wd_run_narrow(ng, src, w, threads=th)
                    assert done and np.array_equal(d, exp), (gid, src, algo, th)


def test_oracle_narrow_c2_matches_reference_digests(oracle, golden):
    """C2 (RMAT s22) end to end in the narrow oracle: graph, BFS levels and
    SSSP distances equal the reference's (big.json, made by the reference)."""
    big = golden["big"]
    if not big:
        pytest.skip("big.json not generated")
    c2 = big["C2"]
    g = oracle.rmat_narrow(22, 16, seed=1, max_weight=255)
    assert gs.digest(g) == c2["graph_digest"]
    assert gs.dist_digest(oracle.narrow_distances(g, 0, "bfs")) == c2["bfs_digest"]
    assert gs.dist_digest(oracle.narrow_distances(g, 0, "sssp")) == c2["sssp_digest"]
    # a time-bounded run_bs sample stops early with partial work counted
    _, it, ops, done = oracle.bs_run_narrow(g, 0, True, max_seconds=1e-6)
    assert not done and it >= 1 and ops >= 1
    d, _, _, done = oracle.wd_run_narrow(g, 0, True)
    assert done and gs.dist_digest(d) == c2["sssp_digest"]
