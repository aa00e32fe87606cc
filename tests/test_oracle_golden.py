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
