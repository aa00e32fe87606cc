"""Graph files (io.py:26-170): the native readers against fixtures written and
parsed by the reference itself (tests/golden/make_io_golden.py)."""

import json
from pathlib import Path

import numpy as np
import pytest

import paper_1711_00231_b200 as pkg
from paper_1711_00231_b200 import _lib

IO = Path(__file__).resolve().parent / "golden" / "io"
EXP = json.loads((IO / "expected.json").read_text())


def check_graph(g, e):
    assert (g.num_nodes, g.num_edges) == (e["n"], e["m"])
    assert g.row_offsets.tolist() == e["row"] and g.col_indices.tolist() == e["col"]
    assert (None if g.weights is None else g.weights.tolist()) == e["w"]


@pytest.mark.parametrize("key", [k for k in EXP if not k.endswith(".csrg")])
def test_text_readers_match_reference(key):
    name, _, weighted = key.partition("|")
    path = IO / name
    e = EXP[key]

    def load():
        if name.endswith(".gr"):
            return pkg.load_dimacs_gr(path)
        return pkg.load_edge_list(path, weighted=weighted == "1")

    if "error" in e:
        with pytest.raises(pkg.ParseError) as ei:
            load()
        assert str(ei.value) == e["error"].replace("{path}", str(path))
        assert ei.value.line_no == e["line"] and ei.value.path == str(path)
        assert isinstance(ei.value, ValueError)
    else:
        check_graph(load(), e)


def test_csr_cache_host_path_and_writer(tmp_path):
    for gid in ("rmat8", "unw"):
        g = pkg.read_csr_bin(IO / f"{gid}.csrg")
        check_graph(g, EXP[f"{gid}.csrg"])
        out = tmp_path / f"{gid}.csrg"
        pkg.write_csr_bin(g, out)
        assert out.read_bytes() == (IO / f"{gid}.csrg").read_bytes()  # byte-identical to the reference
    with pytest.raises(pkg.ParseError, match="bad magic"):
        pkg.read_csr_bin(IO / "bad_magic.csrg")
    with pytest.raises(ValueError):
        pkg.read_csr_bin(IO / "truncated.csrg")


def test_native_reader_scales(tmp_path):
    # a larger DIMACS file round-trips through the native reader
    rng = np.random.default_rng(1)
    n, m = 2000, 20000
    src, dst, w = rng.integers(1, n + 1, m), rng.integers(1, n + 1, m), rng.integers(0, 100, m)
    lines = ["c generated", f"p sp {n} {m}"] + [f"a {a} {b} {c}" for a, b, c in zip(src, dst, w)]
    (tmp_path / "g.gr").write_text("\n".join(lines) + "\n")
    g = pkg.load_dimacs_gr(tmp_path / "g.gr")
    ref = pkg.CsrGraph.from_edges(n, src - 1, dst - 1, w)
    assert np.array_equal(g.row_offsets, ref.row_offsets)
    assert np.array_equal(g.col_indices, ref.col_indices)
    assert np.array_equal(g.weights, ref.weights)


@pytest.mark.gpu
def test_csr_cache_straight_to_hbm(oracle):
    for gid in ("rmat8", "unw"):
        dg = pkg.read_csr_bin(IO / f"{gid}.csrg", device=0)
        assert isinstance(dg, pkg.DeviceCsrGraph)
        check_graph(dg.to_host(), EXP[f"{gid}.csrg"])
        h = pkg.read_csr_bin(IO / f"{gid}.csrg")
        for algo in ("bfs", "sssp"):
            exp = oracle.oracle_distances(h, 0, algo)
            for tag in pkg.STRATEGY_TAGS:
                r = pkg.run_strategy(tag, dg, 0, pkg.RelaxOp(algo), pkg.KernelConfig())
                assert np.array_equal(r.dist.array, exp), (gid, algo, tag)
    for name, msg in (("bad_magic.csrg", "bad magic"), ("truncated.csrg", "truncated")):
        with pytest.raises(pkg.ParseError, match=msg):
            pkg.read_csr_bin(IO / name, device=0)
    _lib.lib()
