"""Golden fixtures for the graph-file readers, produced by the REFERENCE's own
io.py (run here, where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_io_golden.py

Writes small .gr / edge-list / .csrg files plus the arrays and ParseError
messages the reference returns for them into tests/golden/io/.
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import graphlb  # noqa: E402

OUT = Path(__file__).resolve().parent / "io"
OUT.mkdir(exist_ok=True)

files = {
    "small.gr": "c tiny road-like graph\np sp 5 7\na 1 2 4\na 1 3 1\na 3 2 1\nc mid comment\n"
                "a 2 4 5\na 3 4 8\na 4 5 3\na 1 2 9\n",
    "zero.gr": "p sp 3 0\n",
    "edges.txt": "# u v w\n0 1 5\n0 2 3  # trailing comment\n\n2 1 1\n1 3 7\n3 0 2\n5 5 0\n",
    "bad_arc_before_p.gr": "a 1 2 3\np sp 2 1\n",
    "bad_dup_p.gr": "p sp 2 0\np sp 2 0\n",
    "bad_range.gr": "p sp 2 1\na 1 3 1\n",
    "bad_neg_w.gr": "p sp 2 1\na 1 2 -4\n",
    "bad_count.gr": "p sp 2 2\na 1 2 1\n",
    "bad_kind.gr": "p sp 2 1\nx 1 2 1\n",
    "bad_noproblem.gr": "c nothing\n",
    "bad_malformed_p.gr": "p sq 2 1\n",
    "bad_short.txt": "0 1\n7\n",
    "bad_tok.txt": "0 x\n",
}
expect = {}
for name, text in files.items():
    (OUT / name).write_text(text)
for name in files:
    path = OUT / name
    rel = f"io/{name}"
    for weighted in ((False, True) if name.endswith(".txt") else (None,)):
        key = name if weighted is None else f"{name}|{int(weighted)}"
        try:
            g = graphlb.load_dimacs_gr(path) if weighted is None else graphlb.load_edge_list(path, weighted)
            expect[key] = {"n": g.num_nodes, "m": g.num_edges, "row": g.row_offsets.tolist(),
                           "col": g.col_indices.tolist(),
                           "w": None if g.weights is None else g.weights.tolist()}
        except graphlb.ParseError as e:
            expect[key] = {"error": str(e).replace(str(path), "{path}"), "line": e.line_no}
# the binary cache, written by the reference
for gid, g in {"rmat8": graphlb.generate_rmat(8, 8, seed=3, max_weight=255),
               "unw": graphlb.CsrGraph.from_edges(4, [0, 0, 2, 3], [1, 3, 0, 2])}.items():
    graphlb.write_csr_bin(g, OUT / f"{gid}.csrg")
    expect[f"{gid}.csrg"] = {"n": g.num_nodes, "m": g.num_edges, "row": g.row_offsets.tolist(),
                             "col": g.col_indices.tolist(),
                             "w": None if g.weights is None else g.weights.tolist()}
(OUT / "bad_magic.csrg").write_bytes(b"XXXX" + bytes(40))
(OUT / "truncated.csrg").write_bytes((OUT / "rmat8.csrg").read_bytes()[:100])
for name in ("bad_magic.csrg", "truncated.csrg"):
    try:
        graphlb.read_csr_bin(OUT / name)
    except ValueError as e:  # ParseError, or numpy's ValueError on a short buffer
        expect[name] = {"error": str(e).replace(str(OUT / name), "{path}"),
                        "line": getattr(e, "line_no", None), "type": type(e).__name__}
(OUT / "expected.json").write_text(json.dumps(expect, indent=0))
print(len(expect), "fixtures")
