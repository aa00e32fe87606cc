"""Graph corpus shared by the golden-vector generator and the parity tests.

Every spec is rebuilt through the generators of a graphlb-compatible module
(the reference itself in tests/golden/make_golden.py, the drop-in package in
the tests); tests/golden/generators.json pins that both produce identical
arrays.
"""

from __future__ import annotations

import numpy as np

SKEWED = (0.7, 0.15, 0.10, 0.05)

# gid -> spec
CORPUS = {
    "rmat10_s1": dict(kind="rmat", scale=10, edge_factor=8, seed=1, max_weight=255),
    "rmat10_s2": dict(kind="rmat", scale=10, edge_factor=8, seed=2, max_weight=255),
    "rmat10_s3": dict(kind="rmat", scale=10, edge_factor=8, seed=3, max_weight=255),
    "rmat10_unw": dict(kind="rmat", scale=10, edge_factor=16, seed=1, weighted=False),
    "rmat10_skew": dict(kind="rmat", scale=10, edge_factor=16, seed=1, max_weight=255,
                        params=SKEWED),
    "rmat12_s4": dict(kind="rmat", scale=12, edge_factor=8, seed=4),
    "er1024": dict(kind="er", num_nodes=1024, num_edges=4096, seed=3),
    "er_empty": dict(kind="er", num_nodes=300, num_edges=0, seed=5),
    "path17": dict(kind="path", n=17, weighted=True, seed=2),
    "star65": dict(kind="star", n=65, weighted=True, seed=3),
    "ring33": dict(kind="ring", n=33),
    "degrees": dict(kind="degrees", degrees=[1181] + [1] * 100, weighted=True, seed=1),
    "grid24": dict(kind="grid", k=24, seed=1),
    "quirks": dict(kind="edges", n=6,
                   src=[0, 0, 0, 1, 1, 2, 2, 3, 3, 5, 5],
                   dst=[0, 1, 1, 2, 1, 3, 3, 4, 4, 5, 0],
                   w=[0, 4, 2, 0, 7, 5, 1, 0, 3, 0, 9]),
}

# sources per graph (clipped to the node count)
def sources_for(n: int) -> list[int]:
    out = [0]
    for s in (n // 3, n - 1):
        if 0 <= s < n and s not in out:
            out.append(s)
    return out


def build(mod, spec: dict):
    """Build `spec` with module `mod` (graphlb or paper_1711_00231_b200)."""
    k = spec["kind"]
    if k == "rmat":
        kw = dict(seed=spec["seed"], weighted=spec.get("weighted", True))
        if "max_weight" in spec:
            kw["max_weight"] = spec["max_weight"]
        if "params" in spec:
            kw["params"] = tuple(spec["params"])
        return mod.generate_rmat(spec["scale"], spec["edge_factor"], **kw)
    if k == "er":
        return mod.generate_er(spec["num_nodes"], spec["num_edges"], seed=spec["seed"])
    if k == "path":
        return mod.path_graph(spec["n"], weighted=spec.get("weighted", False), seed=spec.get("seed", 0))
    if k == "star":
        return mod.star_graph(spec["n"], weighted=spec.get("weighted", False), seed=spec.get("seed", 0))
    if k == "ring":
        return mod.ring_graph(spec["n"], weighted=spec.get("weighted", False), seed=spec.get("seed", 0))
    if k == "degrees":
        return mod.graph_from_degrees(spec["degrees"], weighted=spec.get("weighted", False),
                                      seed=spec.get("seed", 0))
    if k == "edges":
        return mod.CsrGraph.from_edges(spec["n"], spec["src"], spec["dst"], spec.get("w"))
    if k == "grid":
        # the reference has no grid generator: build it with the drop-in's
        # grid_graph and hand the arrays to mod.CsrGraph
        import paper_1711_00231_b200 as pkg

        g = pkg.grid_graph(spec["k"], seed=spec["seed"])
        return mod.CsrGraph(g.num_nodes, g.num_edges, np.array(g.row_offsets),
                            np.array(g.col_indices), np.array(g.weights))
    raise ValueError(k)


def digest(g) -> str:
    import hashlib

    h = hashlib.sha256()
    for a in (g.row_offsets, g.col_indices, g.weights):
        if a is None:
            h.update(b"none")
        else:
            h.update(np.ascontiguousarray(a, dtype="<i8").tobytes())
    return h.hexdigest()


def dist_digest(a) -> str:
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").tobytes()).hexdigest()
