"""The sharded (multi-GPU) protocol on CPU: world_size-2 gloo processes run the
real bsp_loop + DistTransport of paper_1711_00231_b200.sharded with a numpy
test double of the glb_shard_* contract, and must reproduce the oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

INF = (1 << 63) - 1
INF32 = 0xFFFFFFFF


class NumpyShard:
    """Host double of one rank's glb_shard_* calls (test-only)."""

    def __init__(self, row, col, w, bounds, rank, source):
        self.row, self.col, self.w = row, col, w
        self.bounds, self.rank = bounds, rank
        self.lo, self.hi = int(bounds[rank]), int(bounds[rank + 1])
        n = len(row) - 1
        self.dist = np.full(n, INF32, dtype=np.int64)  # owned cells + remote shadows
        self.mark = np.zeros(n, dtype=np.int64)
        self.gen = 1
        self.dist[source] = 0
        self.front = [source] if self.lo <= source < self.hi else []
        self.out = []

    def _owner(self, v):
        return int(np.searchsorted(self.bounds, v, side="right") - 1)

    def _relax(self, v, cand):
        if cand < self.dist[v]:
            self.dist[v] = cand
            if self.mark[v] != self.gen:
                self.mark[v] = self.gen
                self.out.append(v)

    def local(self):
        for u in self.front:
            du = self.dist[u]
            for e in range(self.row[u], self.row[u + 1]):
                self._relax(int(self.col[e]), int(du + (self.w[e] if self.w is not None else 1)))
        parts = len(self.bounds) - 1
        buckets = [[] for _ in range(parts)]
        keep = []
        for v in self.out:
            o = self._owner(v)
            if o == self.rank:
                keep.append(v)
            else:
                buckets[o].append((int(self.dist[v]) << 32) | v)
        self.out = keep
        counts = np.array([len(b) for b in buckets], dtype=np.int64)
        flat = [x for b in buckets for x in b]
        return counts, torch.tensor(flat + [0], dtype=torch.int64), len(keep)

    def apply(self, recv, n):
        for x in recv[:n].tolist():
            self._relax(x & 0xFFFFFFFF, x >> 32)

    def advance(self):
        self.front, self.out = self.out, []
        self.gen += 1
        return len(self.front)

    def finish(self):
        d = self.dist[self.lo:self.hi].copy()
        d[d == INF32] = INF
        return d


def _worker(rank, world, port, spec, algo, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1711_00231_b200 as pkg
        from paper_1711_00231_b200 import sharded
        from tests import graph_specs as gs

        g = gs.build(pkg, spec)
        deg = np.diff(g.row_offsets)
        # edge-balanced bounds, the same rule as glb_graph_partition
        bounds = [0]
        for r in range(1, world):
            bounds.append(max(bounds[-1], int(np.searchsorted(g.row_offsets[:-1], g.num_edges * r // world))))
        bounds.append(g.num_nodes)
        bounds = np.array(bounds, dtype=np.int64)
        w = g.weights if algo == "sssp" else None
        sh = NumpyShard(g.row_offsets, g.col_indices, w, bounds, rank, 0)
        it = sharded.bsp_loop(sh, sharded.DistTransport(torch), "cpu", max_iterations=10_000)
        out = torch.tensor(sh.finish())
        sizes = [int(bounds[r + 1] - bounds[r]) for r in range(world)]
        parts = [torch.empty(s, dtype=torch.int64) for s in sizes]
        dist.all_gather(parts, out) if len(set(sizes)) == 1 else [
            dist.broadcast(parts[r].copy_(out) if r == rank else parts[r], src=r) for r in range(world)]
        if rank == 0:
            q.put((np.concatenate([p.numpy() for p in parts]), it, deg.sum()))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("gid,algo", [("rmat10_s1", "sssp"), ("rmat10_skew", "bfs"),
                                      ("grid24", "sssp"), ("quirks", "sssp")])
def test_bsp_loop_gloo_world2_matches_oracle(gid, algo, oracle):
    import paper_1711_00231_b200 as pkg
    from tests import graph_specs as gs

    spec = gs.CORPUS[gid]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, spec, algo, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, it, _ = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = gs.build(pkg, spec)
    assert np.array_equal(got, oracle.oracle_distances(g, 0, algo))
    assert it >= 1
