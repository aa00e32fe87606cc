"""Multi-GPU BFS/SSSP: 1-D vertex partition with a per-iteration exchange.

Each rank owns a contiguous, edge-balanced vertex range [lo, hi) and holds the
graph over the GLOBAL id space with only its own rows (``glb_graph_restrict``),
so the single-GPU strategy kernels (BS, WD, HP) run unchanged on the owned
frontier.

Two transports run the same bulk-synchronous iteration:

* ``"peer"`` (default, the product path): the whole loop runs inside the
  library (``glb_peer_run``).  Ranks write remote improvements straight into
  each other's HBM over NVLink / NVSwitch (CUDA IPC between processes, plain
  device pointers between ranks of one process), synchronise through
  release/acquire mailboxes in that memory, and the host reads one control
  block per iteration.  ``PeerExchange`` sets it up (IPC handles gathered
  with torch.distributed).
* ``"torch"``: the step-by-step ``glb_shard_*`` protocol below, exchanged
  with torch.distributed collectives (NCCL between GPUs, gloo staged through
  the host); kept as the portable form and for CPU tests of the protocol.

Per iteration of the ``"torch"`` form:

1. ``local``   -- the rank relaxes its frontier to the iteration boundary;
                  candidates for remote vertices are min-combined on the
                  sender (shadow cells) and bucketed by owner;
2. ``exchange``-- the (dist << 32 | v) buckets go to their owners: NCCL
                  all-to-all over NVLink (one process per GPU), or device
                  slices when several virtual ranks share one GPU;
3. ``apply``   -- received entries are relaxed with the same generation, so
                  local and remote improvements deduplicate together;
4. ``advance`` -- worklists swap; the run ends when the all-reduced frontier
                  is empty.

Relaxation is confluent (engine.py:7-9), so any partition and exchange order
reaches the reference's fixpoint: distances are bit-identical to a
single-device run.  This module is orchestration only; the kernels, the
split into buckets and the relaxation of received updates are CUDA
(glb_shard_* in libgraphlb_b200.so).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .graph import DeviceCsrGraph, generate_rmat
from .runtime import KernelConfig
from .strategies import RelaxOp, _ID_OF

SHARD_TAGS = ("BS", "WD", "HP")


@dataclass
class ShardGraph:
    """One rank's part of a partitioned graph (resident on `device`)."""

    graph: DeviceCsrGraph
    bounds: np.ndarray  # int64[parts + 1], edge-balanced vertex ranges
    rank: int
    device: int
    peer: "PeerExchange | None" = None  # connected peer transport (cached by run_sharded)
    mdt: int = 0  # HP's window of the WHOLE graph (0: each rank computes its own)

    @property
    def parts(self) -> int:
        return int(self.bounds.shape[0] - 1)

    @property
    def lo(self) -> int:
        return int(self.bounds[self.rank])

    @property
    def hi(self) -> int:
        return int(self.bounds[self.rank + 1])

    @property
    def num_nodes(self) -> int:
        return self.graph.num_nodes


def global_mdt(g, bins: int = 10) -> int:
    """compute_mdt(build_histogram(g, bins)) of the full graph (degrees.py:45-76),
    taken before a shard is restricted: every rank then runs HP with the
    reference's window, not one derived from its own rows."""
    from .analysis import build_histogram, compute_mdt

    return compute_mdt(build_histogram(g, bins))


def partition_bounds(g, parts: int) -> np.ndarray:
    """Edge-balanced contiguous vertex ranges of a device graph."""
    b = np.empty(parts + 1, dtype=np.int64)
    _lib.check(_lib.lib().glb_graph_partition(g.device_graph(), parts, _lib.ptr64(b)),
               "glb_graph_partition")
    return b


def shard_rmat(scale: int, edge_factor: int, parts: int, rank: int, device: int, *,
               params=(0.45, 0.15, 0.15, 0.25), seed: int = 1, weighted: bool = True,
               max_weight: int = 255) -> ShardGraph:
    """Generate the R-MAT graph on `device` (bit-identical to generate_rmat),
    cut the edge-balanced partition and keep this rank's rows."""
    g = generate_rmat(scale, edge_factor, params=params, seed=seed, weighted=weighted,
                      max_weight=max_weight, device=device, download=False)
    bounds = partition_bounds(g, parts)
    mdt = global_mdt(g)
    _lib.check(_lib.lib().glb_graph_restrict(g.device_graph(), int(bounds[rank]),
                                             int(bounds[rank + 1])), "glb_graph_restrict")
    m = ctypes.c_int64()
    _lib.check(_lib.lib().glb_graph_info(g.device_graph(), None, ctypes.byref(m), None, None))
    g.num_edges = int(m.value)
    return ShardGraph(g, bounds, rank, device, mdt=mdt)


def shard_graph(g, parts: int, rank: int, device: int) -> ShardGraph:
    """This rank's part of a host CsrGraph (uploaded, then restricted)."""
    h = ctypes.c_void_p()
    _lib.check(_lib.lib().glb_graph_create(_lib.ptr64(g.row_offsets), _lib.ptr64(g.col_indices),
                                           _lib.ptr64(g.weights), g.num_nodes, g.num_edges,
                                           device, ctypes.byref(h)), "glb_graph_create")
    dg = DeviceCsrGraph(h.value, g.num_nodes, g.num_edges, g.weights is not None, device)
    bounds = partition_bounds(dg, parts)
    mdt = global_mdt(dg)
    _lib.check(_lib.lib().glb_graph_restrict(h.value, int(bounds[rank]), int(bounds[rank + 1])),
               "glb_graph_restrict")
    return ShardGraph(dg, bounds, rank, device, mdt=mdt)


def restrict_host(g, bounds: np.ndarray, rank: int):
    """Host CSR arrays of rank `rank`'s shard over the global id space: the
    owned rows keep their edges, every other row is empty (what
    glb_graph_restrict leaves on the device)."""
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    row = np.asarray(g.row_offsets)
    e_lo, e_hi = int(row[lo]), int(row[hi])
    r = np.clip(row, e_lo, e_hi) - e_lo
    r[: lo + 1] = 0
    r[hi:] = e_hi - e_lo
    col = np.ascontiguousarray(g.col_indices[e_lo:e_hi])
    w = None if g.weights is None else np.ascontiguousarray(g.weights[e_lo:e_hi])
    return np.ascontiguousarray(r, dtype=np.int64), col, w


def shard_host_graph(g, bounds: np.ndarray, rank: int, device: int, mdt: int = 0) -> ShardGraph:
    """Upload only this rank's rows of a host CsrGraph (the sharded form of
    glb_graph_create): 1/P of the edges cross PCIe on every rank.  `mdt`: the
    whole graph's HP window (global_mdt), 0 = per rank."""
    row, col, w = restrict_host(g, bounds, rank)
    h = ctypes.c_void_p()
    _lib.check(_lib.lib().glb_graph_create(_lib.ptr64(row), _lib.ptr64(col), _lib.ptr64(w),
                                           g.num_nodes, int(col.shape[0]), device, ctypes.byref(h)),
               "glb_graph_create")
    dg = DeviceCsrGraph(h.value, g.num_nodes, int(col.shape[0]), w is not None, device)
    return ShardGraph(dg, np.asarray(bounds, dtype=np.int64), rank, device, mdt=mdt)


# ----------------------------------------------------------------- backends
class CudaShard:
    """glb_shard_* calls for one rank; buffers are torch tensors on its device."""

    def __init__(self, sg: ShardGraph, tag: str, source: int, op: RelaxOp, cfg: KernelConfig,
                 torch):
        if tag.upper() not in SHARD_TAGS:
            raise ValueError(f"sharded runs support {SHARD_TAGS}, not {tag!r}")
        self.sg = sg
        self.torch = torch
        self.h = sg.graph.device_graph()
        p = _lib.RunParams()
        p.strategy = _ID_OF[tag.upper()]
        p.algo = _lib.GLB_BFS if op.kind == "bfs" else _lib.GLB_SSSP
        p.source = source
        p.bins = 10
        p.mdt = sg.mdt
        p.chunked = 1
        p.max_cells = 1 << 62
        p.block_size = cfg.block_size
        p.hp_fallback = 1
        p.record_timing = 1 if cfg.record_timing else 0
        self.dev = torch.device("cuda", sg.device)
        self.send = torch.empty(sg.num_nodes, dtype=torch.int64, device=self.dev)
        _lib.check(_lib.lib().glb_shard_begin(self.h, ctypes.byref(p), _lib.ptr64(sg.bounds),
                                              sg.parts, sg.rank), "glb_shard_begin")

    def local(self):
        """Relax to the iteration boundary; returns (per-owner send counts, send
        buffer, number of owned vertices already in the next frontier)."""
        counts = np.zeros(self.sg.parts, dtype=np.int64)
        nxt = ctypes.c_int64()
        _lib.check(_lib.lib().glb_shard_local(self.h, _lib.ptr64(counts),
                                              ctypes.c_void_p(self.send.data_ptr()),
                                              self.send.numel(), ctypes.byref(nxt)),
                   "glb_shard_local")
        return counts, self.send, int(nxt.value)

    def apply(self, recv, n: int):
        if n:
            _lib.check(_lib.lib().glb_shard_apply(self.h, ctypes.c_void_p(recv.data_ptr()), n),
                       "glb_shard_apply")

    def advance(self) -> int:
        f = ctypes.c_int64()
        _lib.check(_lib.lib().glb_shard_advance(self.h, ctypes.byref(f)), "glb_shard_advance")
        return int(f.value)

    def finish(self):
        out = np.empty(self.sg.hi - self.sg.lo, dtype=np.int64)
        st = _lib.RunStats()
        _lib.check(_lib.lib().glb_shard_finish(self.h, _lib.ptr64(out), ctypes.byref(st)),
                   "glb_shard_finish")
        return out, {f: getattr(st, f) for f, _ in _lib.RunStats._fields_}


# -------------------------------------------------------- peer transport
class PeerExchange:
    """One rank's exchange region (glb_peer_*), connected to its peers."""

    def __init__(self, sg: ShardGraph):
        self.sg = sg
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().glb_peer_create(sg.graph.device_graph(), _lib.ptr64(sg.bounds),
                                              sg.parts, sg.rank, ctypes.byref(h)),
                   "glb_peer_create")
        self.h = h.value

    def handle(self) -> bytes:
        buf = ctypes.create_string_buffer(_lib.GLB_PEER_HANDLE_BYTES)
        _lib.check(_lib.lib().glb_peer_handle(self.h, buf), "glb_peer_handle")
        return buf.raw

    def connect(self, handles: list[bytes]) -> None:
        """Map every other rank's region (handles in rank order)."""
        if len(handles) != self.sg.parts:
            raise ValueError("one handle per rank")
        blob = b"".join(handles)
        _lib.check(_lib.lib().glb_peer_connect(self.h, blob), "glb_peer_connect")

    @staticmethod
    def connect_local(peers: list["PeerExchange"]) -> None:
        arr = (ctypes.c_void_p * len(peers))(*[p.h for p in peers])
        _lib.check(_lib.lib().glb_peer_connect_local(arr, len(peers)), "glb_peer_connect_local")

    @classmethod
    def over(cls, sg: ShardGraph, group=None) -> "PeerExchange":
        """Create this rank's region and connect it to every rank of the
        torch.distributed group (IPC handles all-gathered)."""
        import torch.distributed as dist

        px = cls(sg)
        handles: list = [None] * sg.parts
        dist.all_gather_object(handles, px.handle(), group=group)
        px.connect(handles)
        dist.barrier(group=group)
        return px

    def run(self, tag: str, source: int, op: RelaxOp, cfg: KernelConfig | None = None):
        """This rank's part of a sharded run: int64 distances of [lo, hi) and
        stats (run stats + exchange stats under ``"exchange"``)."""
        cfg = cfg or KernelConfig()
        p = _shard_params(tag, source, op, cfg, self.sg.mdt)
        out = np.empty(self.sg.hi - self.sg.lo, dtype=np.int64)
        st = _lib.RunStats()
        xs = _lib.PeerStats()
        _lib.check(_lib.lib().glb_peer_run(self.h, ctypes.byref(p), _lib.ptr64(out),
                                           ctypes.byref(st), ctypes.byref(xs)), "glb_peer_run")
        return out, _stats(st, xs)

    def close(self) -> None:
        if self.h:
            _lib.lib().glb_peer_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _shard_params(tag: str, source: int, op: RelaxOp, cfg: KernelConfig, mdt: int = 0):
    if tag.upper() not in SHARD_TAGS:
        raise ValueError(f"sharded runs support {SHARD_TAGS}, not {tag!r}")
    p = _lib.RunParams()
    p.strategy = _ID_OF[tag.upper()]
    p.algo = _lib.GLB_BFS if op.kind == "bfs" else _lib.GLB_SSSP
    p.source = source
    p.bins = 10
    p.mdt = mdt
    p.chunked = 1
    p.max_cells = 1 << 62
    p.block_size = cfg.block_size
    p.hp_fallback = 1
    p.dist_bits = cfg.dist_bits
    p.loop_mode = _lib.GLB_LOOP_GRAPH
    p.record_timing = 1 if cfg.record_timing else 0
    return p


def _stats(st, xs=None) -> dict:
    d = {f: getattr(st, f) for f, _ in _lib.RunStats._fields_}
    if xs is not None:
        d["exchange"] = {f: getattr(xs, f) for f, _ in _lib.PeerStats._fields_}
        d["bsp_iterations"] = xs.bsp_iterations
    return d


def run_virtual_peer(tag: str, shards: list[ShardGraph], source: int, op: RelaxOp,
                     cfg: KernelConfig | None = None, peers: list[PeerExchange] | None = None):
    """Every rank in this process over the peer transport (glb_peer_run_local):
    virtual ranks sharing one GPU, or one process driving several GPUs.
    Returns the full int64 distance array and the per-rank stats."""
    cfg = cfg or KernelConfig()
    if peers is None:
        peers = [PeerExchange(sg) for sg in shards]
        PeerExchange.connect_local(peers)
    parts = len(shards)
    p = _shard_params(tag, source, op, cfg, shards[0].mdt)
    outs = [np.empty(sg.hi - sg.lo, dtype=np.int64) for sg in shards]
    arr = (ctypes.c_void_p * parts)(*[px.h for px in peers])
    dptr = (_lib._p64 * parts)(*[_lib.ptr64(o) for o in outs])
    st = (_lib.RunStats * parts)()
    xs = (_lib.PeerStats * parts)()
    _lib.check(_lib.lib().glb_peer_run_local(arr, parts, ctypes.byref(p), dptr, st, xs),
               "glb_peer_run_local")
    return np.concatenate(outs), [_stats(st[r], xs[r]) for r in range(parts)]


# --------------------------------------------------------------- transports
class DistTransport:
    """All-to-all of the owner buckets + all-reduce of frontiers through
    torch.distributed (NCCL over NVLink between GPUs; gloo works on CPU)."""

    def __init__(self, torch, group=None):
        import torch.distributed as dist

        self.torch = torch
        self.dist = dist
        self.group = group
        # gloo moves host tensors only: stage device buffers through the host
        self.host = dist.get_backend(group) == "gloo"

    def exchange(self, counts: np.ndarray, send, work: int = 0):
        """All-to-all of the owner buckets.  The count exchange also carries each
        rank's pending work (next-frontier vertices it keeps + updates it sends),
        so the caller learns the global total without a separate all-reduce."""
        torch, dist = self.torch, self.dist
        dev = torch.device("cpu") if self.host else send.device
        c2 = np.empty((counts.shape[0], 2), dtype=np.int64)
        c2[:, 0] = counts
        c2[:, 1] = work
        c_send = torch.as_tensor(c2).to(dev)
        c_recv = torch.empty_like(c_send)
        dist.all_to_all_single(c_recv, c_send, group=self.group)
        c_host = c_recv.cpu()
        self.global_work = int(c_host[:, 1].sum())
        in_split = [int(x) for x in counts]
        out_split = [int(x) for x in c_host[:, 0]]
        total_out = sum(out_split)
        recv = torch.empty(max(total_out, 1), dtype=torch.int64, device=dev)
        dist.all_to_all_single(recv[:total_out], send[:sum(in_split)].to(dev), out_split,
                               in_split, group=self.group)
        return recv.to(send.device), total_out

    def allreduce_sum(self, x: int, device) -> int:
        dev = "cpu" if self.host else device
        t = self.torch.tensor([x], dtype=self.torch.int64, device=dev)
        self.dist.all_reduce(t, group=self.group)
        return int(t.item())


def bsp_loop(shard, transport, device, max_iterations: int | None = None) -> int:
    """One rank of the bulk-synchronous loop; returns the iteration count.

    Termination rides on the bucket-count exchange: when no rank keeps a
    next-frontier vertex and none sends an update, every frontier is empty
    after this iteration (one all-to-all per iteration, no all-reduce)."""
    it = 0
    while True:
        counts, send, keep = shard.local()
        recv, n = transport.exchange(counts, send, keep + int(counts.sum()))
        shard.apply(recv, n)
        shard.advance()
        it += 1
        if transport.global_work == 0:
            return it
        if max_iterations is not None and it >= max_iterations:
            raise RuntimeError("sharded run did not converge")


def run_sharded(tag: str, sg: ShardGraph, source: int, op: RelaxOp,
                cfg: KernelConfig | None = None, transport=None, group=None):
    """This rank's part of a sharded run (one process per GPU).  Returns the
    int64 distances of the owned range [sg.lo, sg.hi) and device stats.

    transport: ``"peer"`` (default; a PeerExchange is created once per shard
    and cached on it), a connected ``PeerExchange``, ``"torch"`` or a
    DistTransport-like object for the step-by-step protocol."""
    import torch

    cfg = cfg or KernelConfig()
    if transport is None or transport == "peer" or isinstance(transport, PeerExchange):
        px = transport if isinstance(transport, PeerExchange) else getattr(sg, "peer", None)
        if px is None:
            px = PeerExchange.over(sg, group)
            sg.peer = px
        return px.run(tag, source, op, cfg)
    if transport == "torch":
        transport = DistTransport(torch, group)
    shard = CudaShard(sg, tag, source, op, cfg, torch)
    it = bsp_loop(shard, transport, shard.dev)
    dist, info = shard.finish()
    info["bsp_iterations"] = it
    return dist, info


def run_virtual(tag: str, shards: list[ShardGraph], source: int, op: RelaxOp,
                cfg: KernelConfig | None = None, transport: str = "peer"):
    """All ranks in one process (e.g. several virtual ranks on one GPU).
    Returns the full int64 distance array and the BSP iteration count.
    ``"peer"``: glb_peer_run_local; ``"torch"``: the step-by-step protocol
    with device-side slicing as the exchange."""
    if transport == "peer":
        d, stats = run_virtual_peer(tag, shards, source, op, cfg)
        return d, stats[0]["bsp_iterations"]
    import torch

    cfg = cfg or KernelConfig()
    ranks = [CudaShard(sg, tag, source, op, cfg, torch) for sg in shards]
    parts = len(shards)
    iters = 0
    while True:
        outs = [r.local()[:2] for r in ranks]
        offs = []
        for me, (counts, _) in enumerate(outs):
            o, run = np.zeros(parts, dtype=np.int64), 0
            for d in range(parts):
                o[d] = run
                if d != me:
                    run += counts[d]
            offs.append(o)
        for d, r in enumerate(ranks):
            pieces = [outs[s][1][offs[s][d]: offs[s][d] + outs[s][0][d]]
                      for s in range(parts) if s != d and outs[s][0][d] > 0]
            if pieces:
                recv = torch.cat([p.to(r.dev) for p in pieces])
                r.apply(recv, int(recv.numel()))
        fronts = [r.advance() for r in ranks]
        iters += 1
        if sum(fronts) == 0:
            break
    dist = np.concatenate([r.finish()[0] for r in ranks])
    return dist, iters
