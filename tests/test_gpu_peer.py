"""GPU parity of the peer-memory sharded path (glb_peer_*): the whole BSP loop
inside the library, remote updates written straight into the owners' HBM.

* virtual ranks of one process (glb_peer_run_local) on the golden corpus and
  on device-generated R-MATs, every shard strategy, both distance tiers that
  the auto choice can pick plus the pinned 24 / 64-bit tiers;
* a global overflow promotes every rank to the next tier at once;
* two real processes sharing GPU 0 exchange through CUDA IPC handles
  (gathered with torch.distributed/gloo) -- the same code path as one
  process per GPU, bit-exact against the single-GPU result.
"""

import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_1711_00231_b200 as pkg
from paper_1711_00231_b200 import _lib, sharded
from tests import graph_specs as gs

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    _lib.lib()
    assert _lib.device_count() > 0, "no CUDA device visible to libgraphlb_b200.so"


def test_peer_virtual_ranks_match_golden(golden):
    for gid in ("rmat10_s1", "rmat10_skew", "grid24", "quirks", "rmat12_s4", "degrees"):
        g = gs.build(pkg, gs.CORPUS[gid])
        full_mdt = pkg.compute_mdt(pkg.build_histogram(g, 10))
        for parts in (1, 2, 3, 5):
            shards = [sharded.shard_graph(g, parts, r, 0) for r in range(parts)]
            assert all(sg.mdt == full_mdt for sg in shards)
            for algo in ("bfs", "sssp"):
                exp = golden["corpus"][f"{gid}|0|{algo}"]
                for tag in sharded.SHARD_TAGS:
                    d, st = sharded.run_virtual_peer(tag, shards, 0, pkg.RelaxOp(algo))
                    assert np.array_equal(d, exp), (gid, parts, algo, tag)
                    iters = {s["bsp_iterations"] for s in st}
                    assert len(iters) == 1, iters  # every rank stopped after the same iteration
                    sent = sum(s["exchange"]["sent_entries"] for s in st)
                    recv = sum(s["exchange"]["recv_entries"] for s in st)
                    assert sent == recv, (sent, recv)
                    if tag == "HP":  # every rank windows by the whole graph's MDT
                        assert {s["mdt"] for s in st} == {shards[0].mdt}, (gid, parts)


def test_peer_and_torch_transports_agree_on_rmat():
    shards = [sharded.shard_rmat(14, 8, 4, r, 0, seed=3) for r in range(4)]
    h = pkg.generate_rmat(14, 8, seed=3, max_weight=255)
    for algo in ("bfs", "sssp"):
        exp = pkg.run_wd(h, 0, pkg.RelaxOp(algo), pkg.KernelConfig()).dist.array
        for tag in sharded.SHARD_TAGS:
            d, _ = sharded.run_virtual(tag, shards, 0, pkg.RelaxOp(algo), transport="peer")
            assert np.array_equal(d, exp), ("peer", algo, tag)
            d, _ = sharded.run_virtual(tag, shards, 0, pkg.RelaxOp(algo), transport="torch")
            assert np.array_equal(d, exp), ("torch", algo, tag)


@pytest.mark.parametrize("bits", [24, 32, 64])
def test_peer_pinned_tiers(bits, oracle):
    g = pkg.generate_rmat(13, 8, seed=7, max_weight=255)
    shards = [sharded.shard_graph(g, 3, r, 0) for r in range(3)]
    for algo in ("bfs", "sssp"):
        exp = oracle.oracle_distances(g, 5, algo)
        for tag in sharded.SHARD_TAGS:
            d, st = sharded.run_virtual_peer(tag, shards, 5, pkg.RelaxOp(algo),
                                             pkg.KernelConfig(dist_bits=bits))
            assert np.array_equal(d, exp), (bits, algo, tag)
            assert all(s["dist_bits"] == bits for s in st)
            assert all(s["exchange"]["entry_bytes"] == (16 if bits == 64 else 8) for s in st)


def test_peer_overflow_promotes_every_rank(oracle):
    # a path whose distances pass 2^32: the 32-bit tier overflows on one
    # rank, and every rank restarts at 64 bits at the same iteration
    n = 64
    src = np.arange(n - 1)
    g = pkg.CsrGraph.from_edges(n, src, src + 1, np.full(n - 1, 0xF0000000, dtype=np.int64))
    shards = [sharded.shard_graph(g, 4, r, 0) for r in range(4)]
    exp = oracle.oracle_distances(g, 0, "sssp")
    for tag in sharded.SHARD_TAGS:
        d, st = sharded.run_virtual_peer(tag, shards, 0, pkg.RelaxOp("sssp"))
        assert np.array_equal(d, exp), tag
        assert all(s["dist_bits"] == 64 for s in st)
        with pytest.raises(OverflowError):
            sharded.run_virtual_peer(tag, shards, 0, pkg.RelaxOp("sssp"),
                                     pkg.KernelConfig(dist_bits=32))


def test_peer_24bit_renormalisation_across_ranks(oracle):
    # > 128 BSP iterations at the 24-bit tier: the push tags are reset on
    # every rank between iterations (k_renorm inside the resumed loop graph)
    g = pkg.grid_graph(96, seed=2, max_weight=255)
    shards = [sharded.shard_graph(g, 2, r, 0) for r in range(2)]
    for algo in ("bfs", "sssp"):
        exp = oracle.oracle_distances(g, 0, algo)
        for tag in sharded.SHARD_TAGS:
            d, st = sharded.run_virtual_peer(tag, shards, 0, pkg.RelaxOp(algo),
                                             pkg.KernelConfig(dist_bits=24))
            assert np.array_equal(d, exp), (algo, tag)
            assert st[0]["bsp_iterations"] > 128


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_peer_two_processes_over_cuda_ipc(tmp_path):
    """Two ranks in two processes sharing GPU 0: regions mapped with CUDA IPC,
    handles all-gathered over gloo -- the one-process-per-GPU code path."""
    port = _free_port()
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE="2",
               GLB_PEER_TIMEOUT_S="60", PYTHONPATH=str(ROOT))
    procs = []
    for r in range(2):
        e = dict(env, RANK=str(r), LOCAL_RANK=str(r))
        procs.append(subprocess.Popen([sys.executable, str(ROOT / "tests" / "peer_worker.py"),
                                       str(tmp_path)], env=e, cwd=str(ROOT)))
    rcs = []
    for p in procs:
        try:
            rcs.append(p.wait(timeout=600))
        except subprocess.TimeoutExpired:
            p.kill()
            rcs.append(-9)
    assert rcs == [0, 0], rcs
    res = (tmp_path / "result.txt").read_text().split()
    assert res == ["ok"] * 6, res


def test_peer_missing_rank_times_out_instead_of_hanging(monkeypatch):
    """Rank 0 runs, rank 1 never does: rank 0's mailbox poll gives up after
    GLB_PEER_TIMEOUT_S, the call fails with DeviceError, the peer refuses
    further runs (lockstep lost) and the GPU stays usable."""
    import time

    monkeypatch.setenv("GLB_PEER_TIMEOUT_S", "2")
    g = pkg.generate_rmat(10, 8, seed=1, max_weight=255)
    shards = [sharded.shard_graph(g, 2, r, 0) for r in range(2)]
    peers = [sharded.PeerExchange(sg) for sg in shards]
    sharded.PeerExchange.connect_local(peers)
    t0 = time.time()
    with pytest.raises(_lib.DeviceError, match="did not publish"):
        peers[0].run("WD", 0, pkg.RelaxOp("bfs"))
    assert time.time() - t0 < 60
    with pytest.raises(_lib.DeviceError, match="lockstep"):
        peers[0].run("WD", 0, pkg.RelaxOp("bfs"))
    for p in peers:
        p.close()
    # the device is healthy: a fresh run on the same GPU is bit-exact
    r = pkg.run_wd(g, 0, pkg.RelaxOp("bfs"), pkg.KernelConfig())
    h = pkg.generate_rmat(10, 8, seed=1, max_weight=255)
    exp = pkg.run_bs(h, 0, pkg.RelaxOp("bfs"), pkg.KernelConfig()).dist.array
    assert np.array_equal(r.dist.array, exp)
