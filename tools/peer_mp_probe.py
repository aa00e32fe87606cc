"""Probe: N processes sharing GPU 0 over the peer transport (gloo gathers the
IPC handles).  Launch: torchrun --nproc-per-node N tools/peer_mp_probe.py SCALE [ref]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch.distributed as dist
import paper_1711_00231_b200 as pkg
from paper_1711_00231_b200 import _lib, sharded

scale = int(sys.argv[1])
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
def log(*a):
    print(f"[r{rank} {time.time() % 1000:.3f}]", *a, flush=True)
g = pkg.generate_rmat(scale, 16, seed=1, max_weight=255, device=0, download=False)
log("generated")
if rank == 0 and "ref" in sys.argv:
    ref = pkg.run_strategy("WD", g, 0, pkg.RelaxOp("sssp"), pkg.KernelConfig(instrument=False)).dist.array
    log("ref done")
bounds = sharded.partition_bounds(g, world)
mdt = sharded.global_mdt(g)
_lib.check(_lib.lib().glb_graph_restrict(g.device_graph(), int(bounds[rank]), int(bounds[rank + 1])))
sg = sharded.ShardGraph(g, bounds, rank, 0, mdt=mdt)
px = sharded.PeerExchange.over(sg)
log("connected")
for algo in ("bfs", "sssp"):
    for tag in ("BS", "WD"):
        t = time.time()
        d, info = px.run(tag, 0, pkg.RelaxOp(algo))
        log(algo, tag, round(time.time() - t, 3), info["bsp_iterations"], info["exchange"])
px.close()
dist.barrier()
log("done")
