"""One rank of test_gpu_peer.test_peer_two_processes_over_cuda_ipc (GPU 0 shared
by both processes; torch.distributed gloo only gathers the IPC handles)."""
import sys
from pathlib import Path

import numpy as np
import torch.distributed as dist

import paper_1711_00231_b200 as pkg
from paper_1711_00231_b200 import sharded


def main(out_dir: str) -> None:
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    g = pkg.generate_rmat(14, 8, seed=3, max_weight=255, device=0, download=False)
    exp = {a: pkg.run_wd(g, 0, pkg.RelaxOp(a), pkg.KernelConfig()).dist.array for a in ("bfs", "sssp")}
    bounds = sharded.partition_bounds(g, world)
    mdt = sharded.global_mdt(g)
    from paper_1711_00231_b200 import _lib
    _lib.check(_lib.lib().glb_graph_restrict(g.device_graph(), int(bounds[rank]),
                                             int(bounds[rank + 1])))
    sg = sharded.ShardGraph(g, bounds, rank, 0, mdt=mdt)
    res = []
    for algo in ("bfs", "sssp"):
        for tag in sharded.SHARD_TAGS:
            d, info = sharded.run_sharded(tag, sg, 0, pkg.RelaxOp(algo))
            assert info["exchange"]["transport"] == 1  # CUDA IPC
            full = [None] * world
            dist.all_gather_object(full, d)
            res.append("ok" if np.array_equal(np.concatenate(full), exp[algo]) else
                       f"bad:{algo}:{tag}")
    if rank == 0:
        Path(out_dir, "result.txt").write_text(" ".join(res))
    sg.peer.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
