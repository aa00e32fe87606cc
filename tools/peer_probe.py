"""Quick probe of the peer path with virtual ranks on one GPU (short timeout)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1711_00231_b200 as pkg
from paper_1711_00231_b200 import sharded
g = pkg.generate_rmat(12, 8, seed=3, max_weight=255)
exp = pkg.run_wd(g, 0, pkg.RelaxOp("sssp"), pkg.KernelConfig()).dist.array
for parts in (1, 2, 3):
    shards = [sharded.shard_graph(g, parts, r, 0) for r in range(parts)]
    for tag in sharded.SHARD_TAGS:
        t = time.time()
        d, st = sharded.run_virtual_peer(tag, shards, 0, pkg.RelaxOp("sssp"))
        print(parts, tag, np.array_equal(d, exp), st[0]["bsp_iterations"], round(time.time() - t, 3),
              st[0]["exchange"], flush=True)
