"""Per-phase time of the cluster loop's iterations (build with -DGLB_SMALL_TRACE:
tools/build_variant.sh trace -DGLB_SMALL_TRACE; the kernel prints one line per
launch from CTA 0 / thread 0: its own relax work, counter atomics, the cluster
barrier wait, and the single-thread control transition).

    GRAPHLB_B200_LIB=_exp/trace.so python tools/small_trace.py --tags BS,EP,WD --algo bfs
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1711_00231_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--k", type=int, default=4096)
ap.add_argument("--tags", default="BS,EP,WD")
ap.add_argument("--algo", default="bfs")
a = ap.parse_args()
g = pkg.grid_graph(a.k, seed=1, max_weight=255)
for tag in a.tags.split(","):
    r = pkg.run_strategy(tag, g, 0, pkg.RelaxOp(a.algo), pkg.KernelConfig(loop="graph"))
    sys.stdout.flush()
    print(f"== {tag} {a.algo}: device {r.device['device_ms']:.2f} ms", flush=True)
