import sys, time
sys.path.insert(0, ".")
import paper_1711_00231_b200 as pkg
from tests import graph_specs as gs
import json
for scale in (22, 26):
    t = time.time()
    g = pkg.generate_rmat(scale, 16, seed=1, max_weight=255, device=0, download=(scale == 22))
    print(scale, "device gen+download" if scale == 22 else "device gen", round(time.time() - t, 2), "s")
    if scale == 22:
        big = json.load(open("tests/golden/big.json"))
        print("C2 digest match:", gs.digest(g) == big["C2"]["graph_digest"])
    del g
