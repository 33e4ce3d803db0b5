"""One hierarchy; between repeats the memory pool is churned by a small setup (its freed workspaces hold
garbage); compares level-0 RAS, RAS-T, the V-cycle and PCG with their first results. det_churn.py [grid] [reps]"""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2601_04112_b200 import configs, lsamgdd
grid = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 60
cfg = configs.config("c2", grid)
h = lsamgdd.setup(cfg, lsamgdd.params_for(cfg))
small = configs.config("c2", 384)
ps = lsamgdd.params_for(small)
r = cfg.rhs
ref = None
bad = {"ras": 0, "rast": 0, "vcycle": 0, "pcg": 0}
for i in range(reps):
    hs = lsamgdd.setup(small, ps)
    del hs
    cur = {"ras": lsamgdd.apply(h, 0, r, lsamgdd.RAS), "rast": lsamgdd.apply(h, 0, r, lsamgdd.RAST),
           "vcycle": lsamgdd.vcycle(h, r), "pcg": lsamgdd.pcg(h, r, 1e-8, 1000)[0]}
    if ref is None:
        ref = cur
        continue
    for k in bad:
        if not np.array_equal(cur[k], ref[k]):
            bad[k] += 1
            d = cur[k] != ref[k]
            print("rep", i, k, "differs in", int(d.sum()), "entries, max abs", float(np.abs(cur[k] - ref[k]).max()),
                  "first index", int(np.argmax(d)), flush=True)
print("mismatches of", reps - 1, ":", bad)
