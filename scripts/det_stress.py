import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2601_04112_b200 import configs, lsamgdd
grid = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cfg = configs.config("c2", grid)
h = lsamgdd.setup(cfg, lsamgdd.params_for(cfg))
r = cfg.rhs
rng = np.random.default_rng(0)
x0 = lsamgdd.pcg(h, r)[0]
v0 = lsamgdd.vcycle(h, r)
t0 = lsamgdd.apply(h, 0, r, lsamgdd.RAST)
bad = [0, 0, 0]
for i in range(reps):
    a = rng.uniform(-1, 1, cfg.n)
    lsamgdd.vcycle(h, a)  # disturb the pool / caches between repeats
    if not np.array_equal(lsamgdd.apply(h, 0, r, lsamgdd.RAST), t0):
        bad[0] += 1
    if not np.array_equal(lsamgdd.vcycle(h, r), v0):
        bad[1] += 1
    x = lsamgdd.pcg(h, r)[0]
    if not np.array_equal(x, x0):
        bad[2] += 1
        print("rep", i, "pcg differs: max", float(np.abs(x - x0).max()), "count", int((x != x0).sum()))
print("mismatches (rast, vcycle, pcg) of", reps, ":", bad)
