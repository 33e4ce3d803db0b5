"""Bit-identical reruns of the V-cycle and PCG on small instances of every config (row-layout and
lane-layout sweeps, colour-ordered RAS-T with programmatic dependent launch): det_small_configs.py [reps]"""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2601_04112_b200 import configs, lsamgdd
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 150
cases = [("c1", 64, {}), ("c2", 192, {}), ("c3", 128, {"thresh_override": 10.0}), ("c4", 48, {}), ("c5", 12, {})]
total_bad = 0
for name, scale, over in cases:
    cfg = configs.config(name, scale)
    h = lsamgdd.setup(cfg, lsamgdd.params_for(cfg, **over))
    v0 = lsamgdd.vcycle(h, cfg.rhs)
    x0, rep0 = lsamgdd.pcg(h, cfg.rhs, 1e-8, 1000)
    bad = [0, 0]
    for i in range(reps):
        if not np.array_equal(lsamgdd.vcycle(h, cfg.rhs), v0):
            bad[0] += 1
        x, rep = lsamgdd.pcg(h, cfg.rhs, 1e-8, 1000)
        if not np.array_equal(x, x0):
            bad[1] += 1
    print(name, scale, "levels", h.num_levels, "iterations", rep0.iterations, "mismatches (vcycle, pcg) of", reps, ":", bad,
          flush=True)
    total_bad += sum(bad)
    del h
print("total mismatches", total_bad)
