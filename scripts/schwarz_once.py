"""Level-0 Schwarz sweeps of a config through lsamgdd.apply (ncu target): schwarz_once.py [config] [grid] [reps]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2601_04112_b200 import configs, lsamgdd

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
grid = int(sys.argv[2]) if len(sys.argv) > 2 else None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = configs.config(name, grid)
h = lsamgdd.setup(cfg, lsamgdd.params_for(cfg, probe_levels=1))
r = cfg.rhs
for mode in (lsamgdd.RAS, lsamgdd.RAST):
    for _ in range(reps):
        t = time.perf_counter()
        y = lsamgdd.apply(h, 0, r, mode)
        dt = time.perf_counter() - t
    print("mode", mode, "norm", float(np.linalg.norm(y)), "host call %.2f ms" % (dt * 1e3))
