"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck / synccheck):
config 1 at 64² (warp and CTA classes, lane-layout Schwarz) and config 2 at 96²
(TMA Schwarz sweep, RAS-T slots, multi-level Galerkin), setup + PCG each, plus
the on-device generator. usage: compute-sanitizer --tool memcheck python scripts/sanitize_small.py"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2601_04112_b200 import configs, lsamgdd

for name, scale in (("c1", 64), ("c2", 96)):
    cfg = configs.config(name, scale)
    h = lsamgdd.setup(cfg, lsamgdd.params_for(cfg))
    x, rep = lsamgdd.pcg(h, cfg.rhs, 1e-8, 200)
    print(name, scale, "levels", h.num_levels, "iterations", rep.iterations, "converged", rep.converged, flush=True)
    del h
g = lsamgdd.generate_stencil_rows(*configs.config_stencil("c2", 96))
cfg = configs.config("c2", 96)
assert np.array_equal(g.to_host().values, cfg.g_vals)
g.close()
print("done")
