"""Config 3 at its full 4096² grid, level-0 stages only (probe_levels = 1), from a factor generated on
the device: stage times, level sizes and the level-0 Schwarz sweep times. usage: c3_full_level0.py [grid]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2601_04112_b200 import configs, lsamgdd

grid = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
t = time.perf_counter()
g = lsamgdd.generate_stencil_rows(*configs.config_stencil("c3", grid))
print(f"generated c3 {grid}^2 on the device: {g.n_rows} x {g.n_cols}, nnz {g.nnz}, {time.perf_counter() - t:.3f} s", flush=True)
part, nagg = configs.block_partition_2d(grid, grid, 8, 8)
p = lsamgdd.LevelParams(thresh_override=20.0, level0_overlap=2, probe_levels=1, level0_partition=part,
                        level0_n_aggregates=nagg)
for rep in range(2):
    t = time.perf_counter()
    h = lsamgdd.setup(g, p)
    print(f"setup (level-0 stages) {time.perf_counter() - t:.3f} s", [(a, round(b, 1)) for a, b in h.timings()], flush=True)
    if rep == 0:
        del h
for l, s in enumerate(h.summary):
    print(l, "dim", s.dim, "nnzA", s.nnz, "aggs", s.n_aggregates, "modes", s.modes_kept, "thresh", s.thresh)
r = np.random.default_rng(0).uniform(-1, 1, g.n_cols)
for mode in (lsamgdd.RAS, lsamgdd.RAST):
    for _ in range(3):
        t = time.perf_counter()
        y = lsamgdd.apply(h, 0, r, mode)
        dt = time.perf_counter() - t
    print("mode", mode, "norm", float(np.linalg.norm(y)), "host call %.2f ms" % (dt * 1e3), flush=True)
