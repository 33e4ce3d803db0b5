"""One setup of a config: per-level stage times and level sizes."""
import sys
sys.path.insert(0, '/root/repo')
from paper_2601_04112_b200 import configs, lsamgdd
cfg = configs.config(sys.argv[1] if len(sys.argv) > 1 else "c2", int(sys.argv[2]) if len(sys.argv) > 2 else None)
for rep in range(2):
    h = lsamgdd.setup(cfg, lsamgdd.params_for(cfg))
print("levels", h.num_levels)
from paper_2601_04112_b200 import abi
import numpy as np
for l, s in enumerate(h.summary):
    g = h._sizes(l, abi.EXPORT_G)
    line = f"{l} dim {s.dim} nnzA {s.nnz} aggs {s.n_aggregates} kc {s.k_c} modes {s.modes_kept} G {g[0]}x{g[1]} nnzG {g[2]}"
    if l + 1 < h.num_levels:
        topo = h.levels[l].topology
        nw = np.array([len(o) for o in topo.omega]); ng = np.array([len(o) for o in topo.gamma])
        line += f" | nw max {nw.max()} mean {nw.mean():.0f} ng max {ng.max()} mean {ng.mean():.0f}"
    print(line)
lvl = -1
for name, ms in h.timings():
    if name == "aggregation_topology":
        lvl += 1
    print(f"L{max(lvl, 0)} {name:24s} {ms:9.1f}")
print("total_ms", round(sum(ms for _, ms in h.timings()), 1))
