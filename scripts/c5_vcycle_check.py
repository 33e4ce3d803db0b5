import sys
sys.path.insert(0, ".")
import numpy as np
from oracle import refbind
from paper_2601_04112_b200 import configs, lsamgdd
cfg = configs.config("c5", 12)
h = lsamgdd.setup(cfg, lsamgdd.params_for(cfg))
ho = refbind.oracle().setup(cfg, refbind.params_for(cfg))
r = cfg.rhs
e, eo = lsamgdd.vcycle(h, r), ho.vcycle(r)
print("vcycle rel err", np.linalg.norm(e - eo) / np.linalg.norm(eo))
for l in range(h.num_levels - 1):
    rr = np.random.default_rng(l).uniform(-1, 1, h.summary[l].dim)
    for mode in (lsamgdd.RAS, lsamgdd.RAST):
        y, yo = lsamgdd.apply(h, l, rr, mode), ho.schwarz_apply(rr, l, mode)
        print("level", l, "mode", mode, "schwarz rel err", np.linalg.norm(y - yo) / np.linalg.norm(yo), "dim", h.summary[l].dim, "aggs", h.summary[l].n_aggregates)
x, rep = lsamgdd.pcg(h, r); xo, repo = ho.pcg(r)
print("iters", rep.iterations, repo["iterations"], "x err", np.linalg.norm(x - xo) / np.linalg.norm(xo))
