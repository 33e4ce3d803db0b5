"""Repeat [setup -> pcg -> vcycle x2 -> pcg] and compare the two PCG results bit for bit (the pattern of
test_full_size_config2): det_setup_stress.py [grid] [reps]"""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2601_04112_b200 import configs, lsamgdd
grid = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = configs.config("c2", grid)
p = lsamgdd.params_for(cfg)
rng = np.random.default_rng(3)
xref = None
bad = 0
for i in range(reps):
    h = lsamgdd.setup(cfg, p)
    x, rep = lsamgdd.pcg(h, cfg.rhs, 1e-8, 1000)
    a = rng.uniform(-1, 1, cfg.n)
    lsamgdd.vcycle(h, a)
    lsamgdd.vcycle(h, a)
    x2, rep2 = lsamgdd.pcg(h, cfg.rhs, 1e-8, 1000)
    if xref is None:
        xref = x
        href = rep.residual_history.copy()
    for nm, rr in (("first", rep), ("second", rep2)):
        hh = rr.residual_history
        if len(hh) != len(href) or not np.array_equal(hh, href):
            m = min(len(hh), len(href))
            dif = np.nonzero(hh[:m] != href[:m])[0]
            k0 = int(dif[0]) if len(dif) else m
            print("rep", i, nm, "history differs from iteration", k0, "rel", float(abs(hh[k0] - href[k0]) / href[k0]) if k0 < m else -1,
                  "len", len(hh), len(href), flush=True)
    d1, d2 = int((x != x2).sum()), int((x != xref).sum())
    if d1 or d2:
        bad += 1
        print("   max |x - xref| / max|xref|", float(np.abs(x - xref).max() / np.abs(xref).max()),
              float(np.abs(x2 - xref).max() / np.abs(xref).max()))
        print("rep", i, "first vs second pcg differ in", d1, "entries; first vs rep 0 in", d2, "second vs rep 0 in",
              int((x2 != xref).sum()), "iters", rep.iterations, flush=True)
    del h
print("mismatching repeats:", bad, "of", reps)
