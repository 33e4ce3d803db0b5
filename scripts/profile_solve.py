"""Setup config 2 once, then run V-cycles and one PCG solve (ncu target)."""
import sys
import numpy as np
sys.path.insert(0, '/root/repo')
from paper_2601_04112_b200 import configs, lsamgdd
cfg = configs.config(sys.argv[1] if len(sys.argv) > 1 else "c2", int(sys.argv[2]) if len(sys.argv) > 2 else None)
h = lsamgdd.setup(cfg, lsamgdd.params_for(cfg))
for _ in range(3):
    e = lsamgdd.vcycle(h, cfg.rhs)
x, rep = lsamgdd.pcg(h, cfg.rhs)
print("levels", h.num_levels, "iters", rep.iterations, "converged", rep.converged)
