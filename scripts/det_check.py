import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2601_04112_b200 import configs, lsamgdd
grid = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
cfg = configs.config("c2", grid)
h = lsamgdd.setup(cfg, lsamgdd.params_for(cfg))
r = cfg.rhs
for mode in (lsamgdd.RAS, lsamgdd.RAST):
    ys = [lsamgdd.apply(h, 0, r, mode) for _ in range(4)]
    print("mode", mode, "identical", [bool(np.array_equal(ys[0], y)) for y in ys[1:]], "max diff", max(float(np.abs(ys[0] - y).max()) for y in ys[1:]))
vs = [lsamgdd.vcycle(h, r) for _ in range(3)]
print("vcycle identical", [bool(np.array_equal(vs[0], v)) for v in vs[1:]], max(float(np.abs(vs[0] - v).max()) for v in vs[1:]))
xs = [lsamgdd.pcg(h, r)[0] for _ in range(3)]
print("pcg identical", [bool(np.array_equal(xs[0], x)) for x in xs[1:]], max(float(np.abs(xs[0] - x).max()) for x in xs[1:]))
