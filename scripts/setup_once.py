"""One setup of a config (ncu launch-list target)."""
import sys
sys.path.insert(0, '/root/repo')
from paper_2601_04112_b200 import configs, lsamgdd
cfg = configs.config(sys.argv[1] if len(sys.argv) > 1 else "c2", int(sys.argv[2]) if len(sys.argv) > 2 else None)
h = lsamgdd.setup(cfg, lsamgdd.params_for(cfg))
print("levels", h.num_levels, [(a, round(b, 1)) for a, b in h.timings()])
