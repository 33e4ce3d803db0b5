"""Scaling probe: setup + PCG of a config at several grid sizes on the GPU."""
import sys, time
import numpy as np
sys.path.insert(0, '/root/repo')
from paper_2601_04112_b200 import configs, lsamgdd

name = sys.argv[1]
for scale in [int(s) for s in sys.argv[2:]]:
    t = time.time(); cfg = configs.config(name, scale); tg = time.time() - t
    p = lsamgdd.params_for(cfg)
    t = time.time(); h = lsamgdd.setup(cfg, p); ts = time.time() - t
    t = time.time(); x, rep = lsamgdd.pcg(h, cfg.rhs, 1e-8, 1000); tsol = time.time() - t
    t = time.time(); h2 = lsamgdd.setup(cfg, p); ts2 = time.time() - t
    t = time.time(); x, rep, st = lsamgdd.pcg(h2, cfg.rhs, 1e-8, 1000, stats=True); tsol2 = time.time() - t
    print(f"{name} {scale}: n={cfg.n} gen {tg:.2f}s levels={h.num_levels} opcx={lsamgdd.operator_complexity(h):.4f} "
          f"iters={rep.iterations} conv={rep.converged} setup {ts:.3f}s/{ts2:.3f}s solve {tsol:.3f}s/{tsol2:.3f}s "
          f"unk/s={cfg.n/(ts2+tsol2):.3e}", flush=True)
    print("   stats", st)
    print("   levels", [(s.dim, s.nnz, s.n_aggregates, s.modes_kept) for s in h.summary])
    print("   timings", [(a, round(b, 1)) for a, b in h2.timings()], flush=True)
    del h, h2
