"""GPU vs oracle on small C3/C5 instances (hierarchy sizes, opcx, PCG), plus
GPU-only timing of larger instances. Diagnostic."""
import sys, time
import numpy as np
sys.path.insert(0, '/root/repo')
from paper_2601_04112_b200 import configs, lsamgdd
from oracle import refbind
orc = refbind.oracle()
for name, scale, over, check in [("c5", 16, {}, True), ("c5", 32, {}, True), ("c3", 128, {"thresh_override": 10.0}, True),
                                  ("c5", 64, {}, False), ("c3", 512, {"thresh_override": 10.0}, False)]:
    cfg = configs.config(name, scale)
    t = time.time(); h = lsamgdd.setup(cfg, lsamgdd.params_for(cfg, **over)); ts = time.time() - t
    t = time.time(); x, rep = lsamgdd.pcg(h, cfg.rhs, 1e-8, 1000); tsol = time.time() - t
    msg = f"{name} {scale} n={cfg.n} levels={h.num_levels} opcx={lsamgdd.operator_complexity(h):.4f} it={rep.iterations} conv={rep.converged} setup={ts:.2f}s solve={tsol:.2f}s"
    if check:
        ho = orc.setup(cfg, refbind.params_for(cfg, **over))
        xo, repo = ho.pcg(cfg.rhs, 1e-8, 1000)
        same = h.num_levels == ho.num_levels and all(h.summary[l].nnz == ho.summary(l)["nnz"] for l in range(h.num_levels))
        msg += f" | oracle levels={ho.num_levels} opcx={ho.operator_complexity():.4f} it={repo['iterations']} sizes_match={same} xerr={np.linalg.norm(x-xo)/np.linalg.norm(xo):.2e}"
    print(msg, flush=True)
