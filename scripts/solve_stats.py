"""Level-0 Schwarz sweep and PCG-operator (Gᵀ(G p)) throughput of config 2,
from the library's event-timed kernel stats; one run per argument (the
argument is exported as LSB_LANE_CH for schedule experiments)."""
import os, sys, time
import numpy as np
sys.path.insert(0, '/root/repo')
from paper_2601_04112_b200 import configs, lsamgdd

scale = int(os.environ.get("SCALE", "1024"))
cfg = configs.config("c2", scale)
p = lsamgdd.params_for(cfg)
x0 = None
for var in sys.argv[1:]:
    os.environ["LSB_LANE_CH"] = var
    h = lsamgdd.setup(cfg, p)
    for _ in range(2):
        x, rep, st = lsamgdd.pcg(h, cfg.rhs, 1e-8, 1000, stats=True)
    if x0 is None:
        x0 = x
    d = float(np.max(np.abs(x - x0)))
    gbs = st["schwarz_bytes"] / (st["schwarz_ms"] / 1e3) / 1e9
    sp = st["spmv_bytes"] / (st["spmv_ms"] / 1e3) / 1e9 if st["spmv_ms"] > 0 else 0.0
    print(f"spmv (Gᵀ(G p)) {sp:.0f} GB/s over {st['spmv_launches']} launches, {st['spmv_ms']:.2f} ms")
    print(f"ch={var}: iters={rep.iterations} solve={rep.solve_seconds*1e3:.2f} ms stats={st} schwarz {gbs:.0f} GB/s max|dx|={d:.3e}", flush=True)
    del h
