"""Per-level shape statistics of a hierarchy (aggregate, ω and Γ sizes) and the
per-level setup stage timings. Diagnostic only."""
import sys, time, json
import numpy as np
sys.path.insert(0, '/root/repo')
from paper_2601_04112_b200 import configs, lsamgdd, abi

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
grid = int(sys.argv[2]) if len(sys.argv) > 2 else None
cfg = configs.config(name, grid)
t = time.time()
h = lsamgdd.setup(cfg, lsamgdd.params_for(cfg))
print("setup wall %.2f s" % (time.time() - t))
print("timings", [(a, round(b, 1)) for a, b in h.timings()])
for l in range(h.num_levels - 1):
    s = h.summary[l]
    go, _ = h._export_offsets(l, abi.EXPORT_GAMMA)
    part = h._export_vec(l, abi.EXPORT_PARTITION)[0]
    ng = np.diff(go)
    nw = np.bincount(part)
    print(f"L{l}: dim={s.dim} nnz={s.nnz} aggs={s.n_aggregates} kc={s.k_c} modes={s.modes_kept} "
          f"nw max={nw.max()} mean={nw.mean():.1f}  ng max={ng.max()} mean={ng.mean():.1f} "
          f"sum ng^3={float((ng.astype(float)**3).sum()):.3e} n(ng>=48)={(ng>=48).sum()} n(ng>=200)={(ng>=200).sum()}")
    big = np.sort(ng)[-8:]
    print("     largest ng:", big.tolist())
