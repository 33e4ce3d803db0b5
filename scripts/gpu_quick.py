import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2601_04112_b200 import configs, lsamgdd, abi
from oracle import refbind
orc = refbind.oracle()
for name, scale in [("c1", None), ("c2", 32), ("c2", 64), ("c2", 128), ("c3", 64)]:
    cfg = configs.config(name, scale)
    over = dict(keep_spectra=True)
    if name == "c3": over["thresh_override"] = 10.0
    t = time.time(); h = lsamgdd.setup(cfg, lsamgdd.params_for(cfg, **over)); ts = time.time() - t
    ho = orc.setup(cfg, refbind.params_for(cfg, keep_spectra=1, **({"thresh_override": 10.0} if name=="c3" else {})))
    ok = h.num_levels == ho.num_levels
    bad = []
    for l in range(min(h.num_levels, ho.num_levels)):
        whats = [abi.EXPORT_A, abi.EXPORT_G] + ([abi.EXPORT_P, abi.EXPORT_PARTITION, abi.EXPORT_GAMMA, abi.EXPORT_COLORS, abi.EXPORT_SPECTRA, abi.EXPORT_MULTIPLICITY] if l + 1 < ho.num_levels else [])
        for w in whats:
            b = ho.export(l, w)
            if w in (abi.EXPORT_A, abi.EXPORT_G, abi.EXPORT_P):
                m = h._export_csr(l, w); a = (m.row_offsets, m.col_indices, m.values)
                same = all(np.array_equal(x, y) for x, y in zip(a, b[:3]))
            elif w in (abi.EXPORT_PARTITION, abi.EXPORT_COLORS, abi.EXPORT_MULTIPLICITY):
                a = h._export_vec(l, w); same = np.array_equal(a[0], b[0]) and a[1] == b[1]
            elif w == abi.EXPORT_GAMMA:
                a = h._export_offsets(l, w); same = np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
            else:
                a = h._export_offsets(l, w, with_vals=True); same = np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
            if not same: bad.append((l, w))
    r = cfg.rhs
    e1 = lsamgdd.vcycle(h, r); e2 = ho.vcycle(r)
    verr = np.linalg.norm(e1 - e2) / np.linalg.norm(e2)
    t = time.time(); x, rep = lsamgdd.pcg(h, r); tsol = time.time() - t
    xo, repo = ho.pcg(r)
    print(name, scale, "levels", h.num_levels, ho.num_levels, "mismatch", bad, "vcycle rel %.2e" % verr,
          "iters", rep.iterations, repo["iterations"], "xerr %.2e" % (np.linalg.norm(x - xo) / np.linalg.norm(xo)),
          "setup %.3f s solve %.3f s" % (ts, tsol), flush=True)
    print("   timings", [(a, round(b, 2)) for a, b in h.timings()])
