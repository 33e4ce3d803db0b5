#!/usr/bin/env python3
"""Golden fixture of a whole hierarchy for cases whose CPU run is too slow for
the test suite: the plain-C oracle (pinned bit-for-bit to the reference, see
tests/test_oracle_pins.py) builds the hierarchy and runs PCG once here; the
per-level SHA-256 hashes of every exported stage, the level summaries, the
operator complexity, the PCG iteration count, the final residual and the
solution (as a .npy next to the JSON) are committed under tests/golden/.

usage: make_hierarchy_fixture.py c5 16
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import refbind  # noqa: E402
from paper_2601_04112_b200 import configs  # noqa: E402
from tests import _hashes  # noqa: E402


def main():
    name, grid = sys.argv[1], int(sys.argv[2])
    cfg = configs.config(name, grid)
    orc = refbind.oracle()
    t0 = time.perf_counter()
    h = orc.setup(cfg, refbind.params_for(cfg, keep_spectra=1))
    t_setup = time.perf_counter() - t0
    x, rep = h.pcg(cfg.rhs, 1e-8, 1000)
    levels = []
    for l in range(h.num_levels):
        names = ["A", "G"] + (["P", "partition", "gamma", "colors", "spectra", "multiplicity"] if l + 1 < h.num_levels else [])
        lv = {}
        for nm in names:
            sizes, arrays = _hashes.cpu_stage(h, l, nm)
            lv[nm] = {"sizes": sizes, "sha256": _hashes.digest(arrays)}
        levels.append(lv)
    fx = {"config": name, "grid": grid, "n": int(cfg.n), "m": int(cfg.m), "oracle_setup_s": t_setup,
          "num_levels": h.num_levels, "operator_complexity": h.operator_complexity(),
          "summary": [h.summary(l) for l in range(h.num_levels)], "levels": levels,
          "pcg_iterations": int(rep["iterations"]), "pcg_converged": bool(rep["converged"]),
          "residual_first": float(rep["residual_history"][0]), "residual_last": float(rep["residual_history"][-1])}
    base = os.path.join(ROOT, "tests", "golden", f"hier_{name}_{grid}")
    with open(base + ".json", "w") as f:
        json.dump(fx, f, indent=1)
    np.save(base + "_x.npy", x)
    print("wrote", base + ".json", "setup %.1f s" % t_setup, "iters", rep["iterations"])


if __name__ == "__main__":
    main()
