#!/usr/bin/env python3
"""Full-size stage-wise fixture: runs the compiled reference (oracle/_ref, the
unmodified headers) on the level-0 stages of a BASELINE config at its full
grid (probe_levels = 1: no coarse levels, which the reference cannot finish at
this size) and stores SHA-256 hashes of every exported stage array plus the
reference's stage times. tests/test_gpu_parity.py compares the GPU exports of
the same stages with these hashes.

usage: make_level0_fixture.py c2 1024 [threads]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import refbind  # noqa: E402
from paper_2601_04112_b200 import abi, configs  # noqa: E402

from tests import _hashes  # noqa: E402


def level_hashes(hier, level: int, names) -> dict:
    out = {}
    for nm in names:
        sizes, arrays = _hashes.cpu_stage(hier, level, nm)
        out[nm] = {"sizes": sizes, "sha256": _hashes.digest(arrays)}
    return out


def main():
    name, grid = sys.argv[1], int(sys.argv[2])
    threads = int(sys.argv[3]) if len(sys.argv) > 3 else (os.cpu_count() or 1)
    os.environ["LSAMGDD_REF_THREADS"] = str(threads)
    cfg = configs.config(name, grid)
    p = refbind.params_for(cfg, probe_levels=1, keep_spectra=1)
    chk = refbind.reference()
    t0 = time.perf_counter()
    h = chk.setup(cfg, p)
    wall = time.perf_counter() - t0
    fx = {"config": name, "grid": grid, "n": int(cfg.n), "m": int(cfg.m), "reference_threads_local_gevp": threads,
          "reference_wall_s": wall, "reference_stage_s": [[a, b] for a, b in h.timings()],
          "level0": level_hashes(h, 0, ["A", "G", "P", "partition", "gamma", "colors", "spectra", "multiplicity"]),
          "level1": level_hashes(h, 1, ["A", "G"]),
          "summary0": h.summary(0)}
    path = os.path.join(ROOT, "tests", "golden", f"level0_{name}_{grid}.json")
    with open(path, "w") as f:
        json.dump(fx, f, indent=1)
    print("wrote", path, "wall %.1f s" % wall, fx["reference_stage_s"])


if __name__ == "__main__":
    main()
