"""Canonical SHA-256 digests of exported hierarchy stages, shared by the
fixture generator (scripts/make_level0_fixture.py, CPU reference) and the GPU
parity test that checks the full-size fixtures."""
from __future__ import annotations

import hashlib

import numpy as np

from paper_2601_04112_b200 import abi

STAGES = {"A": abi.EXPORT_A, "G": abi.EXPORT_G, "P": abi.EXPORT_P, "partition": abi.EXPORT_PARTITION,
          "gamma": abi.EXPORT_GAMMA, "colors": abi.EXPORT_COLORS, "spectra": abi.EXPORT_SPECTRA,
          "multiplicity": abi.EXPORT_MULTIPLICITY}


def digest(arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def cpu_stage(ho, level: int, name: str):
    """(sizes, arrays) of one stage of an oracle/refbind CpuHierarchy."""
    w = STAGES[name]
    out = ho.export(level, w)
    if w in (abi.EXPORT_A, abi.EXPORT_G, abi.EXPORT_P):
        rp, c, v, shape = out
        return [int(shape[0]), int(shape[1]), int(c.shape[0])], [rp, c, v]
    if w in (abi.EXPORT_PARTITION, abi.EXPORT_COLORS, abi.EXPORT_MULTIPLICITY):
        a, cnt = out
        return [int(a.shape[0]), int(cnt)], [a]
    a0, a1 = out
    return [int(a0.shape[0] - 1), int(a1.shape[0])], [a0, a1]


def gpu_stage(h, level: int, name: str):
    """(sizes, arrays) of one stage of a paper_2601_04112_b200.lsamgdd.Hierarchy."""
    w = STAGES[name]
    if w in (abi.EXPORT_A, abi.EXPORT_G, abi.EXPORT_P):
        m = h._export_csr(level, w)
        return [int(m.n_rows), int(m.n_cols), int(m.col_indices.shape[0])], [m.row_offsets, m.col_indices, m.values]
    if w in (abi.EXPORT_PARTITION, abi.EXPORT_COLORS, abi.EXPORT_MULTIPLICITY):
        a, cnt = h._export_vec(level, w)
        return [int(a.shape[0]), int(cnt)], [a]
    a0, a1 = h._export_offsets(level, w, with_vals=(w == abi.EXPORT_SPECTRA))
    return [int(a0.shape[0] - 1), int(a1.shape[0])], [a0, a1]
