"""Small hand-built inputs mirroring the reference's unit-test fixtures
(proj/tests/test_util.hpp and the per-suite helpers)."""
from __future__ import annotations

import numpy as np

from paper_2601_04112_b200 import abi, configs


def csr_from_dense(d: np.ndarray):
    rows, cols = np.nonzero(d)
    vals = d[rows, cols]
    rowptr = np.zeros(d.shape[0] + 1, np.int64)
    np.add.at(rowptr, rows + 1, 1)
    return np.cumsum(rowptr).astype(np.int64), cols.astype(np.int64), vals.astype(np.float64)


def chain_factor(n: int, shift: float = 0.0):
    """test_splitting.cpp:21-28: row k couples nodes k and k+1 (-1, +1);
    optional sqrt(shift)·I rows make A = GᵀG + shift·I definite."""
    m = n - 1 + (n if shift > 0 else 0)
    d = np.zeros((m, n))
    for k in range(n - 1):
        d[k, k] = -1.0
        d[k, k + 1] = 1.0
    if shift > 0:
        for k in range(n):
            d[n - 1 + k, k] = np.sqrt(shift)
    rp, c, v = csr_from_dense(d)
    return rp, c, v, n


def gradient_factor_2d(nx: int, ny: int):
    """test_util.hpp:119-132: two forward-difference rows per node, h = 1/(n+1)."""
    hx, hy = 1.0 / (nx + 1), 1.0 / (ny + 1)
    n = nx * ny
    d = np.zeros((2 * n, n))
    for j in range(ny):
        for i in range(nx):
            node = j * nx + i
            d[2 * node, node] = -1.0 / hx
            if i + 1 < nx:
                d[2 * node, node + 1] = 1.0 / hx
            d[2 * node + 1, node] = -1.0 / hy
            if j + 1 < ny:
                d[2 * node + 1, node + nx] = 1.0 / hy
    rp, c, v = csr_from_dense(d)
    return rp, c, v, n


def rotated_aniso_ref(nx: int, ny: int, eps: float, theta: float):
    """The reference's own generator (problems.hpp:84-132): two rows per node
    Bᵀ·∇⁺ with Bᵀ = sqrt(diag(eps,1))·Qᵀ, Dirichlet closure."""
    c, s = np.cos(theta), np.sin(theta)
    se = np.sqrt(eps)
    bt = [se * c, se * s, -s, c]
    hx, hy = 1.0 / (nx + 1), 1.0 / (ny + 1)
    n = nx * ny
    rows, cols, vals = [], [], []
    for j in range(ny):
        for i in range(nx):
            node = j * nx + i
            for r in range(2):
                cx, cy = bt[2 * r] / hx, bt[2 * r + 1] / hy
                row = 2 * node + r
                rows.append(row); cols.append(node); vals.append(-cx - cy)
                if i + 1 < nx:
                    rows.append(row); cols.append(node + 1); vals.append(cx)
                if j + 1 < ny:
                    rows.append(row); cols.append(node + nx); vals.append(cy)
    rp, cc, vv = configs._assemble_rows(2 * n, np.array(rows), np.array(cols), np.array(vals, dtype=np.float64), n)
    return rp, cc, vv, n


def params(**kw) -> abi.Params:
    part = kw.pop("partition", None)
    if part is not None:
        part = np.ascontiguousarray(part, dtype=np.int64)
        kw["level0_partition"] = part.ctypes.data
        kw["level0_n_aggregates"] = int(part.max()) + 1
    p = abi.default_params(**kw)
    p._keep = part  # keep the partition alive with the struct
    return p
