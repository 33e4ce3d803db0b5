"""Synthetic inputs for the BASELINE.json configs.

Every generator returns the factor G as int64/float64 CSR arrays plus the
level-0 partition and the LevelParams extensions the config asks for. The
same arrays are handed to the product (C ABI), the plain-C oracle and the
compiled reference harness, so all sides see identical bits.

The right-hand side follows the reference CLI recipe
(``lsamgdd_cli.cpp:103-107``): ``std::mt19937_64(seed)`` fed through
``std::uniform_real_distribution<double>(-1, 1)``. ``mt19937_64_uniform``
restates libstdc++'s engine and ``generate_canonical<double,53>`` in
vectorised numpy; tests pin it bit-for-bit against the real
``std::mt19937_64`` compiled into oracle/_ref.

Matrices are assembled like ``csr_from_triplets`` (``sparse.hpp:79-108``):
columns ascending within a row and exact-zero entries dropped, which is what
the reference would hold after ``mm_read`` of the same triplets.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_U64 = np.uint64
_MASK64 = (1 << 64) - 1


def _mt64_seed(seed: int) -> np.ndarray:
    mt = [0] * 312
    mt[0] = seed & _MASK64
    for i in range(1, 312):
        prev = mt[i - 1]
        mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & _MASK64
    return np.array(mt, dtype=np.uint64)


def _mt64_twist(mt: np.ndarray) -> np.ndarray:
    n, m = 312, 156
    upper = _U64(0xFFFFFFFF80000000)
    lower = _U64(0x7FFFFFFF)
    a = _U64(0xB5026F5AA96619E9)
    new = mt.copy()

    def step(lo: int, hi: int, src_next: np.ndarray, src_m: np.ndarray) -> None:
        x = (new[lo:hi] & upper) | (src_next & lower)
        xa = x >> _U64(1)
        xa = np.where((x & _U64(1)) != 0, xa ^ a, xa)
        new[lo:hi] = src_m ^ xa

    # i in [0, n-m): mt[i+1] old, mt[i+m] old
    step(0, n - m, mt[1 : n - m + 1], mt[m:n])
    # i in [n-m, n-1): mt[i+1] old, mt[i+m-n] new
    step(n - m, n - 1, mt[n - m + 1 : n], new[0 : m - 1])
    # i = n-1: mt[0] new, mt[m-1] new
    step(n - 1, n, new[0:1], new[m - 1 : m])
    return new


def _mt64_temper(y: np.ndarray) -> np.ndarray:
    y = y ^ ((y >> _U64(29)) & _U64(0x5555555555555555))
    y = y ^ ((y << _U64(17)) & _U64(0x71D67FFFEDA60000))
    y = y ^ ((y << _U64(37)) & _U64(0xFFF7EEE000000000))
    y = y ^ (y >> _U64(43))
    return y


def mt19937_64_raw(seed: int, count: int) -> np.ndarray:
    """First ``count`` outputs of std::mt19937_64(seed)."""
    state = _mt64_seed(seed)
    out = np.empty(count, dtype=np.uint64)
    done = 0
    while done < count:
        state = _mt64_twist(state)
        take = min(312, count - done)
        out[done : done + take] = _mt64_temper(state[:take])
        done += take
    return out


def _u64_to_f64_rn(x: np.ndarray) -> np.ndarray:
    """uint64 -> double rounded to nearest-even (numpy uses the C conversion)."""
    return x.astype(np.float64)


def mt19937_64_uniform(seed: int, count: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """std::uniform_real_distribution<double>(lo, hi) over std::mt19937_64(seed).

    libstdc++: generate_canonical<double,53> takes one 64-bit draw x and returns
    double(x) / 2^64 (clamped below 1), then the distribution returns
    canon * (hi - lo) + lo.
    """
    raw = mt19937_64_raw(seed, count)
    canon = _u64_to_f64_rn(raw) / 18446744073709551616.0
    one_minus = np.nextafter(1.0, 0.0)
    canon = np.where(canon >= 1.0, one_minus, canon)
    return canon * (hi - lo) + lo


@dataclass
class ConfigInput:
    """One BASELINE config instance: factor, rhs and setup hooks."""

    name: str
    n: int
    g_rowptr: np.ndarray
    g_cols: np.ndarray
    g_vals: np.ndarray
    rhs: np.ndarray
    level0_partition: np.ndarray | None
    level0_n_aggregates: int
    params: dict = field(default_factory=dict)
    meta: dict = field(default_factory=dict)

    @property
    def m(self) -> int:
        return int(self.g_rowptr.shape[0] - 1)

    @property
    def nnz(self) -> int:
        return int(self.g_cols.shape[0])


def _assemble_rows(n_rows: int, rows: np.ndarray, cols: np.ndarray, vals: np.ndarray, n_cols: int):
    """CSR from triplets (row, col unique per entry), columns sorted, exact zeros dropped."""
    keep = vals != 0.0
    rows, cols, vals = rows[keep], cols[keep], vals[keep]
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    rowptr = np.zeros(n_rows + 1, dtype=np.int64)
    np.add.at(rowptr, rows + 1, 1)
    np.cumsum(rowptr, out=rowptr)
    return rowptr, cols.astype(np.int64), vals.astype(np.float64)


def block_partition_2d(nx: int, ny: int, bx: int, by: int) -> tuple[np.ndarray, int]:
    """Geometric bx×by blocks on a lexicographic (j*nx+i) grid; block ids
    lexicographic by block row, then block column."""
    nbx = -(-nx // bx)
    nby = -(-ny // by)
    j, i = np.divmod(np.arange(nx * ny, dtype=np.int64), nx)
    return (j // by) * nbx + (i // bx), nbx * nby


def block_partition_3d(n: int, b: int) -> tuple[np.ndarray, int]:
    nb = -(-n // b)
    idx = np.arange(n * n * n, dtype=np.int64)
    k, rem = np.divmod(idx, n * n)
    j, i = np.divmod(rem, n)
    return ((k // b) * nb + (j // b)) * nb + (i // b), nb * nb * nb


def poisson_edges_2d(nx: int, ny: int, shift: float) -> tuple[np.ndarray, np.ndarray, np.ndarray, int]:
    """Config 1 factor: one ±1 row per interior edge (horizontal edges, then
    vertical edges, lexicographic), then sqrt(shift)·I rows, so
    A = GᵀG + shift·I."""
    n = nx * ny
    jj, ii = np.meshgrid(np.arange(ny), np.arange(nx - 1), indexing="ij")
    h_node = (jj * nx + ii).ravel()
    jj, ii = np.meshgrid(np.arange(ny - 1), np.arange(nx), indexing="ij")
    v_node = (jj * nx + ii).ravel()
    nh, nv = h_node.size, v_node.size
    m = nh + nv + (n if shift > 0 else 0)
    rows = [np.repeat(np.arange(nh), 2), np.repeat(nh + np.arange(nv), 2)]
    cols = [np.stack([h_node, h_node + 1], 1).ravel(), np.stack([v_node, v_node + nx], 1).ravel()]
    vals = [np.tile([-1.0, 1.0], nh), np.tile([-1.0, 1.0], nv)]
    if shift > 0:
        rows.append(nh + nv + np.arange(n))
        cols.append(np.arange(n))
        vals.append(np.full(n, math.sqrt(shift)))
    rowptr, c, v = _assemble_rows(m, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals), n)
    return rowptr, c, v, m


def rotated_aniso_2d(nx: int, ny: int, eps: float, theta: float):
    """9-point factorised rotated-anisotropy factor (configs 2 and 3).

    K = R(θ)·diag(1, ε)·R(θ)ᵀ on the interior nodes of a unit-square grid,
    h = 1/(n+1), homogeneous Dirichlet closure. Four rows per node:
    (1/√2)·Bᵀ∇⁺ and (1/√2)·Bᵀ∇^{+-} with Bᵀ = diag(1, √ε)·R(θ)ᵀ, where ∇⁺
    uses forward differences in x and y and ∇^{+-} forward in x, backward
    in y. The two halves couple the NW-SE and NE-SW diagonals respectively,
    so A = GᵀG is the full 9-point stencil and consistent with -∇·K∇.
    Rows touch at most three nodes; m = 4n.
    """
    n = nx * ny
    h = 1.0 / (nx + 1)
    hy = 1.0 / (ny + 1)
    c, s = math.cos(theta), math.sin(theta)
    se = math.sqrt(eps)
    w = 1.0 / math.sqrt(2.0)
    # direction rows: (bx, by) multiplies (∂x, ∂y)
    dirs = [(w * c, w * s), (w * se * -s, w * se * c)]
    node = np.arange(n, dtype=np.int64)
    j, i = np.divmod(node, nx)
    has_e = i + 1 < nx
    has_n = j + 1 < ny
    has_s = j > 0
    rows_l, cols_l, vals_l = [], [], []
    for half in range(2):  # 0: ∂y forward, 1: ∂y backward
        for d, (bx, by) in enumerate(dirs):
            r = 4 * node + 2 * half + d
            cx, cy = bx / h, by / hy
            if half == 0:
                # cx(u_E - u) + cy(u_N - u)
                rows_l += [r, r[has_e], r[has_n]]
                cols_l += [node, node[has_e] + 1, node[has_n] + nx]
                vals_l += [np.full(n, -cx - cy), np.full(int(has_e.sum()), cx), np.full(int(has_n.sum()), cy)]
            else:
                # cx(u_E - u) + cy(u - u_S)
                rows_l += [r, r[has_e], r[has_s]]
                cols_l += [node, node[has_e] + 1, node[has_s] - nx]
                vals_l += [np.full(n, -cx + cy), np.full(int(has_e.sum()), cx), np.full(int(has_s.sum()), -cy)]
    m = 4 * n
    rowptr, cc, vv = _assemble_rows(m, np.concatenate(rows_l), np.concatenate(cols_l), np.concatenate(vals_l), n)
    return rowptr, cc, vv, m


def rotated_aniso_3d(nn: int, eps: float, alpha: float, beta: float):
    """Config 5 factor: 7-point forward differences, K = R(α,β)·diag(1,ε,ε)·Rᵀ,
    three rows per node Bᵀ∇⁺ with Bᵀ = diag(1,√ε,√ε)·Rᵀ (R = Rz(α)·Ry(β)),
    homogeneous Dirichlet closure, h = 1/(n+1)."""
    n = nn ** 3
    h = 1.0 / (nn + 1)
    ca, sa, cb, sb = math.cos(alpha), math.sin(alpha), math.cos(beta), math.sin(beta)
    rz = np.array([[ca, -sa, 0.0], [sa, ca, 0.0], [0.0, 0.0, 1.0]])
    ry = np.array([[cb, 0.0, sb], [0.0, 1.0, 0.0], [-sb, 0.0, cb]])
    R = rz @ ry
    bt = np.diag([1.0, math.sqrt(eps), math.sqrt(eps)]) @ R.T
    node = np.arange(n, dtype=np.int64)
    k, rem = np.divmod(node, nn * nn)
    j, i = np.divmod(rem, nn)
    nb = [(i + 1 < nn, 1), (j + 1 < nn, nn), (k + 1 < nn, nn * nn)]
    rows_l, cols_l, vals_l = [], [], []
    for d in range(3):
        r = 3 * node + d
        coef = bt[d] / h
        rows_l.append(r)
        cols_l.append(node)
        vals_l.append(np.full(n, -coef.sum()))
        for axis, (mask, stride) in enumerate(nb):
            rows_l.append(r[mask])
            cols_l.append(node[mask] + stride)
            vals_l.append(np.full(int(mask.sum()), coef[axis]))
    m = 3 * n
    rowptr, cc, vv = _assemble_rows(m, np.concatenate(rows_l), np.concatenate(cols_l), np.concatenate(vals_l), n)
    return rowptr, cc, vv, m


ANNULUS_R0, ANNULUS_R1 = 0.5, 1.0
ANNULUS_MODES = 4


def annulus_field(n_phi: int, n_r: int, seed: int = 3, amplitude: float = 0.05):
    """Unit field b = (b_r, b_φ) of config 4 on the annulus nodes.

    Closed circular field lines (b = e_φ) with a smooth seeded radial
    perturbation p(r, φ) = amplitude · Σ_k a_k sin(kφ + ψ_k) · sin(π(r−r0)/(r1−r0))
    / Σ_k |a_k|, k = 1..4, so |p| ≤ amplitude and p vanishes on both
    Dirichlet circles; a_k ∈ uniform[-1,1), ψ_k = π·(u_k + 1) with u_k the
    next draw, all from std::mt19937_64(seed) (the RHS recipe of
    lsamgdd_cli.cpp:103-107). b = (p, 1)/√(1+p²). Nodes are lexicographic
    j·n_phi + i (i the periodic angle index, j the radial index); radii are
    interior nodes r_j = r0 + (j+1)·Δr, Δr = (r1−r0)/(n_r+1), angles φ_i = i·Δφ.
    """
    draws = mt19937_64_uniform(seed, 2 * ANNULUS_MODES)
    a = draws[0::2]
    psi = math.pi * (draws[1::2] + 1.0)
    dr = (ANNULUS_R1 - ANNULUS_R0) / (n_r + 1)
    dphi = 2.0 * math.pi / n_phi
    r = ANNULUS_R0 + (np.arange(n_r, dtype=np.float64) + 1.0) * dr
    phi = np.arange(n_phi, dtype=np.float64) * dphi
    ang = np.zeros(n_phi)
    for k in range(ANNULUS_MODES):
        ang += a[k] * np.sin((k + 1) * phi + psi[k])
    ang *= amplitude / np.abs(a).sum()
    bump = np.sin(math.pi * (r - ANNULUS_R0) / (ANNULUS_R1 - ANNULUS_R0))
    p = bump[:, None] * ang[None, :]  # [n_r, n_phi]
    norm = np.sqrt(1.0 + p * p)
    return p / norm, 1.0 / norm, r, dr, dphi


def annulus_heat(n_phi: int, n_r: int, eps_perp: float, seed: int = 3):
    """Config 4 factor: G = [√D1; D2^{-1/2}·B], D1 = ε⊥·h²·I, D2 = I, so
    A = GᵀG = D1 + BᵀD2⁻¹B (BASELINE.json configs[3]).

    B is the first-order upwinded directional derivative b·∇u =
    b_r ∂u/∂r + (b_φ/r) ∂u/∂φ: the angular part is a backward difference
    (b_φ > 0 everywhere) that wraps periodically, the radial part a backward
    difference where b_r ≥ 0 and a forward one where b_r < 0, with
    homogeneous Dirichlet closure on both circles (the missing neighbour is
    dropped). h = Δr. Rows 0..n−1 are √D1, rows n..2n−1 are B; m = 2n and
    every B row touches at most three nodes.
    """
    if n_phi < 2 or n_r < 1:
        raise ValueError("annulus_heat: need n_phi >= 2 and n_r >= 1")
    br, bphi, r, dr, dphi = annulus_field(n_phi, n_r, seed)
    n = n_phi * n_r
    node = np.arange(n, dtype=np.int64)
    j, i = np.divmod(node, n_phi)
    br, bphi = br.ravel(), bphi.ravel()
    c_phi = bphi / (r[j] * dphi)
    c_r = br / dr
    west = j * n_phi + (i - 1) % n_phi
    up = br >= 0.0
    has_in = up & (j > 0)
    has_out = ~up & (j + 1 < n_r)
    rb = n + node
    rows = [node, rb, rb, rb[has_in], rb[has_out]]
    cols = [node, node, west, node[has_in] - n_phi, node[has_out] + n_phi]
    vals = [np.full(n, math.sqrt(eps_perp) * dr), c_phi + np.abs(c_r), -c_phi, -c_r[has_in], c_r[has_out]]
    m = 2 * n
    rowptr, cc, vv = _assemble_rows(m, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals), n)
    return rowptr, cc, vv, m


def config(name: str, scale: int | None = None, eps_perp: float = 1e-6) -> ConfigInput:
    """Build config ``c1``..``c5`` (BASELINE.json configs[0..4]).

    ``scale`` overrides the grid edge for parity tests at sizes the oracle
    finishes in seconds; the bench always uses the full size. ``eps_perp``
    picks the point of config 4's ε⊥ sweep {1e-3, 1e-6, 1e-9}.
    """
    name = name.lower()
    if name == "c1":
        nx = scale or 64
        rp, c, v, m = poisson_edges_2d(nx, nx, 1e-6)
        part, nagg = block_partition_2d(nx, nx, 4, 4)
        rhs = mt19937_64_uniform(0, nx * nx)
        return ConfigInput(
            "c1", nx * nx, rp, c, v, rhs, part, nagg,
            params=dict(thresh_override=10.0, level0_overlap=1),
            meta=dict(grid=nx, tau=0.1, ref_thresh=10.0, blocks="4x4", overlap=1, seed=0),
        )
    if name == "c2":
        nx = scale or 1024
        rp, c, v, m = rotated_aniso_2d(nx, nx, 1e-3, math.pi / 6)
        part, nagg = block_partition_2d(nx, nx, 3, 3)
        rhs = mt19937_64_uniform(1, nx * nx)
        return ConfigInput(
            "c2", nx * nx, rp, c, v, rhs, part, nagg,
            params=dict(level0_overlap=1, level0_max_modes=6),
            meta=dict(grid=nx, eps=1e-3, theta=math.pi / 6, blocks="3x3", overlap=1, max_modes=6, seed=1),
        )
    if name == "c3":
        nx = scale or 4096
        theta = float(mt19937_64_uniform(2, 1, 0.0, math.pi)[0])
        rp, c, v, m = rotated_aniso_2d(nx, nx, 1e-6, theta)
        part, nagg = block_partition_2d(nx, nx, 8, 8)
        rhs = mt19937_64_uniform(2, nx * nx + 1)[1:]
        return ConfigInput(
            "c3", nx * nx, rp, c, v, rhs, part, nagg,
            params=dict(thresh_override=20.0, level0_overlap=2),
            meta=dict(grid=nx, eps=1e-6, theta=theta, blocks="8x8", overlap=2, tau=0.05, ref_thresh=20.0, seed=2),
        )
    if name == "c4":
        nx = scale or 2048
        rp, c, v, m = annulus_heat(nx, nx, eps_perp, seed=3)
        part, nagg = block_partition_2d(nx, nx, 6, 6)
        rhs = mt19937_64_uniform(3, nx * nx + 2 * ANNULUS_MODES)[2 * ANNULUS_MODES:]
        return ConfigInput(
            "c4", nx * nx, rp, c, v, rhs, part, nagg,
            params=dict(level0_overlap=2),
            meta=dict(grid=nx, eps_perp=eps_perp, r0=ANNULUS_R0, r1=ANNULUS_R1, perturbation=0.05,
                      blocks="6x6", overlap=2, seed=3),
        )
    if name == "c5":
        nn = scale or 256
        rp, c, v, m = rotated_aniso_3d(nn, 1e-4, math.pi / 4, math.pi / 5)
        part, nagg = block_partition_3d(nn, 4)
        rhs = mt19937_64_uniform(4, nn ** 3)
        return ConfigInput(
            "c5", nn ** 3, rp, c, v, rhs, part, nagg,
            params=dict(level0_overlap=1, level0_max_modes=12, max_levels=3),
            meta=dict(grid=nn, eps=1e-4, alpha=math.pi / 4, beta=math.pi / 5, blocks="4x4x4", max_modes=12, seed=4),
        )
    raise ValueError(f"unknown config {name!r}")


# ---- stencil-row descriptions for the on-device generator (lsamgdd_generate_stencil_rows) ----


def rotated_aniso_2d_stencil(nx: int, ny: int, eps: float, theta: float):
    """The factor of :func:`rotated_aniso_2d` as (grid, offsets[4][3][3], coefs[4][3]):
    row 4·node + 2·half + d, same coefficient arithmetic, so the device-generated
    CSR equals the host one bit for bit."""
    h = 1.0 / (nx + 1)
    hy = 1.0 / (ny + 1)
    c, s = math.cos(theta), math.sin(theta)
    se = math.sqrt(eps)
    w = 1.0 / math.sqrt(2.0)
    dirs = [(w * c, w * s), (w * se * -s, w * se * c)]
    offsets = np.zeros((4, 3, 3), dtype=np.int32)
    coefs = np.zeros((4, 3), dtype=np.float64)
    for half in range(2):
        for d, (bx, by) in enumerate(dirs):
            k = 2 * half + d
            cx, cy = bx / h, by / hy
            if half == 0:
                offsets[k] = [[0, 0, 0], [1, 0, 0], [0, 1, 0]]
                coefs[k] = [-cx - cy, cx, cy]
            else:
                offsets[k] = [[0, 0, 0], [1, 0, 0], [0, -1, 0]]
                coefs[k] = [-cx + cy, cx, -cy]
    return (nx, ny, 1), offsets, coefs


def rotated_aniso_3d_stencil(nn: int, eps: float, alpha: float, beta: float):
    """The factor of :func:`rotated_aniso_3d` as (grid, offsets[3][4][3], coefs[3][4])."""
    h = 1.0 / (nn + 1)
    ca, sa, cb, sb = math.cos(alpha), math.sin(alpha), math.cos(beta), math.sin(beta)
    rz = np.array([[ca, -sa, 0.0], [sa, ca, 0.0], [0.0, 0.0, 1.0]])
    ry = np.array([[cb, 0.0, sb], [0.0, 1.0, 0.0], [-sb, 0.0, cb]])
    R = rz @ ry
    bt = np.diag([1.0, math.sqrt(eps), math.sqrt(eps)]) @ R.T
    offsets = np.zeros((3, 4, 3), dtype=np.int32)
    coefs = np.zeros((3, 4), dtype=np.float64)
    for d in range(3):
        coef = bt[d] / h
        offsets[d] = [[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]]
        coefs[d] = [-coef.sum(), coef[0], coef[1], coef[2]]
    return (nn, nn, nn), offsets, coefs


def stencil_rows_host(grid, offsets: np.ndarray, coefs: np.ndarray):
    """numpy statement of lsamgdd_generate_stencil_rows' contract (test helper):
    neighbours outside the grid and exact zeros dropped, columns ascending."""
    nx, ny, nz = (int(g) for g in grid)
    n = nx * ny * nz
    R, E = coefs.shape
    node = np.arange(n, dtype=np.int64)
    x, y, z = node % nx, (node // nx) % ny, node // (nx * ny)
    rows_l, cols_l, vals_l = [], [], []
    for k in range(R):
        for e in range(E):
            dx, dy, dz = (int(v) for v in offsets[k, e])
            ok = (x + dx >= 0) & (x + dx < nx) & (y + dy >= 0) & (y + dy < ny) & (z + dz >= 0) & (z + dz < nz)
            rows_l.append(R * node[ok] + k)
            cols_l.append(node[ok] + (dz * ny + dy) * nx + dx)
            vals_l.append(np.full(int(ok.sum()), coefs[k, e]))
    rowptr, cc, vv = _assemble_rows(R * n, np.concatenate(rows_l), np.concatenate(cols_l), np.concatenate(vals_l), n)
    return rowptr, cc, vv


def config_stencil(name: str, scale: int | None = None):
    """(grid, offsets, coefs) of a config whose factor the device can generate (c2, c3, c5), else None."""
    name = name.lower()
    if name == "c2":
        nx = scale or 1024
        return rotated_aniso_2d_stencil(nx, nx, 1e-3, math.pi / 6)
    if name == "c3":
        nx = scale or 4096
        theta = float(mt19937_64_uniform(2, 1, 0.0, math.pi)[0])
        return rotated_aniso_2d_stencil(nx, nx, 1e-6, theta)
    if name == "c5":
        nn = scale or 256
        return rotated_aniso_3d_stencil(nn, 1e-4, math.pi / 4, math.pi / 5)
    return None
