"""Generator properties of config 4 (the annulus, BASELINE.json configs[3]).

The oracle-vs-reference and CUDA-vs-oracle parity of the hierarchy built
from it lives in test_oracle_pins.py / test_gpu_parity.py; these check that
the factor is the operator the config names."""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_2601_04112_b200 import configs


def _dense(rp, c, v, n):
    d = np.zeros((len(rp) - 1, n))
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    d[rows, c] = v
    return d


def test_field_is_unit_and_perturbation_bounded():
    br, bphi, r, dr, dphi = configs.annulus_field(64, 40)
    assert np.allclose(br * br + bphi * bphi, 1.0, rtol=0, atol=1e-15)
    p = br / bphi
    assert np.abs(p).max() <= 0.05 + 1e-15 and np.abs(p).max() > 0.01
    assert (bphi > 0).all()
    assert r[0] == pytest.approx(configs.ANNULUS_R0 + dr) and r[-1] == pytest.approx(configs.ANNULUS_R1 - dr)


@pytest.mark.parametrize("eps", [1e-3, 1e-6, 1e-9])
def test_factor_structure(eps):
    cfg = configs.config("c4", 12, eps_perp=eps)
    n = cfg.n
    assert n == 144 and cfg.m == 2 * n
    d = _dense(cfg.g_rowptr, cfg.g_cols, cfg.g_vals, n)
    dr = (configs.ANNULUS_R1 - configs.ANNULUS_R0) / 13
    assert np.array_equal(d[:n], np.eye(n) * (math.sqrt(eps) * dr))
    b = d[n:]
    assert (np.count_nonzero(b, axis=1) <= 3).all()
    # B annihilates constants away from the Dirichlet circles (a pure derivative)
    ones = b @ np.ones(n)
    j = np.arange(n) // 12
    interior = (j > 0) & (j < 11)
    assert np.abs(ones[interior]).max() < 1e-9 * np.abs(b).max()
    # the angular difference wraps: node (j, 0) couples to (j, n_phi - 1)
    assert all(b[jj * 12, jj * 12 + 11] < 0 for jj in range(12))
    # columns ascending within rows (csr_from_triplets order)
    for row in range(cfg.m):
        cs = cfg.g_cols[cfg.g_rowptr[row]:cfg.g_rowptr[row + 1]]
        assert (np.diff(cs) > 0).all()


def test_normal_matrix_is_definite_and_sweep_changes_only_d1():
    a = configs.config("c4", 10, eps_perp=1e-3)
    b = configs.config("c4", 10, eps_perp=1e-9)
    assert np.array_equal(a.g_cols, b.g_cols) and np.array_equal(a.rhs, b.rhs)
    n = a.n
    assert np.array_equal(a.g_vals[a.g_rowptr[n]:], b.g_vals[b.g_rowptr[n]:])
    g = _dense(a.g_rowptr, a.g_cols, a.g_vals, n)
    assert np.linalg.eigvalsh(g.T @ g).min() > 0


def test_partition_is_6x6_blocks_with_ragged_edge():
    cfg = configs.config("c4", 20)
    part = cfg.level0_partition
    assert cfg.level0_n_aggregates == 16 and part.max() == 15
    sizes = np.bincount(part)
    assert sorted(set(sizes.tolist())) == [4, 12, 36]
    assert cfg.params == {"level0_overlap": 2}


@pytest.mark.parametrize("name,scale", [("c2", 1), ("c2", 2), ("c2", 33), ("c3", 20), ("c5", 1), ("c5", 2), ("c5", 7)])
def test_stencil_description_equals_host_generator(name, scale):
    """configs.config_stencil (the input of the on-device generator,
    lsamgdd_generate_stencil_rows) describes exactly the factor the host
    generator assembles: same rows, columns and value bits."""
    cfg = configs.config(name, scale)
    grid, offsets, coefs = configs.config_stencil(name, scale)
    rp, cc, vv = configs.stencil_rows_host(grid, offsets, coefs)
    assert np.array_equal(rp, cfg.g_rowptr)
    assert np.array_equal(cc, cfg.g_cols)
    assert np.array_equal(vv, cfg.g_vals)
