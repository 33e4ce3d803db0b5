"""Pins of the CPU oracle (no GPU): the reference's own golden vectors and
known-answer tests, bit-for-bit agreement with the compiled reference
(oracle/_ref), and the RHS generator against std::mt19937_64."""
from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import refbind
from paper_2601_04112_b200 import abi, configs

from . import _cases


def _lap1d(n):
    d = np.zeros((n, n))
    for i in range(n):
        d[i, i] = 2.0
        if i + 1 < n:
            d[i, i + 1] = d[i + 1, i] = -1.0
    return _cases.csr_from_dense(d)


# ---- RNG (lsamgdd_cli.cpp:103-107) ----------------------------------------------------------


def test_mt19937_64_uniform_matches_std(ref_lib, oracle_lib):
    for seed in (0, 1, 2, 4, 2024):
        want = ref_lib.uniform(seed, 5000)
        assert np.array_equal(configs.mt19937_64_uniform(seed, 5000), want)
        assert np.array_equal(oracle_lib.uniform(seed, 5000), want)


def test_config3_theta_is_first_draw():
    cfg = configs.config("c3", 16)
    assert 0.0 <= cfg.meta["theta"] < math.pi
    assert cfg.meta["theta"] == configs.mt19937_64_uniform(2, 1, 0.0, math.pi)[0]


# ---- golden vectors of the reference unit suites -----------------------------------------------


def test_aggregation_chain_golden(oracle_lib):
    """test_aggregation.cpp:57-63: 1D chain of nine -> {0,0,1,1,1,2,2,2,2}."""
    rp, c, v = _lap1d(9)
    asg, nagg = oracle_lib.standard_aggregation(rp, c, v)
    assert nagg == 3
    assert asg.tolist() == [0, 0, 1, 1, 1, 2, 2, 2, 2]


def test_aggregation_diagonal_singletons(oracle_lib):
    """test_aggregation.cpp:65-70."""
    rp, c, v = _cases.csr_from_dense(np.diag([1.0, 2.0, 3.0, 4.0, 5.0]))
    asg, nagg = oracle_lib.standard_aggregation(rp, c, v)
    assert nagg == 5 and asg.tolist() == [0, 1, 2, 3, 4]


def test_topology_chain_golden(oracle_lib):
    """test_aggregation.cpp:139-156 on the chain pattern: Γ0={3}, Γ1={2,6},
    Γ2={5}, two colours; subdomain(1) = {3,4,5,2,6}."""
    g = _cases.chain_factor(9, shift=0.25)
    p = _cases.params(partition=[0, 0, 0, 1, 1, 1, 2, 2, 2], max_levels=2, coarse_size=1)
    h = oracle_lib.setup(g, p)
    goff, gam = h.export(0, abi.EXPORT_GAMMA)
    gammas = [gam[goff[i]:goff[i + 1]].tolist() for i in range(3)]
    assert gammas == [[3], [2, 6], [5]]
    colors, ncol = h.export(0, abi.EXPORT_COLORS)
    assert ncol == 2 and colors[0] != colors[1] and colors[1] != colors[2]


def test_row_multiplicity_golden(oracle_lib):
    """test_splitting.cpp:37-58: split chain of six; row 2 is shared (M=2)."""
    g = _cases.chain_factor(6)
    p = _cases.params(partition=[0, 0, 0, 1, 1, 1], max_levels=2, coarse_size=1)
    h = oracle_lib.setup(g, p)
    mult, n_mult = h.export(0, abi.EXPORT_MULTIPLICITY)
    assert mult.tolist() == [1, 1, 2, 1, 1] and n_mult == 2


def test_eigen_threshold_golden(oracle_lib):
    """test_splitting.cpp:143-147."""
    assert oracle_lib.eigen_threshold(50.0, 4, 2) == pytest.approx(5.75, abs=1e-14)
    assert oracle_lib.eigen_threshold(50.0, 49, 100) == pytest.approx(0.1, abs=1e-14)
    assert oracle_lib.eigen_threshold(50.0, 2, 1) == pytest.approx(24.0, abs=1e-14)


def test_sym_eig_golden(oracle_lib):
    """test_eigen.cpp:33-57: sorted diagonal; closed form 2±√2."""
    vals, vecs = oracle_lib.sym_eig(np.diag([3.0, 1.0, 2.0]))
    assert np.allclose(vals, [1, 2, 3], atol=1e-14)
    assert abs(abs(vecs[1, 0]) - 1) < 1e-13 and abs(abs(vecs[2, 1]) - 1) < 1e-13
    rp, c, v = _lap1d(3)
    d = np.zeros((3, 3))
    d[np.repeat(np.arange(3), np.diff(rp)), c] = v
    vals, _ = oracle_lib.sym_eig(d)
    r2 = math.sqrt(2.0)
    assert np.allclose(vals, [2 - r2, 2, 2 + r2], rtol=1e-13)


def test_sym_eig_reconstructs(oracle_lib):
    rng = np.random.default_rng(90)
    a = rng.uniform(-1, 1, (20, 20))
    a = 0.5 * (a + a.T)
    vals, vecs = oracle_lib.sym_eig(a)
    assert np.all(np.diff(vals) >= 0)
    assert np.linalg.norm(vecs @ np.diag(vals) @ vecs.T - a) / np.linalg.norm(a) < 1e-11
    assert np.abs(vecs.T @ vecs - np.eye(20)).max() < 1e-12


def test_sym_eig_rejects_nan(oracle_lib):
    a = np.zeros((2, 2))
    a[0, 1] = np.nan
    with pytest.raises(abi.LsamgddError) as e:
        oracle_lib.sym_eig(a)
    assert e.value.name == "EigError"


def test_spsd_gevp_golden(oracle_lib):
    """test_eigen.cpp:81-92 (diagonal pencil), :152-174 (∞ modes, discards)."""
    vals, _, disc = oracle_lib.spsd_gevp(np.diag([2.0, 8.0]), np.diag([1.0, 2.0]))
    assert vals.tolist() == pytest.approx([4.0, 2.0], rel=1e-12) and disc == 0
    vals, vecs, disc = oracle_lib.spsd_gevp(np.eye(2), np.diag([1.0, 0.0]))
    assert math.isinf(vals[0]) and vals[1] == pytest.approx(1.0, rel=1e-12) and disc == 0
    assert abs(abs(vecs[1, 0]) - 1) < 1e-12 and abs(vecs[0, 0]) < 1e-12
    vals, _, disc = oracle_lib.spsd_gevp(np.diag([1.0, 0.0]), np.diag([1.0, 0.0]))
    assert vals.tolist() == pytest.approx([1.0], rel=1e-12) and disc == 1


def test_pseudo_inverse_golden(oracle_lib):
    """test_eigen.cpp:197-206: pinv(u uᵀ) = u uᵀ / 81 for u = (1,2,2)."""
    u = np.array([1.0, 2.0, 2.0])
    got = oracle_lib.pseudo_inverse(np.outer(u, u))
    assert np.abs(got - np.outer(u, u) / 81.0).max() < 1e-12


def test_smoother_matches_dense_reference(oracle_lib):
    """test_smoother.cpp:79-107: RAS / RAS-T against dense inverses, 1e-12."""
    g = _cases.chain_factor(12, shift=0.5)
    part = [0, 0, 0, 0, 1, 1, 1, 2, 2, 2, 2, 2]
    h = oracle_lib.setup(g, _cases.params(partition=part, max_levels=2, coarse_size=1))
    rp, c, v, s = h.export(0, abi.EXPORT_A)
    A = np.zeros(s)
    A[np.repeat(np.arange(s[0]), np.diff(rp)), c] = v
    goff, gam = h.export(0, abi.EXPORT_GAMMA)
    n = 12
    for mode in (abi.RAS, abi.RAST):
        want = np.zeros((n, n))
        for i in range(3):
            om = [k for k in range(n) if part[k] == i]
            sub = om + gam[goff[i]:goff[i + 1]].tolist()
            inv = np.linalg.inv(A[np.ix_(sub, sub)])
            for r_ in range(len(sub)):
                for c_ in range(len(sub)):
                    w = inv[r_, c_]
                    if mode == abi.RAS and r_ >= len(om):
                        w = 0.0
                    if mode == abi.RAST and c_ >= len(om):
                        w = 0.0
                    want[sub[r_], sub[c_]] += w
        got = np.stack([h.schwarz_apply(np.eye(n)[j], 0, mode) for j in range(n)], axis=1)
        assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12


def test_pcg_contracts(oracle_lib):
    """krylov.hpp:49-54 (zero rhs), :61-81 (maxit stall returns unconverged)."""
    cfg = configs.config("c2", 32)
    h = oracle_lib.setup(cfg, refbind.params_for(cfg))
    x, rep = h.pcg(np.zeros(cfg.n))
    assert rep["converged"] and rep["iterations"] == 0 and not x.any()
    x, rep = h.pcg(cfg.rhs, 1e-14, 2)
    assert not rep["converged"] and rep["iterations"] == 2


def test_setup_input_errors(oracle_lib):
    """hierarchy.hpp:107-117 and the stagnation guard :173-176."""
    g = _cases.chain_factor(12, shift=0.5)
    for kw in (dict(max_levels=1), dict(kappa=1.0), dict(must_keep=1.0), dict(coarsening_ratios=[1])):
        with pytest.raises(abi.LsamgddError) as e:
            oracle_lib.setup(g, _cases.params(**kw))
        assert e.value.name == "InputError"
    ident = _cases.csr_from_dense(np.eye(30)) + (30,)
    with pytest.raises(abi.LsamgddError) as e:
        oracle_lib.setup(ident, _cases.params(coarse_size=10))
    assert e.value.name == "SetupError"


# ---- oracle == compiled reference, bit for bit -------------------------------------------------

_CASES = [("c1", None, {}), ("c2", 32, {}), ("c2", 64, {}), ("c3", 32, {"thresh_override": 0.0}),
          ("c3", 64, {"thresh_override": 10.0}), ("c4", 24, {}), ("c4", 48, {}),
          ("c4", 30, {"eps_perp": 1e-3}), ("c4", 30, {"eps_perp": 1e-9})]


@pytest.mark.parametrize("name,scale,over", _CASES)
def test_oracle_matches_reference_bitwise(ref_lib, oracle_lib, name, scale, over):
    over = dict(over)
    cfg = configs.config(name, scale, **({"eps_perp": over.pop("eps_perp")} if "eps_perp" in over else {}))
    p = refbind.params_for(cfg, keep_spectra=1, **over)
    hr = ref_lib.setup(cfg, p)
    ho = oracle_lib.setup(cfg, p)
    assert hr.num_levels == ho.num_levels
    for l in range(hr.num_levels):
        whats = [abi.EXPORT_A, abi.EXPORT_G]
        if l + 1 < hr.num_levels:
            whats += [abi.EXPORT_P, abi.EXPORT_PARTITION, abi.EXPORT_GAMMA, abi.EXPORT_COLORS, abi.EXPORT_SPECTRA,
                      abi.EXPORT_MULTIPLICITY]
        for w in whats:
            for a, b in zip(hr.export(l, w), ho.export(l, w)):
                if isinstance(a, np.ndarray):
                    assert np.array_equal(a, b), (l, w)
                else:
                    assert a == b, (l, w)
    assert np.array_equal(hr.vcycle(cfg.rhs), ho.vcycle(cfg.rhs))
    xr, rr = hr.pcg(cfg.rhs)
    xo, ro = ho.pcg(cfg.rhs)
    assert np.array_equal(xr, xo) and rr["iterations"] == ro["iterations"]
    assert np.array_equal(rr["residual_history"], ro["residual_history"])


def test_replica_equals_plain_setup(ref_lib):
    """With no hook active the stage replica equals the reference's setup()."""
    g = _cases.rotated_aniso_ref(16, 16, 1e-2, 0.7)
    p = _cases.params(coarse_size=30)
    h1 = ref_lib.setup(g, p, plain=True)
    h2 = ref_lib.setup(g, p, plain=False)
    r = configs.mt19937_64_uniform(7, 256)
    assert np.array_equal(h1.vcycle(r), h2.vcycle(r))
    assert h1.num_levels == h2.num_levels


def test_config1_reference_numbers(oracle_lib):
    """config 1 gives 2 levels, op. complexity 1.0601, 18 iterations."""
    cfg = configs.config("c1")
    h = oracle_lib.setup(cfg, refbind.params_for(cfg))
    _, rep = h.pcg(cfg.rhs)
    assert h.num_levels == 2 and rep["iterations"] == 18
    assert round(h.operator_complexity(), 4) == 1.0601
