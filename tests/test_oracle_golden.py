"""Pin the oracle (oracle/specmc_oracle.c) against the reference's own
known-answer tests (CPU only).  Each test cites the reference test it mirrors
(paths relative to the reference root)."""
import math

import numpy as np
import pytest

from helpers import conjugate, oracle_model, ramp
from paper_2604_03271_b200 import model as M


def test_ess_closed_form(port):  # proj/tests/test_smc.cpp:38-53
    lw = np.log([0.5, 0.25, 0.25])
    assert port.ess(lw) == pytest.approx(8.0 / 3.0, rel=1e-13)
    assert port.ess(lw + 7.0) == pytest.approx(8.0 / 3.0, rel=1e-13)
    assert port.ess(np.zeros(50)) == pytest.approx(50.0, rel=1e-13)
    assert port.ess(np.array([0.0, -np.inf, -np.inf])) == pytest.approx(1.0, rel=1e-13)
    with pytest.raises(RuntimeError):
        port.ess(np.full(4, -np.inf))


def test_next_beta_two_atom(port):  # test_smc.cpp:67-86
    E = np.array([0.0, 10.0])
    delta = -math.log(2.0 - math.sqrt(3.0)) / 10.0
    assert port.next_beta(E, 1.0, 0.0, 0.75) == pytest.approx(delta, rel=1e-4)
    assert port.next_beta(E, 1.0, 0.5, 0.75) == pytest.approx(0.5 + delta, rel=1e-4)
    assert port.next_beta(np.full(5, 3.7), 50.0, 0.3, 0.5) == 1.0


def test_resample_counts_and_unbiasedness(port):  # test_smc.cpp:88-120
    lw = np.log([0.5, 0.25, 0.125, 0.125])
    for rep in range(20):
        idx = port.systematic_resample(lw, 8, port.resample_uniform(5, rep + 1))
        assert np.all(np.diff(idx) >= 0)
        assert list(np.bincount(idx, minlength=4)) == [4, 2, 1, 1]
    lw = np.log([0.7, 0.3])
    tot = 0
    for rep in range(4000):
        idx = port.systematic_resample(lw, 3, port.resample_uniform(11, rep))
        c0 = int((idx == 0).sum())
        assert 2 <= c0 <= 3
        tot += c0
    assert tot / 4000 == pytest.approx(2.1, rel=0.02)


def test_conjugate_free_energy(port):  # test_smc.cpp:122-138
    spec, data, F_exact, *_ = conjugate(20, 404, port)
    om = oracle_model(spec, data)
    r = port.smc_run(om, 2000, 10, 0.6, seed=7)
    assert not r.diverged
    assert abs(r.F - F_exact) < 0.15
    assert r.ladder[-1] == 1.0 and np.all(np.diff(r.ladder) > 0)


def test_single_level_is_importance_sampling(port):  # test_smc.cpp:140-157 (bitwise)
    spec, data, *_ = conjugate(12, 1001, port)
    om = oracle_model(spec, data)
    r = port.smc_run(om, 100, 5, 1e-9, seed=99)
    assert r.levels == 1
    th, E = port.init_ensemble(om, 100, 99)
    assert r.F == -port.log_mean_exp(-1.0 * 12.0 * E)


def test_max_levels_abort(port):  # test_smc.cpp:186-194
    spec, data, *_ = conjugate(200, 5, port)
    with pytest.raises(RuntimeError):
        port.smc_run(oracle_model(spec, data), 100, 5, 0.95, max_levels=2)


def test_data_energy_closed_forms(port):  # test_energy.cpp:20-72
    ys, f = np.array([1.0, 2.0]), np.array([0.0, 0.5])
    s2 = 0.49
    assert port.data_energy("gaussian", ys, f, sigma=0.7) == pytest.approx(
        0.5 * math.log(2 * math.pi * s2) + (1.0 + 2.25) / (2 * s2 * 2), rel=1e-14)
    ys, f = np.array([3.0, 0.0]), np.array([2.0, 1.5])
    assert port.data_energy("poisson", ys, f) == pytest.approx(((2 - 3 * math.log(2)) + 1.5) / 2, rel=1e-14)
    assert port.data_energy("poisson", ys, np.array([2.0, 0.0])) == math.inf
    assert port.data_energy("gauss_approx", [10.0], [8.0]) == pytest.approx(
        0.5 * math.log(2 * math.pi * 8) + 4 / 16, rel=1e-14)
    var = 525.0
    assert port.data_energy("xps_hetero", [120.0], [100.0], s0=2, s1=0.1, s2=5) == pytest.approx(
        0.5 * math.log(2 * math.pi * var) + 0.5 * 400 / var, rel=1e-14)
    assert port.data_energy("xps_hetero", [120.0], [100.0], s0=2, s1=0.1, s2=5, paper_literal=True) == pytest.approx(
        0.5 * math.log(2 * math.pi * var) + 400 / var, rel=1e-14)
    assert port.data_energy("xps_hetero", [120.0], [0.0], s0=1, s1=0, s2=0) == math.inf


def test_rm_and_predictor_closed_forms(port):  # test_mcmc.cpp:44-109
    assert port.rm_update(1.0, True, 4) == pytest.approx(math.exp(0.5 / 4 ** 0.6), rel=1e-14)
    assert port.rm_update(1.0, False, 1) == pytest.approx(math.exp(-0.5), rel=1e-14)
    s = 1e-12
    for t in range(1, 11):
        s = port.rm_update(s, False, t)
    assert s == 1e-12
    pk, pa, pb = np.array([0, 0]), np.array([0.0, 0.0]), np.array([4.0, 4.0])
    assert port.predict_step_size([], np.zeros(0), np.zeros(0), 0.5, pk, pa, pb)[0] == 2.0
    p1 = port.predict_step_size([0.01], [0.25, 0.25], [1.0, 1.0], 0.9, pk, pa, pb)
    assert p1[0] == pytest.approx(math.exp(2 * (0.25 - 0.5)), rel=1e-13)
    hb = [0.01, 1.0]
    hs = [[1.0 * b ** -0.5, 3.0 * b ** 0.25] for b in hb]
    p2 = port.predict_step_size(hb, np.full(4, 0.5), np.ravel(hs), 0.25, pk, pa, pb)
    assert p2[0] == pytest.approx(0.25 ** -0.5, rel=1e-12)
    assert p2[1] == pytest.approx(3.0 * 0.25 ** 0.25, rel=1e-12)
    hb = [1e-4, 1e-4, 0.02, 0.05, 0.1, 0.4, 1.0]
    hs = [999.0, 999.0] * 2 + sum(([2 * b ** -0.5] * 2 for b in hb[2:]), [])
    p3 = port.predict_step_size(hb, np.full(14, 0.5), hs, 0.09, pk, pa, pb)
    assert p3[0] == pytest.approx(2 * 0.09 ** -0.5, rel=1e-11)


def test_forward_direct_sums(port):  # test_model.cpp:91-105, :161-175 (xps peaks + Shirley)
    spec = M.gm_model(2, 0, 3, 0.1)
    xs = np.linspace(0, 3, 40)
    om = oracle_model(spec, M.Spectrum(xs, np.zeros(40)))
    th = np.array([0.6, 1.2, 95.0, 1.5, 1.45, 147.0])
    expect = 0.6 * np.exp(-0.5 * 95 * (xs - 1.2) ** 2) + 1.5 * np.exp(-0.5 * 147 * (xs - 1.45) ** 2)
    assert np.allclose(port.forward(om, th), expect, rtol=1e-14, atol=0)
    d = ramp(80, 845.0, 887.0, 300.0, 700.0)
    spec = M.xps_model(2, d)
    om = oracle_model(spec, d)
    th = np.array([1800.0, 858.0, 1.2, 0.4, 2400.0, 872.0, 1.8, 0.6, 310.0, 690.0])
    f = port.forward(om, th)
    assert f[0] == pytest.approx(1800 * (0.4 * math.exp(-math.log(2) * (845 - 858) ** 2 / 1.44) + 0.6 * 1.44 / (
        1.44 + 13 ** 2)) + 2400 * (0.6 * math.exp(-math.log(2) * 27 ** 2 / 3.24) + 0.4 * 3.24 / (3.24 + 27 ** 2))
        + 310.0, rel=1e-13)


def test_mh_stationary_moments(port):  # test_mcmc.cpp:164-182, through smc at beta=1 on the conjugate target
    spec, data, F_exact, mn, vn = conjugate(50, 7, port, truth=1.0, sigma=1.0, m0=0.0, v0=1.0)
    r = port.smc_run(oracle_model(spec, data), 4000, 10, 0.5, seed=3)
    post = r.thetas[:, 0]
    assert abs(post.mean() - mn) < 0.02
    assert abs(post.var() / vn - 1) < 0.15
    assert abs(r.F - F_exact) < 0.1
