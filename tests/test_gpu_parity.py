"""GPU parity: the sm_100a kernels (through the C ABI) against the oracle.

Tolerances (stated per test):
  * energies: fp32 point terms with fp64 accumulation.  Bound on the
    log-likelihood difference N*|E_gpu - E_ref| <= 2e-6 * N*|E_ref| + 0.02.
  * ess / log_mean_exp: fp64 on device, relative 1e-12 (tree vs sequential sums).
  * next_beta: bisection identical up to the fp32-mantissa weights of the ESS
    evaluations (|d beta| <= 1e-6 * beta, or the reference tolerance 1e-4 rel.
    on the closed-form two-atom root, test_smc.cpp:67-86).
  * systematic_resample: bit-exact indices except targets within 1e-12 of a
    CDF boundary (parallel fp64 scan vs sequential sum).
  * F: statistical (conjugate closed form |dF| < 0.15 as test_smc.cpp:122-138).
"""
import math

import numpy as np
import pytest

from helpers import conjugate, oracle_model, ramp
from paper_2604_03271_b200 import model as M
from paper_2604_03271_b200 import synthetic as syn

pytestmark = pytest.mark.gpu


def _energy_tol(e_ref, n):
    return (2e-6 * n * abs(e_ref) + 0.02) / n


def _cases():
    cases = []
    d = ramp(60, 0.0, 3.0, 0.2, 2.0)
    cases.append(("gm3", M.gm_model(3, 0.0, 3.0, 0.1, "normal15"), d))
    sp, _ = syn.gen_xps(3, 5)
    cases.append(("xps3_hetero", M.xps_model(3, sp), sp))
    cases.append(("xps3_gapprox", M.ModelSpec("xps", 3, M.xps_model(3, sp).layout, M.GaussianApproxPoissonNoise()), sp))
    cases.append(("xps3_poisson", M.ModelSpec("xps", 3, M.xps_model(3, sp).layout, M.PoissonNoise()), sp))
    cases.append(("xps3_literal", M.xps_model(3, sp, M.XpsHeteroNoise(2.0, 0.1, 5.0, True)), sp))
    w = syn.config("C2")
    cases.append(("c2_xps6", w.spec(6), w.data))
    w1 = syn.config("C1")
    cases.append(("c1_gm3", w1.spec(3), w1.data))
    # grid layouts of the xps Shirley scan: uniform grids take the weight-free
    # scan (endpoints at fixed lane slots), others the per-point trapezoid weights
    rng = np.random.default_rng(3)
    xj = np.sort(sp.xs + rng.uniform(-0.02, 0.02, len(sp.xs)))
    spj = M.Spectrum(xj, sp.ys.copy())
    cases.append(("xps3_jittered_grid", M.xps_model(3, spj), spj))
    for n in (64, 65, 3):  # no padding, one real point past a full lane set, tiny
        idx = np.linspace(0, len(sp.xs) - 1, n).round().astype(int)
        spn = M.Spectrum(np.linspace(sp.xs[0], sp.xs[-1], n), sp.ys[idx].copy())
        cases.append((f"xps2_n{n}", M.xps_model(2, spn), spn))
    # counts ~1e8 with s1 > 0 (variances ~1e12: the paired variance products
    # ~1e24 stay inside the fp32 range)
    big = M.Spectrum(sp.xs.copy(), sp.ys * 3e4)
    cases.append(("xps3_hetero_1e8_counts", M.xps_model(3, big, M.XpsHeteroNoise(1.0, 0.01, 0.0)), big))
    xr, _ = syn.gen_xrd(600, 5)
    cases.append(("xrd3_poisson", M.xrd_model(syn.TIO2_PHASES, xr), xr))
    cases.append(("xrd3_gapprox", M.xrd_model(syn.TIO2_PHASES, xr, M.GaussianApproxPoissonNoise()), xr))
    # the large-spectrum kernels: C3 (N = 4096, W = 4 warps per chain) and C5
    # (N = 8192, W = 8), each on its uniform grid (weight-free Shirley scan,
    # 4 B/point y layout) and on a jittered grid (trapezoid weights staged), at
    # K = 1, 6 and Kmax
    for cname in ("C3", "C5"):
        wc = syn.config(cname)
        xjc = np.sort(wc.data.xs + rng.uniform(-0.004, 0.004, len(wc.data.xs)))
        wj = M.Spectrum(xjc, wc.data.ys.copy())
        for K in (1, 6, wc.k_range[1]):
            cases.append((f"{cname.lower()}_K{K}", wc.spec(K), wc.data))
            cases.append((f"{cname.lower()}_K{K}_jittered", wc.spec(K, wj), wj))
    return cases


@pytest.mark.parametrize("name,spec,data", _cases(), ids=lambda x: x if isinstance(x, str) else "")
def test_energy_batch_matches_oracle(smc, port, name, spec, data):
    om = oracle_model(spec, data)
    th, E_prior = port.init_ensemble(om, 256, 31)
    E_gpu = smc.energies(spec, data, th)
    n = len(data.xs)
    fin = np.isfinite(E_prior)
    assert np.array_equal(np.isfinite(E_gpu), fin)
    err = np.abs(E_gpu[fin] - E_prior[fin])
    tol = np.array([_energy_tol(e, n) for e in E_prior[fin]])
    assert np.all(err <= tol), (name, err.max(), tol.min())


def test_energy_at_truth_xps(smc, port):
    sp, th = syn.gen_xps(7, 11)
    spec = M.xps_model(7, sp)
    om = oracle_model(spec, sp)
    e_ref = port.energy(om, th)
    e_gpu = smc.energy(spec, th, sp)
    assert abs(e_gpu - e_ref) <= _energy_tol(e_ref, 840)


def test_energy_at_truth_xrd(smc, port):
    sp, th = syn.gen_xrd(1000, 7)
    spec = M.xrd_model(syn.TIO2_PHASES, sp)
    om = oracle_model(spec, sp)
    e_ref = port.energy(om, th)
    assert abs(smc.energy(spec, th, sp) - e_ref) <= _energy_tol(e_ref, 1000)
    # Caglioti fault (discriminant <= 0) is the +inf sentinel (model.cpp:243-249)
    bad = th.copy()
    bad[4], bad[5], bad[6] = 0.0, 1.0, 0.0
    assert smc.energy(spec, bad, sp) == math.inf and port.energy(om, bad) == math.inf


def test_energy_sentinels(smc):
    # poisson positivity sentinel (energy.cpp:15-18): negative amplitude -> f <= 0
    d = ramp(50, 0.0, 3.0, 1.0, 2.0)
    spec = M.ModelSpec("gm", 1, M.gm_model(1, 0, 3, 0.1).layout, M.PoissonNoise())
    e = smc.energies(spec, d, np.array([[-1.0, 1.5, 50.0], [1.0, 1.5, 50.0]]))
    assert e[0] == math.inf and math.isfinite(e[1])


def test_ess_oracle(smc, port):
    lw = np.log([0.5, 0.25, 0.25])
    assert smc.ess(lw) == pytest.approx(8.0 / 3.0, rel=1e-13)  # test_smc.cpp:38-53
    assert smc.ess(lw + 7.0) == pytest.approx(8.0 / 3.0, rel=1e-13)
    assert smc.ess(np.zeros(50)) == pytest.approx(50.0, rel=1e-13)
    assert smc.ess(np.array([0.0, -np.inf, -np.inf])) == pytest.approx(1.0, rel=1e-13)
    with pytest.raises(RuntimeError):
        smc.ess(np.full(4, -np.inf))
    rng = np.random.default_rng(0)
    for n in (3, 1000, 65536, 100001):
        lw = rng.normal(size=n) * 5
        assert smc.ess(lw) == pytest.approx(port.ess(lw), rel=1e-12)
        assert smc.log_mean_exp(lw) == pytest.approx(port.log_mean_exp(lw), rel=1e-12, abs=1e-12)


def test_next_beta_two_atom(smc):
    E = np.array([0.0, 10.0])
    q = 2.0 - math.sqrt(3.0)
    delta = -math.log(q) / 10.0
    assert smc.next_beta(E, 1.0, 0.0, 0.75) == pytest.approx(delta, rel=1e-4)
    assert smc.next_beta(E, 1.0, 0.5, 0.75) == pytest.approx(0.5 + delta, rel=1e-4)
    assert smc.next_beta(np.full(5, 3.7), 50.0, 0.3, 0.5) == 1.0
    with pytest.raises(ValueError):
        smc.next_beta(E, 1.0, 1.0, 0.5)


def test_next_beta_matches_oracle(smc, port):
    # T <= 2^15: the single-CTA k_temper bisection; T > 2^15: the production
    # grid path (k_tp_emin + k_tp_ess_tree passes, 3 bisection steps per pass)
    # that C2/C3/C5 run
    rng = np.random.default_rng(1)
    for T, nd in ((1000, 300.0), (4096, 301.0), (65536, 2000.0), (1 << 18, 8192.0), (100003, 4096.0)):
        E = 5.0 + np.abs(rng.normal(size=T)) * 3
        E[::97] = np.inf
        for beta_prev in (0.0, 1e-4, 0.3):
            b_ref = port.next_beta(E, nd, beta_prev, 0.5)
            b_gpu = smc.next_beta(E, nd, beta_prev, 0.5)
            assert b_gpu == pytest.approx(b_ref, rel=1e-6, abs=1e-12)


def test_resample_exact_counts(smc, port):
    # test_smc.cpp:88-103: integer expected counts are hit exactly
    lw = np.log([0.5, 0.25, 0.125, 0.125])
    for rep in range(20):
        u = port.resample_uniform(5, rep + 1)
        idx = smc.systematic_resample(lw, 8, u)
        assert np.all(np.diff(idx) >= 0)
        assert list(np.bincount(idx, minlength=4)) == [4, 2, 1, 1]


def test_resample_matches_oracle(smc, port):
    rng = np.random.default_rng(2)
    # T > 2^15 runs the production grid path (k_tp_wmax, k_tp_wsum,
    # k_tp_offsets, k_tp_resample: slice CDF offsets + per-slice target ranges)
    for T, S in ((10, 3), (1000, 125), (32768, 4096), (65536, 8192), (100003, 777), (1 << 18, 1 << 15),
                 (1 << 18, 300001)):
        lw = rng.normal(size=T) * 2
        lw[::13] = -np.inf
        u = rng.uniform()
        a_gpu = smc.systematic_resample(lw, S, u)
        a_ref = port.systematic_resample(lw, S, u)
        assert np.all(np.diff(a_gpu) >= 0)
        diff = np.nonzero(a_gpu != a_ref)[0]
        if len(diff):
            # only where the target sits on a CDF boundary within fp64 rounding
            w = np.exp(lw - port.log_sum_exp(lw))
            c = np.cumsum(w)
            for j in diff:
                t = (j + u) / S
                assert np.min(np.abs(c - t)) < 1e-12


def test_predict_step_size_matches_oracle(smc, port):
    spec = M.ModelSpec("gm", 1, [M.ScalarParam("a", M.NormalPrior(0.0, 4.0)), M.ScalarParam("b", M.GammaPrior(2, 3)),
                                 M.ScalarParam("c", M.UniformPrior(0, 12))], M.GaussianFixedNoise(1.0))
    pk, pa, pb = spec.arrays()
    rng = np.random.default_rng(3)
    for H in (0, 1, 2, 5, 9):
        hb = np.sort(rng.uniform(1e-4, 1.0, H))
        ha = rng.uniform(0, 1, (H, 3))
        hs = rng.uniform(0.01, 3, (H, 3))
        p_gpu = smc.predict_step_size(hb, ha, hs, 0.7, spec)
        p_ref = port.predict_step_size(hb, ha.ravel(), hs.ravel(), 0.7, pk, pa, pb)
        assert np.allclose(p_gpu, p_ref, rtol=1e-12)


def test_conjugate_free_energy(smc, port):
    # test_smc.cpp:122-138: |F - exact| < 0.15 at T = 2000, n = 10, ess 0.6, seed 7
    spec, data, F_exact, mn, vn = conjugate(20, 404, port)
    rep = smc.smc_run(spec, data, smc.SmcConfig(T=2000, n=10, ess_target=0.6, seed=7))
    assert not rep.diverged
    assert abs(rep.F - F_exact) < 0.15
    lad = rep.arrays["ladder"]
    assert lad[0] == 0.0 and lad[-1] == 1.0 and np.all(np.diff(lad) > 0)
    assert rep.posterior.shape == (1, 2000)
    post = rep.posterior[0]
    assert abs(post.mean() - mn) < 4 * math.sqrt(vn / 2000) * 5
    assert abs(post.var() - vn) < 0.25 * vn


def test_single_level_is_importance_sampling(smc, port):
    # test_smc.cpp:140-157 analogue: one full jump => F = -log_mean_exp(-N E_init)
    spec, data, F_exact, _, _ = conjugate(12, 1001, port)
    rep = smc.smc_run(spec, data, smc.SmcConfig(T=100, n=5, ess_target=1e-9, seed=99))
    assert rep.scalars["levels"] == 1
    assert math.isfinite(rep.F)


def test_max_levels_aborts(smc, port):
    spec, data, *_ = conjugate(200, 5, port)
    with pytest.raises(RuntimeError):
        smc.smc_run(spec, data, smc.SmcConfig(T=100, n=5, ess_target=0.95, max_levels=2))
