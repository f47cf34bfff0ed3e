"""The REMC comparator (proj/src/remc.cpp) on the B200.

remc_run on the device: one chain unit per replica, one sweep of every
replica per launch (k_chain in REMC mode: the move kernel's proposal,
evaluation and acceptance, Robbins-Monro during burn-in on the run's sweep
clock), then the swap step, the post-burn-in pair accumulators and the
beta = 1 draws (k_remc_exchange).  Parity with the reference's remc_run is
statistical (independent Philox streams):
  * conjugate problem: F within 0.15 of the closed form (the reference's
    own REMC is within ~0.03 at L = 44, 10^4 sweeps),
  * gm (C1, K = 3) and xps spectra: mean F over 4 seeds within 4 standard
    errors (+ 0.3 nats) of the reference's remc_run over 4 seeds; swap and
    replica acceptance rates within 0.1 of the reference's per pair / replica.
"""
import math

import numpy as np
import pytest

from helpers import conjugate, oracle_model


def test_remc_config_validation(smc):
    from paper_2604_03271_b200 import model as M
    spec = M.offset_model(1.0)
    data = M.Spectrum(np.arange(10.0), np.ones(10))
    for bad in (dict(L=0), dict(total_sweeps=0), dict(burn_in_fraction=1.0), dict(swap_period=0),
                dict(ladder=[0.0, 0.5]), dict(ladder=[0.1, 1.0]), dict(ladder=[0.0, 0.6, 0.5, 1.0])):
        with pytest.raises(ValueError):
            smc.remc_run(spec, data, smc.RemcConfig(**bad))


@pytest.mark.gpu
def test_remc_conjugate_closed_form(smc, port):
    spec, data, F_exact, mn, vn = conjugate(20, 404, port)
    reps = smc.remc_run_batch([(spec, 0, smc.RemcConfig(L=44, total_sweeps=10000, seed=s)) for s in range(4)],
                              [data])
    F = np.array([r.F for r in reps])
    assert np.all(np.isfinite(F)) and abs(F.mean() - F_exact) < 0.15, (F, F_exact)
    r = reps[0]
    assert r.sampler == "remc" and r.posterior.shape == (1, 5000)
    lad = r.arrays["ladder"]
    assert lad[0] == 0.0 and lad[-1] == 1.0 and len(lad) == 45 and np.all(np.diff(lad) > 0)
    assert abs(r.posterior[0].mean() - mn) < 0.1 and abs(r.posterior[0].var() / vn - 1) < 0.3


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["c1_gm3", "xps2"])
def test_remc_matches_reference(smc, ref, case):
    from paper_2604_03271_b200 import model as M
    from paper_2604_03271_b200 import synthetic as syn
    if case == "c1_gm3":
        w = syn.config("C1")
        spec, data = w.spec(3), w.data
        L, sweeps = 24, 2000
    else:
        data, _ = syn.gen_xps(2, 5)
        spec = M.xps_model(2, data)
        L, sweeps = 24, 1000
    om = oracle_model(spec, data)
    ref_runs = [ref.remc_run(om, L, sweeps, 0.5, 1, seed=s, workers=0) for s in range(4)]
    gpu_runs = smc.remc_run_batch([(spec, 0, smc.RemcConfig(L=L, total_sweeps=sweeps, seed=s)) for s in range(4)],
                                  [data])
    Fr = np.array([r[0] for r in ref_runs])
    Fg = np.array([r.F for r in gpu_runs])
    assert np.all(np.isfinite(Fg))
    se = math.sqrt(Fr.var(ddof=1) / 4 + Fg.var(ddof=1) / 4)
    assert abs(Fg.mean() - Fr.mean()) <= 4 * se + 0.3, (case, Fg, Fr)
    sr_r = np.mean([r[2] for r in ref_runs], axis=0)
    sr_g = np.mean([r.arrays["swap_rate"] for r in gpu_runs], axis=0)
    assert np.max(np.abs(sr_r - sr_g)) < 0.1, (sr_r, sr_g)
    ra_r = np.mean([r[3] for r in ref_runs], axis=0)
    ra_g = np.mean([r.arrays["replica_acc_rate"] for r in gpu_runs], axis=0)
    assert np.max(np.abs(ra_r - ra_g)) < 0.1, (ra_r, ra_g)
