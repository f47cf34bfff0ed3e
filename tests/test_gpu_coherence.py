"""Cache coherence of the move kernel: the carried energy equals a fresh one.

The reference's contract is that a chain's cached energy always equals a fresh
full evaluation of its state (proj/include/specmc/energy.hpp:27-29; checked
in proj/tests/test_mcmc.cpp:111-135 and test_energy.cpp:81-126).  The move
kernel carries e through fp32 block caches (Q = P - g_b, the amplitude
shortcut Pn = P + (A'/A - 1)(P - Q), in-place commits) and writes it as the
particle's energy.  Here, after whole SMC runs on the BASELINE spectra (C2,
C3 and C5 shapes: W = 2, 4 and 8 warps per chain), every particle's returned
energy is compared with

  * the oracle's fresh fp64 energy of its returned parameters, within the
    energy tolerance of tests/test_gpu_parity.py
    (N |dE| <= 2e-6 N |E| + 0.02 nats), and
  * the device's own fresh full energy (K2) of the same parameters, within
    the same bound.
"""
import numpy as np
import pytest

from helpers import oracle_model
from paper_2604_03271_b200 import synthetic as syn

pytestmark = pytest.mark.gpu


def _tol(e_ref, n):
    return (2e-6 * n * np.abs(e_ref) + 0.02) / n


# (config, K, T, n): small populations so a full run takes seconds
CASES = [("C1", 3, 1024, 8), ("C2", 6, 1024, 8), ("C2", 10, 512, 8), ("C3", 8, 512, 8), ("C5", 20, 256, 16)]


@pytest.mark.parametrize("cfg,K,T,n", CASES, ids=[f"{c}_K{k}" for c, k, _, _ in CASES])
def test_carried_energy_equals_fresh_energy(smc, port, cfg, K, T, n):
    w = syn.config(cfg)
    spec = w.spec(K)
    rep = smc.smc_run(spec, w.data, smc.SmcConfig(T=T, n=n, seed=17))
    assert not rep.diverged
    post = np.ascontiguousarray(rep.posterior.T)  # T x d
    N = len(w.data.xs)
    e_dev = smc.energies(spec, w.data, post)
    e_ref = port.energies(oracle_model(spec, w.data), post)
    e_car = rep.energies
    assert np.all(np.isfinite(e_car)) and np.all(np.isfinite(e_ref))
    tol = _tol(e_ref, N)
    bad_ref = np.abs(e_car - e_ref) > tol
    bad_dev = np.abs(e_car - e_dev) > tol
    assert not bad_ref.any(), (cfg, K, int(bad_ref.sum()), float(np.max(np.abs(e_car - e_ref) * N)))
    assert not bad_dev.any(), (cfg, K, int(bad_dev.sum()), float(np.max(np.abs(e_car - e_dev) * N)))
