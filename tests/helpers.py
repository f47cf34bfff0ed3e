"""Shared test helpers: product ModelSpec -> oracle model, fixtures data."""
from __future__ import annotations

import numpy as np

from oracle.oracle import OracleModel
from paper_2604_03271_b200 import model as M


def oracle_model(spec: M.ModelSpec, data: M.Spectrum) -> OracleModel:
    pk, pa, pb = spec.arrays()
    n = spec.noise
    kw = {}
    if isinstance(n, M.GaussianFixedNoise):
        kw = dict(noise="gaussian", sigma=n.sigma)
    elif isinstance(n, M.PoissonNoise):
        kw = dict(noise="poisson")
    elif isinstance(n, M.GaussianApproxPoissonNoise):
        kw = dict(noise="gauss_approx")
    else:
        kw = dict(noise="xps_hetero", s0=n.s0, s1=n.s1, s2=n.s2, paper_literal=n.paper_literal)
    if spec.family == "xrd":
        ph, mu, ri = spec.reflection_arrays()
        kw.update(refl_phase=ph, refl_mu=mu, refl_int=ri)
    return OracleModel(spec.family, spec.K, pk, pa, pb, data.xs, data.ys, **kw)


def ramp(n, lo, hi, y0, y1) -> M.Spectrum:
    """test_energy.cpp:11-16"""
    return M.Spectrum(np.linspace(lo, hi, n), np.linspace(y0, y1, n))


def conjugate(n, seed, port, truth=1.5, sigma=0.5, m0=0.0, v0=4.0):
    """make_conjugate (tests/conjugate_oracle.hpp:66-77) + closed-form F (:30-40)."""
    ys = truth + sigma * port.normals(seed, n)
    data = M.Spectrum(np.arange(float(n)), ys)
    spec = M.offset_model(sigma, m0, v0)
    N = float(n)
    s2 = sigma * sigma
    vn = 1.0 / (1.0 / v0 + N / s2)
    mn = vn * (m0 / v0 + ys.sum() / s2)
    logz = -0.5 * N * np.log(2 * np.pi * s2) + 0.5 * np.log(vn / v0) + 0.5 * (
        mn * mn / vn - (ys ** 2).sum() / s2 - m0 * m0 / v0)
    return spec, data, -logz, mn, vn
