"""Model description mirroring the reference's C++ interface.

``ModelSpec``, the prior variants, the noise variants and the builders
``gm_model`` / ``xps_model`` follow proj/include/specmc/model.hpp:13-56,
proj/include/specmc/priors.hpp:13-37 and proj/src/model.cpp:121-189 (paths
relative to the reference root).  ``offset_model`` is the conjugate-mean
problem of proj/tests/conjugate_oracle.hpp:19-28 as a device family.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Union

import numpy as np

# ---------------------------------------------------------------- priors
@dataclass(frozen=True)
class NormalPrior:
    mean: float
    var: float


@dataclass(frozen=True)
class GammaPrior:
    shape: float
    rate: float


@dataclass(frozen=True)
class UniformPrior:
    lo: float
    hi: float


PriorSpec = Union[NormalPrior, GammaPrior, UniformPrior]


def prior_code(p: PriorSpec):
    if isinstance(p, NormalPrior):
        return 0, p.mean, p.var
    if isinstance(p, GammaPrior):
        return 1, p.shape, p.rate
    if isinstance(p, UniformPrior):
        return 2, p.lo, p.hi
    raise TypeError(f"unknown prior {p!r}")


def prior_scale(p: PriorSpec) -> float:
    """priors.cpp:44-49"""
    if isinstance(p, NormalPrior):
        return float(np.sqrt(p.var))
    if isinstance(p, GammaPrior):
        return float(np.sqrt(p.shape) / p.rate)
    return float((p.hi - p.lo) / np.sqrt(12.0))


@dataclass(frozen=True)
class ScalarParam:
    name: str
    prior: PriorSpec


# ----------------------------------------------------------------- noise
@dataclass(frozen=True)
class GaussianFixedNoise:
    sigma: float


@dataclass(frozen=True)
class PoissonNoise:
    pass


@dataclass(frozen=True)
class GaussianApproxPoissonNoise:
    pass


@dataclass(frozen=True)
class XpsHeteroNoise:
    s0: float = 1.0
    s1: float = 0.01
    s2: float = 0.0
    paper_literal: bool = False


NoiseSpec = Union[GaussianFixedNoise, PoissonNoise, GaussianApproxPoissonNoise, XpsHeteroNoise]

FAMILY_CODE = {"gm": 0, "xps": 1, "xrd": 2, "offset": 3}


@dataclass(frozen=True)
class Reflection:
    """model.hpp:25-28"""
    mu_ref: float         # degrees 2theta
    rel_intensity: float  # >= 0


@dataclass
class PhaseRef:
    """model.hpp:29-32"""
    name: str
    reflections: List[Reflection]


@dataclass
class Spectrum:
    """proj/include/specmc/spectrum.hpp:16-20"""
    xs: np.ndarray
    ys: np.ndarray

    def __post_init__(self):
        self.xs = np.ascontiguousarray(self.xs, dtype=np.float64)
        self.ys = np.ascontiguousarray(self.ys, dtype=np.float64)


@dataclass
class ModelSpec:
    """proj/include/specmc/model.hpp:50-56; family in {gm, xps, offset}."""
    family: str
    K: int
    layout: List[ScalarParam]
    noise: NoiseSpec
    phases: list = field(default_factory=list)

    @property
    def d(self) -> int:
        return len(self.layout)

    @property
    def param_names(self):
        return [p.name for p in self.layout]

    def arrays(self):
        codes = [prior_code(p.prior) for p in self.layout]
        pk = np.array([c[0] for c in codes], dtype=np.int32)
        pa = np.array([c[1] for c in codes], dtype=np.float64)
        pb = np.array([c[2] for c in codes], dtype=np.float64)
        return pk, pa, pb

    def reflection_arrays(self):
        ph = np.array([b for b, p in enumerate(self.phases) for _ in p.reflections], dtype=np.int32)
        mu = np.array([r.mu_ref for p in self.phases for r in p.reflections], dtype=np.float64)
        ri = np.array([r.rel_intensity for p in self.phases for r in p.reflections], dtype=np.float64)
        return ph, mu, ri

    def desc(self):
        """Flat C struct; the returned keep-alive tuple must outlive the struct."""
        from . import _lib  # (deferred: describing a model needs no library)
        pk, pa, pb = self.arrays()
        n = self.noise
        sigma, s0, s1, s2, lit = 1.0, 1.0, 0.0, 0.0, 0
        if isinstance(n, GaussianFixedNoise):
            code, sigma = 0, n.sigma
        elif isinstance(n, PoissonNoise):
            code = 1
        elif isinstance(n, GaussianApproxPoissonNoise):
            code = 2
        elif isinstance(n, XpsHeteroNoise):
            code, s0, s1, s2, lit = 3, n.s0, n.s1, n.s2, int(n.paper_literal)
        else:
            raise TypeError(f"unknown noise {n!r}")
        ph, mu, ri = self.reflection_arrays()
        d = _lib.ModelDesc(FAMILY_CODE[self.family], self.K, len(pk), code, sigma, s0, s1, s2, lit,
                           pk.ctypes.data_as(_lib._ip), pa.ctypes.data_as(_lib._dp), pb.ctypes.data_as(_lib._dp),
                           len(ph), ph.ctypes.data_as(_lib._ip), mu.ctypes.data_as(_lib._dp),
                           ri.ctypes.data_as(_lib._dp))
        return d, (pk, pa, pb, ph, mu, ri)


def model_dim(spec: ModelSpec) -> int:
    """model.cpp:86-93"""
    return {"gm": 3 * spec.K, "xps": 4 * spec.K + 2, "xrd": 9 * spec.K + 4, "offset": 1}[spec.family]


def gm_model(K: int, x_lo: float, x_hi: float, noise_sigma: float, mu_kind: str = "normal15") -> ModelSpec:
    """model.cpp:121-136; mu_kind in {"normal15", "uniform"} (GmMuPrior)."""
    mu = NormalPrior(1.5, 0.2) if mu_kind == "normal15" else UniformPrior(x_lo, x_hi)
    layout = []
    for k in range(1, K + 1):
        layout += [ScalarParam(f"A{k}", GammaPrior(5.0, 5.0)), ScalarParam(f"mu{k}", mu),
                   ScalarParam(f"b{k}", GammaPrior(5.0, 0.04))]
    return ModelSpec("gm", K, layout, GaussianFixedNoise(noise_sigma))


def xps_model(K: int, data: Spectrum, noise: XpsHeteroNoise = XpsHeteroNoise()) -> ModelSpec:
    """model.cpp:169-189"""
    ys, xs = data.ys, data.xs
    ymax, ymin = float(ys.max()), float(ys.min())
    yfirst, ylast = float(ys[0]), float(ys[-1])
    layout = []
    for k in range(1, K + 1):
        layout += [ScalarParam(f"A{k}", UniformPrior(max(0.0, 0.3 * ymin), 1.05 * ymax)),
                   ScalarParam(f"mu{k}", UniformPrior(float(xs[0]), float(xs[-1]))),
                   ScalarParam(f"sigma{k}", UniformPrior(0.1, 15.0)),
                   ScalarParam(f"eta{k}", UniformPrior(0.0, 1.0))]
    layout += [ScalarParam("bg_a", UniformPrior(0.95 * yfirst, 1.01 * yfirst)),
               ScalarParam("bg_b", UniformPrior(0.95 * ylast, 1.01 * ylast))]
    return ModelSpec("xps", K, layout, noise)


def xrd_model(phases: List[PhaseRef], data: Spectrum, noise: NoiseSpec = PoissonNoise()) -> ModelSpec:
    """model.cpp:138-167: K = len(phases) crystalline phases (A, d2t, r, alpha, u, v, w, s, t)
    then the background (bg_a, bg_sigma, bg_r, bg_b)."""
    ys = data.ys
    ymax, ymin = float(ys.max()), float(ys.min())
    if not ymax > ymin:
        raise ValueError("xrd model: degenerate intensity range")
    ymin_pos = ymin if ymin > 0.0 else 0.0
    layout = []
    for k in range(1, len(phases) + 1):
        layout += [ScalarParam(f"A{k}", GammaPrior(4.0, 4.0 / (ymax - ymin))),
                   ScalarParam(f"d2t{k}", NormalPrior(0.0, 0.05 * 0.05)),
                   ScalarParam(f"r{k}", UniformPrior(0.0, 1.0)),
                   ScalarParam(f"alpha{k}", GammaPrior(5.0, 4.0)),
                   ScalarParam(f"u{k}", GammaPrior(1.0, 10.0)),
                   ScalarParam(f"v{k}", GammaPrior(1.0, 10.0)),
                   ScalarParam(f"w{k}", GammaPrior(2.0, 20.0)),
                   ScalarParam(f"s{k}", GammaPrior(2.0, 20.0)),
                   ScalarParam(f"t{k}", GammaPrior(1.0, 10.0))]
    half = float(np.sqrt(ymin_pos))
    if not half > 0.0:
        half = 1.0
    layout += [ScalarParam("bg_a", GammaPrior(2.0, 1.0 / ymax)), ScalarParam("bg_sigma", GammaPrior(2.0, 0.4)),
               ScalarParam("bg_r", UniformPrior(0.0, 1.0)), ScalarParam("bg_b", UniformPrior(ymin - half, ymin + half))]
    return ModelSpec("xrd", len(phases), layout, noise, list(phases))


def apply_prior_overrides(spec: ModelSpec, overrides: dict) -> ModelSpec:
    """Config-file prior overrides (config.cpp:204-222): ``prior.<name>`` by exact
    parameter name first, then by the digit-stripped stem (``prior.eta``
    applies to eta1..etaK); an override matching no parameter is an error."""
    used = set()
    layout = []
    for p in spec.layout:
        stem = p.name.rstrip("0123456789")
        if p.name in overrides:
            p = ScalarParam(p.name, overrides[p.name])
            used.add(p.name)
        elif stem != p.name and stem in overrides:
            p = ScalarParam(p.name, overrides[stem])
            used.add(stem)
        layout.append(p)
    unused = set(overrides) - used
    if unused:
        raise ValueError(f"prior override matches no parameter: prior.{sorted(unused)[0]}")
    return ModelSpec(spec.family, spec.K, layout, spec.noise, list(spec.phases))


def offset_model(sigma: float, m0: float = 0.0, v0: float = 4.0) -> ModelSpec:
    """Conjugate-mean problem (conjugate_oracle.hpp:19-28): f(x) = theta, y ~ N(theta, sigma^2)."""
    return ModelSpec("offset", 1, [ScalarParam("theta", NormalPrior(m0, v0))], GaussianFixedNoise(sigma))
