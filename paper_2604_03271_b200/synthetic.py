"""Synthetic inputs for the BASELINE.json configurations (input synthesis only).

``Rng`` restates the reference generator (xoshiro256++ seeded by splitmix64,
Box-Muller normals with a cached spare; proj/include/specmc/rng.hpp:11-74) so
that ``gen_xps`` reproduces the reference's ``gen_xps`` spectra bit for bit
(proj/src/synthetic.cpp:270-318; pinned against the reference build in
tests/test_synthetic.py).  ``gen_xps_grid`` generalises that recipe to other
grids, peak counts and a Lorentzian-only variant (configs C2, C3, C5);
``gen_gm301`` is the 301-point Gaussian-mixture spectrum of config C1
(truth = proj/data/gm_truth_k3.csv, generator semantics of
synthetic.cpp:178-228).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .model import (GaussianFixedNoise, ModelSpec, PhaseRef, PoissonNoise, Reflection, Spectrum, UniformPrior,
                    XpsHeteroNoise, apply_prior_overrides, gm_model, xps_model)

_M = 0xFFFFFFFFFFFFFFFF


def mix64(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M
    return z ^ (z >> 31)


def hash_combine(h: int, v: int) -> int:
    return mix64(h ^ ((0x9E3779B97F4A7C15 + v + ((h << 6) & _M) + (h >> 2)) & _M))


def trial_seed(base: int, trial: int) -> int:
    """bench.cpp:104-106"""
    return hash_combine(base & _M, trial & _M)


class Rng:
    """xoshiro256++ with value semantics (rng.hpp:28-74)."""

    def __init__(self, seed: int = 0):
        self.key = seed & _M
        sm = self.key
        s = []
        for _ in range(4):
            sm = (sm + 0x9E3779B97F4A7C15) & _M
            s.append(mix64(sm))
        self.s = s
        self.spare = 0.0
        self.has_spare = False

    def substream(self, ids):
        h = self.key
        for i in ids:
            h = hash_combine(h, i)
        return Rng(h)

    def next_u64(self) -> int:
        s = self.s
        rotl = lambda x, k: ((x << k) | (x >> (64 - k))) & _M
        result = (rotl((s[0] + s[3]) & _M, 23) + s[0]) & _M
        t = (s[1] << 17) & _M
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = rotl(s[3], 45)
        return result

    def uniform01(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def poisson(self, mean: float) -> int:
        """rng.hpp:95-124 (Knuth inversion below 10, PTRS above)"""
        if mean <= 0.0:
            return 0
        if mean < 10.0:
            limit = math.exp(-mean)
            k, p = 0, 1.0
            while True:
                k += 1
                p *= self.uniform01()
                if not p > limit:
                    return k - 1
        slam = math.sqrt(mean)
        loglam = math.log(mean)
        b = 0.931 + 2.53 * slam
        a = -0.059 + 0.02483 * b
        inv_alpha = 1.1239 + 1.1328 / (b - 3.4)
        v_r = 0.9277 - 3.6224 / (b - 2.0)
        while True:
            u = self.uniform01() - 0.5
            v = 1.0 - self.uniform01()
            us = 0.5 - abs(u)
            kd = math.floor((2.0 * a / us + b) * u + mean + 0.43)
            if us >= 0.07 and v <= v_r:
                return int(kd)
            if kd < 0.0 or (us < 0.013 and v > us):
                continue
            if math.log(v * inv_alpha / (a / (us * us) + b)) <= kd * loglam - mean - math.lgamma(kd + 1.0):
                return int(kd)

    def normal(self) -> float:
        if self.has_spare:
            self.has_spare = False
            return self.spare
        u1 = self.uniform01()
        u2 = self.uniform01()
        r = math.sqrt(-2.0 * math.log1p(-u1))
        a = 6.283185307179586476925286766559 * u2
        self.spare = r * math.sin(a)
        self.has_spare = True
        return r * math.cos(a)


def _frac(k: int, step: float) -> float:
    v = k * step
    return v - math.floor(v)


def linspace(lo: float, hi: float, n: int) -> np.ndarray:
    """synthetic.cpp:55-60 (lo + (hi-lo) i/(n-1), evaluated in that order)."""
    return np.array([lo + (hi - lo) * float(i) / float(n - 1) for i in range(n)])


def xps_truth(k_true: int, x_lo: float, x_hi: float, margin: float = 13.0, eta_zero: bool = False) -> np.ndarray:
    """synthetic.cpp:288-300 peak recipe (amplitude, centre, width, mixing) + Shirley 6000 -> 6900."""
    th = np.empty(4 * k_true + 2)
    c_lo, c_hi = x_lo + margin, x_hi - margin
    for k in range(1, k_true + 1):
        fr = 0.5 if k_true == 1 else (k - 1) / (k_true - 1)
        th[4 * (k - 1) + 0] = 2400.0 + 800.0 * _frac(k, 0.6180339887498949)
        th[4 * (k - 1) + 1] = c_lo + (c_hi - c_lo) * fr
        th[4 * (k - 1) + 2] = 0.8 + 1.2 * _frac(k, 0.3819660112501051)
        th[4 * (k - 1) + 3] = 0.0 if eta_zero else 0.3 + 0.4 * _frac(k, 0.2360679774997897)
    th[4 * k_true + 0] = 6000.0
    th[4 * k_true + 1] = 6900.0
    return th


def xps_forward_np(theta: np.ndarray, xs: np.ndarray, K: int) -> np.ndarray:
    """model.cpp:269-292 in fp64 (peaks, then the Shirley background), evaluated
    element by element with libm exp in the reference's operation order."""
    n = len(xs)
    ln2 = 0.693147180559945309417232121458176568076
    f = [0.0] * n
    for b in range(K):
        A, mu, sig, eta = (float(v) for v in theta[4 * b:4 * b + 4])
        cg = -ln2 / (sig * sig)
        s2 = sig * sig
        lnum = (1.0 - eta) * (sig * sig)
        for i in range(n):
            dx = float(xs[i]) - mu
            d2 = dx * dx
            blk = A * (eta * math.exp(cg * d2) + lnum / (s2 + d2))
            f[i] = blk if b == 0 else f[i] + blk
    a, bb = float(theta[4 * K]), float(theta[4 * K + 1])
    c = [0.0] * n
    for i in range(1, n):
        c[i] = c[i - 1] + 0.5 * (float(xs[i]) - float(xs[i - 1])) * (f[i] + f[i - 1])
    rng = float(xs[-1]) - float(xs[0])
    total = c[-1]
    if not (total > 1e-12 * max(f) * rng):
        bg = [a + (bb - a) * (float(xs[i]) - float(xs[0])) / rng for i in range(n)]
    else:
        bg = [a + (bb - a) * (c[i] / total) for i in range(n)]
    bg[0], bg[-1] = a, bb
    return np.array([f[i] + bg[i] for i in range(n)])


def gen_xps_grid(k_true: int, seed: int, n: int, x_lo: float, x_hi: float,
                 noise: XpsHeteroNoise = XpsHeteroNoise(), margin: float = 13.0, eta_zero: bool = False):
    """gen_xps (synthetic.cpp:270-318) on an arbitrary grid; returns (Spectrum, truth theta)."""
    xs = linspace(x_lo, x_hi, n)
    th = xps_truth(k_true, x_lo, x_hi, margin, eta_zero)
    f = xps_forward_np(th, xs, k_true)
    rng = Rng(seed)
    ys = np.empty(n)
    for i in range(n):
        var = noise.s0 * noise.s0 * f[i] + noise.s1 * noise.s1 * f[i] * f[i] + noise.s2 * noise.s2
        ys[i] = f[i] + math.sqrt(var) * rng.normal()
    return Spectrum(xs, ys), th


def gen_xps(k_true: int, seed: int, noise: XpsHeteroNoise = XpsHeteroNoise()):
    """The reference's gen_xps: 840 points on [840, 900] eV."""
    return gen_xps_grid(k_true, seed, 840, 840.0, 900.0, noise)


GM3_TRUTH = np.array([0.587, 1.210, 95.689, 1.522, 1.455, 146.837, 1.183, 1.703, 164.469])  # data/gm_truth_k3.csv


def gen_gm(theta: np.ndarray, seed: int, n: int, x_lo: float, x_hi: float, sigma: float, offset: float = 0.0):
    """gen_gaussian_mixture semantics (synthetic.cpp:178-228) on an n-point grid."""
    xs = linspace(x_lo, x_hi, n)
    K = len(theta) // 3
    f = [0.0] * n
    for b in range(K):
        A, mu, bw = (float(v) for v in theta[3 * b:3 * b + 3])
        c = -0.5 * bw
        for i in range(n):
            t = float(xs[i]) - mu
            blk = A * math.exp(c * (t * t))
            f[i] = blk if b == 0 else f[i] + blk
    if sigma > 0:
        rng = Rng(seed)
        for i in range(n):
            f[i] += sigma * rng.normal()
    return Spectrum(xs, np.array(f) + offset)


# proj/data/tio2_synthetic_reflections.csv, xrd_truth_phases.csv, xrd_truth_background.csv
TIO2_PHASES = [
    PhaseRef("rutile", [Reflection(27.45, 1.00), Reflection(36.09, 0.50), Reflection(41.26, 0.25),
                        Reflection(54.32, 0.60), Reflection(56.64, 0.20)]),
    PhaseRef("anatase", [Reflection(25.28, 1.00), Reflection(37.80, 0.20), Reflection(48.05, 0.35),
                         Reflection(53.89, 0.20), Reflection(55.06, 0.20)]),
    PhaseRef("brookite", [Reflection(25.34, 1.00), Reflection(25.69, 0.80), Reflection(30.81, 0.90),
                          Reflection(42.34, 0.30), Reflection(48.01, 0.30)]),
]
# table order (A, d2t, alpha, r, u, v, w, s, t) -> layout order (A, d2t, r, alpha, u, v, w, s, t)
_XRD_TABLE = [(10000, 0.035, 0.6, 0.50, 0.03, 0.03, 0.06, 0.06, 0.03),
              (3500, 0.055, 0.9, 0.65, 0.1, 0.1, 0.2, 0.2, 0.1),
              (1000, 0.04, 1.0, 0.75, 0.1, 0.1, 0.2, 0.2, 0.1)]
XRD_TRUTH = np.array([v for A, d2t, al, r, u, vv, w, s_, t in _XRD_TABLE for v in (A, d2t, r, al, u, vv, w, s_, t)]
                     + [60000.0, 10.0, 0.0, 100.0])


def xrd_forward_np(theta: np.ndarray, xs: np.ndarray, phases) -> np.ndarray:
    """model.cpp:222-267 in fp64, the reference's operation order (libm exp/tan/cos)."""
    K = len(phases)
    k4 = 2.772588722239781237668928485832706272302
    n = len(xs)
    blocks = []
    for b, ph in enumerate(phases):
        A, d2t, r, alpha, u, v, w, s_, t = (float(x) for x in theta[9 * b:9 * b + 9])
        out = [0.0] * n
        for rf in ph.reflections:
            c = rf.mu_ref + d2t
            half = 0.5 * c * (math.pi / 180.0)
            tn = math.tan(half)
            disc = u * tn * tn - v * tn + w
            if not disc > 0.0:
                raise ValueError(f"Caglioti discriminant non-positive at reflection center {c} deg")
            sig0 = math.sqrt(disc)
            om0 = s_ / math.cos(half) + t * tn
            amp = A * rf.rel_intensity
            for i in range(n):
                dx = float(xs[i]) - c
                wg = dx / (alpha * sig0) if dx >= 0.0 else dx / sig0
                wl = dx / (alpha * om0) if dx >= 0.0 else dx / om0
                out[i] += amp * ((1.0 - r) * math.exp((-k4) * (wg * wg)) + r / (1.0 + 4.0 * (wl * wl)))
        blocks.append(out)
    a, sbg, rbg, bg = (float(x) for x in theta[9 * K:9 * K + 4])
    blocks.append([a * ((1.0 - rbg) * math.exp((-k4) * ((float(x) / sbg) ** 2)) + rbg / (1.0 + 4.0 * ((float(x) / sbg)
                                                                                                    ** 2))) + bg
                   for x in xs])
    f = list(blocks[0])
    for blk in blocks[1:]:
        f = [f[i] + blk[i] for i in range(n)]
    return np.array(f)


def gen_xrd(n_points: int, seed: int):
    """gen_xrd (synthetic.cpp:230-268): three TiO2 phases + pV background, Poisson counts on [5, 60]."""
    xs = linspace(5.0, 60.0, n_points)
    f = xrd_forward_np(XRD_TRUTH, xs, TIO2_PHASES)
    rng = Rng(seed)
    ys = np.array([float(rng.poisson(float(v))) for v in f])
    return Spectrum(xs, ys), XRD_TRUTH.copy()


# ------------------------------------------------------------- BASELINE configs
@dataclass
class Workload:
    name: str
    data: Spectrum
    family: str
    k_range: tuple
    T: int
    n: int
    noise: object
    truth_k: int
    prior_overrides: dict = None  # config-file prior overrides (config.cpp:204-222)

    def spec(self, K: int, data: Spectrum | None = None) -> ModelSpec:
        """The fitted model at K peaks (on ``data``, default the workload's spectrum)."""
        data = self.data if data is None else data
        if self.family == "gm":
            s = gm_model(K, float(data.xs[0]), float(data.xs[-1]), self.noise.sigma, "uniform")
        else:
            s = xps_model(K, data, self.noise)
        return apply_prior_overrides(s, self.prior_overrides) if self.prior_overrides else s


def config(name: str, T: int | None = None) -> Workload:
    """BASELINE.json configs."""
    if name == "C1":
        # N = 301, 3 Gaussian peaks; the flat background is a known offset (generated at 0)
        data = gen_gm(GM3_TRUTH, 1, 301, 0.0, 3.0, 0.1)
        return Workload("C1", data, "gm", (1, 5), T or 4096, 8, GaussianFixedNoise(0.1), 3)
    if name == "C2":
        noise = XpsHeteroNoise(1.0, 0.0, 0.0)
        data, _ = gen_xps_grid(6, 2, 2000, 5.0, 60.0, noise)
        return Workload("C2", data, "xps", (1, 10), T or 65536, 8, noise, 6)
    if name == "C3":
        # 8 Lorentzian peaks; fitted with the xps family and the Lorentzian basis
        # pinned by the config override prior.eta = uniform(0, 1e-9) (SURVEY.md
        # Appendix A; config.cpp:204-222, lineshapes.hpp:51)
        noise = XpsHeteroNoise(1.0, 0.0, 0.0)
        data, _ = gen_xps_grid(8, 3, 4096, 5.0, 60.0, noise, eta_zero=True)
        return Workload("C3", data, "xps", (1, 12), T or (1 << 22), 8, noise, 8, {"eta": UniformPrior(0.0, 1e-9)})
    if name == "C5":
        noise = XpsHeteroNoise(1.0, 0.0, 0.0)
        data, _ = gen_xps_grid(20, 5, 8192, 5.0, 105.0, noise, margin=3.0)
        return Workload("C5", data, "xps", (1, 20), T or (1 << 18), 16, noise, 20)
    raise KeyError(name)


def config_c4(n_spectra: int = 1024, T: int | None = None):
    """C4: n_spectra independent gen_xps spectra (k_true = 1 + (i mod 6), seed = i;
    SURVEY.md 8d), each fitted for K = 1..6.  Returns (spectra, k_true list, T, n)."""
    noise = XpsHeteroNoise()
    spectra, ks = [], []
    for i in range(n_spectra):
        sp, _ = gen_xps(1 + (i % 6), i, noise)
        spectra.append(sp)
        ks.append(1 + (i % 6))
    return spectra, ks, T or 16384, 8
