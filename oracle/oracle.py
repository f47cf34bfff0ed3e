"""ctypes bindings for the parity checker (TEST INFRASTRUCTURE ONLY).

``Port`` wraps oracle/liboracle.so (the C restatement, oracle/specmc_oracle.c);
``Ref`` wraps oracle/_ref/libspecmc_ref.so (the unchanged reference sources
built against oracle/eigen_shim by oracle/build_oracle.py).  Both expose the
same Python surface so tests can compare them and the product against them.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs import this module.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libspecmc_ref.so"

FAMILY = {"gm": 0, "xps": 1, "xrd": 2, "offset": 3}
NOISE = {"gaussian": 0, "poisson": 1, "gauss_approx": 2, "xps_hetero": 3}
PRIOR = {"normal": 0, "gamma": 1, "uniform": 2}

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_lp = C.POINTER(C.c_int64)


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a, t=_dp):
    return a.ctypes.data_as(t)


class _Model(C.Structure):
    _fields_ = [
        ("family", C.c_int), ("K", C.c_int), ("d", C.c_int), ("noise", C.c_int),
        ("sigma", C.c_double), ("s0", C.c_double), ("s1", C.c_double), ("s2", C.c_double),
        ("paper_literal", C.c_int),
        ("prior_kind", _ip), ("prior_a", _dp), ("prior_b", _dp),
        ("xs", _dp), ("ys", _dp), ("n", C.c_int64),
        ("n_refl", C.c_int), ("refl_phase", _ip), ("refl_mu", _dp), ("refl_int", _dp),
    ]


@dataclass
class OracleModel:
    """Flat model description shared by both oracle libraries.

    ``family``: gm | xps | offset; ``prior_kind``/``prior_a``/``prior_b`` follow
    the reference layout order (model.hpp:43-49); noise as energy.cpp:7-28."""
    family: str
    K: int
    prior_kind: np.ndarray
    prior_a: np.ndarray
    prior_b: np.ndarray
    xs: np.ndarray
    ys: np.ndarray
    noise: str = "gaussian"
    sigma: float = 0.1
    s0: float = 1.0
    s1: float = 0.01
    s2: float = 0.0
    paper_literal: bool = False
    refl_phase: np.ndarray = None  # xrd: phase index of every reflection (phase order)
    refl_mu: np.ndarray = None
    refl_int: np.ndarray = None

    def struct(self):
        rp = np.ascontiguousarray(self.refl_phase if self.refl_phase is not None else [0], dtype=np.int32)
        rm = _d(self.refl_mu if self.refl_mu is not None else [0.0])
        ri = _d(self.refl_int if self.refl_int is not None else [0.0])
        nr = 0 if self.refl_phase is None else len(self.refl_phase)
        self._keep = [np.ascontiguousarray(self.prior_kind, dtype=np.int32), _d(self.prior_a), _d(self.prior_b),
                      _d(self.xs), _d(self.ys), rp, rm, ri]
        pk, pa, pb, xs, ys = self._keep[:5]
        return _Model(FAMILY[self.family], self.K, len(pk), NOISE[self.noise], self.sigma, self.s0, self.s1,
                      self.s2, int(self.paper_literal), _ptr(pk, _ip), _ptr(pa), _ptr(pb), _ptr(xs), _ptr(ys),
                      len(xs), nr, _ptr(rp, _ip), _ptr(rm), _ptr(ri))

    @property
    def d(self):
        return len(self.prior_kind)


@dataclass
class OracleRun:
    F: float
    diverged: bool
    levels: int
    ladder: np.ndarray
    ess_ratio: np.ndarray
    log_mean_w: np.ndarray
    acc_rate: np.ndarray
    thetas: np.ndarray  # (T, d)
    energies: np.ndarray | None
    wall_seconds: float = 0.0
    proposals: int = 0
    trials: int = 0


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


class Port:
    """The C restatement (oracle/specmc_oracle.c)."""

    class _Res(C.Structure):
        _fields_ = [("F", C.c_double), ("diverged", C.c_int), ("levels", C.c_int),
                    ("ladder", _dp), ("ess_ratio", _dp), ("log_mean_w", _dp), ("acc_rate", _dp),
                    ("thetas", _dp), ("energies", _dp), ("proposals", C.c_longlong), ("trials", C.c_longlong)]

    def __init__(self, path: Path = PORT_SO):
        if not Path(path).exists():
            from oracle.build_oracle import build_port
            build_port()
        L = self.lib = C.CDLL(str(path))
        L.orc_energy.restype = C.c_double
        L.orc_energy.argtypes = [C.POINTER(_Model), _dp]
        L.orc_forward.argtypes = [C.POINTER(_Model), _dp, _dp]
        L.orc_data_energy.restype = C.c_double
        L.orc_data_energy.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int, _dp, _dp,
                                      C.c_int64]
        L.orc_ess.restype = C.c_double
        L.orc_ess.argtypes = [_dp, C.c_int64, _ip]
        L.orc_log_mean_exp.restype = C.c_double
        L.orc_log_mean_exp.argtypes = [_dp, C.c_int64]
        L.orc_log_sum_exp.restype = C.c_double
        L.orc_log_sum_exp.argtypes = [_dp, C.c_int64]
        L.orc_next_beta.restype = C.c_double
        L.orc_next_beta.argtypes = [_dp, C.c_int64, C.c_double, C.c_double, C.c_double, _ip]
        L.orc_systematic_resample.argtypes = [_dp, C.c_int64, C.c_int64, C.c_double, _lp]
        L.orc_resample_uniform.restype = C.c_double
        L.orc_resample_uniform.argtypes = [C.c_uint64, C.c_int]
        L.orc_predict_step_size.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int, C.c_double, _ip, _dp, _dp, _dp]
        L.orc_rm_update.restype = C.c_double
        L.orc_rm_update.argtypes = [C.c_double, C.c_int, C.c_longlong]
        L.orc_smc_run.argtypes = [C.POINTER(_Model), C.c_int64, C.c_int, C.c_double, C.c_int, C.c_uint64,
                                  C.POINTER(self._Res)]
        L.orc_init_ensemble.argtypes = [C.POINTER(_Model), C.c_int64, C.c_uint64, _dp, _dp]
        L.orc_normals.argtypes = [C.c_uint64, C.c_int64, _dp]
        L.orc_prior_logpdf1.restype = C.c_double
        L.orc_prior_logpdf1.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double]
        L.orc_prior_scale.restype = C.c_double
        L.orc_prior_scale.argtypes = [C.c_int, C.c_double, C.c_double]
        L.orc_hash_combine.restype = C.c_uint64
        L.orc_hash_combine.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_validate_smc_config.argtypes = [C.c_int64, C.c_int, C.c_double, C.c_int, C.c_int]
        L.orc_cumtrapz.argtypes = [_dp, _dp, C.c_int64, _dp]

    # --- parity units -------------------------------------------------
    def energy(self, m: OracleModel, theta) -> float:
        s = m.struct()
        th = _d(theta)
        return self.lib.orc_energy(C.byref(s), _ptr(th))

    def energies(self, m: OracleModel, thetas) -> np.ndarray:
        thetas = np.atleast_2d(_d(thetas))
        return np.array([self.energy(m, t) for t in thetas])

    def forward(self, m: OracleModel, theta) -> np.ndarray:
        s = m.struct()
        th = _d(theta)
        f = np.empty(len(m.xs))
        ok = self.lib.orc_forward(C.byref(s), _ptr(th), _ptr(f))
        if not ok:
            raise OracleError(3, "forward fault")
        return f

    def data_energy(self, noise, ys, f, sigma=1.0, s0=1.0, s1=0.0, s2=0.0, paper_literal=False) -> float:
        ys, f = _d(ys), _d(f)
        return self.lib.orc_data_energy(NOISE[noise], sigma, s0, s1, s2, int(paper_literal), _ptr(ys), _ptr(f),
                                        len(ys))

    def ess(self, lw) -> float:
        lw = _d(lw)
        err = C.c_int(0)
        v = self.lib.orc_ess(_ptr(lw), len(lw), C.byref(err))
        if err.value:
            raise OracleError(err.value, "ess: total weight is zero")
        return v

    def log_mean_exp(self, v) -> float:
        v = _d(v)
        return self.lib.orc_log_mean_exp(_ptr(v), len(v))

    def log_sum_exp(self, v) -> float:
        v = _d(v)
        return self.lib.orc_log_sum_exp(_ptr(v), len(v))

    def next_beta(self, E, n_data, beta_prev, target) -> float:
        E = _d(E)
        err = C.c_int(0)
        v = self.lib.orc_next_beta(_ptr(E), len(E), n_data, beta_prev, target, C.byref(err))
        if err.value:
            raise OracleError(err.value, "next_beta")
        return v

    def systematic_resample(self, lw, S, u) -> np.ndarray:
        lw = _d(lw)
        out = np.empty(S, dtype=np.int64)
        rc = self.lib.orc_systematic_resample(_ptr(lw), len(lw), S, u, _ptr(out, _lp))
        if rc:
            raise OracleError(rc, "systematic_resample: total weight is zero")
        return out

    def resample_uniform(self, seed, level) -> float:
        return self.lib.orc_resample_uniform(seed, level)

    def predict_step_size(self, hbeta, hacc, hstep, beta_next, pk, pa, pb) -> np.ndarray:
        hbeta, hacc, hstep = _d(hbeta), _d(hacc), _d(hstep)
        pk = np.ascontiguousarray(pk, dtype=np.int32)
        pa, pb = _d(pa), _d(pb)
        d = len(pk)
        out = np.empty(d)
        self.lib.orc_predict_step_size(_ptr(hbeta), _ptr(hacc), _ptr(hstep), len(hbeta), d, beta_next,
                                       _ptr(pk, _ip), _ptr(pa), _ptr(pb), _ptr(out))
        return out

    def rm_update(self, step, accepted, t) -> float:
        return self.lib.orc_rm_update(step, int(accepted), t)

    def normals(self, seed, n) -> np.ndarray:
        out = np.empty(n)
        self.lib.orc_normals(seed, n, _ptr(out))
        return out

    def init_ensemble(self, m: OracleModel, T, seed):
        s = m.struct()
        th = np.empty((T, m.d))
        E = np.empty(T)
        self.lib.orc_init_ensemble(C.byref(s), T, seed, _ptr(th), _ptr(E))
        return th, E

    def smc_run(self, m: OracleModel, T, n, ess_target=0.5, max_levels=2000, seed=0, keep=True) -> OracleRun:
        import time
        s = m.struct()
        lad, er, lw, ar = (np.zeros(max_levels + 1) for _ in range(4))
        th = np.empty((T, m.d)) if keep else None
        E = np.empty(T) if keep else None
        res = self._Res(0.0, 0, 0, _ptr(lad), _ptr(er), _ptr(lw), _ptr(ar),
                        _ptr(th) if keep else None, _ptr(E) if keep else None, 0, 0)
        t0 = time.perf_counter()
        rc = self.lib.orc_smc_run(C.byref(s), T, n, ess_target, max_levels, seed, C.byref(res))
        wall = time.perf_counter() - t0
        if rc:
            raise OracleError(rc, "smc_run")
        L = res.levels
        return OracleRun(res.F, bool(res.diverged), L, lad[:L + 1].copy(), er[:L].copy(), lw[:L].copy(),
                         ar[:L].copy(), th, E, wall, res.proposals, res.trials)


class Ref:
    """The unchanged reference sources, built against oracle/eigen_shim."""

    class _Res(C.Structure):
        _fields_ = [("F", C.c_double), ("diverged", C.c_int), ("levels", C.c_int), ("wall_seconds", C.c_double),
                    ("ladder", _dp), ("ess_ratio", _dp), ("log_mean_w", _dp), ("acc_rate", _dp),
                    ("thetas", _dp), ("energies", _dp)]

    def __init__(self, path: Path = REF_SO):
        if not Path(path).exists():
            raise FileNotFoundError(f"{path} not built (needs /root/reference; see oracle/build_oracle.py)")
        L = self.lib = C.CDLL(str(path))
        L.ref_energy.restype = C.c_double
        L.ref_energy.argtypes = [C.POINTER(_Model), _dp]
        L.ref_forward.argtypes = [C.POINTER(_Model), _dp, _dp, C.c_char_p, C.c_size_t]
        L.ref_data_energy.restype = C.c_double
        L.ref_data_energy.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int, _dp, _dp,
                                      C.c_int64]
        L.ref_ess.restype = C.c_double
        L.ref_ess.argtypes = [_dp, C.c_int64, _ip]
        L.ref_log_mean_exp.restype = C.c_double
        L.ref_log_mean_exp.argtypes = [_dp, C.c_int64]
        L.ref_next_beta.restype = C.c_double
        L.ref_next_beta.argtypes = [_dp, C.c_int64, C.c_double, C.c_double, C.c_double, _ip]
        L.ref_systematic_resample.argtypes = [_dp, C.c_int64, C.c_int64, C.c_uint64, _lp]
        L.ref_uniform01.restype = C.c_double
        L.ref_uniform01.argtypes = [C.c_uint64]
        L.ref_predict_step_size.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int, C.c_double, _ip, _dp, _dp, _dp]
        L.ref_rm_update.restype = C.c_double
        L.ref_rm_update.argtypes = [C.c_double, C.c_int, C.c_longlong]
        L.ref_smc_run.argtypes = [C.POINTER(_Model), C.c_int64, C.c_int, C.c_double, C.c_int, C.c_uint64, C.c_int,
                                  C.POINTER(self._Res), C.c_char_p, C.c_size_t]
        L.ref_gen_xps.argtypes = [C.c_int, C.c_uint64, C.c_double, C.c_double, C.c_double, _dp, _dp]
        L.ref_xps_model_priors.argtypes = [C.c_int, _dp, _dp, C.c_int64, _ip, _dp, _dp]
        L.ref_gm_model_priors.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_int, _ip, _dp, _dp]
        L.ref_xrd_model_priors.argtypes = [C.c_int, C.c_int, _ip, _dp, _dp, _dp, _dp, C.c_int64, _ip, _dp, _dp]
        L.ref_gen_xrd.argtypes = [C.c_int64, C.c_uint64, _dp, _dp]
        L.ref_model_select.argtypes = [C.c_int, _ip, _dp, _ip, _ip]
        L.ref_remc_run.argtypes = [C.POINTER(_Model), C.c_int, C.c_int64, C.c_double, C.c_int64, C.c_uint64, C.c_int,
                                   _dp, _ip, _dp, _dp, _dp, C.c_char_p, C.c_size_t]
        L.ref_bench_table.argtypes = [C.POINTER(C.c_char_p), C.c_int, C.c_char_p, C.c_char_p, C.c_size_t]
        L.ref_ci_table.argtypes = [C.POINTER(C.c_char_p), C.c_int, C.c_char_p, C.c_char_p, C.c_double, C.c_char_p,
                                   C.c_size_t]
        L.ref_trial_seed.restype = C.c_uint64
        L.ref_trial_seed.argtypes = [C.c_uint64, C.c_int]

    def energy(self, m: OracleModel, theta) -> float:
        s = m.struct()
        th = _d(theta)
        return self.lib.ref_energy(C.byref(s), _ptr(th))

    def energies(self, m: OracleModel, thetas) -> np.ndarray:
        thetas = np.atleast_2d(_d(thetas))
        return np.array([self.energy(m, t) for t in thetas])

    def forward(self, m: OracleModel, theta) -> np.ndarray:
        s = m.struct()
        th = _d(theta)
        f = np.empty(len(m.xs))
        err = C.create_string_buffer(256)
        rc = self.lib.ref_forward(C.byref(s), _ptr(th), _ptr(f), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return f

    def data_energy(self, noise, ys, f, sigma=1.0, s0=1.0, s1=0.0, s2=0.0, paper_literal=False) -> float:
        ys, f = _d(ys), _d(f)
        return self.lib.ref_data_energy(NOISE[noise], sigma, s0, s1, s2, int(paper_literal), _ptr(ys), _ptr(f),
                                        len(ys))

    def ess(self, lw) -> float:
        lw = _d(lw)
        rc = C.c_int(0)
        v = self.lib.ref_ess(_ptr(lw), len(lw), C.byref(rc))
        if rc.value:
            raise OracleError(rc.value, "ess")
        return v

    def log_mean_exp(self, v) -> float:
        v = _d(v)
        return self.lib.ref_log_mean_exp(_ptr(v), len(v))

    def next_beta(self, E, n_data, beta_prev, target) -> float:
        E = _d(E)
        rc = C.c_int(0)
        v = self.lib.ref_next_beta(_ptr(E), len(E), n_data, beta_prev, target, C.byref(rc))
        if rc.value:
            raise OracleError(rc.value, "next_beta")
        return v

    def systematic_resample(self, lw, S, seed) -> np.ndarray:
        lw = _d(lw)
        out = np.empty(S, dtype=np.int64)
        rc = self.lib.ref_systematic_resample(_ptr(lw), len(lw), S, seed, _ptr(out, _lp))
        if rc:
            raise OracleError(rc, "systematic_resample")
        return out

    def uniform01(self, seed) -> float:
        return self.lib.ref_uniform01(seed)

    def predict_step_size(self, hbeta, hacc, hstep, beta_next, pk, pa, pb) -> np.ndarray:
        hbeta, hacc, hstep = _d(hbeta), _d(hacc), _d(hstep)
        pk = np.ascontiguousarray(pk, dtype=np.int32)
        pa, pb = _d(pa), _d(pb)
        d = len(pk)
        out = np.empty(d)
        self.lib.ref_predict_step_size(_ptr(hbeta), _ptr(hacc), _ptr(hstep), len(hbeta), d, beta_next,
                                       _ptr(pk, _ip), _ptr(pa), _ptr(pb), _ptr(out))
        return out

    def rm_update(self, step, accepted, t) -> float:
        return self.lib.ref_rm_update(step, int(accepted), t)

    def smc_run(self, m: OracleModel, T, n, ess_target=0.5, max_levels=2000, seed=0, workers=1,
                keep=True) -> OracleRun:
        s = m.struct()
        lad, er, lw, ar = (np.zeros(max_levels + 1) for _ in range(4))
        th = np.empty((T, m.d)) if keep else None
        E = np.empty(T) if keep else None
        res = self._Res(0.0, 0, 0, 0.0, _ptr(lad), _ptr(er), _ptr(lw), _ptr(ar),
                        _ptr(th) if keep else None, _ptr(E) if keep else None)
        err = C.create_string_buffer(512)
        rc = self.lib.ref_smc_run(C.byref(s), T, n, ess_target, max_levels, seed, workers, C.byref(res), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        L = res.levels
        return OracleRun(res.F, bool(res.diverged), L, lad[:L + 1].copy(), er[:L].copy(), lw[:L].copy(),
                         ar[:L].copy(), th, E if m.family == "offset" else None, res.wall_seconds,
                         int(T) * m.d * L)

    def gen_xps(self, k_true, seed, s0=1.0, s1=0.01, s2=0.0):
        xs, ys = np.empty(840), np.empty(840)
        rc = self.lib.ref_gen_xps(k_true, seed, s0, s1, s2, _ptr(xs), _ptr(ys))
        if rc:
            raise OracleError(rc, "gen_xps")
        return xs, ys

    def xps_model_priors(self, K, xs, ys):
        xs, ys = _d(xs), _d(ys)
        d = 4 * K + 2
        pk = np.empty(d, dtype=np.int32)
        pa, pb = np.empty(d), np.empty(d)
        self.lib.ref_xps_model_priors(K, _ptr(xs), _ptr(ys), len(xs), _ptr(pk, _ip), _ptr(pa), _ptr(pb))
        return pk, pa, pb

    def gm_model_priors(self, K, x_lo, x_hi, sigma, uniform_mu):
        d = 3 * K
        pk = np.empty(d, dtype=np.int32)
        pa, pb = np.empty(d), np.empty(d)
        self.lib.ref_gm_model_priors(K, x_lo, x_hi, sigma, int(uniform_mu), _ptr(pk, _ip), _ptr(pa), _ptr(pb))
        return pk, pa, pb

    def xrd_model_priors(self, K, refl_phase, refl_mu, refl_int, xs, ys):
        rp = np.ascontiguousarray(refl_phase, dtype=np.int32)
        rm, ri, xs, ys = _d(refl_mu), _d(refl_int), _d(xs), _d(ys)
        d = 9 * K + 4
        pk = np.empty(d, dtype=np.int32)
        pa, pb = np.empty(d), np.empty(d)
        self.lib.ref_xrd_model_priors(K, len(rp), _ptr(rp, _ip), _ptr(rm), _ptr(ri), _ptr(xs), _ptr(ys), len(xs),
                                      _ptr(pk, _ip), _ptr(pa), _ptr(pb))
        return pk, pa, pb

    def gen_xrd(self, n_points, seed):
        xs, ys = np.empty(n_points), np.empty(n_points)
        rc = self.lib.ref_gen_xrd(n_points, seed, _ptr(xs), _ptr(ys))
        if rc:
            raise OracleError(rc, "gen_xrd")
        return xs, ys

    def model_select(self, ks, fs, diverged) -> int:
        ks = np.ascontiguousarray(ks, dtype=np.int32)
        fs = _d(fs)
        dv = np.ascontiguousarray(diverged, dtype=np.int32)
        kb = C.c_int(0)
        rc = self.lib.ref_model_select(len(ks), _ptr(ks, _ip), _ptr(fs), _ptr(dv, _ip), C.byref(kb))
        if rc:
            raise OracleError(rc, "model_select")
        return kb.value

    def remc_run(self, m: OracleModel, L=44, total_sweeps=10000, burn_in_fraction=0.5, swap_period=1, seed=0,
                 workers=1):
        """remc_run(problem, cfg) (remc.cpp:78-163): (F, diverged, swap_rate[L], replica_acc[L + 1], wall)"""
        s = m.struct()
        F, dv, wall = C.c_double(), C.c_int(), C.c_double()
        sr, ra = np.zeros(L), np.zeros(L + 1)
        err = C.create_string_buffer(512)
        rc = self.lib.ref_remc_run(C.byref(s), L, total_sweeps, burn_in_fraction, swap_period, seed, workers,
                                   C.byref(F), C.byref(dv), _ptr(sr), _ptr(ra), C.byref(wall), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return F.value, bool(dv.value), sr, ra, wall.value

    def bench_table(self, paths, reference_label="") -> str:
        """bench_table_text(table_from_reports(read_report(p) for p in paths)) (bench.cpp:147-327)"""
        arr = (C.c_char_p * len(paths))(*[str(p).encode() for p in paths])
        buf = C.create_string_buffer(1 << 20)
        n = self.lib.ref_bench_table(arr, len(paths), reference_label.encode(), buf, len(buf))
        if n < 0:
            raise OracleError(3, buf.value.decode())
        return buf.value.decode()

    def ci_table(self, paths, truth_path, param, level=0.95) -> str:
        """ci_table_text(ci_error_curve(...)) (bench.cpp:251-338)"""
        arr = (C.c_char_p * len(paths))(*[str(p).encode() for p in paths])
        buf = C.create_string_buffer(1 << 20)
        n = self.lib.ref_ci_table(arr, len(paths), str(truth_path).encode(), param.encode(), level, buf, len(buf))
        if n < 0:
            raise OracleError(3, buf.value.decode())
        return buf.value.decode()

    def trial_seed(self, base, trial) -> int:
        return self.lib.ref_trial_seed(base, trial)

    # ---- output side (report.cpp, posterior.cpp)
    def format_double(self, v) -> str:
        buf = C.create_string_buffer(64)
        self.lib.ref_format_double.argtypes = [C.c_double, C.c_char_p, C.c_int]
        self.lib.ref_format_double(float(v), buf, 64)
        return buf.value.decode()

    def weighted_quantile(self, s, w, q) -> float:
        s, w = _d(s), _d(w)
        rc = C.c_int(0)
        f = self.lib.ref_weighted_quantile
        f.restype = C.c_double
        f.argtypes = [_dp, _dp, C.c_int64, C.c_double, C.POINTER(C.c_int)]
        v = f(_ptr(s), _ptr(w), len(s), float(q), C.byref(rc))
        if rc.value:
            raise ValueError("weighted_quantile")
        return v

    def sort_peak_blocks(self, post, block, center_off, n_blocks) -> np.ndarray:
        P = np.ascontiguousarray(np.asarray(post, dtype=np.float64).T)  # draw-major
        out = np.empty_like(P)
        rc = self.lib.ref_sort_peak_blocks(_ptr(P), P.shape[1], P.shape[0], block, center_off, n_blocks, _ptr(out))
        if rc:
            raise ValueError("sort_peak_blocks")
        return out.T.copy()

    def write_report(self, path, sampler, label, F, diverged, wall, scalars, arrays, param_names, posterior,
                     max_draws=20000, config_lines=()):
        def strs(xs):
            arr = (C.c_char_p * max(len(xs), 1))()
            for i, x in enumerate(xs):
                arr[i] = x.encode()
            return arr
        sk = list(scalars.keys())
        sv = _d([scalars[k] for k in sk]) if sk else np.zeros(1)
        ak = list(arrays.keys())
        al = np.array([len(arrays[k]) for k in ak] or [0], dtype=np.int64)
        av = _d(np.concatenate([np.asarray(arrays[k], dtype=np.float64).ravel() for k in ak])) if ak else np.zeros(1)
        P = np.ascontiguousarray(np.asarray(posterior, dtype=np.float64).T)
        f = self.lib.ref_write_report
        f.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_double, C.c_int, C.c_double, C.c_int, C.c_void_p, _dp,
                      C.c_int, C.c_void_p, C.POINTER(C.c_int64), _dp, C.c_int, C.c_void_p, C.c_int64, C.c_int64, _dp,
                      C.c_int64, C.c_int, C.c_void_p]
        cl = list(config_lines)
        rc = f(str(path).encode(), sampler.encode(), label.encode(), float(F), int(diverged), float(wall), len(sk),
               strs(sk), _ptr(sv), len(ak), strs(ak), al.ctypes.data_as(C.POINTER(C.c_int64)), _ptr(av),
               len(param_names), strs(param_names), P.shape[1], P.shape[0], _ptr(P), int(max_draws), len(cl), strs(cl))
        if rc:
            raise OracleError(rc, "write_report")


def ref_available() -> bool:
    return REF_SO.exists()
