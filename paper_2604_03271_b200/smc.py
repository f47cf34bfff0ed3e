"""SMC entry points mirroring the reference interface, over the C ABI.

Reference (paths relative to the reference root):
  SmcConfig / validate_smc_config   proj/include/specmc/smc.hpp:12-21, proj/src/smc.cpp:23-32
  smc_run(spec, data, cfg)          proj/include/specmc/smc.hpp:78, proj/src/smc.cpp:218-249
  RunReport                         proj/include/specmc/report.hpp:16-27
  model_select                      proj/src/posterior.cpp:68-104
  parity units                      smc.cpp:61-112 (ess, next_beta, systematic_resample),
                                    math.hpp:28-30 (log_mean_exp), mcmc.cpp:20-53
                                    (predict_step_size), energy.cpp:7-55 (energies)

Errors map like the reference: invalid configuration -> ValueError (the
std::invalid_argument analogue, CLI exit 2), numeric failure -> RuntimeError
(std::runtime_error, CLI exit 3); CUDA failures raise CudaError.  Every
compute call runs hand-written sm_100a kernels; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import math
import weakref
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import lib
from .model import ModelSpec, Spectrum


class CudaError(RuntimeError):
    pass


def _raise(rc: int, err: C.Array):
    msg = err.value.decode(errors="replace")
    if rc == _lib.SPECMC_EINVAL:
        raise ValueError(msg)
    if rc == _lib.SPECMC_ERUNTIME:
        raise RuntimeError(msg)
    if rc == _lib.SPECMC_ECUDA:
        raise CudaError(msg)
    raise RuntimeError(f"specmc error {rc}: {msg}")


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return a.ctypes.data_as(_lib._dp)


@dataclass
class SmcConfig:
    """proj/include/specmc/smc.hpp:12-19 (+ the CUDA device ordinal)."""
    T: int = 10000
    n: int = 10
    ess_target: float = 0.5
    max_levels: int = 2000
    seed: int = 0
    workers: int = 1
    device: int = 0

    def c(self):
        return _lib.SmcConfigC(int(self.T), int(self.n), float(self.ess_target), int(self.max_levels),
                               int(self.seed) & 0xFFFFFFFFFFFFFFFF, int(self.workers), int(self.device))


def validate_smc_config(cfg: SmcConfig) -> None:
    """smc.cpp:23-32 (host-side; needs no GPU)."""
    err = C.create_string_buffer(512)
    c = cfg.c()
    rc = lib.specmc_validate_config(C.byref(c), err, 512)
    if rc:
        _raise(rc, err)


@dataclass
class RunReport:
    """proj/include/specmc/report.hpp:16-27, filled as smc.cpp:218-249 does."""
    sampler: str = "smc"
    label: str = ""
    F: float = math.nan
    diverged: bool = False
    wall_seconds: float = 0.0
    param_names: List[str] = field(default_factory=list)
    scalars: Dict[str, float] = field(default_factory=dict)
    arrays: Dict[str, np.ndarray] = field(default_factory=dict)
    posterior: Optional[np.ndarray] = None  # d x T
    energies: Optional[np.ndarray] = None   # T
    device_seconds: float = 0.0
    proposals: int = 0
    trials: int = 0
    config_lines: List[str] = field(default_factory=list)  # report.hpp:26, the config echo


def _report(spec: ModelSpec, cfg: SmcConfig, n_data: int, r: _lib.SmcResultC) -> RunReport:
    L = r.levels
    rep = RunReport(sampler="smc", F=r.F, diverged=bool(r.diverged), wall_seconds=r.wall_seconds,
                    param_names=spec.param_names, device_seconds=r.device_seconds, proposals=r.proposals,
                    trials=r.trials)
    rep.scalars = {"T": float(cfg.T), "n": float(cfg.n), "ess_target": cfg.ess_target, "seed": float(cfg.seed),
                   "workers": float(cfg.workers), "n_data": float(n_data), "levels": float(L)}
    if not r.ladder:  # distributed entry: a run this rank did not hold (scalars only)
        return rep
    rep.arrays = {
        "ladder": np.ctypeslib.as_array(r.ladder, (L + 1,)).copy(),
        "level_ess_ratio": np.ctypeslib.as_array(r.level_ess_ratio, (max(L, 1),))[:L].copy(),
        "level_log_mean_w": np.ctypeslib.as_array(r.level_log_mean_w, (max(L, 1),))[:L].copy(),
        "level_acc_rate": np.ctypeslib.as_array(r.level_acc_rate, (max(L, 1),))[:L].copy(),
    }
    d, T = r.d, r.T
    # the particle-major block is handed over without a copy: the array owns the
    # malloc'd buffer (freed with specmc_free when the last view goes), and the
    # result's field is cleared so specmc_result_free leaves it alone
    ptr = C.cast(r.posterior, C.c_void_p).value
    block = np.ctypeslib.as_array(r.posterior, (T, d))
    weakref.finalize(block, lib.specmc_free, ptr)
    r.posterior = None
    rep.posterior = block.T  # d x T view
    rep.energies = np.ctypeslib.as_array(r.energies, (T,)).copy()
    return rep


def smc_run(spec: ModelSpec, data: Spectrum, cfg: SmcConfig) -> RunReport:
    """RunReport smc_run(const ModelSpec&, const Spectrum&, const SmcConfig&) -- smc.cpp:218."""
    return smc_run_batch([(spec, 0, cfg)], [data])[0]


def _pack(problems, spectra):
    n = len(problems)
    keep = []
    probs = (_lib.ProblemC * n)()
    for i, (spec, si, cfg) in enumerate(problems):
        desc, k = spec.desc()
        keep.append(k)
        probs[i] = _lib.ProblemC(desc, int(si), cfg.c())
    sps = (_lib.SpectrumC * len(spectra))()
    for j, s in enumerate(spectra):
        keep.append(s)
        sps[j] = _lib.SpectrumC(_p(s.xs), _p(s.ys), len(s.xs))
    return probs, sps, keep


def _collect(problems, spectra, res, raise_on_error):
    out = []
    try:
        for i, (spec, si, cfg) in enumerate(problems):
            r = res[i]
            if r.status != _lib.SPECMC_OK:
                e = RuntimeError("smc: max_levels exceeded before reaching beta = 1 (or total weight is zero)")
                if raise_on_error:
                    raise e
                out.append(e)
            else:
                out.append(_report(spec, cfg, len(spectra[si].xs), r))
        return out
    finally:
        for i in range(len(problems)):
            lib.specmc_result_free(C.byref(res[i]))


def smc_run_batch(problems: Sequence[Tuple[ModelSpec, int, SmcConfig]], spectra: Sequence[Spectrum],
                  raise_on_error: bool = True):
    """Runs every (spec, spectrum index, cfg) concurrently on one GPU.

    Returns a list of RunReport (or, with raise_on_error=False, the exception
    instance for runs that failed, e.g. max_levels exceeded)."""
    probs, sps, keep = _pack(problems, spectra)
    res = (_lib.SmcResultC * len(problems))()
    err = C.create_string_buffer(1024)
    rc = lib.specmc_smc_run_batch(len(problems), probs, len(spectra), sps, res, err, 1024)
    if rc and rc != _lib.SPECMC_ERUNTIME:
        for i in range(len(problems)):
            lib.specmc_result_free(C.byref(res[i]))
        _raise(rc, err)
    return _collect(problems, spectra, res, raise_on_error)


class Session:
    """Device-resident batch (specmc_session_*): inputs stay in HBM across runs."""

    def __init__(self, problems, spectra):
        self.problems, self.spectra = list(problems), list(spectra)
        probs, sps, self._keep = _pack(self.problems, self.spectra)
        self._h = C.c_void_p()
        err = C.create_string_buffer(1024)
        rc = lib.specmc_session_create(len(self.problems), probs, len(self.spectra), sps, C.byref(self._h), err, 1024)
        if rc:
            _raise(rc, err)

    def run(self) -> float:
        """Runs every problem from init_ensemble to beta = 1; returns device seconds."""
        ds = C.c_double()
        err = C.create_string_buffer(1024)
        rc = lib.specmc_session_run(self._h, C.byref(ds), err, 1024)
        if rc:
            _raise(rc, err)
        return ds.value

    def fetch(self, raise_on_error: bool = True):
        res = (_lib.SmcResultC * len(self.problems))()
        err = C.create_string_buffer(1024)
        rc = lib.specmc_session_fetch(self._h, res, err, 1024)
        if rc and rc != _lib.SPECMC_ERUNTIME:
            _raise(rc, err)
        return _collect(self.problems, self.spectra, res, raise_on_error)

    def close(self):
        if self._h:
            lib.specmc_session_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def init_ensemble(spec: ModelSpec, data: Spectrum, cfg: SmcConfig):
    """init_ensemble (smc.cpp:34-53) on the device: the level-0 prior draws (d x T)
    and their energies (T), the same streams smc_run starts from."""
    desc, keep = spec.desc()
    res = _lib.SmcResultC()
    err = C.create_string_buffer(1024)
    rc = lib.specmc_init_ensemble(C.byref(desc), _p(data.xs), _p(data.ys), len(data.xs), C.byref(cfg.c()),
                                  C.byref(res), err, 1024)
    try:
        if rc:
            _raise(rc, err)
        d, T = res.d, res.T
        th = np.ctypeslib.as_array(res.posterior, (T, d)).copy().T
        E = np.ctypeslib.as_array(res.energies, (T,)).copy()
        return th, E
    finally:
        lib.specmc_result_free(C.byref(res))


# ------------------------------------------------------- particle sharding
class Comm:
    """NCCL communicator with one shard per rank (specmc_comm_init_nccl).

    ``Comm.from_torch(device)`` bootstraps it over an initialised
    torch.distributed process group (rank 0 creates the id, a broadcast
    shares it)."""

    def __init__(self, rank: int, world: int, uid: bytes, device: int = 0):
        if len(uid) != _lib.SPECMC_COMM_ID_BYTES:
            raise ValueError("comm: unique id must be 128 bytes")
        self.rank, self.world, self.device = rank, world, device
        self._h = C.c_void_p()
        err = C.create_string_buffer(1024)
        rc = lib.specmc_comm_init_nccl(rank, world, uid, device, C.byref(self._h), err, 1024)
        if rc:
            _raise(rc, err)

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(_lib.SPECMC_COMM_ID_BYTES)
        err = C.create_string_buffer(512)
        rc = lib.specmc_nccl_unique_id(buf, err, 512)
        if rc:
            _raise(rc, err)
        return buf.raw

    @classmethod
    def from_torch(cls, device: int = 0) -> "Comm":
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        box = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        return cls(rank, world, box[0], device)

    def close(self):
        if self._h:
            lib.specmc_comm_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def smc_run_sharded(spec: ModelSpec, data: Spectrum, cfg: SmcConfig, n_virtual: int = 1,
                    comm: Optional[Comm] = None) -> RunReport:
    """One run with its particles split over shards.

    comm=None: ``n_virtual`` shards in this process on cfg.device (the
    exchanges are device kernels); the report holds every particle.  With a
    Comm: this rank's shard; F and the level diagnostics are global, the
    posterior holds this rank's particles."""
    desc, keep = spec.desc()
    res = _lib.SmcResultC()
    err = C.create_string_buffer(1024)
    rc = lib.specmc_smc_run_sharded(C.byref(desc), _p(data.xs), _p(data.ys), len(data.xs), C.byref(cfg.c()),
                                    int(n_virtual), comm._h if comm is not None else None, C.byref(res), err, 1024)
    try:
        if rc:
            _raise(rc, err)
        return _report(spec, cfg, len(data.xs), res)
    finally:
        lib.specmc_result_free(C.byref(res))


def smc_run_sharded_batch(problems: Sequence[Tuple[ModelSpec, int, SmcConfig]], spectra: Sequence[Spectrum],
                          n_virtual: int = 1, comm: Optional[Comm] = None, raise_on_error: bool = True):
    """Every (spec, spectrum index, cfg) split over the same shards, all at once
    (e.g. the K range of a model selection); see smc_run_sharded."""
    probs, sps, keep = _pack(problems, spectra)
    res = (_lib.SmcResultC * len(problems))()
    err = C.create_string_buffer(1024)
    rc = lib.specmc_smc_run_sharded_batch(len(problems), probs, len(spectra), sps, int(n_virtual),
                                          comm._h if comm is not None else None, res, err, 1024)
    if rc and rc != _lib.SPECMC_ERUNTIME:
        for i in range(len(problems)):
            lib.specmc_result_free(C.byref(res[i]))
        _raise(rc, err)
    return _collect(problems, spectra, res, raise_on_error)


def plan(costs, T, n, world: int):
    """specmc_plan: placement of runs on `world` ranks -> (rank0, shards, rank_load, makespan)."""
    costs = _d(costs)
    m = len(costs)
    Ta = np.ascontiguousarray(T, dtype=np.int64) if np.ndim(T) else np.full(m, T, dtype=np.int64)
    na = np.ascontiguousarray(n, dtype=np.int32) if np.ndim(n) else np.full(m, n, dtype=np.int32)
    r0 = np.empty(m, dtype=np.int32)
    sh = np.empty(m, dtype=np.int32)
    load = np.empty(world)
    mk = C.c_double()
    rc = lib.specmc_plan(m, _p(costs), Ta.ctypes.data_as(_lib._lp), na.ctypes.data_as(_lib._ip), int(world),
                         r0.ctypes.data_as(_lib._ip), sh.ctypes.data_as(_lib._ip), _p(load), C.byref(mk))
    if rc:
        raise ValueError("plan: invalid arguments")
    return r0, sh, load, mk.value


def smc_run_distributed(problems: Sequence[Tuple[ModelSpec, int, SmcConfig]], spectra: Sequence[Spectrum],
                        comm: "Comm", raise_on_error: bool = True):
    """Every problem of the batch placed on the ranks of ``comm`` (specmc_smc_run_distributed):
    returns (reports, rank0, shards).  Every report carries F / levels / trials; posterior
    and diagnostics only where this rank ran (part of) the run."""
    probs, sps, keep = _pack(problems, spectra)
    m = len(problems)
    res = (_lib.SmcResultC * m)()
    r0 = np.empty(m, dtype=np.int32)
    sh = np.empty(m, dtype=np.int32)
    err = C.create_string_buffer(1024)
    rc = lib.specmc_smc_run_distributed(m, probs, len(spectra), sps, comm._h, r0.ctypes.data_as(_lib._ip),
                                        sh.ctypes.data_as(_lib._ip), res, err, 1024)
    if rc and rc != _lib.SPECMC_ERUNTIME:
        for i in range(m):
            lib.specmc_result_free(C.byref(res[i]))
        _raise(rc, err)
    return _collect(problems, spectra, res, raise_on_error), r0, sh


# ------------------------------------------------- replica exchange (REMC)
@dataclass
class RemcConfig:
    """proj/include/specmc/remc.hpp:14-22 (+ the CUDA device ordinal)."""
    L: int = 44
    ladder: Optional[Sequence[float]] = None
    total_sweeps: int = 10000
    burn_in_fraction: float = 0.5
    swap_period: int = 1
    seed: int = 0
    workers: int = 1
    device: int = 0

    def c(self):
        lad = None if self.ladder is None else _d(self.ladder)
        cc = _lib.RemcConfigC(int(self.L), _p(lad) if lad is not None else None, 0 if lad is None else len(lad),
                              int(self.total_sweeps), float(self.burn_in_fraction), int(self.swap_period),
                              int(self.seed) & 0xFFFFFFFFFFFFFFFF, int(self.workers), int(self.device))
        return cc, lad


def remc_run_batch(problems: Sequence[Tuple[ModelSpec, int, RemcConfig]], spectra: Sequence[Spectrum],
                   raise_on_error: bool = True):
    """Every (spec, spectrum index, RemcConfig) concurrently on one GPU
    (specmc_remc_run_batch): RunReports as remc_run(spec, data, cfg) fills them
    (remc.cpp:170-190): sampler 'remc', scalars L / total_sweeps /
    burn_in_fraction / swap_period / seed / workers / n_data, arrays ladder /
    swap_rate / replica_acc_rate, the beta = 1 draws as posterior (d x draws)."""
    n = len(problems)
    probs = (_lib.RemcProblemC * n)()
    keep = []
    for i, (spec, si, cfg) in enumerate(problems):
        desc, k = spec.desc()
        cc, lad = cfg.c()
        keep += [k, lad]
        probs[i] = _lib.RemcProblemC(desc, int(si), cc)
    sps = (_lib.SpectrumC * len(spectra))()
    for j, sp in enumerate(spectra):
        sps[j] = _lib.SpectrumC(_p(sp.xs), _p(sp.ys), len(sp.xs))
    res = (_lib.RemcResultC * n)()
    err = C.create_string_buffer(1024)
    rc = lib.specmc_remc_run_batch(n, probs, len(spectra), sps, res, err, 1024)
    try:
        if rc:
            _raise(rc, err)
        out = []
        for i, (spec, si, cfg) in enumerate(problems):
            r = res[i]
            rep = RunReport(sampler="remc", F=r.F, diverged=bool(r.diverged), wall_seconds=r.wall_seconds,
                            param_names=spec.param_names, device_seconds=r.device_seconds)
            R = r.R
            rep.scalars = {"L": float(R - 1), "total_sweeps": float(cfg.total_sweeps),
                           "burn_in_fraction": float(cfg.burn_in_fraction), "swap_period": float(cfg.swap_period),
                           "seed": float(cfg.seed), "workers": float(cfg.workers),
                           "n_data": float(len(spectra[si].xs))}
            rep.arrays = {"ladder": np.ctypeslib.as_array(r.ladder, (R,)).copy(),
                          "swap_rate": np.ctypeslib.as_array(r.swap_rate, (max(R - 1, 1),))[:R - 1].copy(),
                          "replica_acc_rate": np.ctypeslib.as_array(r.replica_acc, (R,)).copy()}
            rep.posterior = np.ctypeslib.as_array(r.posterior, (int(r.draws), r.d)).copy().T
            out.append(rep)
        return out
    finally:
        for i in range(n):
            lib.specmc_remc_result_free(C.byref(res[i]))


def remc_run(spec: ModelSpec, data: Spectrum, cfg: RemcConfig) -> RunReport:
    """RunReport remc_run(const ModelSpec&, const Spectrum&, const RemcConfig&) -- remc.cpp:170-190."""
    return remc_run_batch([(spec, 0, cfg)], [data])[0]


def probe_mufu(device: int = 0) -> float:
    """Measured MUFU ex2 throughput (ops/s) of the device."""
    v = C.c_double()
    err = C.create_string_buffer(512)
    rc = lib.specmc_probe_mufu(device, C.byref(v), err, 512)
    if rc:
        _raise(rc, err)
    return v.value


# ---------------------------------------------------------------- parity units
def energies(spec: ModelSpec, data: Spectrum, thetas, device: int = 0) -> np.ndarray:
    """Batched BlockEvaluator::full + data_energy (energy.cpp:7-55) on the device (K2)."""
    th = _d(np.atleast_2d(thetas))
    if th.shape[1] != spec.d:
        raise ValueError("theta length mismatch")
    desc, keep = spec.desc()
    out = np.empty(th.shape[0])
    err = C.create_string_buffer(512)
    rc = lib.specmc_energy_batch(C.byref(desc), _p(data.xs), _p(data.ys), len(data.xs), _p(th), th.shape[0],
                                 device, _p(out), err, 512)
    if rc:
        _raise(rc, err)
    return out


def energy(spec: ModelSpec, theta, data: Spectrum, device: int = 0) -> float:
    """double energy(spec, theta, data) -- energy.cpp:130-132"""
    return float(energies(spec, data, np.atleast_2d(theta), device)[0])


def ess(log_weights, device: int = 0) -> float:
    lw = _d(log_weights)
    out = C.c_double()
    err = C.create_string_buffer(512)
    rc = lib.specmc_ess(_p(lw), len(lw), device, C.byref(out), err, 512)
    if rc:
        _raise(rc, err)
    return out.value


def log_mean_exp(v, device: int = 0) -> float:
    v = _d(v)
    out = C.c_double()
    err = C.create_string_buffer(512)
    rc = lib.specmc_log_mean_exp(_p(v), len(v), device, C.byref(out), err, 512)
    if rc:
        _raise(rc, err)
    return out.value


def next_beta(energies_, n_data: float, beta_prev: float, ess_target: float, device: int = 0) -> float:
    E = _d(energies_)
    out = C.c_double()
    err = C.create_string_buffer(512)
    rc = lib.specmc_next_beta(_p(E), len(E), n_data, beta_prev, ess_target, device, C.byref(out), err, 512)
    if rc:
        _raise(rc, err)
    return out.value


def systematic_resample(log_weights, S: int, u: float, device: int = 0) -> np.ndarray:
    lw = _d(log_weights)
    out = np.empty(S, dtype=np.int64)
    err = C.create_string_buffer(512)
    rc = lib.specmc_systematic_resample(_p(lw), len(lw), S, u, device, out.ctypes.data_as(_lib._lp), err, 512)
    if rc:
        _raise(rc, err)
    return out


def predict_step_size(hist_beta, hist_acc, hist_step, beta_next: float, spec: ModelSpec,
                      device: int = 0) -> np.ndarray:
    hb, ha, hs = _d(hist_beta), _d(hist_acc), _d(hist_step)
    desc, keep = spec.desc()
    out = np.empty(spec.d)
    err = C.create_string_buffer(512)
    rc = lib.specmc_predict_step_size(_p(hb), _p(ha), _p(hs), len(hb), C.byref(desc), beta_next, device, _p(out),
                                      err, 512)
    if rc:
        _raise(rc, err)
    return out


# ------------------------------------------------------------ model selection
@dataclass
class ModelChoiceRow:
    K: int
    F: float = math.nan
    trial_std: float = math.nan
    trials: int = 0
    excluded: bool = False


@dataclass
class ModelChoice:
    K_best: int = 0
    table: List[ModelChoiceRow] = field(default_factory=list)


def model_select(reports: Sequence[Tuple[int, RunReport]]) -> ModelChoice:
    """posterior.cpp:68-104: argmin of mean F per K; non-finite/diverged K
    excluded; ties keep the smaller K; RuntimeError if every K is excluded."""
    if not reports:
        raise ValueError("model_select: no reports")
    by_k: Dict[int, List[float]] = {}
    bad = set()
    for k, rep in reports:
        by_k.setdefault(k, []).append(rep.F)
        if not math.isfinite(rep.F) or rep.diverged:
            bad.add(k)
    out = ModelChoice()
    best = None
    for k in sorted(by_k):
        fs = by_k[k]
        row = ModelChoiceRow(K=k, trials=len(fs), excluded=k in bad)
        if not row.excluded:
            mean = sum(fs) / len(fs)
            row.F = mean
            if len(fs) > 1:
                row.trial_std = math.sqrt(sum((f - mean) ** 2 for f in fs) / (len(fs) - 1))
            if best is None or mean < best:
                best = mean
                out.K_best = k
        out.table.append(row)
    if best is None:
        raise RuntimeError("model_select: every candidate diverged")
    return out


def stats():
    s = _lib.StatsC()
    lib.specmc_stats_get(C.byref(s))
    return {"kernel_launches": s.kernel_launches, "move_kernel_ms": s.move_kernel_ms,
            "move_launches": s.move_launches, "point_evals": s.point_evals, "move_mufu_ops": s.move_mufu_ops}


def stats_reset():
    lib.specmc_stats_reset()


def launch_shape(n_points: int):
    W, P, U = C.c_int32(), C.c_int32(), C.c_int32()
    lib.specmc_launch_shape(n_points, C.byref(W), C.byref(P), C.byref(U))
    return W.value, P.value, U.value


def device_count() -> int:
    return lib.specmc_device_count()
