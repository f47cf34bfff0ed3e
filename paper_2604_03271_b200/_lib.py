"""ctypes binding of libspecmc_b200.so (the C ABI in include/specmc_b200.h).

The library is built in-tree by paper_2604_03271_b200/build.py (nvcc,
sm_100a).  There is no CPU fallback: if the shared library is missing the
import fails loudly, and every compute entry point returns SPECMC_ECUDA
when no CUDA device is present.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("SPECMC_LIB", str(PKG / "libspecmc_b200.so")))  # override: tuning experiments

SPECMC_OK, SPECMC_EINVAL, SPECMC_ERUNTIME, SPECMC_ECUDA, SPECMC_ECOMM = 0, 2, 3, 4, 5

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)


class ModelDesc(C.Structure):
    _fields_ = [("family", C.c_int32), ("K", C.c_int32), ("d", C.c_int32), ("noise", C.c_int32),
                ("noise_sigma", C.c_double), ("s0", C.c_double), ("s1", C.c_double), ("s2", C.c_double),
                ("paper_literal", C.c_int32), ("prior_kind", _ip), ("prior_a", _dp), ("prior_b", _dp),
                ("n_refl", C.c_int32), ("refl_phase", _ip), ("refl_mu", _dp), ("refl_int", _dp)]


class SmcConfigC(C.Structure):
    _fields_ = [("T", C.c_int64), ("n", C.c_int32), ("ess_target", C.c_double), ("max_levels", C.c_int32),
                ("seed", C.c_uint64), ("workers", C.c_int32), ("device", C.c_int32)]


class SmcResultC(C.Structure):
    _fields_ = [("status", C.c_int32), ("F", C.c_double), ("diverged", C.c_int32), ("wall_seconds", C.c_double),
                ("device_seconds", C.c_double), ("levels", C.c_int32), ("d", C.c_int32), ("T", C.c_int64),
                ("ladder", _dp), ("level_ess_ratio", _dp), ("level_log_mean_w", _dp), ("level_acc_rate", _dp),
                ("posterior", _dp), ("energies", _dp), ("proposals", C.c_int64), ("trials", C.c_int64)]


class RemcConfigC(C.Structure):
    _fields_ = [("L", C.c_int32), ("ladder", _dp), ("n_ladder", C.c_int32), ("total_sweeps", C.c_int64),
                ("burn_in_fraction", C.c_double), ("swap_period", C.c_int64), ("seed", C.c_uint64),
                ("workers", C.c_int32), ("device", C.c_int32)]


class RemcResultC(C.Structure):
    _fields_ = [("status", C.c_int32), ("F", C.c_double), ("diverged", C.c_int32), ("wall_seconds", C.c_double),
                ("device_seconds", C.c_double), ("R", C.c_int32), ("d", C.c_int32), ("draws", C.c_int64),
                ("ladder", _dp), ("swap_rate", _dp), ("replica_acc", _dp), ("posterior", _dp)]


class ProblemC(C.Structure):
    _fields_ = [("model", ModelDesc), ("spectrum", C.c_int32), ("cfg", SmcConfigC)]


class SpectrumC(C.Structure):
    _fields_ = [("xs", _dp), ("ys", _dp), ("n", C.c_int64)]


class RemcProblemC(C.Structure):
    _fields_ = [("model", ModelDesc), ("spectrum", C.c_int32), ("cfg", RemcConfigC)]


class StatsC(C.Structure):
    _fields_ = [("kernel_launches", C.c_int64), ("move_kernel_ms", C.c_double), ("move_launches", C.c_int64),
                ("point_evals", C.c_double), ("move_mufu_ops", C.c_double)]


# every symbol include/specmc_b200.h declares (tests/test_abi.py checks the header agrees)
EXPORTS = [
    "specmc_smc_run", "specmc_smc_run_batch", "specmc_result_free", "specmc_free", "specmc_energy_batch", "specmc_ess",
    "specmc_log_mean_exp", "specmc_next_beta", "specmc_systematic_resample", "specmc_predict_step_size",
    "specmc_validate_config", "specmc_validate_problem", "specmc_stats_get", "specmc_stats_reset",
    "specmc_launch_shape", "specmc_device_count", "specmc_version", "specmc_session_create", "specmc_session_run",
    "specmc_session_fetch", "specmc_session_destroy", "specmc_probe_mufu", "specmc_smc_run_sharded",
    "specmc_nccl_unique_id", "specmc_comm_init_nccl", "specmc_comm_destroy", "specmc_init_ensemble",
    "specmc_smc_run_sharded_batch", "specmc_smc_run_distributed", "specmc_plan", "specmc_remc_run_batch",
    "specmc_remc_result_free",
]
SPECMC_COMM_ID_BYTES = 128


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a). There is no CPU fallback.")
    lib = C.CDLL(str(LIB_PATH))
    E = C.c_char_p
    Z = C.c_size_t
    lib.specmc_smc_run.argtypes = [C.POINTER(ModelDesc), _dp, _dp, C.c_int64, C.POINTER(SmcConfigC),
                                   C.POINTER(SmcResultC), E, Z]
    lib.specmc_smc_run_batch.argtypes = [C.c_int32, C.POINTER(ProblemC), C.c_int32, C.POINTER(SpectrumC),
                                         C.POINTER(SmcResultC), E, Z]
    lib.specmc_session_create.argtypes = [C.c_int32, C.POINTER(ProblemC), C.c_int32, C.POINTER(SpectrumC),
                                          C.POINTER(C.c_void_p), E, Z]
    lib.specmc_session_run.argtypes = [C.c_void_p, _dp, E, Z]
    lib.specmc_session_fetch.argtypes = [C.c_void_p, C.POINTER(SmcResultC), E, Z]
    lib.specmc_session_destroy.argtypes = [C.c_void_p]
    lib.specmc_session_destroy.restype = None
    lib.specmc_probe_mufu.argtypes = [C.c_int32, _dp, E, Z]
    lib.specmc_init_ensemble.argtypes = [C.POINTER(ModelDesc), _dp, _dp, C.c_int64, C.POINTER(SmcConfigC),
                                         C.POINTER(SmcResultC), E, Z]
    if hasattr(lib, "specmc_smc_run_sharded"):  # (older builds under SPECMC_LIB A/B experiments lack it)
        lib.specmc_smc_run_sharded.argtypes = [C.POINTER(ModelDesc), _dp, _dp, C.c_int64, C.POINTER(SmcConfigC),
                                               C.c_int32, C.c_void_p, C.POINTER(SmcResultC), E, Z]
        lib.specmc_smc_run_sharded_batch.argtypes = [C.c_int32, C.POINTER(ProblemC), C.c_int32,
                                                     C.POINTER(SpectrumC), C.c_int32, C.c_void_p,
                                                     C.POINTER(SmcResultC), E, Z]
        lib.specmc_nccl_unique_id.argtypes = [C.c_char_p, E, Z]
        lib.specmc_comm_init_nccl.argtypes = [C.c_int32, C.c_int32, C.c_char_p, C.c_int32, C.POINTER(C.c_void_p),
                                              E, Z]
        lib.specmc_comm_destroy.argtypes = [C.c_void_p]
        lib.specmc_comm_destroy.restype = None
    if hasattr(lib, "specmc_plan"):
        lib.specmc_smc_run_distributed.argtypes = [C.c_int32, C.POINTER(ProblemC), C.c_int32, C.POINTER(SpectrumC),
                                                   C.c_void_p, _ip, _ip, C.POINTER(SmcResultC), E, Z]
        lib.specmc_plan.argtypes = [C.c_int32, _dp, _lp, _ip, C.c_int32, _ip, _ip, _dp, _dp]
    if hasattr(lib, "specmc_remc_run_batch"):
        lib.specmc_remc_run_batch.argtypes = [C.c_int32, C.POINTER(RemcProblemC), C.c_int32, C.POINTER(SpectrumC),
                                              C.POINTER(RemcResultC), E, Z]
        lib.specmc_remc_result_free.argtypes = [C.POINTER(RemcResultC)]
        lib.specmc_remc_result_free.restype = None
    lib.specmc_result_free.argtypes = [C.POINTER(SmcResultC)]
    lib.specmc_result_free.restype = None
    lib.specmc_free.argtypes = [C.c_void_p]
    lib.specmc_free.restype = None
    lib.specmc_energy_batch.argtypes = [C.POINTER(ModelDesc), _dp, _dp, C.c_int64, _dp, C.c_int64, C.c_int32, _dp,
                                        E, Z]
    lib.specmc_ess.argtypes = [_dp, C.c_int64, C.c_int32, _dp, E, Z]
    lib.specmc_log_mean_exp.argtypes = [_dp, C.c_int64, C.c_int32, _dp, E, Z]
    lib.specmc_next_beta.argtypes = [_dp, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_int32, _dp, E, Z]
    lib.specmc_systematic_resample.argtypes = [_dp, C.c_int64, C.c_int64, C.c_double, C.c_int32, _lp, E, Z]
    lib.specmc_predict_step_size.argtypes = [_dp, _dp, _dp, C.c_int32, C.POINTER(ModelDesc), C.c_double, C.c_int32,
                                             _dp, E, Z]
    lib.specmc_validate_config.argtypes = [C.POINTER(SmcConfigC), E, Z]
    lib.specmc_validate_problem.argtypes = [C.POINTER(ModelDesc), _dp, _dp, C.c_int64, E, Z]
    lib.specmc_stats_get.argtypes = [C.POINTER(StatsC)]
    lib.specmc_stats_reset.argtypes = []
    lib.specmc_stats_reset.restype = None
    lib.specmc_launch_shape.argtypes = [C.c_int64, _ip, _ip, _ip]
    lib.specmc_device_count.argtypes = []
    lib.specmc_version.restype = C.c_char_p
    return lib


lib = _load()
