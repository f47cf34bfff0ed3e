"""C ABI checks that need no GPU: the library loads, exports every symbol
include/specmc_b200.h declares, validates like the reference (error codes
2 = invalid_argument) and reports a missing device as a CUDA error instead of
falling back to the CPU."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2604_03271_b200 as S
from paper_2604_03271_b200 import _lib
from paper_2604_03271_b200 import synthetic as syn

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    txt = (ROOT / "include" / "specmc_b200.h").read_text()
    return sorted(set(re.findall(r"\b(specmc_[a-z_]+)\s*\(", txt)))


def test_header_declares_exactly_the_bound_exports():
    assert _declared() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    syms = {l.split()[-1] for l in out.splitlines() if l.strip()}
    for name in _declared():
        assert name in syms, name
        assert hasattr(_lib.lib, name)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("kw,msg", [
    (dict(T=1), "T must be >= 2"), (dict(T=1001, n=10), "divisible"), (dict(T=10, n=10), "S = T/n"),
    (dict(ess_target=1.0), "ess_target"), (dict(ess_target=0.0), "ess_target"), (dict(max_levels=0), "max_levels"),
    (dict(workers=-1), "workers")])
def test_config_validation(kw, msg):  # proj/tests/test_smc.cpp:11-36
    S.validate_smc_config(S.SmcConfig())
    with pytest.raises(ValueError, match=msg):
        S.validate_smc_config(S.SmcConfig(**kw))


def test_problem_validation_without_device():
    sp, _ = syn.gen_xps(2, 1)
    spec = S.xps_model(2, sp)
    desc, keep = spec.desc()
    err = C.create_string_buffer(256)
    xs, ys = sp.xs.copy(), sp.ys.copy()
    dp = _lib._dp
    assert _lib.lib.specmc_validate_problem(C.byref(desc), xs.ctypes.data_as(dp), ys.ctypes.data_as(dp), len(xs), err,
                                            256) == 0
    xs[5] = xs[4]
    assert _lib.lib.specmc_validate_problem(C.byref(desc), xs.ctypes.data_as(dp), ys.ctypes.data_as(dp), len(xs), err,
                                            256) == 2
    assert b"strictly increasing" in err.value
    desc.d = 7
    assert _lib.lib.specmc_validate_problem(C.byref(desc), sp.xs.ctypes.data_as(dp), sp.ys.ctypes.data_as(dp),
                                            len(xs), err, 256) == 2


def test_invalid_config_is_reported_before_touching_the_device():
    sp, _ = syn.gen_xps(1, 1)
    with pytest.raises(ValueError):
        S.smc_run(S.xps_model(1, sp), sp, S.SmcConfig(T=1001, n=10))


def test_launch_shapes_cover_the_configs():
    for n, (W, P) in {301: (1, 10), 840: (1, 28), 2000: (2, 32), 4096: (4, 32), 8192: (8, 32), 50: (1, 2)}.items():
        w, p, u = S.launch_shape(n)
        assert (w, p) == (W, P) and 32 * w * p >= n and u >= 1


@pytest.mark.skipif(S.device_count() > 0, reason="needs a machine without a GPU")
def test_no_device_fails_loudly():
    sp, _ = syn.gen_xps(1, 1)
    with pytest.raises(S.CudaError, match="no CUDA device"):
        S.smc_run(S.xps_model(1, sp), sp, S.SmcConfig(T=100, n=5))
    with pytest.raises(S.CudaError):
        S.ess(np.zeros(4))
