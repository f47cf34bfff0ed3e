"""The drop-in boundary proven from the reference side.

integration/smc_b200.cpp is the adapter of INTEGRATION.md section 1, written
against the REFERENCE's own types (specmc::ModelSpec / Spectrum / SmcConfig /
RunReport, proj/include) and compiled by integration/build_adapter.py with the
reference headers and sources (Eigen3 -> oracle/eigen_shim).  Its caller
integration/model_select_b200.cpp is a reference-style model selection: the
reference's gen_xps, xps_model, model_select (posterior.cpp:68-104) and
write_report (report.cpp) around the adapter's smc_run_b200 (one run at a
time, the CLI's K x trials loop, specmc_main.cpp:147-170) or
smc_run_batch_b200 (the whole loop as one batched call).
"""
import re
import subprocess
from pathlib import Path

import pytest

import paper_2604_03271_b200 as S

ROOT = Path(__file__).resolve().parent.parent
EXE = ROOT / "oracle" / "_ref" / "model_select_b200"


def _exe():
    if not EXE.exists():
        from integration.build_adapter import build
        if build() is None:
            pytest.skip("adapter not built (needs /root/reference to compile)")
    return EXE


def _run(*args, timeout=600):
    return subprocess.run([str(_exe()), *map(str, args)], capture_output=True, text=True, timeout=timeout)


@pytest.mark.skipif(S.device_count() > 0, reason="CPU-only behaviour")
def test_adapter_without_device_fails_like_the_cli():
    r = _run(3, 5, 2, 4, 1024, 8, 1, "batch")
    assert r.returncode == 3 and "no CUDA device" in r.stderr  # runtime_error -> CLI exit 3


def test_adapter_invalid_config_is_invalid_argument():
    r = _run(3, 5, 2, 4, 1001, 8, 1, "serial")  # T % n != 0 (smc.cpp:23-32)
    assert r.returncode == 2, r.stderr


def _parse(out):
    runs = {(int(m[1]), int(m[2])): float(m[3]) for m in re.finditer(r"run K=(\d+) trial=(\d+) F=(\S+)", out)}
    sel = int(re.search(r"selected K=(\d+)", out)[1])
    return runs, sel


@pytest.mark.gpu
def test_adapter_model_selection_on_gpu(tmp_path):
    rep = tmp_path / "best.report"
    b = _run(3, 5, 1, 5, 4096, 8, 2, "batch", rep)
    s = _run(3, 5, 1, 5, 4096, 8, 2, "serial")
    assert b.returncode == 0 and s.returncode == 0, b.stderr + s.stderr
    rb, kb = _parse(b.stdout)
    rs, ks = _parse(s.stdout)
    assert kb == ks == 3  # gen_xps(k_true = 3) selects K = 3
    assert rb.keys() == rs.keys() and len(rb) == 10
    for k in rb:  # one batched call == the serial drop-in, run for run (same Philox streams)
        assert rb[k] == rs[k]
    r = S.read_report(str(rep))  # the reference's write_report output, read by this repo's reader
    assert r.sampler == "smc" and r.F == rb[(3, 0)] and r.posterior.shape[0] == 4 * 3 + 2
