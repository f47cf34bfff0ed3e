"""The reference CLI's fit / model-select on the B200 backend (SURVEY.md 8f
rank 1): integration/specmc_b200_cli.cpp, built against the reference's own
config, spectrum, posterior and report code (integration/build_adapter.py).
Exit codes as the reference CLI (specmc_main.cpp:17-19): 2 config / usage,
3 numeric or no device."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2604_03271_b200 as S
from paper_2604_03271_b200 import synthetic as syn

ROOT = Path(__file__).resolve().parent.parent
CLI = ROOT / "oracle" / "_ref" / "specmc_b200"


def _cli():
    if not CLI.exists():
        from integration.build_adapter import build
        build()
    if not CLI.exists():
        pytest.skip("CLI not built (needs /root/reference to compile)")
    return CLI


def _files(tmp_path, cfg_text, k_true=3, seed=5):
    sp, _ = syn.gen_xps(k_true, seed)
    data = tmp_path / "spec.csv"
    data.write_text("x,y\n" + "".join(f"{float(a)!r},{float(b)!r}\n" for a, b in zip(sp.xs, sp.ys)))
    cfg = tmp_path / "run.cfg"
    cfg.write_text(cfg_text)
    return cfg, data


def _run(*args):
    return subprocess.run([str(_cli()), *map(str, args)], capture_output=True, text=True, timeout=900)


def test_cli_usage_and_config_errors(tmp_path):
    cfg, data = _files(tmp_path, "family = xps\nK = 3\nsmc.levels = 5\n")  # unknown key
    assert _run("fit", "--config", cfg, "--data", data, "--out", tmp_path / "r").returncode == 2
    assert _run("frobnicate").returncode == 2
    cfg2, _ = _files(tmp_path, "family = xps\nK = 3\n")
    r = _run("model-select", "--config", cfg2, "--data", data, "--k-range", "3..1", "--out", tmp_path / "t")
    assert r.returncode == 2 and "k-range" in r.stderr


@pytest.mark.skipif(S.device_count() > 0, reason="CPU-only behaviour")
def test_cli_without_device_is_numeric_failure(tmp_path):
    cfg, data = _files(tmp_path, "family = xps\nK = 3\nsmc.T = 256\nsmc.n = 8\n")
    r = _run("fit", "--config", cfg, "--data", data, "--out", tmp_path / "r")
    assert r.returncode == 3 and "no CUDA device" in r.stderr


@pytest.mark.gpu
def test_cli_model_select_and_fit_on_gpu(tmp_path):
    cfg, data = _files(tmp_path, "family = xps\nK = 3\nsmc.T = 4096\nsmc.n = 8\nseed = 11\n")
    table = tmp_path / "ms.tsv"
    r = _run("model-select", "--config", cfg, "--data", data, "--k-range", "1..5", "--trials", "2", "--out", table)
    assert r.returncode == 0, r.stderr
    lines = table.read_text().splitlines()
    assert lines[0] == "# model selection over K = 1..5, sampler smc, trials 2"
    assert lines[-1] == "chosen\t3" and "chosen K = 3" in r.stdout
    rows = [l.split("\t") for l in lines if l and l[0].isdigit()]
    assert [int(x[0]) for x in rows] == [1, 2, 3, 4, 5] and all(x[3] == "2" and x[4] == "ok" for x in rows)
    rep = tmp_path / "fit.report"
    r = _run("fit", "--config", cfg, "--data", data, "--out", rep, "--label", "gpu-fit")
    assert r.returncode == 0, r.stderr
    back = S.read_report(str(rep))
    assert back.sampler == "smc" and back.label == "gpu-fit" and np.isfinite(back.F)
    assert back.config_lines[:2] == ["family = xps", "K = 3"]
    mu = back.arrays["post_mean"][[1, 5, 9]]  # peak centres, sorted by the reference's sort_peak_blocks
    assert np.all(np.diff(mu) > 0)
    assert np.all(back.arrays["ci95_lo"] <= back.arrays["ci95_hi"])
