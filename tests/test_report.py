"""The output side of the path against the reference itself (oracle/_ref):
RunReport files byte for byte, shortest round-trip number formatting, weighted
quantiles / credible intervals and peak-block sorting (report.cpp,
posterior.cpp).  CPU only."""
import math

import numpy as np
import pytest

from paper_2604_03271_b200 import report as R
from paper_2604_03271_b200.smc import RunReport


def _specials():
    return [0.0, -0.0, 1.0, -1.0, 0.1, 0.5, 1e-5, 1e-4, 1e-3, 123456789.0, 1e15, 1e16, 1e17, 1.5e300, 5e-324,
            2.2250738585072014e-308, 1.7976931348623157e308, 3.141592653589793, 1 / 3, 100.0, 1e21, 1e22, 12345.678,
            0.001234, 9.999999999999999e-05, math.inf, -math.inf, 27.908959116354943, 65536.0, 2000.0]


def test_format_double_matches_to_chars(ref):  # report.cpp:10-14
    rng = np.random.default_rng(0)
    vals = _specials()
    vals += list(rng.normal(size=300) * 10.0 ** rng.integers(-30, 30, size=300))
    vals += list(rng.integers(-10**9, 10**9, size=100).astype(float))
    vals += list(np.round(rng.uniform(0, 1000, size=100), 3))
    for v in vals:
        assert R.format_double(v) == ref.format_double(v), v
        assert R.parse_double(R.format_double(v)) == v or (math.isnan(v))


def test_nan_format(ref):
    assert R.format_double(math.nan) == ref.format_double(math.nan)


def _report(rng, d=5, m=37):
    rep = RunReport(sampler="smc", label="trial_3", F=27.964921243765353, diverged=False, wall_seconds=0.0390005,
                    param_names=[f"p{i}" for i in range(d)])
    rep.scalars = {"T": 4096.0, "n": 8.0, "ess_target": 0.5, "seed": 7.0, "workers": 1.0, "n_data": 301.0,
                   "levels": 11.0}
    rep.arrays = {"ladder": np.concatenate([[0.0], np.sort(rng.uniform(size=10)), [1.0]]),
                  "level_ess_ratio": rng.uniform(size=11), "level_log_mean_w": -rng.exponential(size=11),
                  "level_acc_rate": rng.uniform(size=11), "empty": np.zeros(0)}
    rep.posterior = rng.normal(size=(d, m)) * 3.0
    return rep


@pytest.mark.parametrize("max_draws", [20000, 10, 7, 0])
def test_write_report_is_byte_identical(ref, tmp_path, max_draws):  # report.cpp:33-72
    rng = np.random.default_rng(max_draws)
    rep = _report(rng)
    cfg = ["[smc]", "T = 4096", "seed = 7"]
    ours, theirs = tmp_path / "ours.txt", tmp_path / "ref.txt"
    R.write_report(rep, str(ours), max_draws, cfg)
    ref.write_report(theirs, rep.sampler, rep.label, rep.F, rep.diverged, rep.wall_seconds, rep.scalars,
                     rep.arrays, rep.param_names, rep.posterior, max_draws, cfg)
    assert ours.read_bytes() == theirs.read_bytes()


def test_report_round_trip(tmp_path):  # report.cpp:74-136: bit-exact read back
    rep = _report(np.random.default_rng(5), d=3, m=12)
    p = tmp_path / "r.txt"
    R.write_report(rep, str(p), 0, ["a = 1"])
    back = R.read_report(str(p))
    assert back.F == rep.F and back.wall_seconds == rep.wall_seconds and back.label == rep.label
    assert back.scalars == rep.scalars and back.param_names == rep.param_names
    for k, v in rep.arrays.items():
        assert np.array_equal(back.arrays[k], v)
    assert np.array_equal(back.posterior, rep.posterior) and back.config_lines == ["a = 1"]
    with pytest.raises(RuntimeError):
        bad = tmp_path / "bad.txt"
        bad.write_text("specmc-report 2\n")
        R.read_report(str(bad))


def test_weighted_quantile_matches_reference(ref):  # posterior.cpp:11-57
    rng = np.random.default_rng(1)
    for n in (1, 2, 7, 100, 1000):
        s = rng.normal(size=n)
        s[::5] = s[0]  # ties (stable order)
        w = rng.exponential(size=n)
        w[1::7] = 0.0  # zero-mass atoms
        if not w.sum() > 0:
            w[0] = 1.0
        for q in (0.0, 0.025, 0.1, 0.5, 0.9, 0.975, 1.0, 0.3333):
            assert R.weighted_quantile(s, w, q) == ref.weighted_quantile(s, w, q), (n, q)
    lo, hi = R.credible_interval([1.0, 2.0, 3.0], [1.0, 1.0, 1.0], 0.5)
    assert (lo, hi) == (ref.weighted_quantile([1, 2, 3], [1, 1, 1], 0.25), ref.weighted_quantile([1, 2, 3], [1, 1, 1], 0.75))
    for bad in (([], [], 0.5), ([1.0], [1.0, 2.0], 0.5), ([1.0], [1.0], 1.5), ([1.0], [0.0], 0.5), ([math.nan], [1.0], 0.5)):
        with pytest.raises(ValueError):
            R.weighted_quantile(*bad)


def test_sort_peak_blocks_matches_reference(ref):  # posterior.cpp:106-125
    rng = np.random.default_rng(2)
    post = rng.normal(size=(4 * 3 + 2, 50))
    for b in range(3):
        post[4 * b + 1] += rng.uniform(-5, 5)
    out = R.sort_peak_blocks(post, 4, 1, 3)
    assert np.array_equal(out, ref.sort_peak_blocks(post, 4, 1, 3))
    assert np.all(np.diff([out[4 * b + 1].mean() for b in range(3)]) >= 0)
    with pytest.raises(ValueError):
        R.sort_peak_blocks(post, 4, 4, 3)
