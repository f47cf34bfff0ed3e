"""Benchmark harness on the B200 backend.

The reference's harness (proj/src/bench.cpp, proj/include/specmc/bench.hpp)
runs a grid of sampler conditions x trials with seeds trial_seed(base, t)
(bench.cpp:104-106), tabulates F mean/std, the |F - F_ref| error against the
reference condition (the largest-T SMC condition unless named), timings, and
the matched-error speedup by log-log interpolation of the SMC error-time curve
(:47-63, :135-249); ci_error_curve scores credible-interval endpoints against
a reference report (:251-311).  Here the SMC conditions run on the GPU:

* ``benchmark(spec, data, grid, trials, base_seed, ...)``: every condition x
  trial through the C ABI.  ``batched=False`` (default) runs them one call
  at a time, so each run's ``wall_seconds`` is its own (timings comparable);
  ``batched=True`` runs the whole grid as ONE specmc_smc_run_batch call and,
  like the reference's parallel_trials, marks the timings non-comparable.
* ``table_from_reports`` / ``ci_error_curve`` / ``bench_table_text`` /
  ``ci_table_text`` / ``time_at_error`` / ``median_of`` restate the
  reference's table arithmetic and text format (checked byte for byte against
  the reference build in tests/test_harness.py), so tables regenerated from
  persisted reports (report.py) match the reference's.
REMC conditions (the paper's comparator, remc.cpp) run on the GPU as well
(smc.remc_run: one chain unit per replica), so the matched-|dF| speedup of
SMC over REMC (bench.cpp:227-247) is measured on one device.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import synthetic
from .report import credible_interval, format_double
from .smc import RemcConfig, RunReport, SmcConfig, remc_run, remc_run_batch, smc_run, smc_run_batch

NAN = float("nan")


@dataclass
class BenchCondition:
    """bench.hpp:9-14"""
    label: str
    sampler: str = "smc"
    smc: SmcConfig = field(default_factory=SmcConfig)
    remc: RemcConfig = field(default_factory=RemcConfig)


@dataclass
class BenchRow:
    label: str = ""
    sampler: str = ""
    trials: int = 0
    divergent: int = 0
    f_mean: float = NAN
    f_std: float = 0.0
    time_mean: float = NAN
    time_std: float = 0.0
    df_mean: float = NAN
    df_median: float = NAN


@dataclass
class BenchTable:
    reference_label: str = ""
    f_ref: float = NAN
    speedup: float = NAN
    timings_comparable: bool = True
    rows: List[BenchRow] = field(default_factory=list)


@dataclass
class BenchResult:
    table: BenchTable
    runs: List[RunReport]


@dataclass
class CiErrRow:
    label: str = ""
    trials: int = 0
    divergent: int = 0
    time_mean: float = NAN
    time_std: float = 0.0
    err_mean: float = NAN
    err_std: float = 0.0
    err_median: float = NAN


def trial_seed(base: int, trial: int) -> int:
    """bench.cpp:104-106"""
    return synthetic.trial_seed(base, trial)


def _mean(v):
    if not v:
        return NAN
    s = 0.0
    for x in v:
        s += x
    return s / float(len(v))


def _std(v, mean):
    if len(v) < 2:
        return 0.0
    ss = 0.0
    for x in v:
        ss += (x - mean) * (x - mean)
    return math.sqrt(ss / float(len(v) - 1))


def median_of(v) -> float:
    """bench.cpp:108-113 (empty input gives NaN)."""
    v = sorted(v)
    n = len(v)
    if n == 0:
        return NAN
    return v[n // 2] if n % 2 == 1 else 0.5 * (v[n // 2 - 1] + v[n // 2])


def time_at_error(pts: Sequence[Tuple[float, float]], err: float) -> float:
    """bench.cpp:47-63: log-log interpolation of time at the target error,
    clamped to the curve's ends; points without positive finite coordinates dropped."""
    p = sorted((e, t) for e, t in pts if e > 0.0 and t > 0.0 and math.isfinite(e) and math.isfinite(t))
    if not p:
        return NAN
    if not (err > 0.0) or err <= p[0][0]:
        return p[0][1]
    if err >= p[-1][0]:
        return p[-1][1]
    i = 1
    while p[i][0] < err:
        i += 1
    e0, e1 = math.log(p[i - 1][0]), math.log(p[i][0])
    t0, t1 = math.log(p[i - 1][1]), math.log(p[i][1])
    if e1 == e0:
        return p[i][1]
    w = (math.log(err) - e0) / (e1 - e0)
    return math.exp(t0 + w * (t1 - t0))


def _report_of(spec, cond: BenchCondition, seed: int, rep: RunReport, trial: int, parallel: bool) -> RunReport:
    """run_once (bench.cpp:65-100) fields of a condition's run."""
    r = RunReport(sampler=cond.sampler, label=cond.label, F=rep.F, diverged=rep.diverged,
                  wall_seconds=rep.wall_seconds, param_names=list(spec.param_names), posterior=rep.posterior,
                  energies=rep.energies, device_seconds=rep.device_seconds, proposals=rep.proposals,
                  trials=rep.trials)
    if cond.sampler == "smc":
        r.scalars = {"T": float(cond.smc.T), "n": float(cond.smc.n)}
    else:
        r.scalars = {"L": rep.scalars.get("L", float(cond.remc.L)), "total_sweeps": float(cond.remc.total_sweeps)}
    r.scalars.update({"seed": float(seed), "trial": float(trial), "parallel_trials": 1.0 if parallel else 0.0})
    return r


def _cfg_with_seed(cond: BenchCondition, seed: int):
    if cond.sampler == "smc":
        c = cond.smc
        return SmcConfig(T=c.T, n=c.n, ess_target=c.ess_target, max_levels=c.max_levels, seed=seed,
                         workers=c.workers, device=c.device)
    c = cond.remc
    return RemcConfig(L=c.L, ladder=c.ladder, total_sweeps=c.total_sweeps, burn_in_fraction=c.burn_in_fraction,
                      swap_period=c.swap_period, seed=seed, workers=c.workers, device=c.device)


def benchmark(spec, data, grid: Sequence[BenchCondition], trials: int, base_seed: int,
              reference_label: str = "", batched: bool = False) -> BenchResult:
    """bench.cpp:115-145 on the GPU: runs are condition-major, then trial order."""
    if trials < 2:
        raise ValueError("benchmark: trials must be >= 2")
    if not grid:
        raise ValueError("benchmark: empty condition grid")
    for c in grid:
        if c.sampler not in ("smc", "remc"):
            raise ValueError(f"benchmark: unknown sampler '{c.sampler}' (expected smc|remc)")
    jobs = [(c, t, trial_seed(base_seed, t)) for c in grid for t in range(trials)]
    reps: List[RunReport] = [None] * len(jobs)
    if batched:  # one call per sampler for the whole grid (the reference's parallel_trials analogue)
        for sampler, call in (("smc", smc_run_batch), ("remc", remc_run_batch)):
            sel = [i for i, (c, _, _) in enumerate(jobs) if c.sampler == sampler]
            if not sel:
                continue
            out = call([(spec, 0, _cfg_with_seed(jobs[i][0], jobs[i][2])) for i in sel], [data],
                       **({"raise_on_error": False} if sampler == "smc" else {}))
            for i, rep in zip(sel, out):
                reps[i] = rep
    else:
        for i, (c, t, seed) in enumerate(jobs):
            try:
                reps[i] = (smc_run if c.sampler == "smc" else remc_run)(spec, data, _cfg_with_seed(c, seed))
            except RuntimeError:
                reps[i] = None
    runs = []
    for (c, t, seed), rep in zip(jobs, reps):
        if rep is None or isinstance(rep, Exception):
            rep = RunReport(F=NAN, diverged=True)
        runs.append(_report_of(spec, c, seed, rep, t, batched))
    return BenchResult(table_from_reports(runs, reference_label), runs)


def table_from_reports(runs: Sequence[RunReport], reference_label: str = "") -> BenchTable:
    """bench.cpp:147-249 (the table, rebuilt from persisted reports)."""
    if not runs:
        raise ValueError("table_from_reports: no runs")
    order: List[str] = []
    groups: Dict[str, dict] = {}
    parallel_seen = False
    for r in runs:
        g = groups.get(r.label)
        if g is None:
            order.append(r.label)
            g = groups[r.label] = dict(sampler=r.sampler, total=0, divergent=0, fs=[], times=[], smc_T=-math.inf,
                                       remc_sweeps=-math.inf)
        if g["sampler"] != r.sampler:
            raise ValueError("table_from_reports: mixed samplers under label " + r.label)
        g["total"] += 1
        if r.diverged or not math.isfinite(r.F):
            g["divergent"] += 1
        else:
            g["fs"].append(r.F)
            g["times"].append(r.wall_seconds)
        if r.sampler == "smc":
            g["smc_T"] = max(g["smc_T"], r.scalars.get("T", -math.inf))
        if r.sampler == "remc":
            g["remc_sweeps"] = max(g["remc_sweeps"], r.scalars.get("total_sweeps", -math.inf))
        if r.scalars.get("parallel_trials", 0.0) != 0.0:
            parallel_seen = True
    t = BenchTable(timings_comparable=not parallel_seen)
    if not reference_label:
        best = -math.inf
        for label in order:
            g = groups[label]
            if g["sampler"] == "smc" and g["smc_T"] > best:
                best = g["smc_T"]
                t.reference_label = label
        if not t.reference_label:
            raise ValueError("table_from_reports: no SMC condition for the auto reference")
    else:
        if reference_label not in groups:
            raise ValueError("table_from_reports: unknown reference label " + reference_label)
        t.reference_label = reference_label
    ref = groups[t.reference_label]
    if not ref["fs"]:
        raise RuntimeError("table_from_reports: every reference trial diverged")
    t.f_ref = _mean(ref["fs"])
    for label in order:
        g = groups[label]
        row = BenchRow(label=label, sampler=g["sampler"], trials=g["total"], divergent=g["divergent"])
        if g["fs"]:
            row.f_mean = _mean(g["fs"])
            row.f_std = _std(g["fs"], row.f_mean)
            row.time_mean = _mean(g["times"])
            row.time_std = _std(g["times"], row.time_mean)
            dfs = [abs(f - t.f_ref) for f in g["fs"]]
            row.df_mean = _mean(dfs)
            row.df_median = median_of(dfs)
        t.rows.append(row)
    remc_big, best_sweeps = None, -math.inf
    for row in t.rows:
        if row.sampler != "remc":
            continue
        sw = groups[row.label]["remc_sweeps"]
        if sw > best_sweeps:
            best_sweeps, remc_big = sw, row
    if remc_big is not None and math.isfinite(remc_big.df_mean) and math.isfinite(remc_big.time_mean):
        curve = [(row.df_mean, row.time_mean) for row in t.rows if row.sampler == "smc"]
        t_smc = time_at_error(curve, remc_big.df_mean)
        if math.isfinite(t_smc) and t_smc > 0.0:
            t.speedup = remc_big.time_mean / t_smc
    return t


def _match_rows(names: Sequence[str], param: str) -> List[int]:
    out = []
    for i, n in enumerate(names):
        if n == param or (len(n) > len(param) and n.startswith(param) and n[len(param):].isdigit()):
            out.append(i)
    return out


def ci_error_curve(runs: Sequence[RunReport], truth_ref: RunReport, param: str, level: float = 0.95) -> List[CiErrRow]:
    """bench.cpp:251-311: per condition, the equal-tailed interval endpoint error
    of `param` (a bare stem averages every '<stem><digits>' component)."""
    ref_rows = _match_rows(truth_ref.param_names, param)
    if not ref_rows:
        raise ValueError(f"ci_error_curve: unknown parameter '{param}'")
    if truth_ref.posterior is None or truth_ref.posterior.shape[1] == 0:
        raise ValueError("ci_error_curve: reference report has no posterior draws")
    w_ref = np.ones(truth_ref.posterior.shape[1])
    ref_ci = [credible_interval(truth_ref.posterior[r], w_ref, level) for r in ref_rows]
    order: List[str] = []
    rows: Dict[str, CiErrRow] = {}
    errs: Dict[str, List[float]] = {}
    times: Dict[str, List[float]] = {}
    for run in runs:
        row = rows.get(run.label)
        if row is None:
            order.append(run.label)
            row = rows[run.label] = CiErrRow(label=run.label)
        row.trials += 1
        if run.diverged or not math.isfinite(run.F) or run.posterior is None or run.posterior.shape[1] == 0:
            row.divergent += 1
            continue
        run_rows = _match_rows(run.param_names, param)
        if len(run_rows) != len(ref_rows):
            raise ValueError("ci_error_curve: parameter set differs from the reference")
        w = np.ones(run.posterior.shape[1])
        err = 0.0
        for m, r in enumerate(run_rows):
            lo, hi = credible_interval(run.posterior[r], w, level)
            err += abs(lo - ref_ci[m][0]) + abs(hi - ref_ci[m][1])
        errs.setdefault(run.label, []).append(err / float(len(run_rows)))
        times.setdefault(run.label, []).append(run.wall_seconds)
    out = []
    for label in order:
        row = rows[label]
        e, t = errs.get(label, []), times.get(label, [])
        if e:
            row.err_mean = _mean(e)
            row.err_std = _std(e, row.err_mean)
            row.err_median = median_of(e)
            row.time_mean = _mean(t)
            row.time_std = _std(t, row.time_mean)
        out.append(row)
    return out


def bench_table_text(t: BenchTable) -> str:
    """bench.cpp:313-327"""
    fd = format_double
    s = f"# reference {t.reference_label} F_ref {fd(t.f_ref)} speedup {fd(t.speedup)}\n"
    if not t.timings_comparable:
        s += "# timings non-comparable (parallel trials)\n"
    s += "label\tsampler\ttrials\tdivergent\tF_mean\tF_std\tdF_mean\tdF_median\ttime_mean\ttime_std\n"
    for r in t.rows:
        s += (f"{r.label}\t{r.sampler}\t{r.trials}\t{r.divergent}\t{fd(r.f_mean)}\t{fd(r.f_std)}\t{fd(r.df_mean)}\t"
              f"{fd(r.df_median)}\t{fd(r.time_mean)}\t{fd(r.time_std)}\n")
    return s


def ci_table_text(rows: Sequence[CiErrRow]) -> str:
    """bench.cpp:329-338"""
    fd = format_double
    s = "condition\ttrials\tdivergent\ttime_mean\ttime_std\terr_mean\terr_std\terr_median\n"
    for r in rows:
        s += (f"{r.label}\t{r.trials}\t{r.divergent}\t{fd(r.time_mean)}\t{fd(r.time_std)}\t{fd(r.err_mean)}\t"
              f"{fd(r.err_std)}\t{fd(r.err_median)}\n")
    return s
