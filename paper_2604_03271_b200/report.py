"""RunReport file format and posterior summaries (the output side of the path).

The on-disk contract of the reference's reports (proj/src/report.cpp:10-136,
proj/include/specmc/report.hpp:12-34): a line-oriented document of scalars,
named arrays, a posterior draw block (downsampled by a deterministic stride to
at most ``max_draws`` columns) and the verbatim config echo.  Numbers use the
shortest round-trip form of ``std::to_chars`` (the shorter of fixed and
scientific, fixed on ties), so a written report reads back bit for bit and a
report written here is byte-identical to the reference's for the same
RunReport (tests/test_report.py checks both against oracle/_ref).

Posterior summaries follow proj/src/posterior.cpp:11-66 (weighted quantiles,
credible intervals) and :106-125 (peak-block sorting by centre); model_select
lives in smc.py.
"""
from __future__ import annotations

import math
from typing import Iterable, List, Sequence, Tuple

import numpy as np

from .smc import RunReport


# ------------------------------------------------------------ number format
def format_double(v: float) -> str:
    """std::to_chars(double) without a format: report.cpp:10-14."""
    v = float(v)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    neg = math.copysign(1.0, v) < 0
    a = -v if neg else v
    if a == 0.0:
        return "-0" if neg else "0"
    # shortest round-trip significand digits and decimal exponent from repr
    r = repr(a)
    if "e" in r:
        mant, ex = r.split("e")
        e10 = int(ex)
    else:
        mant, e10 = r, 0
    if "." in mant:
        ip, fp = mant.split(".")
    else:
        ip, fp = mant, ""
    digits = (ip + fp).lstrip("0")
    # value = 0.<ip fp> * 10^(len(ip) + e10); leading zeros shift the point
    lead = len(ip + fp) - len((ip + fp).lstrip("0"))
    point = len(ip) + e10 - lead  # value = 0.digits * 10^point
    digits = digits.rstrip("0") or "0"
    nd = len(digits)
    # scientific: d.ddd e±XX (at least two exponent digits)
    x = point - 1
    sci = digits[0] + ("." + digits[1:] if nd > 1 else "") + ("e-" if x < 0 else "e+") + f"{abs(x):02d}"
    # fixed
    if point >= nd:  # an integer: printf-style fixed prints its exact digits
        fix = str(int(a))
    elif point > 0:
        fix = digits[:point] + "." + digits[point:]
    else:
        fix = "0." + "0" * (-point) + digits
    s = fix if len(fix) <= len(sci) else sci
    return ("-" if neg else "") + s


def parse_double(s: str) -> float:
    """report.cpp:16-21 (std::from_chars)."""
    try:
        return float(s)
    except ValueError:
        raise RuntimeError("bad number in report: " + s) from None


# ------------------------------------------------------------- write / read
def write_report(r: RunReport, path: str, max_draws: int = 20000, config_lines: Iterable[str] = ()) -> None:
    """report.cpp:33-72: header, sampler, label, diverged, F, wall_seconds, the
    scalars and arrays in key order, param names, the strided posterior block
    (draw per line, d values), then the config echo."""
    fd = format_double
    out: List[str] = ["specmc-report 1", f"sampler {r.sampler}"]
    if r.label:
        out.append(f"label {r.label}")
    out.append(f"diverged {1 if r.diverged else 0}")
    out.append(f"scalar F {fd(r.F)}")
    out.append(f"scalar wall_seconds {fd(r.wall_seconds)}")
    for k in sorted(r.scalars, key=lambda s: s.encode()):
        out.append(f"scalar {k} {fd(r.scalars[k])}")
    if r.param_names:
        out.append("param_names " + " ".join(r.param_names))
    for k in sorted(r.arrays, key=lambda s: s.encode()):
        v = np.asarray(r.arrays[k], dtype=np.float64).ravel()
        out.append(" ".join([f"array {k} {v.size}"] + [fd(x) for x in v]))
    post = r.posterior
    if post is not None:
        post = np.asarray(post, dtype=np.float64)
        d, m = post.shape
        keep, stride = m, 1
        if max_draws > 0 and m > max_draws:
            stride = (m + max_draws - 1) // max_draws
            keep = (m + stride - 1) // stride
        if d > 0 and keep > 0:
            out.append(f"posterior {keep} {d}")
            for j in range(keep):
                col = post[:, j * stride]
                out.append(" ".join(fd(x) for x in col))
    lines = list(config_lines) if config_lines else list(getattr(r, "config_lines", []) or [])
    out.append("config_begin")
    out.extend(lines)
    out.append("config_end")
    with open(path, "w") as f:
        f.write("\n".join(out) + "\n")


def read_report(path: str) -> RunReport:
    """report.cpp:74-136."""
    with open(path) as f:
        lines = f.read().split("\n")
    if not lines or lines[0] != "specmc-report 1":
        raise RuntimeError("not a specmc report: " + path)
    r = RunReport(sampler="", scalars={}, arrays={})
    r.config_lines = []
    i = 1
    n = len(lines)
    while i < n:
        line = lines[i]
        i += 1
        tok = line.split()
        if not tok:
            continue
        tag = tok[0]
        if tag == "sampler":
            r.sampler = tok[1] if len(tok) > 1 else ""
        elif tag == "label":
            r.label = tok[1] if len(tok) > 1 else ""
        elif tag == "diverged":
            r.diverged = int(tok[1]) != 0
        elif tag == "scalar":
            x = parse_double(tok[2])
            if tok[1] == "F":
                r.F = x
            elif tok[1] == "wall_seconds":
                r.wall_seconds = x
            else:
                r.scalars[tok[1]] = x
        elif tag == "param_names":
            r.param_names = tok[1:]
        elif tag == "array":
            k, cnt = tok[1], int(tok[2])
            if len(tok) < 3 + cnt:
                raise RuntimeError("short array in report: " + k)
            r.arrays[k] = np.array([parse_double(t) for t in tok[3:3 + cnt]], dtype=np.float64)
        elif tag == "posterior":
            rows, d = int(tok[1]), int(tok[2])
            post = np.empty((d, rows))
            for j in range(rows):
                if i >= n:
                    raise RuntimeError("short posterior block")
                vals = lines[i].split()
                i += 1
                if len(vals) < d:
                    raise RuntimeError("short posterior row")
                post[:, j] = [parse_double(t) for t in vals[:d]]
            r.posterior = post
        elif tag == "config_begin":
            while i < n and lines[i] != "config_end":
                r.config_lines.append(lines[i])
                i += 1
            i += 1
        else:
            raise RuntimeError("unknown report tag: " + tag)
    return r


# ------------------------------------------------------- posterior summaries
def weighted_quantile(samples: Sequence[float], weights: Sequence[float], q: float) -> float:
    """posterior.cpp:11-57: quantile of the weighted empirical distribution with
    plotting positions p_i = C_{i-1} / (1 - w_last) over the positive-mass
    atoms sorted by value (stable), linear interpolation between them."""
    s = np.asarray(samples, dtype=np.float64).ravel()
    w = np.asarray(weights, dtype=np.float64).ravel()
    n = s.size
    if n == 0:
        raise ValueError("weighted_quantile: empty input")
    if w.size != n:
        raise ValueError("weighted_quantile: size mismatch")
    if not (0.0 <= q <= 1.0):
        raise ValueError("weighted_quantile: q outside [0, 1]")
    total = 0.0
    for i in range(n):
        if not math.isfinite(s[i]):
            raise ValueError("weighted_quantile: non-finite sample")
        if not (w[i] >= 0.0) or not math.isfinite(w[i]):
            raise ValueError("weighted_quantile: bad weight")
        total += float(w[i])
    if not total > 0.0:
        raise ValueError("weighted_quantile: zero total weight")
    idx = [i for i in range(n) if w[i] > 0.0]
    idx.sort(key=lambda i: s[i])  # stable
    m = len(idx)
    if q >= 1.0:
        return float(s[idx[-1]])
    w_last = float(w[idx[-1]]) / total
    denom = 1.0 - w_last
    p = np.empty(m)
    c = 0.0
    for k, i in enumerate(idx):
        p[k] = c / denom if denom > 0.0 else 0.0
        c += float(w[i]) / total
    if q <= p[0]:
        return float(s[idx[0]])
    if q >= p[m - 1]:
        return float(s[idx[m - 1]])
    hi = int(np.searchsorted(p, q, side="right"))
    lo = hi - 1
    t = (q - p[lo]) / (p[hi] - p[lo])
    return float(s[idx[lo]] + t * (s[idx[hi]] - s[idx[lo]]))


def credible_interval(samples, weights, level: float) -> Tuple[float, float]:
    """posterior.cpp:59-66."""
    if not (0.0 < level < 1.0):
        raise ValueError("credible_interval: level outside (0, 1)")
    tail = 0.5 * (1.0 - level)
    return weighted_quantile(samples, weights, tail), weighted_quantile(samples, weights, 1.0 - tail)


def sort_peak_blocks(posterior: np.ndarray, block: int, center_off: int, n_blocks: int) -> np.ndarray:
    """posterior.cpp:106-125: reorder the peak blocks of a d x draws posterior by
    the posterior mean of each block's centre (stable), label-switching aid."""
    post = np.asarray(posterior, dtype=np.float64)
    if block < 1 or center_off < 0 or center_off >= block or n_blocks < 0:
        raise ValueError("sort_peak_blocks: bad block geometry")
    if block * n_blocks > post.shape[0]:
        raise ValueError("sort_peak_blocks: blocks exceed the layout")
    if post.shape[1] == 0 or n_blocks < 2:
        return post.copy()
    # Eigen row mean = sequential sum / size
    means = [float(np.cumsum(post[b * block + center_off])[-1] / post.shape[1]) for b in range(n_blocks)]
    order = sorted(range(n_blocks), key=lambda b: means[b])
    out = post.copy()
    for b, src in enumerate(order):
        out[b * block:(b + 1) * block] = post[src * block:(src + 1) * block]
    return out
