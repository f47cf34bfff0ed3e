"""Multi-GPU host logic (torch.distributed; NCCL on the GPU box, gloo in tests).

Two sharding levels of SURVEY.md 8e:

* Trials / K groups / spectra are independent SMC runs: each rank runs its own
  share and only the final F values are exchanged (``gather_selection``), for
  ``model_select`` over every trial (posterior.cpp:68-104).
* Particles of one large run (C3/C5) shard by chain; a level then needs the
  global ESS/evidence normalisers (``allreduce_weight_stats``) and the
  exclusive scan of per-rank weight totals that places each rank's slice of
  the global systematic-resampling comb (``global_resample_range``,
  smc.cpp:95-112 over the concatenated per-rank CDFs).
"""
from __future__ import annotations

import math
from typing import List, Sequence, Tuple

import torch
import torch.distributed as dist

from .smc import RunReport, model_select


def _dev(group=None):
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device(
        "cpu")


def reduce_timing(elapsed: float, evals: float, group=None) -> Tuple[float, float]:
    """Max over ranks of the device time, sum of the work (bench.py contract)."""
    d = _dev(group)
    t = torch.tensor([elapsed], dtype=torch.float64, device=d)
    e = torch.tensor([evals], dtype=torch.float64, device=d)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(e, op=dist.ReduceOp.SUM, group=group)
    return float(t.item()), float(e.item())


def gather_selection(ks: Sequence[int], Fs: Sequence[float], group=None):
    """All-gather every rank's F per K and run model_select over all trials.

    Returns (K_best or None, table of (K, mean F, trials))."""
    d = _dev(group)
    ws = dist.get_world_size(group)
    local = torch.tensor([float(f) for f in Fs], dtype=torch.float64, device=d)
    out = [torch.empty_like(local) for _ in range(ws)]
    dist.all_gather(out, local, group=group)
    rows = [(k, RunReport(F=float(f))) for t in out for k, f in zip(ks, t.tolist())]
    try:
        choice = model_select(rows)
        return choice.K_best, [(r.K, r.F, r.trials) for r in choice.table]
    except RuntimeError:
        return None, []


def allreduce_weight_stats(local_max: float, local_s1: float, local_s2: float, group=None):
    """Global (max lw, sum e^(lw-max), sum e^(2(lw-max))) from per-rank partials
    (the ESS / log-mean-w reduction of smc.cpp:61-66 across particle shards)."""
    d = _dev(group)
    m = torch.tensor([local_max], dtype=torch.float64, device=d)
    dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
    gm = float(m.item())
    scale = math.exp(local_max - gm) if math.isfinite(local_max) else 0.0
    s = torch.tensor([local_s1 * scale, local_s2 * scale * scale], dtype=torch.float64, device=d)
    dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
    return gm, float(s[0].item()), float(s[1].item())


def count_le(x: float, u: float, S: int) -> int:
    """#{j in [0, S): (j + u) / S <= x} with the reference's fp64 comparison."""
    j = math.floor(x * S - u)
    j = max(-1, min(S - 1, j))
    while j + 1 < S and (float(j + 1) + u) / S <= x:
        j += 1
    while j >= 0 and (float(j) + u) / S > x:
        j -= 1
    return j + 1


def global_resample_range(local_total: float, u: float, S: int, group=None) -> Tuple[int, int, float]:
    """This rank's slice [j0, j1) of the global systematic comb.

    local_total is the rank's share of the normalised weights (sum over its
    particles of exp(lw - lse_global)); ranks own consecutive particle ranges
    in rank order.  Returns (j0, j1, cdf_offset): targets j0..j1-1 resolve to
    local particles via the local CDF shifted by cdf_offset (the exclusive scan
    of the totals of lower ranks).  The last rank takes every remaining target
    (the i < T-1 guard of smc.cpp:103)."""
    d = _dev(group)
    ws, rank = dist.get_world_size(group), dist.get_rank(group)
    t = torch.tensor([local_total], dtype=torch.float64, device=d)
    totals = [torch.empty_like(t) for _ in range(ws)]
    dist.all_gather(totals, t, group=group)
    tv = [float(x.item()) for x in totals]
    offset = 0.0
    for r in range(rank):
        offset += tv[r]
    end = offset + tv[rank]
    j0 = 0 if rank == 0 else count_le(offset, u, S)
    j1 = S if rank == ws - 1 else count_le(end, u, S)
    return j0, max(j0, j1), offset
