"""Multi-GPU host helpers over torch.distributed (NCCL on the GPU box, gloo in tests).

The split of one model selection over the ranks is native: placement
(``specmc_plan``), particle-sharded runs on sub-communicators and the final
all-reduce of the per-run scalars all happen inside
``specmc_smc_run_distributed`` (host.cu).  Python only bootstraps the NCCL
communicator (``Comm.from_torch``) and, for the bench, reduces its timing:

* ``reduce_timing``: max over ranks of the device time, sum of the work
  (bench.py contract);
* ``gather_selection``: the trials mode (one independent model-selection
  trial per rank, bench.cpp:104-106 seeds) gathers every rank's F per K and
  runs model_select over all trials (posterior.cpp:68-104).
"""
from __future__ import annotations

from typing import Sequence, Tuple

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
