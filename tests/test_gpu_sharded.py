"""Particle-sharded runs on one GPU: the shards of a run live on
one device and exchange through kernels; the NCCL path uses the same phases.

Tolerances:
  * one shard == the unsharded grid-tempering path (T > 2^15): bitwise.
  * G shards vs the conjugate closed form: |F - F_exact| < 0.05 at T = 2^15
    (the reference's own tolerance is 0.15 at T = 2000, test_smc.cpp:122-138).
  * G shards vs one shard on the xps family: |dF| < 1.0 (Monte-Carlo error of
    F at T = 8192 is ~0.1-0.3).
"""
import math

import numpy as np
import pytest

from helpers import conjugate
from paper_2604_03271_b200 import model as M
from paper_2604_03271_b200 import synthetic as syn

pytestmark = pytest.mark.gpu


def test_one_shard_is_the_grid_path_bitwise(smc, port):
    spec, data, F_exact, mn, vn = conjugate(40, 77, port, truth=1.0, sigma=1.0, m0=0.0, v0=1.0)
    cfg = smc.SmcConfig(T=1 << 18, n=8, seed=5)
    a = smc.smc_run(spec, data, cfg)
    b = smc.smc_run_sharded(spec, data, cfg, n_virtual=1)
    assert a.F == b.F
    assert np.array_equal(a.arrays["ladder"], b.arrays["ladder"])
    assert np.array_equal(a.posterior, b.posterior)


@pytest.mark.parametrize("G", [2, 4, 8])
def test_virtual_shards_conjugate(smc, port, G):
    spec, data, F_exact, mn, vn = conjugate(30, 404, port)
    rep = smc.smc_run_sharded(spec, data, smc.SmcConfig(T=1 << 15, n=8, ess_target=0.5, seed=11), n_virtual=G)
    assert not rep.diverged and abs(rep.F - F_exact) < 0.05
    lad = rep.arrays["ladder"]
    assert lad[0] == 0.0 and lad[-1] == 1.0 and np.all(np.diff(lad) > 0)
    post = rep.posterior[0]
    assert rep.posterior.shape == (1, 1 << 15)  # the shards' particles together are the population
    assert abs(post.mean() - mn) < 5 * math.sqrt(vn / 4096) and abs(post.var() / vn - 1.0) < 0.1
    # global ESS at every level but the last matches the target (bisection on global sums)
    assert np.all(np.abs(rep.arrays["level_ess_ratio"][:-1] - 0.5) < 1e-5)


def test_virtual_shards_xps_match_unsharded(smc):
    sp, _ = syn.gen_xps(3, 5)
    spec = M.xps_model(3, sp)
    one = [smc.smc_run_sharded(spec, sp, smc.SmcConfig(T=8192, n=8, seed=s), n_virtual=1).F for s in (1, 2)]
    four = [smc.smc_run_sharded(spec, sp, smc.SmcConfig(T=8192, n=8, seed=s), n_virtual=4).F for s in (1, 2)]
    assert abs(np.mean(one) - np.mean(four)) < 1.0, (one, four)


def test_virtual_shards_replay_bitwise(smc):
    w = syn.config("C1")
    cfg = smc.SmcConfig(T=4096, n=8, seed=3)
    a = smc.smc_run_sharded(w.spec(3), w.data, cfg, n_virtual=4)
    b = smc.smc_run_sharded(w.spec(3), w.data, cfg, n_virtual=4)
    assert a.F == b.F and np.array_equal(a.posterior, b.posterior)


def test_sharded_argument_errors(smc, port):
    spec, data, *_ = conjugate(10, 3, port)
    with pytest.raises(ValueError):
        smc.smc_run_sharded(spec, data, smc.SmcConfig(T=1000, n=10, seed=1), n_virtual=3)  # T % shards
    with pytest.raises(ValueError):
        smc.smc_run_sharded(spec, data, smc.SmcConfig(T=1000, n=10, seed=1), n_virtual=0)


def test_nccl_single_rank_equals_one_virtual_shard(smc):
    # the NCCL exchange path (ncclAllReduce / ncclAllGather on the level stream)
    # with a one-rank communicator must reproduce the in-process exchange bitwise
    w = syn.config("C1")
    cfg = smc.SmcConfig(T=4096, n=8, seed=8)
    comm = smc.Comm(0, 1, smc.Comm.unique_id(), 0)
    try:
        a = smc.smc_run_sharded(w.spec(3), w.data, cfg, comm=comm)
    finally:
        comm.close()
    b = smc.smc_run_sharded(w.spec(3), w.data, cfg, n_virtual=1)
    assert a.F == b.F and np.array_equal(a.posterior, b.posterior)


def test_sharded_batch_equals_single_sharded_runs(smc):
    # all K of a selection split over the same shards at once == one call per K, bitwise
    w = syn.config("C1")
    cfgs = {K: smc.SmcConfig(T=2048, n=8, seed=40 + K) for K in (1, 2, 3)}
    batch = smc.smc_run_sharded_batch([(w.spec(K), 0, cfgs[K]) for K in (1, 2, 3)], [w.data], n_virtual=4)
    for K, b in zip((1, 2, 3), batch):
        one = smc.smc_run_sharded(w.spec(K), w.data, cfgs[K], n_virtual=4)
        assert b.F == one.F and np.array_equal(b.posterior, one.posterior)
    assert smc.model_select(list(zip((1, 2, 3), batch))).K_best == 3


def test_distributed_one_rank_equals_batch(smc):
    """specmc_smc_run_distributed on a one-rank NCCL communicator: the plan keeps
    every run local, so the results equal specmc_smc_run_batch bitwise; the
    per-run scalars come back through the NCCL all-reduce."""
    w = syn.config("C1")
    probs = [(w.spec(K), 0, smc.SmcConfig(T=2048, n=8, seed=9)) for K in (1, 2, 3)]
    comm = smc.Comm(0, 1, smc.Comm.unique_id(), 0)
    try:
        reps, r0, sh = smc.smc_run_distributed(probs, [w.data], comm)
        again, _, _ = smc.smc_run_distributed(probs, [w.data], comm)  # cached communicator state reused
    finally:
        comm.close()
    ref = smc.smc_run_batch(probs, [w.data])
    assert list(r0) == [0, 0, 0] and list(sh) == [1, 1, 1]
    for a, b, c in zip(reps, ref, again):
        assert a.F == b.F == c.F and a.trials == b.trials and a.proposals == b.proposals
        assert np.array_equal(a.posterior, b.posterior)
        assert a.scalars["levels"] == b.scalars["levels"]


def test_distributed_sharded_path_one_rank_equals_unsharded(smc, monkeypatch):
    """The distributed entry's sharded branch on one GPU: SPECMC_DIST_SHARD_ALL
    sends every run through an ncclCommSplit sub-communicator and the NCCL
    exchanges of the particle-sharded level loop (one-rank block); with one
    shard that is the unsharded grid-tempering path, bitwise (T > 2^15)."""
    w = syn.config("C1", 1 << 16)
    probs = [(w.spec(K), 0, smc.SmcConfig(T=1 << 16, n=8, seed=21)) for K in (2, 3)]
    ref = smc.smc_run_batch(probs, [w.data])
    monkeypatch.setenv("SPECMC_DIST_SHARD_ALL", "1")
    comm = smc.Comm(0, 1, smc.Comm.unique_id(), 0)
    try:
        reps, r0, sh = smc.smc_run_distributed(probs, [w.data], comm)
    finally:
        comm.close()
    for a, b in zip(reps, ref):
        assert a.F == b.F and a.trials == b.trials and a.scalars["levels"] == b.scalars["levels"]
        assert np.array_equal(a.arrays["ladder"], b.arrays["ladder"])
        assert np.array_equal(a.posterior, b.posterior)
