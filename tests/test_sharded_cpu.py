"""Particle-sharding host plumbing without a GPU: NCCL bootstrap ids and the
no-fallback behaviour of the sharded entry (the device path is in
test_gpu_sharded.py; the cross-rank host arithmetic in test_dist_gloo.py)."""
import pytest

import paper_2604_03271_b200 as S
from helpers import conjugate


@pytest.mark.skipif(S.device_count() > 0, reason="CPU-only behaviour")
def test_nccl_unique_id_bootstrap():
    a, b = S.Comm.unique_id(), S.Comm.unique_id()
    assert len(a) == len(b) == 128 and a != b
    with pytest.raises(S.CudaError):  # a communicator needs a device
        S.Comm(0, 1, a, 0)
    with pytest.raises(ValueError):
        S.Comm(0, 1, a[:64], 0)


@pytest.mark.skipif(S.device_count() > 0, reason="CPU-only behaviour")
def test_sharded_run_without_device_fails_loudly(port):
    spec, data, *_ = conjugate(10, 3, port)
    with pytest.raises(S.CudaError):
        S.smc_run_sharded(spec, data, S.SmcConfig(T=1024, n=8, seed=1), n_virtual=2)
