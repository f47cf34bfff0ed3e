"""Input synthesis and host-side builders against the reference (CPU only)."""
import numpy as np
import pytest

from paper_2604_03271_b200 import model as M
from paper_2604_03271_b200 import synthetic as syn


@pytest.mark.parametrize("k,seed", [(1, 0), (3, 5), (6, 2), (7, 11)])
def test_gen_xps_bitwise(ref, k, seed):  # synthetic.cpp:270-318
    xs, ys = ref.gen_xps(k, seed)
    sp, _ = syn.gen_xps(k, seed)
    assert np.array_equal(xs, sp.xs) and np.array_equal(ys, sp.ys)


def test_rng_normals_bitwise(port):  # rng.hpp:28-74
    r = syn.Rng(404)
    assert np.array_equal(np.array([r.normal() for _ in range(64)]), port.normals(404, 64))


def test_trial_seed(ref):  # bench.cpp:104-106
    for t in range(5):
        assert syn.trial_seed(4242, t) == ref.trial_seed(4242, t)


@pytest.mark.parametrize("K", [1, 4, 10])
def test_xps_model_priors(ref, K):  # model.cpp:169-189
    w = syn.config("C2")
    pk, pa, pb = M.xps_model(K, w.data).arrays()
    rk, ra, rb = ref.xps_model_priors(K, w.data.xs, w.data.ys)
    assert np.array_equal(pk, rk) and np.array_equal(pa, ra) and np.array_equal(pb, rb)


@pytest.mark.parametrize("uniform", [False, True])
def test_gm_model_priors(ref, uniform):  # model.cpp:121-136
    pk, pa, pb = M.gm_model(3, 0.0, 3.0, 0.1, "uniform" if uniform else "normal15").arrays()
    rk, ra, rb = ref.gm_model_priors(3, 0.0, 3.0, 0.1, uniform)
    assert np.array_equal(pk, rk) and np.array_equal(pa, ra) and np.array_equal(pb, rb)


def test_config_shapes():
    for name, (N, kmax) in {"C1": (301, 5), "C2": (2000, 10)}.items():
        w = syn.config(name)
        assert len(w.data.xs) == N and w.k_range[1] == kmax and w.T % w.n == 0
        assert np.all(np.diff(w.data.xs) > 0) and np.all(np.isfinite(w.data.ys))


def test_gen_xrd_bitwise(ref):  # synthetic.cpp:230-268 (Poisson counts, PTRS)
    xs, ys = ref.gen_xrd(1000, 5)
    sp, _ = syn.gen_xrd(1000, 5)
    assert np.array_equal(xs, sp.xs) and np.array_equal(ys, sp.ys)


def test_xrd_model_priors(ref):  # model.cpp:138-167
    sp, _ = syn.gen_xrd(500, 2)
    spec = M.xrd_model(syn.TIO2_PHASES, sp)
    ph, mu, ri = spec.reflection_arrays()
    rk, ra, rb = ref.xrd_model_priors(3, ph, mu, ri, sp.xs, sp.ys)
    pk, pa, pb = spec.arrays()
    assert np.array_equal(pk, rk) and np.array_equal(pa, ra) and np.array_equal(pb, rb)
