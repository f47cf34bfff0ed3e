"""Grid-level tempering (T > 2^15): the tree ESS passes (k_tp_ess_tree, three
next_beta bisection steps per pass over E) against one bisection step per
pass (SPECMC_ESS_DEPTH=1, the order of the reference's loop, smc.cpp:68-93).

Tolerance: bitwise.  Every delta, per-slot sum and fin_ess step is the same in
both schedules, so F, the tempering ladder and the posterior must be equal bit
for bit — for an unsharded run and for a run split over 2 in-process shards
(one exchange of all slots per pass vs one per step).
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent

_SCRIPT = r"""
import hashlib, json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2604_03271_b200 as S
from paper_2604_03271_b200 import model as M
from paper_2604_03271_b200 import synthetic as syn
sp, _ = syn.gen_xps(3, 5)
spec = M.xps_model(2, sp)
cfg = S.SmcConfig(T=1 << 16, n=4, seed=11)
out = {}
S.stats_reset()
for name, r in (("grid", S.smc_run(spec, sp, cfg)), ("shard2", S.smc_run_sharded(spec, sp, cfg, n_virtual=2))):
    out[name] = dict(F=r.F.hex(), levels=len(r.arrays["ladder"]),
                     ladder=hashlib.sha256(np.ascontiguousarray(r.arrays["ladder"]).tobytes()).hexdigest(),
                     post=hashlib.sha256(np.ascontiguousarray(r.posterior).tobytes()).hexdigest())
out["launches"] = S.stats()["kernel_launches"]
print(json.dumps(out))
"""


def _run(depth):
    env = dict(os.environ)
    env.pop("SPECMC_ESS_DEPTH", None)
    if depth is not None:
        env["SPECMC_ESS_DEPTH"] = str(depth)
    cp = subprocess.run([sys.executable, "-c", _SCRIPT, str(ROOT)], env=env, capture_output=True, text=True, timeout=600)
    assert cp.returncode == 0, cp.stderr[-3000:]
    import json
    return json.loads(cp.stdout.strip().splitlines()[-1])


def test_tree_ess_passes_equal_single_steps_bitwise():
    tree, single = _run(None), _run(1)
    assert tree["grid"]["levels"] > 3
    # the schedules differ (25 vs 65 tempering launches per unsharded level) ...
    assert tree.pop("launches") < single.pop("launches")
    # ... the results do not
    assert tree == single, (tree, single)


def test_grid_and_single_cta_next_beta_agree():
    """The same energies through the single-CTA bisection (k_temper's
    block_next_beta, T <= 2^15) and through the production grid launches
    (k_tp_emin + k_tp_ess_tree, forced with SPECMC_GRID_T in a subprocess):
    both replay the reference's bisection exactly, so beta_next agrees to the
    fp64 rounding of the differently ordered weight sums."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    import numpy as np
    import paper_2604_03271_b200 as S

    rng = np.random.default_rng(5)
    cases = []
    for T, nd, bp in ((4096, 301.0, 0.0), (20000, 2000.0, 1e-4), (30000, 840.0, 0.2)):
        E = 5.0 + np.abs(rng.normal(size=T)) * 3
        E[::101] = np.inf
        cases.append((E, nd, bp))
    block = [S.next_beta(E, nd, bp, 0.5) for E, nd, bp in cases]
    root = Path(__file__).resolve().parent.parent
    code = ("import sys, json, numpy as np; sys.path.insert(0, %r); import paper_2604_03271_b200 as S; "
            "rng = np.random.default_rng(5); out = []\n"
            "for T, nd, bp in ((4096, 301.0, 0.0), (20000, 2000.0, 1e-4), (30000, 840.0, 0.2)):\n"
            "    E = 5.0 + np.abs(rng.normal(size=T)) * 3; E[::101] = np.inf; out.append(S.next_beta(E, nd, bp, 0.5))\n"
            "print(json.dumps(out))") % str(root)
    env = dict(os.environ, SPECMC_GRID_T="1024")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stderr
    grid = json.loads(r.stdout.strip().splitlines()[-1])
    for b, g in zip(block, grid):
        assert g == pytest.approx(b, rel=1e-12), (block, grid)
