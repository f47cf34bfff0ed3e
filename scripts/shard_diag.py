import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from oracle.build_oracle import build_port
from oracle.oracle import Port
import paper_2604_03271_b200 as S
from helpers import conjugate
port = Port()
spec, data, F_exact, mn, vn = conjugate(30, 404, port)
for G in (0, 1, 2, 4, 8):
    errs = []
    for seed in range(1, 13):
        cfg = S.SmcConfig(T=1 << 15, n=8, ess_target=0.5, seed=seed)
        r = S.smc_run(spec, data, cfg) if G == 0 else S.smc_run_sharded(spec, data, cfg, n_virtual=G)
        errs.append(r.F - F_exact)
    e = np.array(errs)
    print(G, "mean err %.4f sd %.4f  levels %d" % (e.mean(), e.std(), r.scalars["levels"]), np.round(e, 3))
