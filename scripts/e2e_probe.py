"""Phase breakdown of the end-to-end call on C2 (create / run / fetch / close / collect)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2604_03271_b200 as S
from paper_2604_03271_b200 import synthetic as syn
from paper_2604_03271_b200 import smc as M

T = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
w = syn.config("C2", T)
probs = [(w.spec(k), 0, S.SmcConfig(T=w.T, n=w.n, seed=7)) for k in range(1, 11)]
for rep in range(4):
    t0 = time.perf_counter()
    s = M.Session(probs, [w.data])
    t1 = time.perf_counter()
    dev = s.run()
    t2 = time.perf_counter()
    reps = s.fetch(raise_on_error=False)
    t3 = time.perf_counter()
    s.close()
    t4 = time.perf_counter()
    t5 = time.perf_counter()
    rr = S.smc_run_batch(probs, [w.data], raise_on_error=False)
    t6 = time.perf_counter()
    print(f"rep {rep}: create {t1-t0:.3f} run {t2-t1:.3f} (device {dev:.3f}) fetch+collect {t3-t2:.3f} close {t4-t3:.3f} | smc_run_batch {t6-t5:.3f}", flush=True)
