import sys, time
sys.path.insert(0, '.')
import paper_2604_03271_b200 as S
from paper_2604_03271_b200 import synthetic as syn
w = syn.config("C1")
probs = [(w.spec(K), 0, S.SmcConfig(T=4096, n=8, seed=7)) for K in range(1, 6)]
for i in range(6):
    t = time.perf_counter(); r = S.smc_run_batch(probs, [w.data]); t1 = time.perf_counter()
    print(f"call {i}: python wall {1e3*(t1-t):.3f} ms  C wall {1e3*r[0].wall_seconds:.3f} ms  dev {1e3*r[0].device_seconds:.3f} ms", flush=True)
