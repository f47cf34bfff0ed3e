"""bench-like e2e probe: a device-resident Session leg, then repeated smc_run_batch calls
(SPECMC_TRACE=1 prints the C-side phase timings)."""
import gc, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2604_03271_b200 as S
from paper_2604_03271_b200 import synthetic as syn
w = syn.config("C2")
probs = [(w.spec(k), 0, S.SmcConfig(T=w.T, n=w.n, seed=7)) for k in range(1, 11)]
sess = S.Session(probs, [w.data])
for _ in range(2):
    sess.run()
reps = sess.fetch()
sess.close()
S.smc_run_batch(probs, [w.data])
rr = None
for rep in range(6):
    t0 = time.perf_counter()
    rr = S.smc_run_batch(probs, [w.data], raise_on_error=False)
    t1 = time.perf_counter()
    print(f"call {t1 - t0:.3f}  C wall {rr[0].wall_seconds:.3f}  device {rr[0].device_seconds:.3f}  gc {gc.get_count()}", flush=True)
