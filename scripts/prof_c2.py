"""Small C2 model-selection run used for ncu captures."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2604_03271_b200 as S
from paper_2604_03271_b200 import synthetic as syn
T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
kmax = int(sys.argv[2]) if len(sys.argv) > 2 else 10
w = syn.config("C2", T)
probs = [(w.spec(k), 0, S.SmcConfig(T=w.T, n=w.n, seed=7)) for k in range(1, kmax + 1)]
reps = S.smc_run_batch(probs, [w.data])
print("ok", [round(r.F, 2) for r in reps], reps[0].device_seconds)
