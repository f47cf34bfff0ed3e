"""One model-selection run of a BASELINE config for ncu captures.
usage: python scripts/prof_cfg.py CFG T K[,K..]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2604_03271_b200 as S
from paper_2604_03271_b200 import synthetic as syn
name, T, ks = sys.argv[1], int(sys.argv[2]), [int(k) for k in sys.argv[3].split(",")]
w = syn.config(name, T)
probs = [(w.spec(k), 0, S.SmcConfig(T=w.T, n=w.n, seed=7)) for k in ks]
reps = S.smc_run_batch(probs, [w.data])
print("ok", [round(r.F, 2) for r in reps], reps[0].device_seconds)
