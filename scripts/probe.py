"""Exploratory GPU probe: model selection runs on the BASELINE configs."""
import sys, time, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import subprocess
import numpy as np
import paper_2604_03271_b200 as S
from paper_2604_03271_b200 import synthetic as syn

def run(name, T=None, kmax=None, seed=7):
    w = syn.config(name, T)
    ks = list(range(w.k_range[0], (kmax or w.k_range[1]) + 1))
    probs = [(w.spec(k), 0, S.SmcConfig(T=w.T, n=w.n, seed=seed)) for k in ks]
    S.stats_reset()
    t = time.perf_counter()
    reps = S.smc_run_batch(probs, [w.data])
    wall = time.perf_counter() - t
    st = S.stats()
    props = sum(r.proposals for r in reps); trials = sum(r.trials for r in reps)
    choice = S.model_select([(k, r) for k, r in zip(ks, reps)])
    out = dict(cfg=name, T=w.T, wall=round(wall, 3), dev=round(reps[0].device_seconds, 3),
               levels=[int(r.scalars["levels"]) for r in reps], F=[round(r.F, 3) for r in reps],
               K_best=choice.K_best, proposals=props, trials=trials,
               evals_per_s=props / reps[0].device_seconds, move_ms=round(st["move_kernel_ms"], 1),
               pt_evals_per_s_move=st["point_evals"] / (st["move_kernel_ms"] * 1e-3),
               mufu_ops_per_s=st.get("move_mufu_ops", 0.0) / (st["move_kernel_ms"] * 1e-3),
               launches=st["kernel_launches"])
    print(json.dumps(out), flush=True)

def run_c4(n_spec, T):
    spectra, kt, T, n = syn.config_c4(n_spec, T)
    probs = []
    for si, sp in enumerate(spectra):
        for K in range(1, 7):
            probs.append((S.xps_model(K, sp), si, S.SmcConfig(T=T, n=n, seed=si)))
    S.stats_reset()
    t = time.perf_counter()
    reps = S.smc_run_batch(probs, spectra, raise_on_error=False)
    wall = time.perf_counter() - t
    st = S.stats()
    hits = 0
    for si in range(len(spectra)):
        rows = [(K, reps[6 * si + K - 1]) for K in range(1, 7) if not isinstance(reps[6 * si + K - 1], Exception)]
        hits += S.model_select(rows).K_best == kt[si]
    ok = [r for r in reps if not isinstance(r, Exception)]
    props = sum(r.proposals for r in ok)
    print(json.dumps(dict(cfg="C4", spectra=len(spectra), T=T, wall=round(wall, 3), dev=round(ok[0].device_seconds, 3),
                          hits=hits, failed=len(reps) - len(ok), proposals=props,
                          evals_per_s=props / ok[0].device_seconds,
                          pt_evals_per_s_move=st["point_evals"] / (st["move_kernel_ms"] * 1e-3))), flush=True)


def clocks():
    try:
        return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_event_reasons.active",
                               "--format=csv,noheader"], capture_output=True, text=True, timeout=10).stdout.strip()
    except Exception:
        return "?"


if __name__ == "__main__":
    print("clocks before:", clocks(), flush=True)
    for arg in sys.argv[1:]:
        name, T = arg.split(":")
        if name.startswith("C4x"):
            run_c4(int(name[3:]), int(T) if T != "full" else None)
        else:
            run(name, int(T) if T != "full" else None)
