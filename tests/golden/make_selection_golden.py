"""Generates tests/golden/selection_{C1,C2}.json from the reference itself.

TEST INFRASTRUCTURE.  Runs the unchanged reference sources (oracle/_ref,
built from /root/reference by oracle/build_oracle.py) through
``smc_run(spec, data, cfg)`` for every K of a model selection and every seed
trial_seed(4242, t), t = 0..9 (bench.cpp:104-106), as the CLI's
cmd_model_select loop does (proj/tools/specmc_main.cpp:147-170), and records:

  * F per (seed, K), diverged flags, levels;
  * the per-seed selected K (model_select, posterior.cpp:68-104) and the
    modal K over the seeds (acceptance select_k_once / criterion 4,
    proj/tests/acceptance/acceptance_main.cpp:227-262);
  * at K = k_true, the posterior mean and std of every component after
    sorting each particle's peak blocks by centre (label switching).

tests/test_gpu_selection.py compares the B200 sampler against these files.
Usage:  python tests/golden/make_selection_golden.py C1 C2 [--T 4096] [--seeds 10]
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle.oracle import Ref  # noqa: E402
from paper_2604_03271_b200 import synthetic as syn  # noqa: E402
from helpers import oracle_model  # noqa: E402


def canonical(th: np.ndarray, family: str, K: int) -> np.ndarray:
    """(T, d) draws -> the same draws with each particle's peak blocks sorted by centre."""
    stride = 3 if family == "gm" else 4
    out = th.copy()
    blocks = th[:, :stride * K].reshape(len(th), K, stride)
    order = np.argsort(blocks[:, :, 1], axis=1, kind="stable")
    out[:, :stride * K] = np.take_along_axis(blocks, order[:, :, None], axis=1).reshape(len(th), stride * K)
    return out


def run(cfg_name: str, T: int, n_seeds: int, workers: int) -> dict:
    ref = Ref()
    w = syn.config(cfg_name, T)
    ks = list(range(w.k_range[0], w.k_range[1] + 1))
    seeds = [syn.trial_seed(4242, t) for t in range(n_seeds)]
    out = {"config": cfg_name, "T": T, "n": w.n, "ess_target": 0.5, "K_range": [ks[0], ks[-1]],
           "k_true": w.truth_k, "seeds": [str(s) for s in seeds], "F": [], "diverged": [], "levels": [],
           "selected": [], "posterior_mean": [], "posterior_std": [], "wall_seconds": 0.0}
    t0 = time.perf_counter()
    for s in seeds:
        Fs, dv, lv = [], [], []
        for K in ks:
            om = oracle_model(w.spec(K), w.data)
            keep = K == w.truth_k
            r = ref.smc_run(om, T, w.n, 0.5, 2000, s, workers=workers, keep=keep)
            Fs.append(r.F)
            dv.append(int(r.diverged))
            lv.append(r.levels)
            if keep:
                c = canonical(r.thetas, w.family, K)
                out["posterior_mean"].append(c.mean(axis=0).tolist())
                out["posterior_std"].append(c.std(axis=0).tolist())
        out["F"].append(Fs)
        out["diverged"].append(dv)
        out["levels"].append(lv)
        out["selected"].append(ref.model_select(ks, Fs, dv))
        print(f"{cfg_name} seed {s}: K_sel={out['selected'][-1]} F={np.round(Fs, 3).tolist()} "
              f"({time.perf_counter() - t0:.0f} s)", flush=True)
    sel = out["selected"]
    out["modal_K"] = max(set(sel), key=lambda k: (sel.count(k), -k))
    out["wall_seconds"] = time.perf_counter() - t0
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--T", type=int, default=4096)
    ap.add_argument("--seeds", type=int, default=10)
    ap.add_argument("--workers", type=int, default=0)
    a = ap.parse_args()
    for c in a.configs:
        res = run(c, a.T, a.seeds, a.workers)
        p = Path(__file__).resolve().parent / f"selection_{c}.json"
        p.write_text(json.dumps(res, indent=1) + "\n")
        print("wrote", p, "modal K", res["modal_K"])


if __name__ == "__main__":
    main()
