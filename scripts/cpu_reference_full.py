"""One full-size run of the reference CPU path (the unchanged reference sources,
oracle/_ref, Release flags for this host's ISA) on a BASELINE config: the CLI's
serial K loop (specmc_main.cpp:147-170) of smc_run(spec, data, cfg) with
workers = 0 (all host threads, parallel.hpp:37-40).  Writes
profiles/<tag>.json with per-K wall seconds, levels, F, evals, the selected K,
nproc and lscpu; also times the bench's reduced-T sample on the same host so
that the sample-to-full throughput ratio is measured, not assumed.

usage: python scripts/cpu_reference_full.py C2 [--tag r02_cpu_c2_full] [--T-list 512,4096]
"""
import argparse
import json
import os
import platform
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402  (inputs_module: no product library)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--tag", default=None)
    ap.add_argument("--T-list", default="512,4096")
    ap.add_argument("--full-T", type=int, default=None)
    a = ap.parse_args()
    syn = bench.inputs_module()
    from oracle.build_oracle import timing_ref_so
    from oracle.oracle import OracleModel, Ref
    so, build = timing_ref_so()
    ref = Ref(so)
    seed = syn.trial_seed(4242, 0)
    out = {"config": a.config, "build": build, "nproc": os.cpu_count(), "machine": platform.processor(),
           "seed": str(seed), "runs": {}}
    try:
        out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines()[:16]
    except OSError:
        pass
    Ts = [int(t) for t in a.T_list.split(",") if t] + [a.full_T or syn.config(a.config).T]
    for T in Ts:
        b = bench.Bench(syn, a.config, T)
        rows, evals, wall = [], 0, 0.0
        for spec, si, K in b.runs:
            pk, pa, pb = spec.arrays()
            nz = spec.noise
            kw = dict(noise="xps_hetero", s0=nz.s0, s1=nz.s1, s2=nz.s2) if b.family == "xps" else dict(
                noise="gaussian", sigma=nz.sigma)
            om = OracleModel(b.family, K, pk, pa, pb, b.spectra[si].xs, b.spectra[si].ys, **kw)
            t0 = time.perf_counter()
            r = ref.smc_run(om, T, b.n, 0.5, 2000, seed, workers=0, keep=False)
            e = T * spec.d * r.levels
            rows.append({"K": K, "F": r.F, "levels": r.levels, "wall_seconds": r.wall_seconds,
                         "host_seconds": time.perf_counter() - t0, "evals": e, "diverged": r.diverged})
            evals += e
            wall += r.wall_seconds
            print(f"T={T} K={K} F={r.F:.3f} levels={r.levels} {r.wall_seconds:.1f} s", flush=True)
        ks = [x["K"] for x in rows]
        k_sel = ref.model_select(ks, [x["F"] for x in rows], [int(x["diverged"]) for x in rows])
        out["runs"][str(T)] = {"T": T, "per_K": rows, "evals": evals, "time_to_evidence_s": wall,
                               "evals_per_s": evals / wall, "K_selected": k_sel}
    tag = a.tag or f"r02_cpu_{a.config.lower()}_full"
    p = ROOT / "profiles" / f"{tag}.json"
    p.write_text(json.dumps(out, indent=1) + "\n")
    print("wrote", p)


if __name__ == "__main__":
    main()
