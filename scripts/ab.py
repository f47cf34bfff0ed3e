"""A/B timing of library builds on the same GPU box (interleaved, repeated).
usage: python scripts/ab.py REPS CFG[,CFG..] LIB [LIB ...]   (CFG as in probe.py)"""
import json, os, subprocess, sys
from pathlib import Path
reps, cfgs, libs = int(sys.argv[1]), sys.argv[2].split(","), sys.argv[3:]
root = Path(__file__).resolve().parent.parent
res = {}
for r in range(reps):
    for lib in libs:
        env = dict(os.environ, SPECMC_LIB=str((root / lib).resolve()))
        cp = subprocess.run([sys.executable, str(root / "scripts" / "probe.py"), *cfgs], env=env, capture_output=True, text=True)
        out = cp.stdout
        if cp.returncode:
            print(lib, "probe failed:", cp.stderr[-2000:], flush=True)
        for line in out.splitlines():
            if line.startswith("{"):
                d = json.loads(line)
                res.setdefault((lib, d["cfg"]), []).append((d["dev"], d["pt_evals_per_s_move"] / 1e9,
                                                            d.get("mufu_ops_per_s", 0.0) / 1e9))
            elif line.startswith("clocks"):
                print(lib, line, flush=True)
for (lib, cfg), v in sorted(res.items(), key=lambda kv: (kv[0][1], kv[0][0])):
    devs = sorted(x[0] for x in v); pe = sorted(x[1] for x in v)
    mu = sorted(x[2] for x in v)
    print(f"{cfg:4s} {lib:45s} dev_med={devs[len(devs)//2]:.3f} dev_min={devs[0]:.3f}  Gpe/s_med={pe[len(pe)//2]:.1f} max={pe[-1]:.1f}"
          f"  mufu_Gop/s_med={mu[len(mu)//2]:.0f}  reps={[round(x[1] / 1e0, 1) for x in v]}")
