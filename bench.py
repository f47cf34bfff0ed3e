"""bench.py -- headline benchmark of the B200 SMC sampler (driver contract).

Workload (BASELINE.json configs[1], "C2"): synthetic XRD-like spectrum,
N = 2000 points, 6 pseudo-Voigt peaks + Shirley background, heteroscedastic
(GaussApprox-Poisson) noise; full model selection K = 1..10 with the xps
family (d = 4K+2), T = 65536 particles, n = 8 sweeps per chain, ess 0.5.
One "step" = one complete model-selection trial (all ten SMC runs to
beta = 1, log-evidence per K + posterior samples).

Metric: particle-likelihood evals/s, one eval = one MH proposal (the
SURVEY.md 8d unit, counted as sum over levels of T*d = smc.cpp:182 on both the
GPU and the CPU side), plus the time to log-evidence for K = 1..Kmax.

  value   device-resident throughput (specmc_session_run: spectra, priors and
          particles already in HBM), CUDA-event timed per step, L2 flushed
          between steps (256 MiB write), max over ranks.
  e2e     the same metric through the C ABI call specmc_smc_run_batch with host
          buffers: H2D of the spectrum/priors and D2H of every posterior (d x T
          fp64), energies and diagnostics inside the timed region.
  roofline  move kernel (k_chain<xps, PPL, W, move, noise>): point-evals/s from
          CUDA events around every move launch x the algorithmic MUFU ops per
          point of SURVEY.md 8d (pV shape 2 + hetero noise 2 = 4) against the
          measured MUFU ex2 throughput of this GPU (specmc_probe_mufu);
          executed_frac counts the 3 the kernel issues (paired noise terms).
  cpu_baseline  the reference itself (oracle/_ref, the unchanged reference
          sources), smc_run with workers = 0 (all host threads) on a bounded
          sample of the same workload (same spectrum, K = 1..10, T = 256).

Multi-GPU (torchrun): each rank runs its own trial (seed trial_seed(4242, rank),
weak scaling, no data-path collective); F per K is all-gathered for model
selection.  --impl reference: rank 0 times the reference CPU path alone.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# Algorithmic MUFU ops per point-eval (the credited per-unit
# figure): the swept block's shape (xps pseudo-Voigt: ex2 + rcp; gm: ex2) plus
# the noise term (hetero / GaussApprox: lg2 + rcp; Poisson: lg2; Gaussian: none)
# -> 4 for C2.  The kernel itself issues 3 per point for the hetero family: two
# points share one rcp and one lg2; roofline.executed_frac reports that.
MUFU_SHAPE = {"xps": 2.0, "gm": 1.0, "offset": 0.0}
MUFU_NOISE = {"XpsHeteroNoise": 2.0, "GaussianApproxPoissonNoise": 2.0, "PoissonNoise": 1.0,
              "GaussianFixedNoise": 0.0}
MUFU_NOISE_EXECUTED = {"XpsHeteroNoise": 1.0, "GaussianApproxPoissonNoise": 1.0, "PoissonNoise": 1.0,
                       "GaussianFixedNoise": 0.0}
# reference-CPU sample size per config (bounded: a few seconds of CPU per step;
# 64+ chains keep all host threads busy)
CPU_SAMPLE_T = {"C1": 4096, "C2": 512, "C3": 512, "C5": 256}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--T", type=int, default=None, help="override particle count (debug only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--shard", default="trials", choices=["trials", "particles"],
                    help="multi-GPU split: one model-selection trial per GPU (weak scaling, default) or one "
                         "trial with every run's particles split across the GPUs (strong scaling, SURVEY 8e-3)")
    return ap.parse_args()


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.f.flush()
        rows = []
        for line in Path(self.f.name).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        loaded = [v for v in sm if v > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(rows)}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# BASELINE.json config text per workload (synthetic data, see synthetic.config)
WORKLOAD_TEXT = {
    "C1": "synthetic XPS-like spectrum, 3 Gaussian peaks (flat background as a known offset)",
    "C2": "synthetic XRD-like spectrum, 6 pseudo-Voigt peaks + Shirley",
    "C3": "large-population single spectrum, 8 Lorentzian peaks (eta = 0) + Shirley",
    "C5": "Kmax sweep stress test, 20 pseudo-Voigt peaks + Shirley",
}


def inputs_module():
    """The package's input synthesis (synthetic.py / model.py) WITHOUT importing
    the package: the reference arm must not map libspecmc_b200.so.  A bare
    namespace stands in for the package, so its __init__ (which loads the
    library) never runs; model.py defers its library import to desc()."""
    import importlib
    import types
    name = "paper_2604_03271_b200"
    if name not in sys.modules:
        stub = types.ModuleType(name)
        stub.__path__ = [str(ROOT / name)]
        sys.modules[name] = stub
    return importlib.import_module(name + ".synthetic")


def workload_config(args, w, ws):
    """The `config` object of both arms' JSON lines (identical by construction)."""
    ks = list(range(w.k_range[0], w.k_range[1] + 1))
    N = len(w.data.xs)
    return {"workload": f"{args.config}: {WORKLOAD_TEXT.get(args.config, 'synthetic spectrum')}, N={N},"
                        f" {w.family} family K={ks[0]}..{ks[-1]}, T={w.T}, n={w.n}, ess 0.5; 1 trial per GPU",
            "N": N, "K_range": [ks[0], ks[-1]], "T": w.T, "n": w.n, "trials_per_gpu": 1,
            "l2": "flushed between steps (256 MiB write)", "parallelism": f"trials x{ws} (weak)"}


def cpu_reference_sample(workload, seed, T, timing=True):
    """Reference smc_run (oracle/_ref: the unchanged reference sources) for
    K = 1..Kmax at T particles, workers = 0 (all host threads), the CLI's serial
    K loop (specmc_main.cpp:147-170).  timing=True uses the Release-flag build
    for this host's ISA (oracle/build_oracle.timing_ref_so).  Returns
    (evals, seconds, cores, kind, build)."""
    from oracle.oracle import OracleModel, Port, Ref, ref_available
    ks = list(range(workload.k_range[0], workload.k_range[1] + 1))
    kind = "reference" if ref_available() else "port"
    build = "oracle port (1 thread)"
    if kind == "reference":
        from oracle.build_oracle import timing_ref_so
        so, build = timing_ref_so() if timing else (None, "parity build")
        lib = Ref(so) if so is not None else Ref()
    else:
        lib = Port()
    evals, secs = 0, 0.0
    for K in ks:
        spec = workload.spec(K)
        pk, pa, pb = spec.arrays()
        nz = spec.noise
        kw = dict(noise="xps_hetero", s0=nz.s0, s1=nz.s1, s2=nz.s2) if workload.family == "xps" else dict(
            noise="gaussian", sigma=nz.sigma)
        om = OracleModel(workload.family, K, pk, pa, pb, workload.data.xs, workload.data.ys, **kw)
        t0 = time.perf_counter()
        if kind == "reference":
            r = lib.smc_run(om, T, workload.n, 0.5, 2000, seed, workers=0, keep=False)
            secs += r.wall_seconds
        else:
            r = lib.smc_run(om, T, workload.n, 0.5, 2000, seed, keep=False)
            secs += time.perf_counter() - t0
        evals += T * spec.d * r.levels
    cores = os.cpu_count() if kind == "reference" else 1
    return evals, secs, cores, kind, build


def library_mapped():
    try:
        return "libspecmc_b200" in Path("/proc/self/maps").read_text()
    except OSError:
        return False


def run_reference(args, ws, rank):
    if rank != 0:
        return
    syn = inputs_module()
    w = syn.config(args.config)
    T = CPU_SAMPLE_T[args.config]
    seed = syn.trial_seed(4242, 0)
    # warm-up: page the library and the spectrum in (one K at a small T: the
    # CPU has no caches worth warming beyond that)
    w_small = syn.config(args.config, 64)
    w_small.k_range = (w.k_range[0], w.k_range[0])
    for _ in range(args.warmup):
        cpu_reference_sample(w_small, seed, 64)
    ev, secs = 0, 0.0
    for _ in range(args.steps):
        e, s_, cores, kind, build = cpu_reference_sample(w, seed, T)
        ev += e
        secs += s_
    assert not library_mapped(), "reference arm mapped the product library"
    v = ev / secs
    line = {
        "metric": f"particle-likelihood evals/s (K=1..{w.k_range[1]} model selection, {args.config})",
        "value": v, "unit": "evals/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": workload_config(args, w, ws),
        "cpu_baseline": {"value": v, "unit": "evals/s", "cores": cores, "kind": kind,
                         "sample": f"each step: smc_run for K={w.k_range[0]}..{w.k_range[1]} (serial K loop, "
                                   f"workers=0) on the same spectrum at T={T} particles instead of {w.T}; "
                                   f"evals/s = sum T*d*levels / sum wall_seconds; build {build}"},
        "e2e": {"value": v, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "product_library_mapped": False,
    }
    print(json.dumps(line), flush=True)


def run_ours(args, ws, rank, local):
    import torch
    import paper_2604_03271_b200 as S
    from paper_2604_03271_b200 import synthetic as syn

    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = syn.config(args.config, args.T)
    ks = list(range(w.k_range[0], w.k_range[1] + 1))
    seed = syn.trial_seed(4242, rank)
    problems = [(w.spec(K), 0, S.SmcConfig(T=w.T, n=w.n, ess_target=0.5, seed=seed, device=local)) for K in ks]
    N = len(w.data.xs)
    peak_mufu = S.probe_mufu(local)

    sess = S.Session(problems, [w.data])
    for _ in range(args.warmup):
        sess.run()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    clocks = Clocks(local)
    S.stats_reset()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    elapsed = 0.0
    for _ in range(args.steps):
        flush.fill_(1.0)  # L2 flush between timed steps (outside the timed window)
        torch.cuda.synchronize()
        elapsed += sess.run()  # CUDA events on the session's launch stream, first to last kernel
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    st = S.stats()
    reps = sess.fetch(raise_on_error=False)
    sess.close()
    ok = [r for r in reps if not isinstance(r, Exception)]
    evals_step = sum(r.proposals for r in ok)
    trials_step = sum(r.trials for r in ok)

    # ---- e2e: the C ABI call with host buffers (H2D spectrum/priors, D2H posteriors)
    e2e = None
    if not args.no_e2e:
        S.smc_run_batch(problems, [w.data])  # warm-up of the allocation path
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_evals = 0
        e2e_steps = []
        for _ in range(args.steps):
            ts = time.perf_counter()
            rr = S.smc_run_batch(problems, [w.data], raise_on_error=False)
            e2e_evals += sum(r.proposals for r in rr if not isinstance(r, Exception))
            e2e_steps.append(round(time.perf_counter() - ts, 4))
        torch.cuda.synchronize()
        e2e_t = time.perf_counter() - t0
        h2d = 2 * N * 8 + sum(p[0].d * (4 + 8 + 8) for p in problems)
        d2h = sum(p[0].d * w.T * 8 + w.T * 8 for p in problems) + sum(
            int(r.scalars["levels"]) * 4 * 8 for r in rr if not isinstance(r, Exception))
        e2e = {"value": e2e_evals, "t": e2e_t, "h2d": h2d, "d2h": d2h, "steps": e2e_steps}

    # ---- model selection over all trials (ranks); max-over-ranks timing
    Fs = [r.F if not isinstance(r, Exception) else float("nan") for r in reps]
    if dist:
        from paper_2604_03271_b200 import dist as D
        elapsed, total_evals = D.reduce_timing(elapsed, evals_step * args.steps)
        k_sel, _ = D.gather_selection(ks, Fs)
        if e2e:
            e2e["t"], e2e["value"] = D.reduce_timing(e2e["t"], float(e2e["value"]))
    else:
        total_evals = evals_step * args.steps
        try:
            k_sel = S.model_select([(K, S.RunReport(F=F)) for K, F in zip(ks, Fs)]).K_best
        except RuntimeError:
            k_sel = None

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    value = total_evals / elapsed
    move_s = st["move_kernel_ms"] * 1e-3
    pe_rate = st["point_evals"] / move_s if move_s > 0 else 0.0
    mufu_pt = MUFU_SHAPE[w.family] + MUFU_NOISE[type(w.noise).__name__]
    mufu_exec = MUFU_SHAPE[w.family] + MUFU_NOISE_EXECUTED[type(w.noise).__name__]
    achieved = pe_rate * mufu_pt
    traffic = None
    prof = ROOT / "profiles" / "move_kernel_ncu.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    line = {
        "metric": f"particle-likelihood evals/s (K=1..{ks[-1]} model selection, {args.config})",
        "value": value, "unit": "evals/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": elapsed / args.steps * 1e3, "time_to_evidence_s": elapsed / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 point terms / f64 accumulation", "data": "synthetic",
        "config": workload_config(args, w, ws),
        "K_selected": k_sel, "trials_per_step": trials_step, "point_evals_per_s_move": pe_rate,
        "gpu_launches": st["kernel_launches"],
        "roofline": {"bound": "sfu", "achieved": achieved / 1e9, "peak": peak_mufu / 1e9,
                     "unit": "Gop/s (MUFU)", "frac": achieved / peak_mufu if peak_mufu else None,
                     "traffic": traffic,
                     "executed_frac": pe_rate * mufu_exec / peak_mufu if peak_mufu else None,
                     "note": f"move kernel; {mufu_pt:g} algorithmic MUFU ops per point-eval (SURVEY 8d: pV shape "
                             f"ex2 + rcp, hetero noise lg2 + rcp) x point-evals/s from CUDA events on the launch "
                             f"stream; the kernel executes {mufu_exec:g} (two points share the noise rcp and lg2): "
                             "executed_frac; peak = measured ex2 throughput of this GPU (specmc_probe_mufu)"},
        "clocks": clk,
    }
    if e2e:
        line["e2e"] = {"value": e2e["value"] / e2e["t"], "unit": "evals/s", "h2d_bytes_per_step": e2e["h2d"],
                       "d2h_bytes_per_step": e2e["d2h"], "step_seconds": e2e.get("steps")}
    if ws == 1 and not args.no_cpu_baseline:
        Tc = CPU_SAMPLE_T[args.config]
        ev, secs, cores, kind, build = cpu_reference_sample(w, seed, Tc)
        line["cpu_baseline"] = {"value": ev / secs, "unit": "evals/s", "cores": cores, "kind": kind,
                                "sample": f"smc_run K={ks[0]}..{ks[-1]} on the same spectrum at T={Tc} "
                                          f"(n={w.n}, workers=0), {secs:.1f} s; build {build}"}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_particles(args, ws, rank, local):
    """One model-selection trial whose every run is particle-sharded over the ws
    GPUs (smc_run_sharded, NCCL exchanges): strong scaling of one workload."""
    import torch
    import paper_2604_03271_b200 as S
    from paper_2604_03271_b200 import synthetic as syn

    torch.cuda.set_device(local)
    dist = None
    comm = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = S.Comm.from_torch(local)
    w = syn.config(args.config, args.T)
    ks = list(range(w.k_range[0], w.k_range[1] + 1))
    seed = syn.trial_seed(4242, 0)  # the same trial on every rank
    cfgs = {K: S.SmcConfig(T=w.T, n=w.n, ess_target=0.5, seed=seed, device=local) for K in ks}
    N = len(w.data.xs)
    peak_mufu = S.probe_mufu(local)

    problems = [(w.spec(K), 0, cfgs[K]) for K in ks]

    def step():  # all K at once, every run's particles split over the ranks
        rr = S.smc_run_sharded_batch(problems, [w.data], n_virtual=1, comm=comm)
        reps = dict(zip(ks, rr))
        return rr[0].device_seconds, rr[0].wall_seconds, sum(r.proposals for r in rr), reps

    for _ in range(args.warmup):
        step()
    clocks = Clocks(local)
    S.stats_reset()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    elapsed = wall = 0.0
    evals = 0
    for _ in range(args.steps):
        d, wl, e, reps = step()
        elapsed += d
        wall += wl
        evals += e
    clk = clocks.stop()
    st = S.stats()
    if dist:
        from paper_2604_03271_b200 import dist as D
        elapsed, evals = D.reduce_timing(elapsed, float(evals))
        wall, _ = D.reduce_timing(wall, 0.0)
    choice = S.model_select([(K, r) for K, r in reps.items()])
    if rank == 0:
        move_s = st["move_kernel_ms"] * 1e-3
        pe_rate = st["point_evals"] / move_s if move_s > 0 else 0.0
        mufu_pt = MUFU_SHAPE[w.family] + MUFU_NOISE[type(w.noise).__name__]
        line = {
            "metric": f"particle-likelihood evals/s (K=1..{ks[-1]} model selection, {args.config})",
            "value": evals / elapsed, "unit": "evals/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed / args.steps * 1e3, "time_to_evidence_s": elapsed / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 point terms / f64 accumulation", "data": "synthetic",
            "config": {"workload": f"{args.config}: N={N}, K={ks[0]}..{ks[-1]}, T={w.T} particles per run split "
                                   f"over {ws} GPU(s), n={w.n}", "N": N, "K_range": [ks[0], ks[-1]], "T": w.T,
                       "n": w.n, "l2": f"inputs larger than L2 ({w.T} particles x d fp64)",
                       "parallelism": f"particles x{ws} (strong, NCCL per-level exchanges)"},
            "K_selected": choice.K_best, "point_evals_per_s_move": pe_rate, "gpu_launches": st["kernel_launches"],
            "roofline": {"bound": "sfu", "achieved": pe_rate * mufu_pt / 1e9, "peak": peak_mufu / 1e9,
                         "unit": "Gop/s (MUFU)", "frac": pe_rate * mufu_pt / peak_mufu if peak_mufu else None,
                         "traffic": None, "note": f"move kernel, rank 0; {mufu_pt:g} MUFU ops per point-eval"},
            "clocks": clk,
            "e2e": {"value": evals / wall, "unit": "evals/s", "h2d_bytes_per_step": 2 * N * 8,
                    "d2h_bytes_per_step": int(sum(r.posterior.nbytes + r.energies.nbytes for r in reps.values()))},
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if dist:
        dist.destroy_process_group()


def main():
    args = parse()
    ws, rank, local = dist_init()
    if args.impl == "reference":
        run_reference(args, ws, rank)
    elif args.shard == "particles":
        run_particles(args, ws, rank, local)
    else:
        run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
