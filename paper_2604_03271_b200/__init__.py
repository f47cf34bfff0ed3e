"""B200-native waste-free SMC sampler for Bayesian spectral deconvolution.

Drop-in sampling backend for the reference "specmc" (arxiv/paper_2604_03271):
the same ModelSpec / SmcConfig / RunReport interface, executed by
hand-written sm_100a CUDA kernels behind the C ABI of include/specmc_b200.h.
"""
from .model import (GammaPrior, GaussianApproxPoissonNoise, GaussianFixedNoise, ModelSpec, NormalPrior, PhaseRef,
                    PoissonNoise, Reflection, ScalarParam, Spectrum, UniformPrior, XpsHeteroNoise, gm_model,
                    model_dim, offset_model, prior_scale, xps_model, xrd_model)
from .report import (credible_interval, format_double, parse_double, read_report, sort_peak_blocks,
                     weighted_quantile, write_report)
from .smc import (Comm, CudaError, ModelChoice, RunReport, Session, SmcConfig, probe_mufu, device_count, energies, energy, ess,
                  launch_shape, log_mean_exp, model_select, next_beta, predict_step_size, smc_run, smc_run_batch,
                  stats, stats_reset, systematic_resample, validate_smc_config, smc_run_sharded, smc_run_sharded_batch, init_ensemble, smc_run_distributed, plan,
                  RemcConfig, remc_run, remc_run_batch)

__all__ = [
    "GammaPrior", "GaussianApproxPoissonNoise", "GaussianFixedNoise", "ModelSpec", "NormalPrior", "PoissonNoise",
    "ScalarParam", "Spectrum", "UniformPrior", "XpsHeteroNoise", "gm_model", "model_dim", "offset_model",
    "prior_scale", "xps_model", "xrd_model", "PhaseRef", "Reflection", "CudaError", "ModelChoice", "RunReport", "Session", "SmcConfig", "probe_mufu", "device_count", "energies",
    "energy", "ess", "launch_shape", "log_mean_exp", "model_select", "next_beta", "predict_step_size", "smc_run",
    "write_report", "read_report", "format_double", "parse_double", "weighted_quantile", "credible_interval",
    "sort_peak_blocks", "smc_run_batch", "smc_run_sharded", "smc_run_sharded_batch", "init_ensemble", "smc_run_distributed", "plan", "RemcConfig", "remc_run", "remc_run_batch", "Comm", "stats", "stats_reset", "systematic_resample", "validate_smc_config",
]
