/*
 * specmc_b200.h -- C ABI of the B200-native waste-free SMC sampler.
 *
 * Drop-in sampling backend for the reference "specmc" (arxiv/paper_2604_03271,
 * C++20/Eigen, CPU only).  Each entry point replaces one reference interface;
 * the citation is given next to it (paths relative to the reference root).
 * Plain C types only: caller-owned input buffers are borrowed for the duration
 * of the call; result arrays are allocated by the library and released with
 * specmc_result_free().
 *
 * Return codes mirror the reference's error conventions
 * (proj/src/smc.cpp:24-31, :63, :98, :195-196; proj/tools/specmc_main.cpp:17-19):
 *   SPECMC_OK            0
 *   SPECMC_EINVAL        2   std::invalid_argument (config / model / spectrum)
 *   SPECMC_ERUNTIME      3   std::runtime_error (max_levels, zero total weight)
 *   SPECMC_ECUDA         4   CUDA failure (no device, launch/alloc error)
 *   SPECMC_ECOMM         5   collective / communicator failure
 * A non-finite free energy is NOT an error: result.diverged = 1
 * (proj/src/smc.cpp:205-206).  The message of the first failure is written to
 * err (NUL-terminated, at most errlen bytes) when err != NULL.
 */
#ifndef SPECMC_B200_H
#define SPECMC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPECMC_OK 0
#define SPECMC_EINVAL 2
#define SPECMC_ERUNTIME 3
#define SPECMC_ECUDA 4
#define SPECMC_ECOMM 5

/* proj/include/specmc/model.hpp:40 (Family); OFFSET is the conjugate-mean
 * family f(x) = theta_0 of proj/tests/conjugate_oracle.hpp:19-28, so the
 * closed-form evidence oracle runs on the device. */
enum specmc_family { SPECMC_FAMILY_GM = 0, SPECMC_FAMILY_XPS = 1, SPECMC_FAMILY_XRD = 2, SPECMC_FAMILY_OFFSET = 3 };
/* proj/include/specmc/model.hpp:13-23 (NoiseSpec variants) */
enum specmc_noise { SPECMC_NOISE_GAUSSIAN = 0, SPECMC_NOISE_POISSON = 1, SPECMC_NOISE_GAUSS_APPROX = 2, SPECMC_NOISE_XPS_HETERO = 3 };
/* proj/include/specmc/priors.hpp:13-26 (PriorSpec variants) */
enum specmc_prior { SPECMC_PRIOR_NORMAL = 0, SPECMC_PRIOR_GAMMA = 1, SPECMC_PRIOR_UNIFORM = 2 };

/* Flat ModelSpec (proj/include/specmc/model.hpp:50-56).  prior_* have length
 * d = model_dim(spec) in the reference layout order (model.hpp:43-49):
 *   gm:  (A_k, mu_k, b_k) per peak                 d = 3K
 *   xps: (A_k, mu_k, sigma_k, eta_k) per peak, a, b d = 4K + 2
 *   xrd: (A, d2t, r, alpha, u, v, w, s, t) per phase,
 *        then (bg_a, bg_sigma, bg_r, bg_b)          d = 9K + 4
 *   offset: (theta)                                d = 1
 * Normal(a = mean, b = var), Gamma(a = shape, b = rate), Uniform(a = lo, b = hi). */
typedef struct {
  int32_t family;
  int32_t K;
  int32_t d;
  int32_t noise;
  double noise_sigma;       /* GaussianFixedNoise::sigma */
  double s0, s1, s2;        /* XpsHeteroNoise */
  int32_t paper_literal;    /* XpsHeteroNoise::paper_literal */
  const int32_t* prior_kind;
  const double* prior_a;
  const double* prior_b;
  /* xrd only: reflection list of every phase (PhaseRef, model.hpp:25-32),
   * grouped by phase in phase order: phase index, mu_ref (deg 2theta), rel. intensity */
  int32_t n_refl;
  const int32_t* refl_phase;
  const double* refl_mu;
  const double* refl_int;
} specmc_model_desc;

/* SmcConfig (proj/include/specmc/smc.hpp:12-19) plus the device ordinal. */
typedef struct {
  int64_t T;
  int32_t n;
  double ess_target;
  int32_t max_levels;
  uint64_t seed;
  int32_t workers;  /* echoed only (the GPU ignores it) */
  int32_t device;   /* CUDA device ordinal */
} specmc_smc_config;

/* SmcResult + RunReport fields (proj/include/specmc/smc.hpp:32-48,
 * proj/src/smc.cpp:218-249).  posterior is d x T column-major like the
 * reference's MatrixXd (element (i, c) at posterior[c * d + i]). */
typedef struct {
  int32_t status;        /* SPECMC_OK or the per-run error code */
  double F;
  int32_t diverged;
  double wall_seconds;   /* host wall time of the whole call */
  double device_seconds; /* CUDA-event time of the device run (no H2D/D2H) */
  int32_t levels;
  int32_t d;
  int64_t T;
  double* ladder;           /* levels + 1, ladder[0] = 0 */
  double* level_ess_ratio;  /* levels */
  double* level_log_mean_w; /* levels */
  double* level_acc_rate;   /* levels */
  double* posterior;        /* d * T */
  double* energies;         /* T, per-point energies of the final ensemble */
  int64_t proposals;        /* sum over levels of T * d (smc.cpp:182) */
  int64_t trials;           /* finite-prior proposals = Evaluator::trial calls */
} specmc_smc_result;

/* One SMC run of a batch: model + index of its spectrum + config. */
typedef struct {
  specmc_model_desc model;
  int32_t spectrum;
  specmc_smc_config cfg;
} specmc_problem;

/* A spectrum (proj/include/specmc/spectrum.hpp:16-20). */
typedef struct {
  const double* xs;
  const double* ys;
  int64_t n;
} specmc_spectrum;

/* ---- primary entry ------------------------------------------------------
 * Replaces RunReport smc_run(const ModelSpec&, const Spectrum&,
 * const SmcConfig&) (proj/include/specmc/smc.hpp:78; proj/src/smc.cpp:218-249)
 * and the Problem-level smc_run it wraps (smc.cpp:186-216). */
int specmc_smc_run(const specmc_model_desc* model, const double* xs, const double* ys, int64_t n_points,
                   const specmc_smc_config* cfg, specmc_smc_result* out, char* err, size_t errlen);

/* Batched entry: every problem runs concurrently on cfg.device (problems of
 * one batch must share the device).  This is the K-range / trials / spectra
 * loop of cmd_model_select (proj/tools/specmc_main.cpp:148-170) moved onto the
 * GPU.  out[i].status carries each run's own error code; the return value is
 * the first non-OK status (or an ABI-level error). */
int specmc_smc_run_batch(int32_t n_problems, const specmc_problem* problems, int32_t n_spectra,
                         const specmc_spectrum* spectra, specmc_smc_result* out, char* err, size_t errlen);

void specmc_result_free(specmc_smc_result* r);

/* Frees one result array whose ownership the caller took over (it then sets
 * the field to NULL before specmc_result_free): lets a binding hand the
 * posterior block to its own array type without copying it. */
void specmc_free(void* p);

/* ---- device-resident sessions -----------------------------------------
 * specmc_smc_run_batch == create + run + fetch + destroy.  A session keeps the
 * spectra, priors and particle buffers resident in HBM; run() re-runs every
 * problem from init_ensemble (same seeds => same results) without any
 * host<->device traffic besides 48 bytes of state per run and level. */
typedef struct specmc_session specmc_session;
int specmc_session_create(int32_t n_problems, const specmc_problem* problems, int32_t n_spectra,
                          const specmc_spectrum* spectra, specmc_session** out, char* err, size_t errlen);
int specmc_session_run(specmc_session* s, double* device_seconds, char* err, size_t errlen);
int specmc_session_fetch(specmc_session* s, specmc_smc_result* out, char* err, size_t errlen);
void specmc_session_destroy(specmc_session* s);

/* init_ensemble (proj/src/smc.cpp:34-53) alone: the T prior draws of a run
 * and their full energies, exactly as the sampler's level 0 makes them
 * (same Philox streams).  out->posterior = the d x T draws, out->energies =
 * their energies, levels = 0.  Parity unit for the initial ensemble and the
 * importance-sampling identity (acceptance criterion 9a). */
int specmc_init_ensemble(const specmc_model_desc* model, const double* xs, const double* ys, int64_t n_points,
                         const specmc_smc_config* cfg, specmc_smc_result* out, char* err, size_t errlen);

/* ---- particle-sharded runs (multi-GPU) -----------------
 * One run's T particles split over shards that exchange a few scalars per
 * tempering phase (ESS bisection sums, weight max / sums, per-shard weight
 * totals for the global systematic resampling, step statistics).  The
 * reference runs these as one process (smc.cpp:55-183); the split keeps its
 * arithmetic: global ESS / evidence / resampling positions, Philox streams
 * keyed by global particle and chain ids (F is GPU-count invariant up to the
 * order of fp64 sums).
 *   comm == NULL: n_virtual shards on cfg.device in this process (protocol
 *                 check on one GPU); out holds every particle.
 *   comm != NULL: this process is shard `rank` of `world` (one GPU each,
 *                 NCCL collectives); out holds this shard's particles, F and
 *                 the level diagnostics are global.  T % shards == 0. */
typedef struct specmc_comm specmc_comm;
#define SPECMC_COMM_ID_BYTES 128
int specmc_smc_run_sharded(const specmc_model_desc* model, const double* xs, const double* ys, int64_t n_points,
                           const specmc_smc_config* cfg, int32_t n_virtual, specmc_comm* comm,
                           specmc_smc_result* out, char* err, size_t errlen);
/* Batched form: every problem split over the same shards (all K of a model
 * selection at once); out[i] as for specmc_smc_run_sharded. */
int specmc_smc_run_sharded_batch(int32_t n_problems, const specmc_problem* problems, int32_t n_spectra,
                                 const specmc_spectrum* spectra, int32_t n_virtual, specmc_comm* comm,
                                 specmc_smc_result* out, char* err, size_t errlen);
/* NCCL bootstrap: rank 0 creates the id, the host framework broadcasts it
 * (e.g. torch.distributed), every rank then creates its communicator. */
int specmc_nccl_unique_id(uint8_t* out /* SPECMC_COMM_ID_BYTES */, char* err, size_t errlen);
int specmc_comm_init_nccl(int32_t rank, int32_t world, const uint8_t* id, int32_t device, specmc_comm** out,
                          char* err, size_t errlen);
void specmc_comm_destroy(specmc_comm* c);

/* ---- multi-GPU model selection ------------------
 * The reference runs the K range of a model selection serially
 * (cmd_model_select, proj/tools/specmc_main.cpp:147-170).  Here one batch of
 * runs (e.g. every K) is split over the ranks of comm (one GPU each):
 * cost-aware placement (specmc_plan), runs larger than a rank's share
 * particle-sharded over an aligned block of ranks (sub-communicators split
 * from comm with ncclCommSplit and cached in it), everything else one batch per
 * rank; then one all-reduce of the per-run scalars.  Every rank passes the
 * same problem list.  out[i] on every rank: status, F, diverged, levels, d,
 * proposals, trials (summed over shards), device_seconds (CUDA events around
 * this rank's whole call); posterior/energies/diagnostics only on the ranks
 * that ran run i (a shard's particles for a sharded run), NULL elsewhere.
 * plan_rank0 / plan_shards (optional, n_problems each): the placement. */
int specmc_smc_run_distributed(int32_t n_problems, const specmc_problem* problems, int32_t n_spectra,
                               const specmc_spectrum* spectra, specmc_comm* comm, int32_t* plan_rank0,
                               int32_t* plan_shards, specmc_smc_result* out, char* err, size_t errlen);
/* The placement alone (host only, no device): costs[i] (T d N for the
 * distributed entry), T[i] and n[i] (shards keep whole chains) on `world`
 * ranks -> first rank and shard count per run, per-rank load, max load. */
int specmc_plan(int32_t n_runs, const double* costs, const int64_t* T, const int32_t* n_sweeps, int32_t world,
                int32_t* rank0, int32_t* shards, double* rank_load, double* makespan);

/* ---- replica exchange MC: the paper's comparator --
 * RemcConfig (proj/include/specmc/remc.hpp:14-22): L replicas above beta = 0
 * on the geometric ladder (remc.cpp:22-30) unless `ladder` (n_ladder entries,
 * 0 ... 1, strictly increasing) is given; total_sweeps sweeps, the first
 * round(burn_in_fraction * total_sweeps) adapting the step sizes
 * (Robbins-Monro) and discarded; a swap step every swap_period sweeps.
 * Results (RunReport of remc_run, remc.cpp:170-190): F = -sum_l log mean
 * exp(-(beta_{l+1} - beta_l) N E_l) over the retained sweeps, the ladder, the
 * swap rate per pair, the post-burn-in acceptance per replica and the
 * beta = 1 draws (d x draws, column-major).  Every run of a batch executes
 * concurrently: one chain unit per replica, one sweep of every replica per
 * launch.  Parity with the reference's remc_run is statistical (Philox). */
typedef struct {
  int32_t L;
  const double* ladder;
  int32_t n_ladder;
  int64_t total_sweeps;
  double burn_in_fraction;
  int64_t swap_period;
  uint64_t seed;
  int32_t workers; /* echoed only */
  int32_t device;
} specmc_remc_config;

typedef struct {
  specmc_model_desc model;
  int32_t spectrum;
  specmc_remc_config cfg;
} specmc_remc_problem;

typedef struct {
  int32_t status;
  double F;
  int32_t diverged;
  double wall_seconds;
  double device_seconds;
  int32_t R;          /* replicas (ladder entries) */
  int32_t d;
  int64_t draws;      /* retained sweeps */
  double* ladder;     /* R */
  double* swap_rate;  /* R - 1 */
  double* replica_acc; /* R */
  double* posterior;  /* d * draws */
} specmc_remc_result;

int specmc_remc_run_batch(int32_t n_problems, const specmc_remc_problem* problems, int32_t n_spectra,
                          const specmc_spectrum* spectra, specmc_remc_result* out, char* err, size_t errlen);
void specmc_remc_result_free(specmc_remc_result* r);

/* ---- parity units (each runs the same device code as the sampler) ------ */

/* Batched full energies E(theta) for fixed parameters: the K2 kernel.
 * Replaces Problem::energy / BlockEvaluator::full (proj/include/specmc/energy.hpp:47;
 * proj/src/energy.cpp:43-55) composed with data_energy (energy.cpp:7-28).
 * thetas: n_thetas rows of length d (row-major). */
int specmc_energy_batch(const specmc_model_desc* model, const double* xs, const double* ys, int64_t n_points,
                        const double* thetas, int64_t n_thetas, int32_t device, double* energies_out, char* err,
                        size_t errlen);

/* double ess(const ArrayXd& log_weights) -- proj/src/smc.cpp:61-66 */
int specmc_ess(const double* log_weights, int64_t n, int32_t device, double* out, char* err, size_t errlen);

/* double log_mean_exp(const ArrayXd&) -- proj/include/specmc/math.hpp:28-30 */
int specmc_log_mean_exp(const double* v, int64_t n, int32_t device, double* out, char* err, size_t errlen);

/* double next_beta(energies, n_data, beta_prev, ess_target) -- smc.cpp:68-93 */
int specmc_next_beta(const double* energies, int64_t n, double n_data, double beta_prev, double ess_target,
                     int32_t device, double* beta_out, char* err, size_t errlen);

/* std::vector<Index> systematic_resample(log_weights, S, rng) -- smc.cpp:95-112,
 * with the uniform u = rng.uniform01() passed explicitly. */
int specmc_systematic_resample(const double* log_weights, int64_t n, int64_t S, double u, int32_t device,
                               int64_t* ancestors_out, char* err, size_t errlen);

/* VectorXd predict_step_size(history, beta_next, params) -- proj/src/mcmc.cpp:20-53.
 * History arrays are [H][d] row-major, oldest first. */
int specmc_predict_step_size(const double* hist_beta, const double* hist_acc, const double* hist_step, int32_t H,
                             const specmc_model_desc* model, double beta_next, int32_t device, double* out,
                             char* err, size_t errlen);

/* void validate_smc_config(const SmcConfig&) -- smc.cpp:23-32 (host only,
 * no device needed). */
int specmc_validate_config(const specmc_smc_config* cfg, char* err, size_t errlen);

/* validate_model (proj/src/model.cpp:97-113) + validate_spectrum
 * (proj/src/spectrum.cpp:12-23) as make_problem does (energy.cpp:141-143). */
int specmc_validate_problem(const specmc_model_desc* model, const double* xs, const double* ys, int64_t n_points,
                            char* err, size_t errlen);

/* ---- runtime info / instrumentation ------------------------------------ */
typedef struct {
  int64_t kernel_launches;  /* kernels launched by the library since reset */
  double move_kernel_ms;    /* CUDA-event time summed over move-kernel launches */
  int64_t move_launches;
  double point_evals;       /* trials x N summed over move launches */
  double move_mufu_ops;     /* MUFU lane-ops the move kernel executed (shape evaluations and noise
                               terms over the padded point slots; the SFU roofline numerator) */
} specmc_stats;

int specmc_stats_get(specmc_stats* out);
void specmc_stats_reset(void);

/* Launch shape the library picks for a spectrum of n points:
 * warps per chain, points per lane, chains per CTA. */
int specmc_launch_shape(int64_t n_points, int32_t* warps_per_chain, int32_t* points_per_lane,
                        int32_t* chains_per_cta);

/* Measured MUFU (ex2) throughput of the device in operations per second:
 * the SFU roofline denominator of the move kernel (bench.py). */
int specmc_probe_mufu(int32_t device, double* ops_per_second, char* err, size_t errlen);

int specmc_device_count(void);
const char* specmc_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SPECMC_B200_H */
