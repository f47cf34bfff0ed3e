// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNCHANGED reference sources
// (/root/reference/proj/src/*.cpp, compiled by oracle/build_ref.sh against
// oracle/eigen_shim into oracle/_ref/libspecmc_ref.so).  Used by tests/ to pin
// the C restatement (oracle/specmc_oracle.c) and by bench.py's cpu_baseline /
// --impl reference legs as the reference CPU path.  Nothing in the product
// links this.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

#include "specmc/bench.hpp"
#include "specmc/energy.hpp"
#include "specmc/mcmc.hpp"
#include "specmc/posterior.hpp"
#include "specmc/report.hpp"
#include "specmc/smc.hpp"
#include "specmc/synthetic.hpp"

using namespace specmc;

namespace {

enum { FAM_GM = 0, FAM_XPS = 1, FAM_XRD = 2, FAM_OFFSET = 3 };

PriorSpec make_prior(int kind, double a, double b) {
  if (kind == 0) return NormalPrior{a, b};
  if (kind == 1) return GammaPrior{a, b};
  return UniformPrior{a, b};
}

NoiseSpec make_noise(int kind, double sigma, double s0, double s1, double s2, int lit) {
  switch (kind) {
    case 0: return GaussianFixedNoise{sigma};
    case 1: return PoissonNoise{};
    case 2: return GaussianApproxPoissonNoise{};
    default: return XpsHeteroNoise{s0, s1, s2, lit != 0};
  }
}

std::vector<PhaseRef> make_phases(int K, int n_refl, const int* ph, const double* mu, const double* ri) {
  std::vector<PhaseRef> phases(K);
  for (int k = 0; k < K; ++k) phases[k].name = "phase" + std::to_string(k + 1);
  for (int q = 0; q < n_refl; ++q) phases[ph[q]].reflections.push_back(Reflection{mu[q], ri[q]});
  return phases;
}

// layout names exactly as gm_model / xps_model / xrd_model write them (model.cpp:121-189)
ModelSpec make_spec(int family, int K, const int* pk, const double* pa, const double* pb,
                    NoiseSpec noise, int n_refl = 0, const int* ph = nullptr, const double* mu = nullptr,
                    const double* ri = nullptr) {
  ModelSpec s;
  s.family = family == FAM_GM ? Family::GaussianMixture
                              : (family == FAM_XRD ? Family::XrdPseudoVoigt : Family::XpsShirley);
  s.K = K;
  s.noise = noise;
  int i = 0;
  if (family == FAM_XRD) {
    s.phases = make_phases(K, n_refl, ph, mu, ri);
    for (int k = 1; k <= K; ++k)
      for (const char* stem : {"A", "d2t", "r", "alpha", "u", "v", "w", "s", "t"}) {
        s.layout.push_back({std::string(stem) + std::to_string(k), make_prior(pk[i], pa[i], pb[i])});
        ++i;
      }
    for (const char* nm : {"bg_a", "bg_sigma", "bg_r", "bg_b"}) {
      s.layout.push_back({nm, make_prior(pk[i], pa[i], pb[i])});
      ++i;
    }
    validate_model(s);
    return s;
  }
  for (int k = 1; k <= K; ++k) {
    if (family == FAM_GM) {
      for (const char* stem : {"A", "mu", "b"}) {
        s.layout.push_back({std::string(stem) + std::to_string(k), make_prior(pk[i], pa[i], pb[i])});
        ++i;
      }
    } else {
      for (const char* stem : {"A", "mu", "sigma", "eta"}) {
        s.layout.push_back({std::string(stem) + std::to_string(k), make_prior(pk[i], pa[i], pb[i])});
        ++i;
      }
    }
  }
  if (family == FAM_XPS) {
    s.layout.push_back({"bg_a", make_prior(pk[i], pa[i], pb[i])});
    ++i;
    s.layout.push_back({"bg_b", make_prior(pk[i], pa[i], pb[i])});
  }
  validate_model(s);
  return s;
}

Spectrum make_data(const double* xs, const double* ys, int64_t n) {
  Spectrum d;
  d.xs = ArrayXd(xs, n);
  d.ys = ArrayXd(ys, n);
  return d;
}

// the conjugate-mean test problem (tests/conjugate_oracle.hpp:19-28)
Problem conjugate_problem(const double* ys, int64_t n, double sigma, double m0, double v0) {
  const double s2 = sigma * sigma;
  const ArrayXd data(ys, n);
  const double nd = static_cast<double>(n);
  return make_custom_problem({{"theta", NormalPrior{m0, v0}}}, nd,
                             [data, s2, nd](const VectorXd& th) {
                               return 0.5 * std::log(2.0 * M_PI * s2) +
                                      (data - th[0]).square().sum() / (2.0 * s2 * nd);
                             });
}

int fail(const std::exception& e, char* err, size_t errlen) {
  if (err && errlen) {
    std::strncpy(err, e.what(), errlen - 1);
    err[errlen - 1] = 0;
  }
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 2;
  return 3;
}

}  // namespace

extern "C" {

typedef struct {
  int family, K, d, noise;
  double sigma, s0, s1, s2;
  int paper_literal;
  const int* prior_kind;
  const double* prior_a;
  const double* prior_b;
  const double* xs;
  const double* ys;
  int64_t n;
  int n_refl;
  const int* refl_phase;
  const double* refl_mu;
  const double* refl_int;
} ref_model;

#define REF_SPEC(m)                                                                                          \
  make_spec((m)->family, (m)->K, (m)->prior_kind, (m)->prior_a, (m)->prior_b,                               \
            make_noise((m)->noise, (m)->sigma, (m)->s0, (m)->s1, (m)->s2, (m)->paper_literal), (m)->n_refl, \
            (m)->refl_phase, (m)->refl_mu, (m)->refl_int)

typedef struct {
  double F;
  int diverged;
  int levels;
  double wall_seconds;
  double* ladder;      // capacity max_levels + 1
  double* ess_ratio;   // capacity max_levels
  double* log_mean_w;
  double* acc_rate;
  double* thetas;      // d * T (column-major), may be NULL
  double* energies;    // T, may be NULL
} ref_result;

double ref_energy(const ref_model* m, const double* theta) {
  if (m->family == FAM_OFFSET) {
    Problem p = conjugate_problem(m->ys, m->n, m->sigma, 0.0, 1.0);
    VectorXd th(1);
    th[0] = theta[0];
    return p.energy(th);
  }
  ModelSpec spec = REF_SPEC(m);
  VectorXd th(theta, m->d);
  return energy(spec, th, make_data(m->xs, m->ys, m->n));
}

int ref_forward(const ref_model* m, const double* theta, double* f_out, char* err, size_t errlen) {
  try {
    ModelSpec spec = REF_SPEC(m);
    VectorXd th(theta, m->d);
    ArrayXd f = model_forward(spec, th, ArrayXd(m->xs, m->n));
    std::memcpy(f_out, f.data(), sizeof(double) * static_cast<size_t>(m->n));
    return 0;
  } catch (const std::exception& e) {
    return fail(e, err, errlen);
  }
}

double ref_data_energy(int noise, double sigma, double s0, double s1, double s2, int lit,
                       const double* ys, const double* f, int64_t n) {
  return data_energy(make_noise(noise, sigma, s0, s1, s2, lit), ArrayXd(ys, n), ArrayXd(f, n));
}

double ref_ess(const double* lw, int64_t n, int* rc) {
  try {
    return ess(ArrayXd(lw, n));
  } catch (const std::exception& e) {
    *rc = fail(e, nullptr, 0);
    return 0.0;
  }
}

double ref_log_mean_exp(const double* v, int64_t n) { return log_mean_exp(ArrayXd(v, n)); }

double ref_next_beta(const double* E, int64_t T, double n_data, double beta_prev, double target,
                     int* rc) {
  try {
    return next_beta(ArrayXd(E, T), n_data, beta_prev, target);
  } catch (const std::exception& e) {
    *rc = fail(e, nullptr, 0);
    return 0.0;
  }
}

int ref_systematic_resample(const double* lw, int64_t T, int64_t S, uint64_t seed, int64_t* out) {
  try {
    Rng rng(seed);
    auto idx = systematic_resample(ArrayXd(lw, T), S, rng);
    for (int64_t j = 0; j < S; ++j) out[j] = idx[static_cast<size_t>(j)];
    return 0;
  } catch (const std::exception& e) {
    return fail(e, nullptr, 0);
  }
}

double ref_uniform01(uint64_t seed) {
  Rng r(seed);
  return r.uniform01();
}

void ref_predict_step_size(const double* hbeta, const double* hacc, const double* hstep, int H,
                           int d, double beta_next, const int* pk, const double* pa,
                           const double* pb, double* out) {
  std::vector<StepHistoryEntry> hist;
  for (int j = 0; j < H; ++j) {
    StepHistoryEntry h;
    h.beta = hbeta[j];
    h.acc_rate = VectorXd(hacc + static_cast<size_t>(j) * d, d);
    h.step = VectorXd(hstep + static_cast<size_t>(j) * d, d);
    hist.push_back(h);
  }
  std::vector<ScalarParam> params;
  for (int i = 0; i < d; ++i) params.push_back({"p" + std::to_string(i), make_prior(pk[i], pa[i], pb[i])});
  VectorXd p = predict_step_size(hist, beta_next, params);
  for (int i = 0; i < d; ++i) out[i] = p[i];
}

double ref_rm_update(double step, int accepted, long long t) {
  StepState st(VectorXd::Constant(1, step));
  robbins_monro_update(st, 0, accepted != 0, t);
  return st.step[0];
}

// smc_run(spec, data, cfg) (smc.cpp:218) or, for the offset family, the
// Problem-level smc_run over the conjugate problem (smc.cpp:213)
int ref_smc_run(const ref_model* m, int64_t T, int n, double ess_target, int max_levels,
                uint64_t seed, int workers, ref_result* out, char* err, size_t errlen) {
  try {
    SmcConfig cfg;
    cfg.T = T;
    cfg.n = n;
    cfg.ess_target = ess_target;
    cfg.max_levels = max_levels;
    cfg.seed = seed;
    cfg.workers = workers;
    MatrixXd post;
    ArrayXd energies;
    std::vector<double> ladder, less, lmw, lacc;
    if (m->family == FAM_OFFSET) {
      Problem p = conjugate_problem(m->ys, m->n, m->sigma, m->prior_a[0], m->prior_b[0]);
      SmcResult r = smc_run(p, cfg);
      out->F = r.F;
      out->diverged = r.diverged;
      out->wall_seconds = r.wall_seconds;
      ladder.push_back(0.0);
      for (auto& lv : r.levels) {
        ladder.push_back(lv.beta);
        less.push_back(lv.ess_ratio);
        lmw.push_back(lv.log_mean_w);
        lacc.push_back(lv.acc_rate);
      }
      post = std::move(r.thetas);
      energies = std::move(r.energies);
    } else {
      ModelSpec spec = REF_SPEC(m);
      RunReport r = smc_run(spec, make_data(m->xs, m->ys, m->n), cfg);
      out->F = r.F;
      out->diverged = r.diverged;
      out->wall_seconds = r.wall_seconds;
      const auto& lad = r.arrays.at("ladder");
      for (Index i = 0; i < lad.size(); ++i) ladder.push_back(lad[i]);
      const auto& a1 = r.arrays.at("level_ess_ratio");
      const auto& a2 = r.arrays.at("level_log_mean_w");
      const auto& a3 = r.arrays.at("level_acc_rate");
      for (Index i = 0; i < a1.size(); ++i) {
        less.push_back(a1[i]);
        lmw.push_back(a2[i]);
        lacc.push_back(a3[i]);
      }
      post = std::move(r.posterior);
    }
    out->levels = static_cast<int>(less.size());
    for (size_t i = 0; i < ladder.size(); ++i) out->ladder[i] = ladder[i];
    for (size_t i = 0; i < less.size(); ++i) {
      out->ess_ratio[i] = less[i];
      out->log_mean_w[i] = lmw[i];
      out->acc_rate[i] = lacc[i];
    }
    if (out->thetas) std::memcpy(out->thetas, post.data(), sizeof(double) * static_cast<size_t>(post.size()));
    if (out->energies && energies.size() == T)
      std::memcpy(out->energies, energies.data(), sizeof(double) * static_cast<size_t>(T));
    return 0;
  } catch (const std::exception& e) {
    return fail(e, err, errlen);
  }
}

// gen_xps(k_true, seed, noise) (synthetic.cpp:270-318): 840 points
int ref_gen_xps(int k_true, uint64_t seed, double s0, double s1, double s2, double* xs, double* ys) {
  try {
    SyntheticDataset ds = gen_xps(k_true, seed, XpsHeteroNoise{s0, s1, s2, false});
    std::memcpy(xs, ds.data.xs.data(), sizeof(double) * 840);
    std::memcpy(ys, ds.data.ys.data(), sizeof(double) * 840);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, nullptr, 0);
  }
}

// xps_model(K, data, noise) priors (model.cpp:169-189)
int ref_xps_model_priors(int K, const double* xs, const double* ys, int64_t n, int* pk, double* pa,
                         double* pb) {
  ModelSpec s = xps_model(K, make_data(xs, ys, n));
  for (size_t i = 0; i < s.layout.size(); ++i) {
    const auto& p = s.layout[i].prior;
    if (auto* a = std::get_if<NormalPrior>(&p)) { pk[i] = 0; pa[i] = a->mean; pb[i] = a->var; }
    else if (auto* g = std::get_if<GammaPrior>(&p)) { pk[i] = 1; pa[i] = g->shape; pb[i] = g->rate; }
    else { auto& u = std::get<UniformPrior>(p); pk[i] = 2; pa[i] = u.lo; pb[i] = u.hi; }
  }
  return static_cast<int>(s.layout.size());
}

// xrd_model(phases, data, noise) priors (model.cpp:138-167)
int ref_xrd_model_priors(int K, int n_refl, const int* ph, const double* mu, const double* ri, const double* xs,
                         const double* ys, int64_t n, int* pk, double* pa, double* pb) {
  ModelSpec s = xrd_model(make_phases(K, n_refl, ph, mu, ri), make_data(xs, ys, n), PoissonNoise{});
  for (size_t i = 0; i < s.layout.size(); ++i) {
    const auto& p = s.layout[i].prior;
    if (auto* a = std::get_if<NormalPrior>(&p)) { pk[i] = 0; pa[i] = a->mean; pb[i] = a->var; }
    else if (auto* g = std::get_if<GammaPrior>(&p)) { pk[i] = 1; pa[i] = g->shape; pb[i] = g->rate; }
    else { auto& u = std::get<UniformPrior>(p); pk[i] = 2; pa[i] = u.lo; pb[i] = u.hi; }
  }
  return static_cast<int>(s.layout.size());
}

// gen_xrd(n_points, seed) (synthetic.cpp:230-268): three TiO2 phases, Poisson counts
int ref_gen_xrd(int64_t n_points, uint64_t seed, double* xs, double* ys) {
  try {
    SyntheticDataset ds = gen_xrd(n_points, seed);
    std::memcpy(xs, ds.data.xs.data(), sizeof(double) * static_cast<size_t>(n_points));
    std::memcpy(ys, ds.data.ys.data(), sizeof(double) * static_cast<size_t>(n_points));
    return 0;
  } catch (const std::exception& e) {
    return fail(e, nullptr, 0);
  }
}

int ref_gm_model_priors(int K, double x_lo, double x_hi, double sigma, int uniform_mu, int* pk,
                        double* pa, double* pb) {
  ModelSpec s = gm_model(K, x_lo, x_hi, sigma, uniform_mu ? GmMuPrior::UniformRange : GmMuPrior::Normal15);
  for (size_t i = 0; i < s.layout.size(); ++i) {
    const auto& p = s.layout[i].prior;
    if (auto* a = std::get_if<NormalPrior>(&p)) { pk[i] = 0; pa[i] = a->mean; pb[i] = a->var; }
    else if (auto* g = std::get_if<GammaPrior>(&p)) { pk[i] = 1; pa[i] = g->shape; pb[i] = g->rate; }
    else { auto& u = std::get<UniformPrior>(p); pk[i] = 2; pa[i] = u.lo; pb[i] = u.hi; }
  }
  return static_cast<int>(s.layout.size());
}

// model_select over (K, F, diverged) rows (posterior.cpp:68-104)
int ref_model_select(int n, const int* ks, const double* fs, const int* diverged, int* k_best) {
  try {
    std::vector<std::pair<int, RunReport>> reps;
    for (int i = 0; i < n; ++i) {
      RunReport r;
      r.F = fs[i];
      r.diverged = diverged[i] != 0;
      reps.emplace_back(ks[i], r);
    }
    *k_best = model_select(reps).K_best;
    return 0;
  } catch (const std::exception& e) {
    return fail(e, nullptr, 0);
  }
}

uint64_t ref_trial_seed(uint64_t base, int trial) {
  // bench.cpp:104-106
  return hash_combine(base, static_cast<std::uint64_t>(trial));
}

int ref_hardware_workers() { return ThreadPool::hardware_workers(); }

// ---- output side: report file format and posterior summaries (report.cpp, posterior.cpp)
int ref_format_double(double v, char* out, int n) {
  const std::string s = format_double(v);
  std::strncpy(out, s.c_str(), (size_t)n - 1);
  out[n - 1] = 0;
  return (int)s.size();
}

double ref_weighted_quantile(const double* s, const double* w, int64_t n, double q, int* rc) {
  *rc = 0;
  try {
    return weighted_quantile(ArrayXd(s, n), ArrayXd(w, n), q);
  } catch (const std::invalid_argument&) {
    *rc = 2;
  }
  return 0.0;
}

int ref_sort_peak_blocks(const double* post, int64_t d, int64_t m, int block, int center_off, int n_blocks,
                         double* out) {
  try {
    MatrixXd P(d, m);
    for (int64_t j = 0; j < m; ++j)
      for (int64_t i = 0; i < d; ++i) P(i, j) = post[j * d + i];
    const MatrixXd R = sort_peak_blocks(P, block, center_off, n_blocks);
    for (int64_t j = 0; j < m; ++j)
      for (int64_t i = 0; i < d; ++i) out[j * d + i] = R(i, j);
    return 0;
  } catch (const std::invalid_argument&) {
    return 2;
  }
}

// posterior: m draws of d values, draw-major (post[j * d + i])
int ref_write_report(const char* path, const char* sampler, const char* label, double F, int diverged, double wall,
                     int n_scalars, const char* const* skeys, const double* svals, int n_arrays,
                     const char* const* akeys, const int64_t* alens, const double* avals, int n_params,
                     const char* const* pnames, int64_t d, int64_t m, const double* post, int64_t max_draws,
                     int n_cfg, const char* const* cfg) {
  try {
    RunReport r;
    r.sampler = sampler;
    r.label = label;
    r.F = F;
    r.diverged = diverged != 0;
    r.wall_seconds = wall;
    for (int i = 0; i < n_scalars; ++i) r.scalars[skeys[i]] = svals[i];
    int64_t at = 0;
    for (int a = 0; a < n_arrays; ++a) {
      VectorXd v(alens[a]);
      for (int64_t i = 0; i < alens[a]; ++i) v[i] = avals[at + i];
      at += alens[a];
      r.arrays[akeys[a]] = v;
    }
    for (int i = 0; i < n_params; ++i) r.param_names.push_back(pnames[i]);
    r.posterior = MatrixXd(d, m);
    for (int64_t j = 0; j < m; ++j)
      for (int64_t i = 0; i < d; ++i) r.posterior(i, j) = post[j * d + i];
    for (int i = 0; i < n_cfg; ++i) r.config_lines.push_back(cfg[i]);
    write_report(r, path, max_draws);
    return 0;
  } catch (const std::exception&) {
    return 3;
  }
}

// ---- replica exchange (remc.cpp:78-190): F, swap rates, replica acceptance
#include "specmc/remc.hpp"
int ref_remc_run(const ref_model* m, int L, int64_t total_sweeps, double burn, int64_t swap_period, uint64_t seed,
                 int workers, double* F, int* diverged, double* swap_rate, double* replica_acc, double* wall, char* err,
                 size_t errlen) {
  try {
    RemcConfig cfg;
    cfg.L = L;
    cfg.total_sweeps = total_sweeps;
    cfg.burn_in_fraction = burn;
    cfg.swap_period = swap_period;
    cfg.seed = seed;
    cfg.workers = workers;
    RemcResult r;
    if (m->family == FAM_OFFSET) {
      r = remc_run(conjugate_problem(m->ys, m->n, m->sigma, m->prior_a[0], m->prior_b[0]), cfg);
    } else {
      ModelSpec spec = REF_SPEC(m);
      r = remc_run(make_problem(spec, make_data(m->xs, m->ys, m->n)), cfg);
    }
    *F = r.F;
    *diverged = r.diverged;
    *wall = r.wall_seconds;
    for (Index i = 0; i < r.swap_rate.size(); ++i) swap_rate[i] = r.swap_rate[i];
    for (Index i = 0; i < r.replica_acc.size(); ++i) replica_acc[i] = r.replica_acc[i];
    return 0;
  } catch (const std::exception& e) {
    return fail(e, err, errlen);
  }
}

// ---- benchmark tables (bench.cpp:147-338) over persisted reports
namespace {
int copy_out(const std::string& s, char* out, size_t outlen) {
  if (s.size() + 1 > outlen) return -(int)(s.size() + 1);
  std::memcpy(out, s.c_str(), s.size() + 1);
  return (int)s.size();
}
}  // namespace

// table_from_reports + bench_table_text; returns the text length (or -needed)
int ref_bench_table(const char* const* paths, int n, const char* ref_label, char* out, size_t outlen) {
  try {
    std::vector<RunReport> runs;
    for (int i = 0; i < n; ++i) runs.push_back(read_report(paths[i]));
    return copy_out(bench_table_text(table_from_reports(runs, ref_label)), out, outlen);
  } catch (const std::exception& e) {
    copy_out(std::string("error: ") + e.what(), out, outlen);
    return -1000000;
  }
}

// ci_error_curve + ci_table_text
int ref_ci_table(const char* const* paths, int n, const char* truth_path, const char* param, double level, char* out,
                 size_t outlen) {
  try {
    std::vector<RunReport> runs;
    for (int i = 0; i < n; ++i) runs.push_back(read_report(paths[i]));
    return copy_out(ci_table_text(ci_error_curve(runs, read_report(truth_path), param, level)), out, outlen);
  } catch (const std::exception& e) {
    copy_out(std::string("error: ") + e.what(), out, outlen);
    return -1000000;
  }
}

}  // extern "C"
