// specmc_b200.hpp -- header-only C++ mirror of the reference interface over the C ABI.
//
// Same names, argument meaning and error behaviour as the reference
// ("specmc", arxiv/paper_2604_03271; paths relative to the reference root):
//   ModelSpec / priors / noise      proj/include/specmc/{model,priors}.hpp
//   gm_model, xps_model             proj/src/model.cpp:121-136, :169-189
//   SmcConfig, smc_run -> RunReport proj/include/specmc/smc.hpp:12-21, :78; proj/src/smc.cpp:218-249
//   model_select                    proj/src/posterior.cpp:68-104
//   RemcConfig, remc_run            proj/include/specmc/remc.hpp:14-22; proj/src/remc.cpp:170-190
// Vectors replace Eigen types; the posterior is d x T column-major as the
// reference's MatrixXd.  Config/model/spectrum violations throw
// std::invalid_argument, numeric failures (max_levels, zero weight) and CUDA
// failures throw std::runtime_error.  Link with paper_2604_03271_b200/libspecmc_b200.so.
#pragma once

#include <cmath>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "specmc_b200.h"

namespace specmc_b200 {

struct NormalPrior {
  double mean, var;
};
struct GammaPrior {
  double shape, rate;
};
struct UniformPrior {
  double lo, hi;
};
using PriorSpec = std::variant<NormalPrior, GammaPrior, UniformPrior>;

struct ScalarParam {
  std::string name;
  PriorSpec prior;
};

struct GaussianFixedNoise {
  double sigma;
};
struct PoissonNoise {};
struct GaussianApproxPoissonNoise {};
struct XpsHeteroNoise {
  double s0 = 1.0, s1 = 0.01, s2 = 0.0;
  bool paper_literal = false;
};
using NoiseSpec = std::variant<GaussianFixedNoise, PoissonNoise, GaussianApproxPoissonNoise, XpsHeteroNoise>;

enum class Family { GaussianMixture, XrdPseudoVoigt, XpsShirley, ConjugateOffset };

struct Reflection {  // model.hpp:28-31
  double mu_ref;         // degrees 2theta
  double rel_intensity;  // >= 0
};
struct PhaseRef {  // model.hpp:32-35
  std::string name;
  std::vector<Reflection> reflections;
};

struct ModelSpec {  // model.hpp:50-56
  Family family = Family::GaussianMixture;
  int K = 0;  // peaks (gm, xps) or phases (xrd)
  std::vector<PhaseRef> phases;
  std::vector<ScalarParam> layout;
  NoiseSpec noise = GaussianFixedNoise{1.0};
};

struct Spectrum {
  std::vector<double> xs, ys;
};

struct SmcConfig {
  std::int64_t T = 10000;
  int n = 10;
  double ess_target = 0.5;
  int max_levels = 2000;
  std::uint64_t seed = 0;
  int workers = 1;
  int device = 0;
};

struct RunReport {
  std::string sampler = "smc";
  std::string label;
  double F = NAN;
  bool diverged = false;
  double wall_seconds = 0.0;
  double device_seconds = 0.0;
  std::vector<std::string> param_names;
  std::map<std::string, double> scalars;
  std::map<std::string, std::vector<double>> arrays;
  std::vector<double> posterior;  // d x T, column-major
  std::int64_t d = 0, T = 0;
  std::vector<std::string> config_lines;  // report.hpp:26, the config echo
};

enum class GmMuPrior { Normal15, UniformRange };

inline ModelSpec gm_model(int K, double x_lo, double x_hi, double noise_sigma, GmMuPrior mu_kind) {
  ModelSpec s;
  s.family = Family::GaussianMixture;
  s.K = K;
  s.noise = GaussianFixedNoise{noise_sigma};
  const PriorSpec mu = mu_kind == GmMuPrior::Normal15 ? PriorSpec(NormalPrior{1.5, 0.2})
                                                      : PriorSpec(UniformPrior{x_lo, x_hi});
  for (int k = 1; k <= K; ++k) {
    s.layout.push_back({"A" + std::to_string(k), GammaPrior{5.0, 5.0}});
    s.layout.push_back({"mu" + std::to_string(k), mu});
    s.layout.push_back({"b" + std::to_string(k), GammaPrior{5.0, 0.04}});
  }
  return s;
}

inline ModelSpec xps_model(int K, const Spectrum& data, XpsHeteroNoise noise = {}) {
  if (data.ys.empty()) throw std::invalid_argument("xps_model: empty spectrum");
  ModelSpec s;
  s.family = Family::XpsShirley;
  s.K = K;
  s.noise = noise;
  double ymax = data.ys[0], ymin = data.ys[0];
  for (double y : data.ys) {
    ymax = y > ymax ? y : ymax;
    ymin = y < ymin ? y : ymin;
  }
  const double yf = data.ys.front(), yl = data.ys.back();
  for (int k = 1; k <= K; ++k) {
    s.layout.push_back({"A" + std::to_string(k), UniformPrior{std::max(0.0, 0.3 * ymin), 1.05 * ymax}});
    s.layout.push_back({"mu" + std::to_string(k), UniformPrior{data.xs.front(), data.xs.back()}});
    s.layout.push_back({"sigma" + std::to_string(k), UniformPrior{0.1, 15.0}});
    s.layout.push_back({"eta" + std::to_string(k), UniformPrior{0.0, 1.0}});
  }
  s.layout.push_back({"bg_a", UniformPrior{0.95 * yf, 1.01 * yf}});
  s.layout.push_back({"bg_b", UniformPrior{0.95 * yl, 1.01 * yl}});
  return s;
}

// model.cpp:138-167: K = phases.size() phases (A, d2t, r, alpha, u, v, w, s, t),
// then the background block (bg_a, bg_sigma, bg_r, bg_b)
inline ModelSpec xrd_model(std::vector<PhaseRef> phases, const Spectrum& data, NoiseSpec noise = PoissonNoise{}) {
  if (data.ys.empty()) throw std::invalid_argument("xrd_model: empty spectrum");
  ModelSpec s;
  s.family = Family::XrdPseudoVoigt;
  s.K = static_cast<int>(phases.size());
  s.phases = std::move(phases);
  s.noise = noise;
  double ymax = data.ys[0], ymin = data.ys[0];
  for (double y : data.ys) {
    ymax = y > ymax ? y : ymax;
    ymin = y < ymin ? y : ymin;
  }
  if (!(ymax > ymin)) throw std::invalid_argument("xrd model: degenerate intensity range");
  const double ymin_pos = ymin > 0.0 ? ymin : 0.0;
  for (int k = 1; k <= s.K; ++k) {
    const std::string i = std::to_string(k);
    s.layout.push_back({"A" + i, GammaPrior{4.0, 4.0 / (ymax - ymin)}});
    s.layout.push_back({"d2t" + i, NormalPrior{0.0, 0.05 * 0.05}});
    s.layout.push_back({"r" + i, UniformPrior{0.0, 1.0}});
    s.layout.push_back({"alpha" + i, GammaPrior{5.0, 4.0}});
    s.layout.push_back({"u" + i, GammaPrior{1.0, 10.0}});
    s.layout.push_back({"v" + i, GammaPrior{1.0, 10.0}});
    s.layout.push_back({"w" + i, GammaPrior{2.0, 20.0}});
    s.layout.push_back({"s" + i, GammaPrior{2.0, 20.0}});
    s.layout.push_back({"t" + i, GammaPrior{1.0, 10.0}});
  }
  double half = std::sqrt(ymin_pos);
  if (!(half > 0.0)) half = 1.0;
  s.layout.push_back({"bg_a", GammaPrior{2.0, 1.0 / ymax}});
  s.layout.push_back({"bg_sigma", GammaPrior{2.0, 0.4}});
  s.layout.push_back({"bg_r", UniformPrior{0.0, 1.0}});
  s.layout.push_back({"bg_b", UniformPrior{ymin - half, ymin + half}});
  return s;
}

namespace detail {

struct Desc {
  specmc_model_desc d{};
  std::vector<std::int32_t> k;
  std::vector<double> a, b;
  std::vector<std::int32_t> refl_phase;  // xrd reflections, flattened in phase order
  std::vector<double> refl_mu, refl_int;
};

inline Desc to_desc(const ModelSpec& spec) {
  Desc D;
  for (const auto& p : spec.layout) {
    if (auto* n = std::get_if<NormalPrior>(&p.prior)) {
      D.k.push_back(SPECMC_PRIOR_NORMAL);
      D.a.push_back(n->mean);
      D.b.push_back(n->var);
    } else if (auto* g = std::get_if<GammaPrior>(&p.prior)) {
      D.k.push_back(SPECMC_PRIOR_GAMMA);
      D.a.push_back(g->shape);
      D.b.push_back(g->rate);
    } else {
      const auto& u = std::get<UniformPrior>(p.prior);
      D.k.push_back(SPECMC_PRIOR_UNIFORM);
      D.a.push_back(u.lo);
      D.b.push_back(u.hi);
    }
  }
  specmc_model_desc& d = D.d;
  switch (spec.family) {
    case Family::GaussianMixture: d.family = SPECMC_FAMILY_GM; break;
    case Family::XpsShirley: d.family = SPECMC_FAMILY_XPS; break;
    case Family::XrdPseudoVoigt: d.family = SPECMC_FAMILY_XRD; break;
    case Family::ConjugateOffset: d.family = SPECMC_FAMILY_OFFSET; break;
  }
  d.K = spec.K;
  d.d = static_cast<std::int32_t>(spec.layout.size());
  if (auto* g = std::get_if<GaussianFixedNoise>(&spec.noise)) {
    d.noise = SPECMC_NOISE_GAUSSIAN;
    d.noise_sigma = g->sigma;
  } else if (std::holds_alternative<PoissonNoise>(spec.noise)) {
    d.noise = SPECMC_NOISE_POISSON;
  } else if (std::holds_alternative<GaussianApproxPoissonNoise>(spec.noise)) {
    d.noise = SPECMC_NOISE_GAUSS_APPROX;
  } else {
    const auto& h = std::get<XpsHeteroNoise>(spec.noise);
    d.noise = SPECMC_NOISE_XPS_HETERO;
    d.s0 = h.s0;
    d.s1 = h.s1;
    d.s2 = h.s2;
    d.paper_literal = h.paper_literal ? 1 : 0;
  }
  d.prior_kind = D.k.data();
  d.prior_a = D.a.data();
  d.prior_b = D.b.data();
  for (std::size_t b = 0; b < spec.phases.size(); ++b)
    for (const auto& r : spec.phases[b].reflections) {
      D.refl_phase.push_back(static_cast<std::int32_t>(b));
      D.refl_mu.push_back(r.mu_ref);
      D.refl_int.push_back(r.rel_intensity);
    }
  d.n_refl = static_cast<std::int32_t>(D.refl_phase.size());
  d.refl_phase = D.refl_phase.empty() ? nullptr : D.refl_phase.data();
  d.refl_mu = D.refl_mu.empty() ? nullptr : D.refl_mu.data();
  d.refl_int = D.refl_int.empty() ? nullptr : D.refl_int.data();
  return D;
}

[[noreturn]] inline void raise(int rc, const char* err) {
  if (rc == SPECMC_EINVAL) throw std::invalid_argument(err);
  throw std::runtime_error(err);
}

inline RunReport to_report(const ModelSpec& spec, const SmcConfig& cfg, std::size_t n_data,
                           const specmc_smc_result& r) {
  RunReport rep;
  rep.F = r.F;
  rep.diverged = r.diverged != 0;
  rep.wall_seconds = r.wall_seconds;
  rep.device_seconds = r.device_seconds;
  for (const auto& p : spec.layout) rep.param_names.push_back(p.name);
  rep.scalars = {{"T", static_cast<double>(cfg.T)}, {"n", static_cast<double>(cfg.n)},
                 {"ess_target", cfg.ess_target},   {"seed", static_cast<double>(cfg.seed)},
                 {"workers", static_cast<double>(cfg.workers)}, {"n_data", static_cast<double>(n_data)},
                 {"levels", static_cast<double>(r.levels)}};
  rep.arrays["ladder"].assign(r.ladder, r.ladder + r.levels + 1);
  rep.arrays["level_ess_ratio"].assign(r.level_ess_ratio, r.level_ess_ratio + r.levels);
  rep.arrays["level_log_mean_w"].assign(r.level_log_mean_w, r.level_log_mean_w + r.levels);
  rep.arrays["level_acc_rate"].assign(r.level_acc_rate, r.level_acc_rate + r.levels);
  rep.d = r.d;
  rep.T = r.T;
  rep.posterior.assign(r.posterior, r.posterior + r.d * r.T);
  return rep;
}

}  // namespace detail

inline void validate_smc_config(const SmcConfig& cfg) {  // smc.cpp:23-32
  specmc_smc_config c{cfg.T, cfg.n, cfg.ess_target, cfg.max_levels, cfg.seed, cfg.workers, cfg.device};
  char err[512] = {0};
  const int rc = specmc_validate_config(&c, err, sizeof err);
  if (rc) detail::raise(rc, err);
}

// Runs every (spec, spectrum index, cfg) concurrently on one GPU: the K x trials
// loop of cmd_model_select (proj/tools/specmc_main.cpp:148-170) in one call.
struct Problem {
  ModelSpec spec;
  int spectrum = 0;
  SmcConfig cfg;
};

inline std::vector<RunReport> smc_run_batch(const std::vector<Problem>& problems, const std::vector<Spectrum>& spectra) {
  std::vector<detail::Desc> descs;
  descs.reserve(problems.size());
  std::vector<specmc_problem> ps;
  for (const auto& p : problems) {
    descs.push_back(detail::to_desc(p.spec));
    const auto& c = p.cfg;
    ps.push_back({descs.back().d, p.spectrum, {c.T, c.n, c.ess_target, c.max_levels, c.seed, c.workers, c.device}});
  }
  std::vector<specmc_spectrum> ss;
  for (const auto& s : spectra) {
    if (s.xs.size() != s.ys.size()) throw std::invalid_argument("spectrum: xs/ys length mismatch");
    ss.push_back({s.xs.data(), s.ys.data(), static_cast<std::int64_t>(s.xs.size())});
  }
  std::vector<specmc_smc_result> res(problems.size());
  char err[1024] = {0};
  const int rc = specmc_smc_run_batch(static_cast<std::int32_t>(ps.size()), ps.data(),
                                      static_cast<std::int32_t>(ss.size()), ss.data(), res.data(), err, sizeof err);
  if (rc != SPECMC_OK && rc != SPECMC_ERUNTIME) {
    for (auto& r : res) specmc_result_free(&r);
    detail::raise(rc, err);
  }
  std::vector<RunReport> out;
  int first_bad = SPECMC_OK;
  for (std::size_t i = 0; i < problems.size(); ++i) {
    if (res[i].status == SPECMC_OK)
      out.push_back(detail::to_report(problems[i].spec, problems[i].cfg,
                                      spectra[problems[i].spectrum].xs.size(), res[i]));
    else if (first_bad == SPECMC_OK)
      first_bad = res[i].status;
    specmc_result_free(&res[i]);
  }
  if (rc != SPECMC_OK) detail::raise(rc, err);
  return out;
}

// RunReport smc_run(const ModelSpec&, const Spectrum&, const SmcConfig&) -- smc.cpp:218
inline RunReport smc_run(const ModelSpec& spec, const Spectrum& data, const SmcConfig& cfg) {
  return smc_run_batch({Problem{spec, 0, cfg}}, {data}).front();
}

// ---- replica exchange (remc.hpp:14-22, remc.cpp:78-190): the paper's comparator
struct RemcConfig {
  int L = 44;                   // replicas above beta = 0
  std::vector<double> ladder;   // explicit beta_0 .. beta_L; empty = geometric default
  std::int64_t total_sweeps = 10000;
  double burn_in_fraction = 0.5;
  std::int64_t swap_period = 1;  // > total_sweeps disables swaps
  std::uint64_t seed = 0;
  int workers = 1;  // echoed in the report only
  int device = 0;
};

struct RemcProblem {
  ModelSpec spec;
  int spectrum = 0;
  RemcConfig cfg;
};

// every run of the batch concurrently on one GPU (one chain unit per replica)
inline std::vector<RunReport> remc_run_batch(const std::vector<RemcProblem>& problems,
                                             const std::vector<Spectrum>& spectra) {
  std::vector<detail::Desc> descs;
  descs.reserve(problems.size());
  std::vector<specmc_remc_problem> ps;
  for (const auto& p : problems) {
    descs.push_back(detail::to_desc(p.spec));
    const auto& c = p.cfg;
    specmc_remc_config rc{c.L, c.ladder.empty() ? nullptr : c.ladder.data(), static_cast<std::int32_t>(c.ladder.size()),
                          c.total_sweeps, c.burn_in_fraction, c.swap_period, c.seed, c.workers, c.device};
    ps.push_back({descs.back().d, p.spectrum, rc});
  }
  std::vector<specmc_spectrum> ss;
  for (const auto& s : spectra) {
    if (s.xs.size() != s.ys.size()) throw std::invalid_argument("spectrum: xs/ys length mismatch");
    ss.push_back({s.xs.data(), s.ys.data(), static_cast<std::int64_t>(s.xs.size())});
  }
  std::vector<specmc_remc_result> res(problems.size());
  char err[1024] = {0};
  const int rc = specmc_remc_run_batch(static_cast<std::int32_t>(ps.size()), ps.data(),
                                       static_cast<std::int32_t>(ss.size()), ss.data(), res.data(), err, sizeof err);
  std::vector<RunReport> out;
  if (rc == SPECMC_OK) {
    for (std::size_t i = 0; i < problems.size(); ++i) {
      const auto& r = res[i];
      const auto& c = problems[i].cfg;
      RunReport rep;
      rep.sampler = "remc";
      rep.F = r.F;
      rep.diverged = r.diverged != 0;
      rep.wall_seconds = r.wall_seconds;
      rep.device_seconds = r.device_seconds;
      for (const auto& p : problems[i].spec.layout) rep.param_names.push_back(p.name);
      rep.scalars = {{"L", static_cast<double>(r.R - 1)},
                     {"total_sweeps", static_cast<double>(c.total_sweeps)},
                     {"burn_in_fraction", c.burn_in_fraction},
                     {"swap_period", static_cast<double>(c.swap_period)},
                     {"seed", static_cast<double>(c.seed)},
                     {"workers", static_cast<double>(c.workers)},
                     {"n_data", static_cast<double>(spectra[problems[i].spectrum].xs.size())}};
      rep.arrays["ladder"].assign(r.ladder, r.ladder + r.R);
      rep.arrays["swap_rate"].assign(r.swap_rate, r.swap_rate + (r.R > 0 ? r.R - 1 : 0));
      rep.arrays["replica_acc_rate"].assign(r.replica_acc, r.replica_acc + r.R);
      rep.d = r.d;
      rep.T = r.draws;
      rep.posterior.assign(r.posterior, r.posterior + r.d * r.draws);
      out.push_back(std::move(rep));
    }
  }
  for (auto& r : res) specmc_remc_result_free(&r);
  if (rc != SPECMC_OK) detail::raise(rc, err);
  return out;
}

// RunReport remc_run(const ModelSpec&, const Spectrum&, const RemcConfig&) -- remc.cpp:170-190
inline RunReport remc_run(const ModelSpec& spec, const Spectrum& data, const RemcConfig& cfg) {
  return remc_run_batch({RemcProblem{spec, 0, cfg}}, {data}).front();
}

// posterior.cpp:68-104: argmin over K of the mean F; non-finite/diverged K excluded; ties keep the smaller K
inline int model_select(const std::vector<std::pair<int, RunReport>>& reports) {
  if (reports.empty()) throw std::invalid_argument("model_select: no reports");
  std::map<int, std::vector<double>> by_k;
  std::map<int, bool> bad;
  for (const auto& [k, r] : reports) {
    by_k[k].push_back(r.F);
    if (!std::isfinite(r.F) || r.diverged) bad[k] = true;
  }
  int best = 0;
  bool have = false;
  double best_f = INFINITY;
  for (const auto& [k, fs] : by_k) {
    if (bad.count(k)) continue;
    double m = 0.0;
    for (double f : fs) m += f;
    m /= static_cast<double>(fs.size());
    if (!have || m < best_f) {
      have = true;
      best_f = m;
      best = k;
    }
  }
  if (!have) throw std::runtime_error("model_select: every candidate diverged");
  return best;
}

// The on-disk report (report.cpp:33-136) is written and read by the reference's
// own report code: a RunReport filled by smc_run() goes through its
// write_report() unchanged (integration/specmc_b200_cli.cpp links report.cpp).

}  // namespace specmc_b200
