// smc_b200.cpp -- the reference-side adapter of INTEGRATION.md: the
// translation unit a maintainer adds to the reference tree (e.g.
// proj/src/smc_b200.cpp) to run its SMC through this repo's C ABI
// (include/specmc_b200.h).  It uses ONLY the reference's own types
// (specmc::ModelSpec, Spectrum, SmcConfig, RunReport from proj/include) and
// the C ABI; integration/build_adapter.py compiles it against the reference
// headers (and oracle/eigen_shim, Eigen3 being absent here) to prove the
// boundary from the reference side.
//
//   RunReport smc_run_b200(spec, data, cfg, device)      replaces smc_run
//       (proj/include/specmc/smc.hpp:78, proj/src/smc.cpp:218-249)
//   std::vector<RunReport> smc_run_batch_b200(...)        the K x trials loop of
//       cmd_model_select (proj/tools/specmc_main.cpp:147-170) as one batched call
#include "smc_b200.hpp"

#include <cstring>
#include <stdexcept>
#include <variant>

namespace specmc {

namespace {

struct DescBufs {  // storage the descriptor points into
  std::vector<int32_t> k, refl_phase;
  std::vector<double> a, b, refl_mu, refl_int;
};

void to_desc(const ModelSpec& spec, specmc_model_desc& d, DescBufs& s) {
  for (const auto& p : spec.layout) {
    if (const auto* n = std::get_if<NormalPrior>(&p.prior)) {
      s.k.push_back(SPECMC_PRIOR_NORMAL);
      s.a.push_back(n->mean);
      s.b.push_back(n->var);
    } else if (const auto* g = std::get_if<GammaPrior>(&p.prior)) {
      s.k.push_back(SPECMC_PRIOR_GAMMA);
      s.a.push_back(g->shape);
      s.b.push_back(g->rate);
    } else {
      const auto& u = std::get<UniformPrior>(p.prior);
      s.k.push_back(SPECMC_PRIOR_UNIFORM);
      s.a.push_back(u.lo);
      s.b.push_back(u.hi);
    }
  }
  std::memset(&d, 0, sizeof(d));
  d.family = spec.family == Family::GaussianMixture ? SPECMC_FAMILY_GM
             : spec.family == Family::XpsShirley    ? SPECMC_FAMILY_XPS
                                                    : SPECMC_FAMILY_XRD;
  d.K = spec.K;
  d.d = (int32_t)spec.layout.size();
  if (const auto* g = std::get_if<GaussianFixedNoise>(&spec.noise)) {
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
  d.prior_kind = s.k.data();
  d.prior_a = s.a.data();
  d.prior_b = s.b.data();
  for (size_t ph = 0; ph < spec.phases.size(); ++ph)  // xrd: model.hpp:28-35
    for (const auto& r : spec.phases[ph].reflections) {
      s.refl_phase.push_back((int32_t)ph);
      s.refl_mu.push_back(r.mu_ref);
      s.refl_int.push_back(r.rel_intensity);
    }
  d.n_refl = (int32_t)s.refl_phase.size();
  d.refl_phase = s.refl_phase.data();
  d.refl_mu = s.refl_mu.data();
  d.refl_int = s.refl_int.data();
}

specmc_smc_config to_cfg(const SmcConfig& cfg, int device) {
  specmc_smc_config c;
  c.T = cfg.T;
  c.n = cfg.n;
  c.ess_target = cfg.ess_target;
  c.max_levels = cfg.max_levels;
  c.seed = cfg.seed;
  c.workers = cfg.workers;
  c.device = device;
  return c;
}

// rethrow with the reference's exception types (smc.cpp:24-31, :63, :98, :195-196)
void check(int rc, const char* err) {
  if (rc == SPECMC_OK) return;
  if (rc == SPECMC_EINVAL) throw std::invalid_argument(err);
  throw std::runtime_error(err);
}

VectorXd vec(const double* p, Index n) { return Eigen::Map<const VectorXd>(p, n); }

// RunReport fields as smc.cpp:221-247 fills them
RunReport to_report(const ModelSpec& spec, const Spectrum& data, const SmcConfig& cfg, specmc_smc_result& r) {
  RunReport rep;
  rep.sampler = "smc";
  rep.F = r.F;
  rep.diverged = r.diverged != 0;
  rep.wall_seconds = r.wall_seconds;
  for (const auto& p : spec.layout) rep.param_names.push_back(p.name);
  rep.scalars = {{"T", (double)cfg.T},
                 {"n", (double)cfg.n},
                 {"ess_target", cfg.ess_target},
                 {"seed", (double)cfg.seed},
                 {"workers", (double)cfg.workers},
                 {"n_data", (double)data.xs.size()},
                 {"levels", (double)r.levels}};
  rep.arrays["ladder"] = vec(r.ladder, r.levels + 1);
  rep.arrays["level_ess_ratio"] = vec(r.level_ess_ratio, r.levels);
  rep.arrays["level_log_mean_w"] = vec(r.level_log_mean_w, r.levels);
  rep.arrays["level_acc_rate"] = vec(r.level_acc_rate, r.levels);
  rep.posterior.resize(r.d, (Index)r.T);  // d x T column-major, the ABI's layout
  std::memcpy(rep.posterior.data(), r.posterior, sizeof(double) * (size_t)r.d * (size_t)r.T);
  return rep;
}

}  // namespace

RunReport smc_run_b200(const ModelSpec& spec, const Spectrum& data, const SmcConfig& cfg, int device) {
  specmc_model_desc d;
  DescBufs bufs;
  to_desc(spec, d, bufs);
  const specmc_smc_config c = to_cfg(cfg, device);
  specmc_smc_result r;
  std::memset(&r, 0, sizeof(r));
  char err[512] = {0};
  const int rc = specmc_smc_run(&d, data.xs.data(), data.ys.data(), (int64_t)data.xs.size(), &c, &r, err,
                                sizeof err);
  if (rc != SPECMC_OK) {
    specmc_result_free(&r);
    check(rc, err);
  }
  RunReport rep = to_report(spec, data, cfg, r);
  specmc_result_free(&r);
  return rep;
}

std::vector<RunReport> smc_run_batch_b200(const std::vector<ModelSpec>& specs, const Spectrum& data,
                                          const std::vector<SmcConfig>& cfgs, int device) {
  if (specs.size() != cfgs.size()) throw std::invalid_argument("smc_run_batch_b200: specs / cfgs size mismatch");
  const size_t n = specs.size();
  std::vector<DescBufs> bufs(n);
  std::vector<specmc_problem> probs(n);
  for (size_t i = 0; i < n; ++i) {
    to_desc(specs[i], probs[i].model, bufs[i]);
    probs[i].spectrum = 0;
    probs[i].cfg = to_cfg(cfgs[i], device);
  }
  specmc_spectrum sp{data.xs.data(), data.ys.data(), (int64_t)data.xs.size()};
  std::vector<specmc_smc_result> res(n);
  char err[512] = {0};
  const int rc = specmc_smc_run_batch((int32_t)n, probs.data(), 1, &sp, res.data(), err, sizeof err);
  std::vector<RunReport> out;
  int bad = SPECMC_OK;
  for (size_t i = 0; i < n; ++i) {
    if (res[i].status == SPECMC_OK && rc != SPECMC_EINVAL && rc != SPECMC_ECUDA)
      out.push_back(to_report(specs[i], data, cfgs[i], res[i]));
    else if (bad == SPECMC_OK)
      bad = res[i].status != SPECMC_OK ? res[i].status : rc;
    specmc_result_free(&res[i]);
  }
  if (bad != SPECMC_OK) check(bad, err[0] ? err : "smc_run_batch_b200 failed");
  return out;
}

}  // namespace specmc
