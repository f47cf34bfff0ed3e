// specmc_b200_cli.cpp -- the reference CLI's fit and model-select commands with
// the B200 backend (the reference's commands are
// cmd_fit / cmd_model_select, proj/tools/specmc_main.cpp:96-192).
//
// Everything around the sampler is the reference's own code, compiled where it
// lies (integration/build_adapter.py): the config schema and prior overrides
// (config.cpp), spectrum files (spectrum.cpp), peak-block sorting and
// credible intervals (posterior.cpp), model_select, the report and table
// formats (report.cpp, format_double).  The sampling goes through the adapter
// (smc_b200.cpp): fit = one smc_run_b200; model-select = every (K, trial) of
// the range in ONE batched call (specmc_smc_run_batch) instead of the
// reference's serial loop.  Exit codes as the reference: 0 ok, 2 config /
// usage, 3 numeric (non-finite F, every candidate diverged, or no device).
//
//   specmc_b200 fit --config C --data D --out R [--label L] [--device N]
//   specmc_b200 model-select --config C --data D --k-range A..B [--trials N] --out TABLE [--device N]
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "smc_b200.hpp"
#include "specmc/bench.hpp"
#include "specmc/config.hpp"
#include "specmc/posterior.hpp"
#include "specmc/report.hpp"
#include "specmc/spectrum.hpp"

using namespace specmc;

namespace {

struct NumericFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Args {
  std::string cmd;
  std::map<std::string, std::string> opt;
  std::string get(const std::string& k, const std::string& fb = "") const {
    auto it = opt.find(k);
    return it == opt.end() ? fb : it->second;
  }
  std::string need(const std::string& k) const {
    auto it = opt.find(k);
    if (it == opt.end()) throw std::invalid_argument("missing option --" + k);
    return it->second;
  }
};

Args parse(int argc, char** argv) {
  if (argc < 2) throw std::invalid_argument("usage: specmc_b200 fit|model-select --config C --data D ...");
  Args a;
  a.cmd = argv[1];
  for (int i = 2; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0 || i + 1 >= argc) throw std::invalid_argument("bad option: " + k);
    a.opt[k.substr(2)] = argv[++i];
  }
  return a;
}

// the report summaries of a fit: stable peak order (exchangeable labels of the
// mixture and photoemission families), posterior mean, 95% / 99% intervals
void summarise(RunReport& r, const ModelSpec& spec) {
  if (r.posterior.cols() == 0) return;
  if (spec.family == Family::GaussianMixture) r.posterior = sort_peak_blocks(r.posterior, 3, 1, spec.K);
  if (spec.family == Family::XpsShirley) r.posterior = sort_peak_blocks(r.posterior, 4, 1, spec.K);
  const Index d = r.posterior.rows();
  const ArrayXd w = ArrayXd::Ones(r.posterior.cols());
  VectorXd mean(d), l95(d), h95(d), l99(d), h99(d);
  for (Index i = 0; i < d; ++i) {
    ArrayXd x(r.posterior.cols());
    for (Index j = 0; j < r.posterior.cols(); ++j) x[j] = r.posterior(i, j);
    mean[i] = x.mean();
    const auto a = credible_interval(x, w, 0.95), b = credible_interval(x, w, 0.99);
    l95[i] = a.first;
    h95[i] = a.second;
    l99[i] = b.first;
    h99[i] = b.second;
  }
  r.arrays["post_mean"] = mean;
  r.arrays["ci95_lo"] = l95;
  r.arrays["ci95_hi"] = h95;
  r.arrays["ci99_lo"] = l99;
  r.arrays["ci99_hi"] = h99;
}

Index max_draws(const Config& cfg) {
  const long long m = cfg_int(cfg, "report.max_draws", 20000);
  if (m < 1) throw std::invalid_argument("config key report.max_draws: must be >= 1");
  return (Index)m;
}

std::uint64_t base_seed(const Config& cfg) {
  const long long s = cfg_int(cfg, "seed", 0);
  if (s < 0) throw std::invalid_argument("config key seed: must be >= 0");
  return (std::uint64_t)s;
}

int fit(const Args& a) {
  Config cfg = load_config(a.need("config"));
  validate_config_keys(cfg);
  const Spectrum data = load_spectrum(a.need("data"));
  const ModelSpec spec = make_model_spec(cfg, data);
  const std::string out = a.need("out");
  RunReport r = smc_run_b200(spec, data, make_smc_config(cfg), std::stoi(a.get("device", "0")));
  r.label = a.get("label");
  r.config_lines = cfg.lines;
  summarise(r, spec);
  write_report(r, out, max_draws(cfg));
  std::cout << "F = " << format_double(r.F) << "  (" << out << ")\n";
  if (r.diverged || !std::isfinite(r.F)) {
    std::cerr << "error: non-finite free energy (see " << out << ")\n";
    return 3;
  }
  return 0;
}

int model_select_cmd(const Args& a) {
  Config cfg = load_config(a.need("config"));
  validate_config_keys(cfg);
  const std::string kr = a.need("k-range");
  const size_t dots = kr.find("..");
  if (dots == std::string::npos) throw std::invalid_argument("--k-range expects the form A..B, got " + kr);
  int lo = 0, hi = 0;
  try {
    lo = std::stoi(kr.substr(0, dots));
    hi = std::stoi(kr.substr(dots + 2));
  } catch (const std::exception&) {
    throw std::invalid_argument("--k-range expects integers, got " + kr);
  }
  if (lo < 1 || hi < lo) throw std::invalid_argument("--k-range must satisfy 1 <= A <= B");
  const int trials = std::stoi(a.get("trials", "1"));
  if (trials < 1) throw std::invalid_argument("--trials must be >= 1");
  const Spectrum data = load_spectrum(a.need("data"));
  // every candidate competes under the same prior family (the reference pins
  // the mixture centre prior to uniform unless the config names one)
  const bool force_uniform = cfg_str(cfg, "family") == "gm" && !cfg.kv.count("gm.mu_prior");
  std::vector<ModelSpec> specs;
  std::vector<SmcConfig> cfgs;
  std::vector<int> ks;
  for (int t = 0; t < trials; ++t)
    for (int k = lo; k <= hi; ++k) {
      Config ck = cfg;
      ck.kv["K"] = std::to_string(k);
      specs.push_back(make_model_spec(ck, data, force_uniform));
      SmcConfig sc = make_smc_config(cfg);
      sc.seed = trial_seed(base_seed(cfg), t);
      cfgs.push_back(sc);
      ks.push_back(k);
    }
  std::vector<RunReport> reps = smc_run_batch_b200(specs, data, cfgs, std::stoi(a.get("device", "0")));
  std::vector<std::pair<int, RunReport>> rows;
  for (size_t i = 0; i < reps.size(); ++i) {
    reps[i].posterior.resize(0, 0);  // selection consumes F only
    rows.emplace_back(ks[i], std::move(reps[i]));
  }
  ModelChoice choice;
  try {
    choice = model_select(rows);
  } catch (const std::runtime_error& e) {
    throw NumericFailure(e.what());
  }
  const std::string path = a.need("out");
  std::ofstream out(path);
  if (!out) throw std::invalid_argument("cannot write table file: " + path);
  out << "# model selection over K = " << lo << ".." << hi << ", sampler smc, trials " << trials << "\n";
  for (const auto& line : cfg.lines) out << "#cfg " << line << "\n";
  out << "K\tF_mean\tF_std\ttrials\tstatus\n";
  for (const auto& row : choice.table)
    out << row.K << "\t" << format_double(row.F) << "\t" << format_double(row.trial_std) << "\t" << row.trials
        << "\t" << (row.excluded ? "excluded" : "ok") << "\n";
  out << "chosen\t" << choice.K_best << "\n";
  if (!out) throw std::invalid_argument("write failure on table file: " + path);
  std::cout << "chosen K = " << choice.K_best << "  (" << path << ")\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv);
    if (a.cmd == "fit") return fit(a);
    if (a.cmd == "model-select") return model_select_cmd(a);
    throw std::invalid_argument("unknown command: " + a.cmd + " (expected fit|model-select)");
  } catch (const std::invalid_argument& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  }
}
