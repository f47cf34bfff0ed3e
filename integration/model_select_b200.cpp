// model_select_b200.cpp -- a reference-side caller of the adapter: the
// reference's own model selection (cmd_model_select's K x trials loop,
// proj/tools/specmc_main.cpp:147-170, written anew here) with every smc_run
// replaced by the B200 backend, the reference's xps_model / gen_xps /
// model_select / write_report doing everything else.
//
// usage: model_select_b200 <k_true> <data_seed> <K_lo> <K_hi> <T> <n> <trials> <serial|batch> [report_path]
// prints one line per (K, trial) "run K=.. trial=.. F=.. levels=.." and a
// final "selected K=..".  Exit codes as the reference CLI (specmc_main.cpp:17-19):
// 2 invalid argument, 3 runtime / numeric (including no CUDA device).
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "smc_b200.hpp"
#include "specmc/model.hpp"
#include "specmc/posterior.hpp"
#include "specmc/report.hpp"
#include "specmc/rng.hpp"
#include "specmc/synthetic.hpp"

using namespace specmc;

int main(int argc, char** argv) {
  if (argc < 9) {
    std::fprintf(stderr, "usage: %s k_true data_seed K_lo K_hi T n trials serial|batch [report]\n", argv[0]);
    return 2;
  }
  try {
    const int k_true = std::atoi(argv[1]);
    const std::uint64_t data_seed = std::strtoull(argv[2], nullptr, 10);
    const int k_lo = std::atoi(argv[3]), k_hi = std::atoi(argv[4]);
    const long long T = std::atoll(argv[5]);
    const int n = std::atoi(argv[6]), trials = std::atoi(argv[7]);
    const std::string mode = argv[8];
    const XpsHeteroNoise noise{1.0, 0.01, 0.0, false};
    const SyntheticDataset ds = gen_xps(k_true, data_seed, noise);
    std::vector<ModelSpec> specs;
    std::vector<SmcConfig> cfgs;
    std::vector<std::pair<int, int>> tag;  // (K, trial)
    for (int t = 0; t < trials; ++t)
      for (int K = k_lo; K <= k_hi; ++K) {
        SmcConfig cfg;
        cfg.T = T;
        cfg.n = n;
        cfg.seed = hash_combine(4242, (std::uint64_t)t);  // bench.cpp trial_seed semantics
        specs.push_back(xps_model(K, ds.data, noise));
        cfgs.push_back(cfg);
        tag.emplace_back(K, t);
      }
    std::vector<RunReport> reps;
    if (mode == "serial") {
      for (size_t i = 0; i < specs.size(); ++i) reps.push_back(smc_run_b200(specs[i], ds.data, cfgs[i]));
    } else {
      reps = smc_run_batch_b200(specs, ds.data, cfgs);
    }
    std::vector<std::pair<int, RunReport>> rows;
    for (size_t i = 0; i < reps.size(); ++i) {
      std::printf("run K=%d trial=%d F=%.17g levels=%g diverged=%d draws=%ld\n", tag[i].first, tag[i].second,
                  reps[i].F, reps[i].scalars.at("levels"), (int)reps[i].diverged, (long)reps[i].posterior.cols());
      rows.emplace_back(tag[i].first, reps[i]);
    }
    const ModelChoice choice = model_select(rows);
    std::printf("selected K=%d\n", choice.K_best);
    if (argc > 9)
      for (size_t i = 0; i < reps.size(); ++i)
        if (tag[i].first == choice.K_best && tag[i].second == 0) write_report(reps[i], argv[9]);
    return 0;
  } catch (const std::invalid_argument& e) {
    std::fprintf(stderr, "invalid argument: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  }
}
