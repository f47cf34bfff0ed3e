// C++ host-side check of the reference-shaped adapter (include/specmc_b200.hpp).
// Without a GPU: validation errors throw std::invalid_argument exactly as the
// reference (smc.cpp:23-32) and a compute call throws std::runtime_error (no
// CPU fallback).  With a GPU (argv[1] == "gpu"): a gm model selection K = 1..3
// on a 3-peak spectrum picks K = 3.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "specmc_b200.hpp"

using namespace specmc_b200;

static int fails = 0;
#define CHECK(c)                                              \
  do {                                                        \
    if (!(c)) {                                               \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
      ++fails;                                                \
    }                                                         \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  SmcConfig ok;
  CHECK(!throws<std::exception>([&] { validate_smc_config(ok); }));
  SmcConfig bad = ok;
  bad.T = 1001;  // not divisible by n = 10
  CHECK(throws<std::invalid_argument>([&] { validate_smc_config(bad); }));
  bad = ok;
  bad.ess_target = 1.0;
  CHECK(throws<std::invalid_argument>([&] { validate_smc_config(bad); }));

  Spectrum data;
  const double A[3] = {0.587, 1.522, 1.183}, mu[3] = {1.210, 1.455, 1.703}, b[3] = {95.689, 146.837, 164.469};
  for (int i = 0; i < 301; ++i) {
    const double x = 3.0 * i / 300.0;
    double y = 0.0;
    for (int k = 0; k < 3; ++k) y += A[k] * std::exp(-0.5 * b[k] * (x - mu[k]) * (x - mu[k]));
    data.xs.push_back(x);
    data.ys.push_back(y + 0.1 * std::sin(17.0 * i));  // deterministic "noise"
  }
  SmcConfig c;
  c.T = 4096;
  c.n = 8;
  c.seed = 3;
  CHECK(throws<std::invalid_argument>([&] { smc_run(gm_model(2, 0, 3, 0.1, GmMuPrior::UniformRange), data, bad); }));
  if (!gpu) {
    CHECK(throws<std::runtime_error>([&] { smc_run(gm_model(2, 0, 3, 0.1, GmMuPrior::UniformRange), data, c); }));
  } else {
    std::vector<Problem> ps;
    for (int K = 1; K <= 3; ++K) ps.push_back({gm_model(K, 0, 3, 0.1, GmMuPrior::UniformRange), 0, c});
    auto reps = smc_run_batch(ps, {data});
    std::vector<std::pair<int, RunReport>> rows;
    for (int K = 1; K <= 3; ++K) rows.emplace_back(K, reps[K - 1]);
    CHECK(model_select(rows) == 3);
    CHECK(reps[2].posterior.size() == static_cast<size_t>(9 * 4096));
    CHECK(reps[2].arrays.at("ladder").back() == 1.0);
    std::printf("F = %.4f %.4f %.4f\n", reps[0].F, reps[1].F, reps[2].F);
  }
  // xrd family (model.cpp:138-167): one phase with three reflections on a counts spectrum
  Spectrum xr;
  const double refl[3][2] = {{25.3, 100.0}, {37.8, 20.0}, {48.0, 35.0}};
  for (int i = 0; i < 700; ++i) {
    const double x = 20.0 + 40.0 * i / 699.0;
    double y = 30.0;
    for (const auto& r : refl) y += 400.0 * r[1] / 100.0 / (1.0 + ((x - r[0]) / 0.15) * ((x - r[0]) / 0.15));
    xr.xs.push_back(x);
    xr.ys.push_back(std::floor(y + 3.0 * std::sin(11.0 * i)));
  }
  PhaseRef ph{"anatase", {{25.3, 100.0}, {37.8, 20.0}, {48.0, 35.0}}};
  const ModelSpec xs = xrd_model({ph}, xr);
  CHECK(xs.K == 1 && xs.layout.size() == 13 && xs.phases.size() == 1);
  Spectrum flat = xr;
  for (auto& y : flat.ys) y = 5.0;
  CHECK(throws<std::invalid_argument>([&] { xrd_model({ph}, flat); }));
  SmcConfig cx;
  cx.T = 1024;
  cx.n = 8;
  cx.seed = 5;
  if (!gpu) {
    CHECK(throws<std::runtime_error>([&] { smc_run(xs, xr, cx); }));
  } else {
    const RunReport r = smc_run(xs, xr, cx);
    CHECK(std::isfinite(r.F) && !r.diverged);
    CHECK(r.posterior.size() == static_cast<size_t>(13 * 1024));
    std::printf("xrd F = %.4f\n", r.F);
  }
  // replica exchange (remc.cpp:170-190): validation errors are invalid_argument,
  // compute without a GPU is runtime_error; on the GPU a gm run reports the
  // reference's RunReport fields
  {
    RemcConfig rc;
    rc.L = 12;
    rc.total_sweeps = 400;
    rc.seed = 9;
    RemcConfig rbad = rc;
    rbad.burn_in_fraction = 1.5;
    const ModelSpec g3 = gm_model(3, 0, 3, 0.1, GmMuPrior::UniformRange);
    CHECK(throws<std::invalid_argument>([&] { remc_run(g3, data, rbad); }));
    if (!gpu) {
      CHECK(throws<std::runtime_error>([&] { remc_run(g3, data, rc); }));
    } else {
      const RunReport r = remc_run(g3, data, rc);
      CHECK(r.sampler == "remc" && std::isfinite(r.F) && !r.diverged);
      CHECK(r.arrays.at("ladder").size() == 13 && r.arrays.at("swap_rate").size() == 12);
      CHECK(r.arrays.at("replica_acc_rate").size() == 13 && r.scalars.at("L") == 12.0);
      CHECK(r.d == 9 && r.T == 200 && r.posterior.size() == static_cast<size_t>(9 * 200));
      std::printf("remc F = %.4f\n", r.F);
    }
  }
  std::printf("%s (%d failures)\n", fails ? "FAILED" : "OK", fails);
  return fails ? 1 : 0;
}
