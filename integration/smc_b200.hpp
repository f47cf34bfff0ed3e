// smc_b200.hpp -- declarations of the reference-side adapter (smc_b200.cpp).
#pragma once
#include <vector>

#include "specmc/report.hpp"
#include "specmc/smc.hpp"
#include "specmc/spectrum.hpp"
#include "specmc_b200.h"

namespace specmc {

// drop-in for RunReport smc_run(const ModelSpec&, const Spectrum&, const SmcConfig&)
// (proj/include/specmc/smc.hpp:78) on CUDA device `device`
RunReport smc_run_b200(const ModelSpec& spec, const Spectrum& data, const SmcConfig& cfg, int device = 0);

// every (spec_i, cfg_i) concurrently on one GPU: the K x trials loop of cmd_model_select
std::vector<RunReport> smc_run_batch_b200(const std::vector<ModelSpec>& specs, const Spectrum& data,
                                          const std::vector<SmcConfig>& cfgs, int device = 0);

}  // namespace specmc
