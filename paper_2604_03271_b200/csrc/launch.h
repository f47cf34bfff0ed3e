// launch.h -- host-visible launchers for the sm_100a kernels (kernels.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "device.cuh"

namespace smc {

// Launch shape of the chain-parallel kernels for a spectrum of N points:
// W warps cooperate on one chain (unit), each lane owns PPL consecutive
// points in registers, U units share one CTA (and its staged spectrum).
// Spectrum layout in the chain kernels' shared memory (bit flags): bit 0 = the
// trapezoid weights are staged (xps on a non-uniform grid), bit 1 = y at 4 B
// per point (every noise model but poisson).  W <= 2 kernels use the fixed full layout
// (weights + 8 B y: 20 B/point, compile-time offsets); W >= 4 kernels size
// it per launch, which halves the footprint of the large spectra (C3, C5) and
// lets two CTAs share an SM.
constexpr int kLayWeights = 1, kLayY4 = 2, kLayFull = kLayWeights;
// units per CTA of the W = 2 kernels (N <= 2048): 8 (512 threads) or 10 (640
// threads; needs the per-launch layout to fit the units' caches)
#ifndef SPECMC_W2_UNITS
#define SPECMC_W2_UNITS 8
#endif
__host__ __device__ constexpr bool chain_dyn_layout(int W) { return W >= 4 || (W == 2 && SPECMC_W2_UNITS > 8); }

struct Shape {
  int W;
  int PPL;
  int U;
  int lay = kLayFull;
};

// chain-kernel CTA size per unit width W (units per CTA = threads / 32 W):
// W = 2 runs 8 units per 512-thread CTA, one CTA per SM, so the spectrum is
// staged once per SM and the 8 units' P and Q caches fit in shared memory
// W = 8 (N <= 8192): two chains per 512-thread CTA with P in shared memory
// (one spectrum copy per SM); a launch whose spectrum layout leaves no room
// for two chains' P and Q caches (a non-uniform grid's trapezoid weights)
// runs one chain per 256-thread CTA instead (fit_units, host.cu)
__host__ __device__ constexpr int chain_threads(int W) {
  return W >= 8 ? 64 * W : (W == 2 ? 64 * SPECMC_W2_UNITS : 256);
}
// (and W = 1 with wide lanes, PPL >= 20: 512 < N <= 1024)
__host__ __device__ constexpr bool chain_p_in_smem(int W, int PPL) {
  return W == 2 || W == 4 || W == 8 || (W == 1 && PPL >= 20);
}

constexpr size_t kChainSmemMax = 226 * 1024;  // dynamic shared memory per CTA (227 KB less the static descriptor copy)
Shape pick_shape(int64_t N, int dmax);
bool ppl_supported(int ppl);
size_t chain_smem_bytes(const Shape& s, int dmax);

// prior draws for every particle of every listed group (init_ensemble, smc.cpp:34-53)
cudaError_t launch_init_draw(const GroupDesc* d_gds, const int* d_list, int n_list, int Tmax, cudaStream_t st);
// full energies of theta[cur] (BlockEvaluator::full, energy.cpp:43-55), one chain unit per particle
cudaError_t launch_energy(int family, const Shape& s, int dmax, const GroupDesc* d_gds, const int* d_list,
                          const int* d_cta_prefix, int n_list, int total_ctas, cudaStream_t st);
// per-(family, mode) instantiation units (chain_<fam>_<mode>.cu)
#define SMC_DECL_CHAIN(NAME)                                                                                    \
  cudaError_t NAME(const Shape& s, int dmax, const GroupDesc* d_gds, const int* d_list, const int* d_cta_prefix, \
                   int n_list, int total_ctas, cudaStream_t st);
SMC_DECL_CHAIN(launch_chain_gm_energy)
SMC_DECL_CHAIN(launch_chain_xps_energy)
SMC_DECL_CHAIN(launch_chain_xrd_energy)
SMC_DECL_CHAIN(launch_chain_offset_energy)
SMC_DECL_CHAIN(launch_chain_offset_move_dyn)
SMC_DECL_CHAIN(launch_chain_gm_remc)
SMC_DECL_CHAIN(launch_chain_xps_remc)
SMC_DECL_CHAIN(launch_chain_xrd_remc)
SMC_DECL_CHAIN(launch_chain_offset_remc)
#define SMC_DECL_MOVE(FAM) \
  SMC_DECL_CHAIN(launch_chain_##FAM##_move_gauss)  \
  SMC_DECL_CHAIN(launch_chain_##FAM##_move_hetero) \
  SMC_DECL_CHAIN(launch_chain_##FAM##_move_poisson) \
  SMC_DECL_CHAIN(launch_chain_##FAM##_move_hlin)   \
  SMC_DECL_CHAIN(launch_chain_##FAM##_move_hprop)
SMC_DECL_MOVE(gm)
SMC_DECL_MOVE(xps)
SMC_DECL_MOVE(xpsl)
SMC_DECL_MOVE(xrd)
#undef SMC_DECL_MOVE
#undef SMC_DECL_CHAIN
// fused waste-free chain move (wastefree_level chain loop x cw_mh_sweep, smc.cpp:142-156, mcmc.cpp:55-96)
// (one instantiation per kernel family x device noise model, NoiseDev in device.cuh; kernel
// family = the model family, or kFamXpsLorentz for xps with the Lorentzian basis pinned)
constexpr int kFamXpsLorentz = 4;  // == FAM_XPSL (chain.cuh)
cudaError_t launch_move(int family, int noise, const Shape& s, int dmax, const GroupDesc* d_gds, const int* d_list,
                        const int* d_cta_prefix, int n_list, int total_ctas, cudaStream_t st);
// next_beta + weights + evidence + systematic resampling + predict_step_size (one CTA per group)
cudaError_t launch_temper(const GroupDesc* d_gds, const int* d_list, int n_list, cudaStream_t st);
// grid-level tempering for large T: emin, 61 bisection steps, weights, CDF scan,
// resampling + step prediction (66 launches, each over (slices x groups))
cudaError_t launch_temper_grid(const GroupDesc* d_gds, const int* d_list, int n_list, int max_slices, cudaStream_t st);
int temper_grid_launches();
// its halves: emin + the ESS bisection passes (-> ts->beta_next), then weights,
// evidence, CDF offsets and resampling (u_override: parity unit's explicit uniform)
cudaError_t launch_tp_next_beta(const GroupDesc* d_gds, const int* d_list, int n_list, int max_slices,
                                cudaStream_t st);
cudaError_t launch_tp_resample(const GroupDesc* d_gds, const int* d_list, int n_list, int max_slices,
                               const double* u_override, cudaStream_t st);
// ---- particle sharding (shard.cu): one run's particles split over shards that
// exchange a few scalars per tempering phase
enum ExchangeOp : int { XOP_SUM = 0, XOP_MIN = 1, XOP_MAX = 2 };
struct Exchange {
  virtual ~Exchange() = default;
  // reduce `count` doubles of every shard's g.xbuf (buf 0) or g.stat_acc (buf 1)
  // across the shards of each run (count < 0: the run's 2d step statistics);
  // every shard receives the result
  virtual cudaError_t reduce(int buf, int count, int op, cudaStream_t st) = 0;
  // every shard's (xbuf[0], xbuf[1]) into every shard's g.xgat, in shard order
  virtual cudaError_t gather(cudaStream_t st) = 0;
};
// one sharded level's tempering: the k_tp_* phases with an exchange and a
// k_tpf_* finaliser after each cross-shard reduction
cudaError_t launch_temper_sharded(const GroupDesc* d_gds, const int* d_list, int n_list, int max_slices, Exchange& x,
                                  cudaStream_t st);
int temper_sharded_launches();
cudaError_t launch_stats_sharded(const GroupDesc* d_gds, const int* d_list, int n_list, int dmax, Exchange& x,
                                 cudaStream_t st);
// exchange among shards resident on this device (one stream, kernels); d_list
// holds the nsh shards of each of nruns runs, run-major
cudaError_t launch_xreduce(const GroupDesc* d_gds, const int* d_list, int nruns, int nsh, int buf, int count, int op,
                           cudaStream_t st);
cudaError_t launch_xgather(const GroupDesc* d_gds, const int* d_list, int nruns, int nsh, cudaStream_t st);

// step-size statistics, one CTA per (component, group), + per-group finalisation
cudaError_t launch_stats_grid(const GroupDesc* d_gds, const int* d_list, int n_list, int dmax, cudaStream_t st);

// ---- replica exchange (the paper's REMC comparator, remc.cpp): one sweep of
// every replica of every listed run (k_chain in REMC mode), then per run the
// swap step (remc.cpp:53-73), the post-burn-in pair accumulators and beta = 1
// draws, and the sweep counter advance (k_remc_exchange)
cudaError_t launch_remc_sweep(int family, const Shape& s, int dmax, const GroupDesc* d_gds, const int* d_list,
                              const int* d_cta_prefix, int n_list, int total_ctas, cudaStream_t st);
cudaError_t launch_remc_exchange(const GroupDesc* d_gds, const int* d_list, int n_list, cudaStream_t st);

// load every kernel of one class (family, noise, shape) before its timed run
cudaError_t prime_level_kernels(int family, int noise, const Shape& s, int dmax);

// theta [d][tp] -> out [T][d] + shift[i] (result posterior block)
cudaError_t launch_posterior_out(const double* theta, int tp, int d, int T, const double* shift, double* out,
                                 cudaStream_t st);

cudaError_t launch_probe_mufu(float* d_out, int blocks, int iters, cudaStream_t st);

// ---- parity units (single-array versions of the temper building blocks)
cudaError_t launch_unit_ess(const double* d_lw, int64_t n, double* d_out, int* d_err, cudaStream_t st);
cudaError_t launch_unit_log_mean_exp(const double* d_v, int64_t n, double* d_out, cudaStream_t st);
cudaError_t launch_unit_next_beta(const double* d_E, int64_t n, double n_data, double beta_prev, double target,
                                  double* d_out, int* d_err, cudaStream_t st);
cudaError_t launch_unit_resample(const double* d_lw, int64_t n, int64_t S, double u, double* d_wscratch,
                                 int* d_anc, int* d_err, cudaStream_t st);
cudaError_t launch_unit_predict(const double* d_hist, int H, int d, double beta_next, const int* d_pk,
                                const double* d_pa, const double* d_pb, double* d_out, cudaStream_t st);

}  // namespace smc
