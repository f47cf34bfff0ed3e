// device.cuh -- shared device-side types and helpers of the B200 SMC sampler.
//
// Layout in HBM (one "group" = one SMC run = one (spectrum, K, seed)):
//   theta[2]   fp64 SoA [d][T]    particle parameters, double-buffered by level
//   E[2]       fp64 [T]           per-point energies (+inf allowed)
//   anc        int32 [S]          systematic-resampling ancestors of a level
//   ls0        fp64 [d]           log step sizes predicted for a level
//   chain_acc  int32 [d][S]       per-chain accept tallies (component-major)
//   chain_ls   fp64 [d][S]        per-chain final log step sizes
//   wbuf       fp64 [T]           normalised weights (CDF scan input)
//   hist       fp64 [5][1+2d]     step-size history ring (beta, acc[d], step[d])
//   diag       fp64 [max_levels][4] (beta, ess_ratio, log_mean_w, acc_rate)
// The observed spectrum is prepared on the host per launch shape in
// lane-transposed pair-slot order: lane l's points l*PPL + k and
// l*PPL + k + PPL/2 share slot k, stored at [k * L + l] (L = 32 W lanes per
// chain; chain.cuh), so a warp's shared-memory reads of a slot are
// conflict-free 8- or 16-byte accesses.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace smc {

enum Family : int { FAM_GM = 0, FAM_XPS = 1, FAM_XRD = 2, FAM_OFFSET = 3 };
enum NoiseDev : int { NZ_DYN = -1, NZ_GAUSS = 0, NZ_HETERO = 1, NZ_POISSON = 2, NZ_HLIN = 3, NZ_HPROP = 4 };
enum PriorKind : int { PR_NORMAL = 0, PR_GAMMA = 1, PR_UNIFORM = 2 };
enum Role : uint32_t { ROLE_INIT = 1, ROLE_CHAIN = 2, ROLE_RESAMPLE = 3, ROLE_REMC = 4, ROLE_SWAP = 5 };
enum GroupError : int { GE_NONE = 0, GE_MAX_LEVELS = 1, GE_ZERO_WEIGHT = 2 };

constexpr int kHist = 5;       // predict_step_size window (mcmc.cpp:28)
constexpr double kLogStepMin = -27.631021115928547;  // log(1e-12), mcmc.hpp:8
constexpr double kLogStepMax = 27.631021115928547;   // log(1e12),  mcmc.hpp:9

struct GroupState {  // mutable per-group scalars; read back by the host every round
  double beta;
  double neg_log_z;
  int level;
  int cur;
  int active;
  int error;
  int hist_count;
  int T_loc;     // particles held by this group (== T unless the run is particle-sharded)
  int S_loc;     // chains of the current level held by this group
  int chain_lo;  // global index of its first chain (Philox stream: chain_base + chain_lo + c)
  unsigned long long trials;
  unsigned long long shape_evals;  // move kernel: block shape evaluations (block entries + non-amplitude trials)
};

// Grid-level tempering state of one group (multi-CTA path, k_tp_*): the
// bisection state machine of next_beta, slice partial sums and the slice
// offsets of the grid-level CDF scan.
constexpr int kMaxSlices = 512;
// next_beta bisection steps per k_tp_ess_tree launch, and its delta slots
// (slot 0: the full step; 1 .. 2^D - 1: the heap of bisection midpoints)
constexpr int kEssDepth = 3;
constexpr int kEssSlots = 1 << kEssDepth;
struct TemperScratch {
  double emin, lo, hi, full, beta_next;
  double m, lse, u;
  double base;                 // global CDF offset of this group's first particle (sharded runs)
  long long shard_lo, shard_hi;  // global chain range [lo, hi) resolved by this group
  int it, done, err, pad;
  unsigned int counter, pad2;
  double part[kMaxSlices][2];
  double offs[kMaxSlices + 1];
  double tpart[kMaxSlices][2 * kEssSlots];  // k_tp_ess_tree: (sum w, sum w^2) per slice and slot
};

struct GroupDesc {  // immutable per group
  int family, K, d, noise;
  int T, n, S, max_levels;
  double ess_target, n_data;
  uint32_t key0, key1;
  uint32_t chain_base;  // global chain offset (multi-GPU invariance)
  int N;                // real points
  // particle sharding (shard.cu): this group is one shard of a run whose T and
  // S are global; its level-0 particles are global ids [pbase, pbase + T_loc)
  int sharded;
  int pbase;
  int shard, nshards;  // this shard's index and the shard count of the run
  double* xbuf;        // [2 kEssSlots] cross-shard exchange of the tempering phases
  double* xgat;        // [nshards][2] gathered (weight total, particle count) per shard
  // energy: E = e_a0 + e_a1 * sum(l_k); device noise parameters
  double e_a0, e_a1;
  float nz_a0, nz_a1, nz_a2, nz_q;
  // shirley helpers (shifted x)
  float x0s, inv_range, range;
  // xps on a uniform ascending grid (sh_uniform): the trapezoid weights are
  // constant, so the Shirley scan sums Pn alone (no per-point weights).  The
  // spectrum layout then keeps the first and the last real point at fixed lane
  // slots: points 0..N-2 at positions 0..N-2, point N-1 at the last position,
  // padding in between at x = 1e30 (every peak shape is exactly 0 there)
  int sh_uniform;
  float x1s;  // shifted abscissa of the last point (linear-ramp fallback clamp)
  // spectrum (lane-transposed, see header)
  const float* spec_x;   // shifted abscissa x' = x - x_shift
  const float2* spec_c;  // (c_k, h_{k+1}): trapezoid weights of the Shirley scan
  const float2* spec_y;  // (y_k, 1/s_k): observation and inverse noise scale; paired noise
                         // models: (y_2p, y_2p+1) per point pair, then 1/(s_2p s_2p+1)
  float y_last, s_last;  // (y, 1/s) of the last point (padding replicates it)
  // xrd reflections (mu_ref, rel_intensity) grouped by phase: phase b owns [refl_off[b], refl_off[b+1])
  const float2* refl;
  const int* refl_off;
  // priors (layout order, location components already shifted)
  const int* pkind;
  const double* pa;
  const double* pb;
  // buffers.  [d][*] arrays use a padded row pitch (tp for T columns, sp for
  // S): pitch * 8 bytes is an odd multiple of 256 B, so the d rows of one
  // particle (read/written lane-parallel over components by the chain kernel)
  // spread over L2 slices instead of aliasing at a power-of-two stride
  int tp, sp;
  double* theta[2];
  double* E[2];
  int* anc;
  double* ls0;
  int* chain_acc;
  double* chain_ls;
  double* wbuf;
  double* hist;
  double* diag;
  GroupState* st;
  TemperScratch* ts;  // grid-level tempering (large T)
  int nslices;        // slices of the grid-level tempering (0: single-CTA path)
  int slice_len;
  double* stat_acc;   // [2d] per-component accept sums and log-step sums of the level (k_stats_grid)
  // replica-exchange runs (REMC comparator, remc.cpp): one chain unit per
  // replica; T = S = R replicas, st->level = the current sweep t (1-based)
  const double* ladder;  // [R] inverse temperatures beta_0 = 0 < ... < beta_{R-1} = 1
  double* pair_acc;      // [R-1][2] running (max, scaled sum) of exp(tempered_term) after burn-in
  int* swaps;            // [R-1][2] (accepts, attempts)
  double* post;          // [d][draws] beta = 1 draws after burn-in
  long long n_burn, total_sweeps, swap_period;
};

// ----------------------------------------------------------------- Philox4x32-10
struct u32x4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ u32x4 philox(u32x4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = u32x4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// ------------------------------------------------------------------ fast math
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcpf(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2f(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 32-bit uniforms: (0, 1] and [0, 1)
__device__ __forceinline__ float u01_open_lo(uint32_t v) { return (float(v >> 8) + 1.0f) * 5.9604644775390625e-8f; }
__device__ __forceinline__ double u53(uint32_t a, uint32_t b) {
  const uint64_t v = ((uint64_t)a << 32) | b;
  return (double)(v >> 11) * 0x1.0p-53;
}

// Box-Muller in fp32 (MUFU lg2 / cos); u1 in (0,1], angle centred on [-pi, pi)
__device__ __forceinline__ float normal_f32(uint32_t a, uint32_t b) {
  const float u1 = u01_open_lo(a);
  const float u2 = float(b >> 8) * 5.9604644775390625e-8f;
  const float r = sqrtf(-2.0f * 0.69314718056f * lg2f(u1));
  return -r * __cosf(6.283185307179586f * (u2 - 0.5f));
}
// fp64 Box-Muller for prior draws (init only)
__device__ __forceinline__ double normal_f64(u32x4 o) {
  const double u1 = u53(o.x, o.y);
  const double u2 = u53(o.z, o.w);
  return sqrt(-2.0 * log1p(-u1)) * cos(6.283185307179586476925286766559 * u2);
}

// ------------------------------------------------------------ warp reductions
__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_min_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_incl_scan_f(float v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}
__device__ __forceinline__ double warp_incl_scan_d(double v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ----------------------------------------------- bulk async copy (global->smem)
// cp.async.bulk (SASS UBLKCP) completing on an mbarrier: stages the spectrum.
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(phase)
      : "memory");
}

}  // namespace smc
