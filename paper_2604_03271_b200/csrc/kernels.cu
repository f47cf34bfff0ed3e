// kernels.cu -- sm_100a kernels of the B200 waste-free SMC sampler.
//
//   k_init_draw   prior draws, one thread per particle        (smc.cpp:34-53, priors.cpp:105-110)
//   k_chain<E=1>  batched full energies, one chain unit each  (energy.cpp:43-55 + :7-28)   [K2]
//   k_chain<E=0>  fused propose/evaluate/accept move          (smc.cpp:142-156, mcmc.cpp:55-96) [K3]
//   k_temper      ESS bisection, weights, evidence, systematic resampling, step prediction
//                                                             (smc.cpp:55-112, :128-135, mcmc.cpp:20-53)
//   k_stats       step-size statistics and history            (smc.cpp:162-183)
//
// Reference paths are relative to the reference root (proj/...).
//
// A "chain unit" is W warps (32*W lanes).  Lane l owns the PPL consecutive
// spectrum points [l*PPL, (l+1)*PPL) and keeps the committed peak signal P and
// the trial signal Pn for them in registers.  The observed spectrum is staged
// once per CTA into shared memory with cp.async.bulk and read lane-transposed.
// A proposal changes one block (peak), so the trial signal is
// Pn = P + g_new - g_old (2 shape evaluations per point instead of the
// reference's K-block recombination, model.cpp:285-294).  The xps Shirley
// background (lineshapes.hpp:65-83) needs the cumulative trapezoid integral
// of Pn: it is written as C_k = sum_{j<=k} c_j Pn_j - h_{k+1} Pn_k, i.e. one
// lane-local inclusive scan plus one warp (and cross-warp) scan per proposal.
// Energies are summed per lane in fp32 from O(1) centred terms and reduced
// across lanes in fp64; the energy of the committed state is carried in fp64.
#include <cfloat>
#include <cmath>

#include "launch.h"

namespace smc {

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kHalfLn2 = 0.34657359027997264f;
constexpr float kLn2 = 0.6931471805599453f;

// ------------------------------------------------------------ block shapes
// Per-block fp32 constants of one peak; location parameters are in shifted
// coordinates (x' = x - x_shift, mu' = mu - x_shift) on the device.
struct BlockC {
  float mu, c1, c2, c3;
  bool ok;
};

template <int FAM>
__device__ __forceinline__ int block_stride() {
  return FAM == FAM_GM ? 3 : (FAM == FAM_XPS ? 4 : 1);
}

// gm:  g = A exp(-1/2 b (x-mu)^2)                          (model.cpp:216-220)
// xps: g = A [eta 2^(-u) + (1-eta) / (1 + u)], u = (x-mu)^2 / sigma^2
//      (= A [eta exp(-ln2 d^2/s^2) + (1-eta) s^2/(s^2+d^2)], model.cpp:269-280)
// offset: g = theta_0                                      (conjugate_oracle.hpp:22-26)
template <int FAM>
__device__ __forceinline__ BlockC block_consts(const double* p) {
  BlockC c;
  c.ok = true;
  c.c3 = 0.f;
  if (FAM == FAM_GM) {
    c.c1 = (float)p[0];
    c.mu = (float)p[1];
    c.c2 = (float)(-0.5 * p[2] * 1.4426950408889634);
  } else if (FAM == FAM_XPS) {
    const double A = p[0], sig = p[2], eta = p[3];
    c.ok = sig > 0.0;
    c.mu = (float)p[1];
    c.c1 = (float)(A * eta);
    c.c2 = (float)(A * (1.0 - eta));
    c.c3 = (float)(1.0 / (sig * sig));
  } else {
    c.c1 = (float)p[0];
    c.mu = 0.f;
    c.c2 = 0.f;
  }
  return c;
}

template <int FAM>
__device__ __forceinline__ float shape(const BlockC& b, float x) {
  if (FAM == FAM_GM) {
    const float d = x - b.mu;
    return b.c1 * ex2f(b.c2 * (d * d));
  } else if (FAM == FAM_XPS) {
    const float d = x - b.mu;
    const float u = (d * d) * b.c3;
    return fmaf(b.c1, ex2f(-u), b.c2 * rcpf(1.0f + u));
  } else {
    return b.c1;
  }
}

// ------------------------------------------------------------- chain unit
struct Xch {  // per-unit cross-warp exchange, double-buffered by parity
  float2 scan[2][16];
  double en[2][16];
  int flt[2][16];
};

struct UnitCtx {
  const float* sx;
  const float2* sc;
  const float2* sy;
  Xch* xc;
  int lg, L, W, wiu, lane, bar_id, p0;
  int par;
};

__device__ __forceinline__ void unit_sync(const UnitCtx& u) {
  if (u.W > 1) named_bar(u.bar_id, 32 * u.W);
}

// signal without background: P_k = sum_b g_b(x_k), blocks in layout order
// (combine, model.cpp:287-288).  Optional override of one parameter.
template <int FAM, int PPL>
__device__ __forceinline__ bool full_signal(const GroupDesc& g, const double* th, int ovr_i, double ovr_v,
                                            const UnitCtx& u, float (&P)[PPL]) {
#pragma unroll
  for (int k = 0; k < PPL; ++k) P[k] = 0.f;
  const int stride = block_stride<FAM>();
  const int nb = FAM == FAM_OFFSET ? 1 : g.K;
  bool ok = true;
  for (int b = 0; b < nb; ++b) {
    double p[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j < stride) p[j] = (b * stride + j == ovr_i) ? ovr_v : th[b * stride + j];
    const BlockC c = block_consts<FAM>(p);
    ok = ok && c.ok;
#pragma unroll
    for (int k = 0; k < PPL; ++k) P[k] += shape<FAM>(c, u.sx[k * u.L + u.lg]);
  }
  return ok;
}

// trial signal for component i set to v.  Returns false on a shape fault.
template <int FAM, int PPL>
__device__ __forceinline__ bool trial_signal(const GroupDesc& g, const double* th, int i, double v, const UnitCtx& u,
                                             const float (&P)[PPL], bool pvalid, float (&Pn)[PPL]) {
  const int stride = block_stride<FAM>();
  if (FAM == FAM_OFFSET) return full_signal<FAM, PPL>(g, th, i, v, u, Pn);
  if (FAM == FAM_XPS && i >= 4 * g.K) {  // Shirley endpoint: enters combine() only (block -1)
    if (pvalid) {
#pragma unroll
      for (int k = 0; k < PPL; ++k) Pn[k] = P[k];
      return true;
    }
    return full_signal<FAM, PPL>(g, th, i, v, u, Pn);
  }
  if (!pvalid) return full_signal<FAM, PPL>(g, th, i, v, u, Pn);
  const int b = i / stride, j = i - b * stride;
  double po[4], pn[4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (q < stride) {
      po[q] = th[b * stride + q];
      pn[q] = (q == j) ? v : po[q];
    }
  const BlockC cn = block_consts<FAM>(pn);
  if (!cn.ok) return false;
  const BlockC co = block_consts<FAM>(po);
#pragma unroll
  for (int k = 0; k < PPL; ++k) {
    const float x = u.sx[k * u.L + u.lg];
    Pn[k] = P[k] + (shape<FAM>(cn, x) - shape<FAM>(co, x));
  }
  return true;
}

// per-point centred negative log-likelihood term (data_energy, energy.cpp:7-28)
//   gauss:  r^2                                         E = a0 + a1 * sum
//   hetero: 1/2 ln(var/s_k) + q r^2/var, var = a1 f^2 + a0 f + a2  (GaussApprox = (1,0,0))
//   poisson: f - y - y ln(f/y)  (deviance form)
template <int NZ>
__device__ __forceinline__ float noise_term(const GroupDesc& g, float f, float2 yq, bool& flt) {
  const float r = yq.x - f;
  if (NZ == NZ_GAUSS) {
    return r * r;
  } else if (NZ == NZ_HETERO) {
    const float var = fmaf(fmaf(g.nz_a1, f, g.nz_a0), f, g.nz_a2);
    flt = flt || !(var > 0.f);
    return fmaf(kHalfLn2, lg2f(var * yq.y), g.nz_q * (r * r) * rcpf(var));
  } else {
    flt = flt || !(f > 0.f);
    return (f - yq.x) - yq.x * (kLn2 * lg2f(f * yq.y));
  }
}

// fp64 reduction of the lane partials over the unit; identical in every warp
__device__ __forceinline__ double unit_energy(const GroupDesc& g, UnitCtx& u, float acc, bool flt) {
  double s = warp_sum_d((double)acc);
  bool wf = __any_sync(0xffffffffu, flt);
  if (u.W > 1) {
    if (u.lane == 0) {
      u.xc->en[u.par][u.wiu] = s;
      u.xc->flt[u.par][u.wiu] = wf ? 1 : 0;
    }
    unit_sync(u);
    s = 0.0;
    wf = false;
    for (int w = 0; w < u.W; ++w) {
      s += u.xc->en[u.par][w];
      wf = wf || u.xc->flt[u.par][w];
    }
  }
  u.par ^= 1;
  return wf ? dinf() : g.e_a0 + g.e_a1 * s;
}

template <int PPL, int NZ>
__device__ __forceinline__ double eval_plain_nz(const GroupDesc& g, UnitCtx& u, const float (&Pn)[PPL]) {
  float acc = 0.f;
  bool flt = false;
#pragma unroll
  for (int k = 0; k < PPL; ++k) {
    const float2 yq = u.sy[k * u.L + u.lg];
    bool f1 = false;
    const float l = noise_term<NZ>(g, Pn[k], yq, f1);
    if (u.p0 + k < g.N) {
      acc += l;
      flt = flt || f1;
    }
  }
  return unit_energy(g, u, acc, flt);
}

// Shirley background + energy (lineshapes.hpp:65-83, model.cpp:289-292)
template <int PPL, int NZ>
__device__ __forceinline__ double eval_shirley_nz(const GroupDesc& g, UnitCtx& u, const float (&Pn)[PPL], float bga,
                                                  float bgb) {
  float Cn[PPL];
  float run = 0.f, mx = -FLT_MAX;
#pragma unroll
  for (int k = 0; k < PPL; ++k) {
    const float2 c = u.sc[k * u.L + u.lg];
    run = fmaf(c.x, Pn[k], run);
    Cn[k] = fmaf(-c.y, Pn[k], run);
    if (u.p0 + k < g.N) mx = fmaxf(mx, Pn[k]);
  }
  const float incl = warp_incl_scan_f(run, u.lane);
  float prefix = incl - run;
  float total = __shfl_sync(0xffffffffu, incl, 31);
  float gmax = warp_max_f(mx);
  if (u.W > 1) {
    if (u.lane == 0) u.xc->scan[u.par][u.wiu] = make_float2(total, gmax);
    unit_sync(u);
    float pre = 0.f, tot = 0.f, gm = -FLT_MAX;
    for (int w = 0; w < u.W; ++w) {
      const float2 s = u.xc->scan[u.par][w];
      if (w < u.wiu) pre += s.x;
      tot += s.x;
      gm = fmaxf(gm, s.y);
    }
    prefix += pre;
    total = tot;
    gmax = gm;
  }
  const float ba = bgb - bga;
  const bool degen = !(total > 1e-12f * gmax * g.range);
  const float scale = degen ? 0.f : ba / total;
  float acc = 0.f;
  bool flt = false;
#pragma unroll
  for (int k = 0; k < PPL; ++k) {
    const int p = u.p0 + k;
    float B = degen ? fmaf(ba, (u.sx[k * u.L + u.lg] - g.x0s) * g.inv_range, bga) : fmaf(scale, prefix + Cn[k], bga);
    if (p == 0) B = bga;
    if (p == g.N - 1) B = bgb;
    const float2 yq = u.sy[k * u.L + u.lg];
    bool f1 = false;
    const float l = noise_term<NZ>(g, Pn[k] + B, yq, f1);
    if (p < g.N) {
      acc += l;
      flt = flt || f1;
    }
  }
  return unit_energy(g, u, acc, flt);
}

template <int FAM, int PPL>
__device__ __forceinline__ double evaluate(const GroupDesc& g, UnitCtx& u, const float (&Pn)[PPL], float bga,
                                           float bgb) {
  if (FAM == FAM_XPS) {
    switch (g.noise) {
      case NZ_GAUSS: return eval_shirley_nz<PPL, NZ_GAUSS>(g, u, Pn, bga, bgb);
      case NZ_HETERO: return eval_shirley_nz<PPL, NZ_HETERO>(g, u, Pn, bga, bgb);
      default: return eval_shirley_nz<PPL, NZ_POISSON>(g, u, Pn, bga, bgb);
    }
  } else {
    switch (g.noise) {
      case NZ_GAUSS: return eval_plain_nz<PPL, NZ_GAUSS>(g, u, Pn);
      case NZ_HETERO: return eval_plain_nz<PPL, NZ_HETERO>(g, u, Pn);
      default: return eval_plain_nz<PPL, NZ_POISSON>(g, u, Pn);
    }
  }
}

// ------------------------------------------------------------------ priors
// lp_new - lp_old for one component (priors.cpp:22-35); false = -inf (reject)
__device__ __forceinline__ bool prior_delta(int kind, double a, double b, double xo, double xn, double& dlp) {
  if (kind == PR_UNIFORM) {
    if (xn < a || xn > b) return false;
    dlp = (xo < a || xo > b) ? dinf() : 0.0;
    return true;
  }
  if (kind == PR_NORMAL) {
    const double dn = xn - a, dd = xo - a;
    dlp = (dd * dd - dn * dn) / (2.0 * b);
    return true;
  }
  if (!(xn > 0.0)) return false;
  if (!(xo > 0.0)) {
    dlp = dinf();
    return true;
  }
  dlp = (a - 1.0) * (double)__logf((float)(xn / xo)) - b * (xn - xo);
  return true;
}

// ------------------------------------------------------------- CTA -> group
__device__ __forceinline__ int find_group(const int* prefix, int n, int x) {
  int lo = 0, hi = n - 1;  // largest gi with prefix[gi] <= x
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= x)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// ------------------------------------------------------------ chain kernel
// ENERGY = true : unit c evaluates the full energy of particle c of theta[cur]
// ENERGY = false: unit c runs waste-free chain c of the current level
template <int FAM, int PPL, bool ENERGY>
__global__ void __launch_bounds__(256) k_chain(const GroupDesc* __restrict__ gds, const int* __restrict__ list,
                                               const int* __restrict__ cta_prefix, int n_list, int W, int U,
                                               int dpad) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int gi = find_group(cta_prefix, n_list, blockIdx.x);
  const GroupDesc& g = gds[list[gi]];
  const int cta_in_group = blockIdx.x - cta_prefix[gi];
  const int L = 32 * W;
  const int npt = PPL * L;

  // ---- carve shared memory
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  float* sx = reinterpret_cast<float*>(smem + 16);
  float2* sc = reinterpret_cast<float2*>(sx + npt);
  float2* sy = sc + npt;
  unsigned char* wbase = reinterpret_cast<unsigned char*>(sy + npt);
  const int nwarps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* th = reinterpret_cast<double*>(wbase) + (size_t)warp * dpad;
  double* lsv = reinterpret_cast<double*>(wbase) + (size_t)(nwarps + warp) * dpad;
  int* acc = reinterpret_cast<int*>(reinterpret_cast<double*>(wbase) + (size_t)2 * nwarps * dpad) + (size_t)warp * dpad;
  Xch* xcs = reinterpret_cast<Xch*>(reinterpret_cast<int*>(reinterpret_cast<double*>(wbase) + (size_t)2 * nwarps * dpad) +
                                    (size_t)nwarps * dpad);

  // ---- stage the spectrum (cp.async.bulk -> mbarrier)
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    const uint32_t bx = npt * 4u, bc = npt * 8u;
    mbar_expect_tx(bar, bx + 2u * bc);
    bulk_g2s(sx, g.spec_x, bx, bar);
    bulk_g2s(sc, g.spec_c, bc, bar);
    bulk_g2s(sy, g.spec_y, bc, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);

  const int unit = warp / W, wiu = warp - unit * W;
  const int c = cta_in_group * U + unit;
  const int units = ENERGY ? g.T : g.S;
  if (c >= units) return;  // whole unit leaves together; no CTA-wide barrier follows

  UnitCtx u;
  u.sx = sx;
  u.sc = sc;
  u.sy = sy;
  u.xc = xcs + unit;
  u.lg = wiu * 32 + lane;
  u.L = L;
  u.W = W;
  u.wiu = wiu;
  u.lane = lane;
  u.bar_id = 1 + unit;
  u.p0 = u.lg * PPL;
  u.par = 0;

  const GroupState* st = g.st;
  const int cur = st->cur;
  const int d = g.d, T = g.T;
  const double* thc = g.theta[cur];
  const int src = ENERGY ? c : g.anc[c];
  for (int i = lane; i < d; i += 32) {
    th[i] = thc[(size_t)i * T + src];
    if (!ENERGY) {
      lsv[i] = g.ls0[i];
      acc[i] = 0;
    }
  }
  __syncwarp();

  float P[PPL];
  bool pvalid = full_signal<FAM, PPL>(g, th, -1, 0.0, u, P);
  const int ibg = 4 * g.K;
  double e = pvalid ? evaluate<FAM, PPL>(g, u, P, FAM == FAM_XPS ? (float)th[ibg] : 0.f,
                                         FAM == FAM_XPS ? (float)th[ibg + 1] : 0.f)
                    : dinf();
  if (ENERGY) {
    if (wiu == 0 && lane == 0) g.E[cur][c] = e;
    return;
  }

  // ---- waste-free chain: n sweeps at beta_next, keep every post-sweep state
  const int n = g.n, S = g.S;
  const int level = st->level;
  const double beta = st->beta;
  const double nd = g.n_data;
  const int adapt_sweeps = (n + 1) / 2;  // smc.cpp:136
  const uint32_t cg = g.chain_base + (uint32_t)c;
  double* thn = g.theta[cur ^ 1];
  double* En = g.E[cur ^ 1];
  unsigned long long trials = 0;
  float Pn[PPL];

  for (int t = 1; t <= n; ++t) {
    const float gam = (t <= adapt_sweeps) ? exp2f(-0.6f * log2f((float)t)) : 0.f;  // t^-0.6 (mcmc.cpp:15)
    for (int i = 0; i < d; ++i) {
      const u32x4 o = philox(u32x4{cg, (uint32_t)level, (uint32_t)((t - 1) * d + i), ROLE_CHAIN}, g.key0, g.key1);
      const float z = normal_f32(o.x, o.y);
      const double old_i = th[i];
      const double s = (double)__expf((float)lsv[i]);
      const double new_i = old_i + s * (double)z;
      double dlp = 0.0;
      const bool in_support = prior_delta(g.pkind[i], g.pa[i], g.pb[i], old_i, new_i, dlp);
      bool accept = false;
      if (in_support) {
        ++trials;
        const bool nvalid = trial_signal<FAM, PPL>(g, th, i, new_i, u, P, pvalid, Pn);
        float bga = 0.f, bgb = 0.f;
        if (FAM == FAM_XPS) {
          bga = (float)(i == ibg ? new_i : th[ibg]);
          bgb = (float)(i == ibg + 1 ? new_i : th[ibg + 1]);
        }
        const double e_new = nvalid ? evaluate<FAM, PPL>(g, u, Pn, bga, bgb) : dinf();
        // mcmc.cpp:72-80
        double lr;
        const bool inf_new = e_new == dinf(), inf_old = e == dinf();
        if (beta == 0.0 || (inf_new && inf_old))
          lr = dlp;
        else if (inf_new)
          lr = -dinf();
        else if (inf_old)
          lr = dinf();
        else
          lr = -beta * nd * (e_new - e) + dlp;
        accept = lr >= 0.0 || (double)__logf(u01_open_lo(o.z)) < lr;
        if (accept) {
#pragma unroll
          for (int k = 0; k < PPL; ++k) P[k] = Pn[k];
          pvalid = nvalid;
          e = e_new;
          if (lane == 0) {
            th[i] = new_i;
            acc[i] += 1;
          }
        }
      }
      if (t <= adapt_sweeps && lane == 0) {  // robbins_monro_update in log space (mcmc.cpp:14-18)
        double ls = lsv[i] + (double)gam * ((accept ? 1.0 : 0.0) - 0.5);
        lsv[i] = fmin(fmax(ls, kLogStepMin), kLogStepMax);
      }
      __syncwarp();
    }
    const size_t slot = (size_t)c * n + (t - 1);  // smc.cpp:151
    if (wiu == 0) {
      for (int i = lane; i < d; i += 32) thn[(size_t)i * T + slot] = th[i];
      if (lane == 0) En[slot] = e;
    }
  }
  if (wiu == 0) {
    for (int i = lane; i < d; i += 32) {
      g.chain_acc[(size_t)i * S + c] = acc[i];
      g.chain_ls[(size_t)i * S + c] = lsv[i];
    }
    if (lane == 0) atomicAdd(&g.st->trials, trials);
  }
}

// ------------------------------------------------------------- init draws
// rng.hpp:77-92 (Marsaglia-Tsang) in fp64 on a Philox stream
__device__ double gamma_draw(double shape, double rate, uint32_t p, uint32_t& seq, uint32_t k0, uint32_t k1) {
  double boost = 1.0;
  if (shape < 1.0) {
    const u32x4 o = philox(u32x4{p, 0u, seq++, ROLE_INIT}, k0, k1);
    const double u = 1.0 - u53(o.x, o.y);
    boost = pow(u, 1.0 / shape);
    shape += 1.0;
  }
  const double dd = shape - 1.0 / 3.0;
  const double cc = 1.0 / sqrt(9.0 * dd);
  for (int it = 0; it < 1000; ++it) {
    const double x = normal_f64(philox(u32x4{p, 0u, seq++, ROLE_INIT}, k0, k1));
    const double t = 1.0 + cc * x;
    if (t <= 0.0) continue;
    const double v = t * t * t;
    const u32x4 o = philox(u32x4{p, 0u, seq++, ROLE_INIT}, k0, k1);
    const double uu = 1.0 - u53(o.x, o.y);
    if (log(uu) < 0.5 * x * x + dd - dd * v + dd * log(v)) return boost * dd * v / rate;
  }
  return boost * dd / rate;
}

__global__ void k_init_draw(const GroupDesc* __restrict__ gds, const int* __restrict__ list) {
  const GroupDesc& g = gds[list[blockIdx.y]];
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= g.T) return;
  double* th = g.theta[0];
  uint32_t seq = 0;
  const uint32_t pid = g.chain_base * 0u + (uint32_t)p;
  for (int i = 0; i < g.d; ++i) {
    const int kind = g.pkind[i];
    const double a = g.pa[i], b = g.pb[i];
    double v;
    if (kind == PR_NORMAL) {
      v = a + sqrt(b) * normal_f64(philox(u32x4{pid, 0u, seq++, ROLE_INIT}, g.key0, g.key1));
    } else if (kind == PR_GAMMA) {
      v = gamma_draw(a, b, pid, seq, g.key0, g.key1);
    } else {
      const u32x4 o = philox(u32x4{pid, 0u, seq++, ROLE_INIT}, g.key0, g.key1);
      v = a + (b - a) * u53(o.x, o.y);
    }
    th[(size_t)i * g.T + p] = v;
  }
}

// ------------------------------------------------------- block reductions
constexpr int kTemperThreads = 1024;

template <typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, T* sh, Op op, T ident) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < nw ? sh[lane] : ident;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) sh[0] = v;
  }
  __syncthreads();
  return sh[0];
}
struct OpAdd {
  __device__ double operator()(double a, double b) const { return a + b; }
};
struct OpMax {
  __device__ double operator()(double a, double b) const { return fmax(a, b); }
};
struct OpMin {
  __device__ double operator()(double a, double b) const { return a < b ? a : b; }
};
struct OpMaxI {
  __device__ long long operator()(long long a, long long b) const { return a > b ? a : b; }
};

// exp(a) for a <= 0 with fp64 range reduction and an fp32 MUFU mantissa
__device__ __forceinline__ double exp_neg_split(double a) {
  if (!(a > -745.0)) return 0.0;
  const double y = a * 1.4426950408889634074;
  const double yi = floor(y);
  const float yf = (float)(y - yi);
  return scalbn((double)ex2f(yf), (int)yi);
}

struct TemperShared {
  double red[32];
  long long redi[32];
  double bc[4];
  int ibc[4];
};

// (sum w)^2 / sum w^2 / T with w = exp(c (E - emin)) (smc.cpp:61-66, :76-79);
// returns NaN when every weight vanishes
__device__ double ess_ratio_at(const double* E, int64_t T, double emin, double c, TemperShared& sh) {
  double a1 = 0.0, a2 = 0.0;
  for (int64_t i = threadIdx.x; i < T; i += blockDim.x) {
    const double w = exp_neg_split(c * (E[i] - emin));
    a1 += w;
    a2 += w * w;
  }
  const double s1 = block_reduce(a1, sh.red, OpAdd(), 0.0);
  const double s2 = block_reduce(a2, sh.red, OpAdd(), 0.0);
  if (!(s1 > 0.0)) return nan("");
  return (s1 * s1 / s2) / (double)T;
}

__device__ double block_emin(const double* E, int64_t T, TemperShared& sh) {
  double m = dinf();
  for (int64_t i = threadIdx.x; i < T; i += blockDim.x) m = (E[i] < m) ? E[i] : m;
  m = block_reduce(m, sh.red, OpMin(), dinf());
  return isfinite(m) ? m : 0.0;
}

// next_beta (smc.cpp:68-93); err = 1 when every weight vanishes
__device__ double block_next_beta(const double* E, int64_t T, double n_data, double beta_prev, double target,
                                  TemperShared& sh, int& err) {
  err = 0;
  const double emin = block_emin(E, T, sh);
  const double full = 1.0 - beta_prev;
  double r = ess_ratio_at(E, T, emin, -full * n_data, sh);
  if (isnan(r)) {
    err = 1;
    return 0.0;
  }
  if (r >= target) return 1.0;
  double lo = 0.0, hi = full, mid = 0.5 * full;
  for (int it = 0; it < 60; ++it) {
    mid = 0.5 * (lo + hi);
    r = ess_ratio_at(E, T, emin, -mid * n_data, sh);
    if (isnan(r)) {
      err = 1;
      return 0.0;
    }
    if (fabs(r - target) <= 1e-6) break;
    if (r > target)
      lo = mid;
    else
      hi = mid;
  }
  return beta_prev + mid;
}

// incremental weights (smc.cpp:55-59) -> lse, ess ratio, log_mean_w; writes
// normalised weights exp(lw - lse) to wout.  Returns false if all vanish.
__device__ bool block_weights(const double* E, int64_t T, double delta, double n_data, double* wout,
                              TemperShared& sh, double& ess_ratio, double& log_mean_w) {
  const double c = -delta * n_data;
  double m = -dinf();
  for (int64_t i = threadIdx.x; i < T; i += blockDim.x) {
    const double lw = delta == 0.0 ? 0.0 : c * E[i];
    m = fmax(m, lw);
  }
  m = block_reduce(m, sh.red, OpMax(), -dinf());
  if (m == -dinf()) return false;
  double a1 = 0.0, a2 = 0.0;
  for (int64_t i = threadIdx.x; i < T; i += blockDim.x) {
    const double lw = delta == 0.0 ? 0.0 : c * E[i];
    const double w = exp(lw - m);
    a1 += w;
    a2 += w * w;
  }
  const double s1 = block_reduce(a1, sh.red, OpAdd(), 0.0);
  const double s2 = block_reduce(a2, sh.red, OpAdd(), 0.0);
  const double lse = m + log(s1);
  ess_ratio = (s1 * s1 / s2) / (double)T;
  log_mean_w = lse - log((double)T);
  if (wout)
    for (int64_t i = threadIdx.x; i < T; i += blockDim.x) {
      const double lw = delta == 0.0 ? 0.0 : c * E[i];
      wout[i] = exp(lw - lse);
    }
  __syncthreads();
  return true;
}

// #{j in [0,S): (j+u)/S <= x}, with the reference's fp64 comparison (smc.cpp:103-106)
__device__ __forceinline__ long long count_le(double x, double u, long long S) {
  const double Sd = (double)S;
  double jm = floor(x * Sd - u);
  long long j = jm < -1.0 ? -1 : (jm > (double)(S - 1) ? S - 1 : (long long)jm);
  while (j + 1 < S && ((double)(j + 1) + u) / Sd <= x) ++j;
  while (j >= 0 && ((double)j + u) / Sd > x) --j;
  return j + 1;
}

// systematic resampling over normalised weights w (smc.cpp:95-112): block fp64
// scan of the CDF, then every element i writes the targets
// j with c_{i-1} < (j+u)/S <= c_i (running max keeps ranges disjoint).
__device__ void block_resample(const double* w, int64_t T, long long S, double u, int* anc, TemperShared& sh) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t chunk = (T + nt - 1) / nt;
  const int64_t b0 = (int64_t)tid * chunk < T ? (int64_t)tid * chunk : T;
  const int64_t b1 = b0 + chunk < T ? b0 + chunk : T;
  double loc = 0.0;
  for (int64_t i = b0; i < b1; ++i) loc += w[i];
  // block exclusive scan of loc (fp64)
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  double incl = warp_incl_scan_d(loc, lane);
  __syncthreads();
  if (lane == 31) sh.red[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    double v = lane < nw ? sh.red[lane] : 0.0;
    const double vi = warp_incl_scan_d(v, lane);
    if (lane < nw) sh.red[lane] = vi - v;  // exclusive warp offsets
  }
  __syncthreads();
  const double prefix = sh.red[warp] + (incl - loc);
  // running boundary counts; per-thread maximum then block exclusive max-scan
  long long mymax = 0;
  {
    double cc = prefix;
    for (int64_t i = b0; i < b1; ++i) {
      cc += w[i];
      long long k = (i == T - 1) ? S : count_le(cc, u, S);
      mymax = k > mymax ? k : mymax;
    }
  }
  long long v = mymax;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v = v > t ? v : t;
  }
  __syncthreads();
  if (lane == 31) sh.redi[warp] = v;
  __syncthreads();
  if (warp == 0) {
    long long x = lane < nw ? sh.redi[lane] : 0;
    long long xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long t = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi = xi > t ? xi : t;
    }
    const long long ex = __shfl_up_sync(0xffffffffu, xi, 1);
    if (lane < nw) sh.redi[lane] = lane == 0 ? 0 : ex;
  }
  __syncthreads();
  long long excl_lane = __shfl_up_sync(0xffffffffu, v, 1);
  if (lane == 0) excl_lane = 0;
  long long lo = sh.redi[warp] > excl_lane ? sh.redi[warp] : excl_lane;
  double cc = prefix;
  for (int64_t i = b0; i < b1; ++i) {
    cc += w[i];
    long long k = (i == T - 1) ? S : count_le(cc, u, S);
    if (k < lo) k = lo;
    for (long long j = lo; j < k; ++j) anc[j] = (int)i;
    lo = k;
  }
  __syncthreads();
}

// predict_step_size (mcmc.cpp:20-53) for component i; hist is the ring of
// the last min(H, 5) levels, entry = (beta, acc[d], step[d]); returns log step
__device__ double predict_log_step(const double* hist, int H, int d, int i, double beta_next, int kind, double a,
                                   double b) {
  if (H == 0) {
    double s = kind == PR_NORMAL ? sqrt(b) : (kind == PR_GAMMA ? sqrt(a) / b : (b - a) / sqrt(12.0));
    s = fmin(fmax(s, 1e-12), 1e12);
    return log(s);
  }
  const int m = H < kHist ? H : kHist;
  const int stride = 1 + 2 * d;
  double sx = 0, sy = 0, sxx = 0, sxy = 0;
  for (int jj = H - m; jj < H; ++jj) {
    const double* h = hist + (size_t)(jj % kHist) * stride;
    const double x = log(h[0]);
    const double y = log(h[1 + d + i]) + 2.0 * (h[1 + i] - 0.5);
    sx += x;
    sy += y;
    sxx += x * x;
    sxy += x * y;
  }
  double pred;
  const double denom = m * sxx - sx * sx;
  if (m < 2 || fabs(denom) < 1e-12 * (m * sxx + sx * sx + 1e-300)) {
    pred = sy / m;
  } else {
    const double slope = (m * sxy - sx * sy) / denom;
    const double icept = (sy - slope * sx) / m;
    pred = icept + slope * log(beta_next);
  }
  const double s = fmin(fmax(exp(pred), 1e-12), 1e12);
  return log(s);
}

// one CTA per active group: tempering + evidence + resampling + step prediction
__global__ void __launch_bounds__(kTemperThreads) k_temper(const GroupDesc* __restrict__ gds,
                                                           const int* __restrict__ list) {
  __shared__ TemperShared sh;
  const GroupDesc& g = gds[list[blockIdx.x]];
  GroupState* st = g.st;
  const int level = st->level;
  if (level >= g.max_levels) {  // smc.cpp:195-196
    if (threadIdx.x == 0) {
      st->error = GE_MAX_LEVELS;
      st->active = 0;
    }
    return;
  }
  const double* E = g.E[st->cur];
  const int64_t T = g.T;
  const double beta_prev = st->beta;
  int err = 0;
  const double beta_next = block_next_beta(E, T, g.n_data, beta_prev, g.ess_target, sh, err);
  double ess_ratio = 0.0, lmw = 0.0;
  bool ok = !err && block_weights(E, T, beta_next - beta_prev, g.n_data, g.wbuf, sh, ess_ratio, lmw);
  if (!ok) {
    if (threadIdx.x == 0) {
      st->error = GE_ZERO_WEIGHT;
      st->active = 0;
    }
    return;
  }
  const u32x4 o = philox(u32x4{0u, (uint32_t)(level + 1), 0u, ROLE_RESAMPLE}, g.key0, g.key1);
  const double u = u53(o.x, o.y);
  block_resample(g.wbuf, T, g.S, u, g.anc, sh);
  for (int i = threadIdx.x; i < g.d; i += blockDim.x)
    g.ls0[i] = predict_log_step(g.hist, st->hist_count, g.d, i, beta_next, g.pkind[i], g.pa[i], g.pb[i]);
  __syncthreads();
  if (threadIdx.x == 0) {
    double* dg = g.diag + (size_t)level * 4;
    dg[0] = beta_next;
    dg[1] = ess_ratio;
    dg[2] = lmw;
    st->neg_log_z -= lmw;  // smc.cpp:201
    st->beta = beta_next;
    st->level = level + 1;
  }
}

// one CTA per active group: pooled acceptance, geometric-mean step (smc.cpp:162-183)
__global__ void __launch_bounds__(256) k_stats(const GroupDesc* __restrict__ gds, const int* __restrict__ list) {
  __shared__ TemperShared sh;
  const GroupDesc& g = gds[list[blockIdx.x]];
  GroupState* st = g.st;
  const int d = g.d, S = g.S, H = st->hist_count;
  const int stride = 1 + 2 * d;
  double* h = g.hist + (size_t)(H % kHist) * stride;
  double acc_all = 0.0;
  for (int i = 0; i < d; ++i) {
    double a = 0.0, l = 0.0;
    for (int c = threadIdx.x; c < S; c += blockDim.x) {
      a += (double)g.chain_acc[(size_t)i * S + c];
      l += g.chain_ls[(size_t)i * S + c];
    }
    a = block_reduce(a, sh.red, OpAdd(), 0.0);
    l = block_reduce(l, sh.red, OpAdd(), 0.0);
    if (threadIdx.x == 0) {
      const double prop = (double)S * g.n;
      h[1 + i] = prop > 0 ? a / prop : 0.0;
      h[1 + d + i] = exp(l / (double)S);
    }
    acc_all += a;
  }
  if (threadIdx.x == 0) {
    const double beta = st->beta;
    h[0] = beta;
    const double prop_all = (double)S * g.n * d;
    g.diag[(size_t)(st->level - 1) * 4 + 3] = prop_all > 0 ? acc_all / prop_all : 0.0;
    st->hist_count = H + 1;
    st->cur ^= 1;
    if (beta >= 1.0) st->active = 0;
  }
}

// ---------------------------------------------------------- unit kernels
__global__ void __launch_bounds__(kTemperThreads) k_unit_ess(const double* lw, int64_t n, double* out, int* err) {
  __shared__ TemperShared sh;
  double m = -dinf();
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, lw[i]);
  m = block_reduce(m, sh.red, OpMax(), -dinf());
  if (m == -dinf()) {
    if (threadIdx.x == 0) *err = 1;
    return;
  }
  double a1 = 0.0, a2 = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double w = exp(lw[i] - m);
    a1 += w;
    a2 += w * w;
  }
  a1 = block_reduce(a1, sh.red, OpAdd(), 0.0);
  a2 = block_reduce(a2, sh.red, OpAdd(), 0.0);
  if (threadIdx.x == 0) {
    *out = a1 * a1 / a2;
    *err = 0;
  }
}

__global__ void __launch_bounds__(kTemperThreads) k_unit_lme(const double* v, int64_t n, double* out) {
  __shared__ TemperShared sh;
  double m = -dinf();
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, v[i]);
  m = block_reduce(m, sh.red, OpMax(), -dinf());
  if (!isfinite(m)) {
    if (threadIdx.x == 0) *out = m;
    return;
  }
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a += exp(v[i] - m);
  a = block_reduce(a, sh.red, OpAdd(), 0.0);
  if (threadIdx.x == 0) *out = m + log(a) - log((double)n);
}

__global__ void __launch_bounds__(kTemperThreads) k_unit_next_beta(const double* E, int64_t n, double n_data,
                                                                   double beta_prev, double target, double* out,
                                                                   int* err) {
  __shared__ TemperShared sh;
  int e = 0;
  const double b = block_next_beta(E, n, n_data, beta_prev, target, sh, e);
  if (threadIdx.x == 0) {
    *out = b;
    *err = e;
  }
}

__global__ void __launch_bounds__(kTemperThreads) k_unit_resample(const double* lw, int64_t n, long long S, double u,
                                                                  double* wscr, int* anc, int* err) {
  __shared__ TemperShared sh;
  double m = -dinf();
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, lw[i]);
  m = block_reduce(m, sh.red, OpMax(), -dinf());
  if (m == -dinf()) {
    if (threadIdx.x == 0) *err = 1;
    return;
  }
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a += exp(lw[i] - m);
  a = block_reduce(a, sh.red, OpAdd(), 0.0);
  const double lse = m + log(a);
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) wscr[i] = exp(lw[i] - lse);
  __syncthreads();
  block_resample(wscr, n, S, u, anc, sh);
  if (threadIdx.x == 0) *err = 0;
}

__global__ void k_unit_predict(const double* hist, int H, int d, double beta_next, const int* pk, const double* pa,
                               const double* pb, double* out) {
  for (int i = threadIdx.x; i < d; i += blockDim.x)
    out[i] = exp(predict_log_step(hist, H, d, i, beta_next, pk[i], pa[i], pb[i]));
}

// ============================================================== launchers
static const int kPPL[] = {2, 4, 6, 8, 10, 12, 14, 16};

bool ppl_supported(int ppl) {
  for (int p : kPPL)
    if (p == ppl) return true;
  return false;
}

Shape pick_shape(int64_t N) {
  int W = 1;
  while (W < 16 && (int64_t)32 * W * 16 < N) W *= 2;
  int ppl = 16;
  for (int p : kPPL)
    if ((int64_t)32 * W * p >= N) {
      ppl = p;
      break;
    }
  Shape s;
  s.W = W;
  s.PPL = ppl;
  s.U = W >= 8 ? 1 : 8 / W;
  return s;
}

size_t chain_smem_bytes(const Shape& s, int dmax) {
  const int dpad = (dmax + 1) & ~1;
  const int L = 32 * s.W;
  const int nwarps = s.W * s.U;
  size_t b = 16;                         // mbarrier
  b += (size_t)s.PPL * L * (4 + 8 + 8);  // sx, sc, sy
  b += (size_t)nwarps * dpad * (8 + 8 + 4);
  b = (b + 15) & ~(size_t)15;
  b += (size_t)s.U * sizeof(Xch);
  return b;
}

template <int FAM, int PPL, bool ENERGY>
static cudaError_t launch_chain_t(const Shape& s, int dmax, const GroupDesc* gds, const int* list, const int* prefix,
                                  int n_list, int total_ctas, cudaStream_t st) {
  const size_t smem = chain_smem_bytes(s, dmax);
  auto kern = k_chain<FAM, PPL, ENERGY>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int dpad = (dmax + 1) & ~1;
  kern<<<total_ctas, 32 * s.W * s.U, smem, st>>>(gds, list, prefix, n_list, s.W, s.U, dpad);
  return cudaGetLastError();
}

template <bool ENERGY>
static cudaError_t launch_chain(int family, const Shape& s, int dmax, const GroupDesc* gds, const int* list,
                                const int* prefix, int n_list, int total_ctas, cudaStream_t st) {
#define SMC_PPL_CASE(FAM, P) \
  case P: return launch_chain_t<FAM, P, ENERGY>(s, dmax, gds, list, prefix, n_list, total_ctas, st);
#define SMC_FAM_CASE(FAM)                                                                                      \
  switch (s.PPL) {                                                                                             \
    SMC_PPL_CASE(FAM, 2)                                                                                       \
    SMC_PPL_CASE(FAM, 4)                                                                                       \
    SMC_PPL_CASE(FAM, 6)                                                                                       \
    SMC_PPL_CASE(FAM, 8)                                                                                       \
    SMC_PPL_CASE(FAM, 10)                                                                                      \
    SMC_PPL_CASE(FAM, 12)                                                                                      \
    SMC_PPL_CASE(FAM, 14)                                                                                      \
    SMC_PPL_CASE(FAM, 16)                                                                                      \
    default: return cudaErrorInvalidValue;                                                                     \
  }
  switch (family) {
    case FAM_GM: SMC_FAM_CASE(FAM_GM)
    case FAM_XPS: SMC_FAM_CASE(FAM_XPS)
    case FAM_OFFSET: SMC_FAM_CASE(FAM_OFFSET)
    default: return cudaErrorInvalidValue;
  }
#undef SMC_FAM_CASE
#undef SMC_PPL_CASE
}

cudaError_t launch_energy(int family, const Shape& s, int dmax, const GroupDesc* gds, const int* list,
                          const int* prefix, int n_list, int total_ctas, cudaStream_t st) {
  return launch_chain<true>(family, s, dmax, gds, list, prefix, n_list, total_ctas, st);
}
cudaError_t launch_move(int family, const Shape& s, int dmax, const GroupDesc* gds, const int* list,
                        const int* prefix, int n_list, int total_ctas, cudaStream_t st) {
  return launch_chain<false>(family, s, dmax, gds, list, prefix, n_list, total_ctas, st);
}

cudaError_t launch_init_draw(const GroupDesc* gds, const int* list, int n_list, int Tmax, cudaStream_t st) {
  dim3 grid((Tmax + 255) / 256, n_list);
  k_init_draw<<<grid, 256, 0, st>>>(gds, list);
  return cudaGetLastError();
}
cudaError_t launch_temper(const GroupDesc* gds, const int* list, int n_list, cudaStream_t st) {
  k_temper<<<n_list, kTemperThreads, 0, st>>>(gds, list);
  return cudaGetLastError();
}
cudaError_t launch_stats(const GroupDesc* gds, const int* list, int n_list, cudaStream_t st) {
  k_stats<<<n_list, 256, 0, st>>>(gds, list);
  return cudaGetLastError();
}
cudaError_t launch_unit_ess(const double* lw, int64_t n, double* out, int* err, cudaStream_t st) {
  k_unit_ess<<<1, kTemperThreads, 0, st>>>(lw, n, out, err);
  return cudaGetLastError();
}
cudaError_t launch_unit_log_mean_exp(const double* v, int64_t n, double* out, cudaStream_t st) {
  k_unit_lme<<<1, kTemperThreads, 0, st>>>(v, n, out);
  return cudaGetLastError();
}
cudaError_t launch_unit_next_beta(const double* E, int64_t n, double n_data, double beta_prev, double target,
                                  double* out, int* err, cudaStream_t st) {
  k_unit_next_beta<<<1, kTemperThreads, 0, st>>>(E, n, n_data, beta_prev, target, out, err);
  return cudaGetLastError();
}
cudaError_t launch_unit_resample(const double* lw, int64_t n, int64_t S, double u, double* wscr, int* anc, int* err,
                                 cudaStream_t st) {
  k_unit_resample<<<1, kTemperThreads, 0, st>>>(lw, n, S, u, wscr, anc, err);
  return cudaGetLastError();
}
cudaError_t launch_unit_predict(const double* hist, int H, int d, double beta_next, const int* pk, const double* pa,
                                const double* pb, double* out, cudaStream_t st) {
  k_unit_predict<<<1, 128, 0, st>>>(hist, H, d, beta_next, pk, pa, pb, out);
  return cudaGetLastError();
}

}  // namespace smc
