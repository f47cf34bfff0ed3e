// chain.cuh -- the chain-parallel kernel of the B200 SMC sampler (K2 + K3).
//
//   k_chain<FAM, PPL, W, ENERGY=true>   batched full energies, one chain unit
//                                       per particle (BlockEvaluator::full,
//                                       energy.cpp:43-55 + data_energy :7-28)
//   k_chain<FAM, PPL, W, ENERGY=false>  fused propose/evaluate/accept move of
//                                       a waste-free level (smc.cpp:142-156
//                                       x cw_mh_sweep, mcmc.cpp:55-96)
// Reference paths are relative to the reference root (proj/...).
//
// A chain unit is W warps (L = 32 W lanes, compile-time).  Lane l owns the PPL
// consecutive points [l*PPL, (l+1)*PPL) of the spectrum and keeps, in
// registers,
//   P[k]  committed peak signal  sum_b g_b(x)      (combine, model.cpp:287-288)
//   Q[k]  P minus g_b(x) of the block being swept (shared memory, lane-transposed)
// A proposal changes one block: the trial signal is Pn = Q + g_new, and an
// amplitude proposal needs no transcendental at all (Pn = P + (A'/A - 1)(P - Q)).
// The Shirley background (lineshapes.hpp:65-83) needs the cumulative
// trapezoid of Pn: C_k = sum_{j<=k} c_j Pn_j - h_{k+1} Pn_k with
// c_j = h_j + h_{j+1}, h_j = (x_j - x_{j-1})/2, i.e. a lane-local scan and one
// warp (and cross-warp) scan per proposal.  Energy terms are O(1)-centred,
// summed per lane in fp32 and across lanes in fp64.  Padding points replicate
// the last real point with weight 0, so no per-point masks are needed; a
// forward/noise fault shows up as a non-finite sum (=> E = +inf, the
// reference's rejection sentinel).
#pragma once
#include <cfloat>
#include <cmath>

#include "launch.h"

namespace smc {

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }

constexpr float kHalfLn2 = 0.34657359027997264f;
constexpr float kLn2 = 0.6931471805599453f;

struct BlockC {
  float mu, c1, c2, c3;
  bool ok;
};

template <int FAM>
__device__ __forceinline__ constexpr int block_stride() {
  return FAM == FAM_GM ? 3 : (FAM == FAM_XPS ? 4 : (FAM == FAM_XRD ? 9 : 1));
}

// gm:  g = A exp(-b/2 (x-mu)^2) = c1 2^(c2 d^2)                   (model.cpp:216-220)
// xps: g = c1 2^(-u) + 1 / (c2 (1 + u)), u = t^2, t = x/sigma - mu/sigma = fma(x, c3, mu'),
//      c1 = A eta, c2 = 1 / (A (1-eta)) (the Lorentzian amplitude folded into its
//      reciprocal: one FMUL less per point; a zero Lorentzian amplitude becomes
//      c2 = 1e30, i.e. a contribution <= 1e-30)
//      (= A [eta exp(-ln2 d^2/s^2) + (1-eta) s^2/(s^2+d^2)], model.cpp:269-280)
// offset: g = theta_0                              (conjugate_oracle.hpp:22-26)
template <int FAM>
__device__ __forceinline__ BlockC block_consts(const float* p) {  // p: fp32 shadow of the block's parameters
  BlockC c;
  c.ok = true;
  c.c3 = 0.f;
  if (FAM == FAM_GM) {
    c.c1 = p[0];
    c.mu = p[1];
    c.c2 = p[2] * -0.72134752044448170f;  // -b/2 * log2(e)
  } else if (FAM == FAM_XPS) {
    const float A = p[0], sig = p[2], eta = p[3];
    c.ok = sig > 0.f;
    c.c3 = rcpf(sig);
    c.mu = -p[1] * c.c3;
    c.c1 = A * eta;
    const float aL = A - c.c1;
    c.c2 = aL != 0.f ? rcpf(aL) : 1e30f;
  } else {
    c.c1 = p[0];
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
    const float t = fmaf(x, b.c3, b.mu);
    const float nu = t * -t;  // -u: the negation rides on the FMUL (MUFU.EX2 takes no negate)
    return fmaf(b.c1, ex2f(nu), rcpf(fmaf(nu, -b.c2, b.c2)));
  } else {
    return b.c1;
  }
}

struct Xch {  // per-unit cross-warp exchange, double-buffered by parity
  float scan[2][16];
  int4 lim[2][16];  // energy partial sums: three fixed-point limbs + fault flag
};

// Per-CTA shared memory (dynamic):
//   [0,16)     mbarrier of the spectrum bulk copy
//   sx  float  [PPL][L]   shifted abscissa
//   sc  float2 [PPL][L]   (c_k, h_{k+1})
//   sy  float2 [PPL][L]   (y_k, 1/s_k)   (20 B per point: N = 8192 fits)
//   per unit: th f64, ls f64, acc i32, proposal f64, dlp f64, log u f32, flags i32,
//             fp32 shadows of th and of the proposal  (x dpad); every warp of the
//             unit computes and writes identical values (idempotent), one unit
//             barrier per sweep orders the sweep-level rewrites
//   per unit: Xch, then G float [PPL][L] (cached g_b(x) of the block being swept)
// committed peak signal P: shared memory for W = 2 and 4 (one trial signal in
// registers leaves the allocator room: no spills at 128 registers), registers
// for W = 1 and 8; see chain_p_in_smem (launch.h)
template <int W, int PPL>
__host__ __device__ constexpr bool p_in_smem() { return chain_p_in_smem(W, PPL); }

template <int PPL, int W>
struct Smem {
  static constexpr int L = 32 * W;
  static constexpr int NPT = PPL * L;
  // lay: spectrum layout flags (launch.h); W <= 2 always uses kLayFull
  __host__ __device__ static constexpr int layout(int lay) { return chain_dyn_layout(W) ? lay : kLayFull; }
  static constexpr size_t off_x = 16;
  static constexpr size_t off_c = off_x + (size_t)NPT * 4;
  __host__ __device__ static constexpr size_t off_y(int lay) {
    return off_c + ((layout(lay) & kLayWeights) ? (size_t)NPT * 8 : 0);
  }
  __host__ __device__ static constexpr size_t y_bytes(int lay) { return (layout(lay) & kLayY4) ? 4 : 8; }
  __host__ __device__ static constexpr size_t off_w(int lay) { return off_y(lay) + (size_t)NPT * y_bytes(lay); }
  __host__ __device__ static size_t per_unit(int dpad) { return (size_t)dpad * (8 + 8 + 4 + 8 + 8 + 4 + 4 + 4 + 4); }
  __host__ __device__ static size_t bytes(int U, int dpad, int lay) {
    size_t b = off_w(lay) + (size_t)U * per_unit(dpad);
    b = (b + 15) & ~(size_t)15;
    return b + (size_t)U * sizeof(Xch) + (size_t)U * NPT * (p_in_smem<W, PPL>() ? 8 : 4);  // + caches Q (and P)
  }
};

template <int PPL, int W>
struct Unit {
  static constexpr int L = 32 * W;
  static constexpr int NPT = PPL * L;
  const float* sx;
  const float2* sc;
  const float2* sy;
  int nv;      // leading real (non-padding) points of this lane
  float npad;  // padding points of this lane
  bool tail;   // uniform xps layout: this lane's last slot holds the last real point
  Xch* xc;
  int lg, wiu, lane, bar_id;
  int par;
  __device__ __forceinline__ float x(int k) const { return sx[k * L + lg]; }
  __device__ __forceinline__ float2 c(int k) const { return sc[k * L + lg]; }
  __device__ __forceinline__ float2 y(int k) const { return sy[k * L + lg]; }
  // paired noise layout (nz_pairs): (y_2p, y_2p+1) per point pair p
  __device__ __forceinline__ float2 y2(int p) const { return sy[p * L + lg]; }
  __device__ __forceinline__ void sync() const {
    if (W > 1) named_bar(bar_id, L);
  }
};

// ---- block geometry and block signals -----------------------------------
// Component i belongs to block b (a peak, an xrd phase, or the xrd background
// block K), is parameter j of it, and the block's parameters start at off.
template <int FAM>
struct BlockIdx {
  int b, j, off, np;  // np: parameters of the block
};
template <int FAM>
__device__ __forceinline__ BlockIdx<FAM> block_of(const GroupDesc& g, int i) {
  BlockIdx<FAM> r;
  if (FAM == FAM_XRD) {
    if (i < 9 * g.K) {
      r.b = i / 9;
      r.off = 9 * r.b;
      r.np = 9;
    } else {
      r.b = g.K;
      r.off = 9 * g.K;
      r.np = 4;
    }
  } else {
    constexpr int stride = block_stride<FAM>();
    r.b = i / stride;
    r.off = r.b * stride;
    r.np = stride;
  }
  r.j = i - r.off;
  return r;
}
template <int FAM>
__device__ __forceinline__ int n_blocks(const GroupDesc& g) {
  return FAM == FAM_OFFSET ? 1 : (FAM == FAM_XRD ? g.K + 1 : g.K);
}
template <int FAM>
__device__ __forceinline__ int block_off(const GroupDesc& g, int b) {
  return FAM == FAM_XRD ? 9 * b : b * block_stride<FAM>();
}

// acc_k += sign * g_b(x_k) for block b with (fp32) parameters p.  Returns false
// on an evaluation fault (model.cpp:226-258, :272-275): the block then adds nothing.
//   xrd phase b (model.cpp:235-267): sum over its reflections of
//     A ri [(1-r) 2^(-(2 dx/wg)^2) + r / (1 + (2 dx/wl)^2)],  c = mu_ref + d2t,
//     wg = sqrt(u tan^2 - v tan + w), wl = s / cos + t tan (theta = c/2), both x alpha for dx >= 0
//   xrd background (model.cpp:223-234): a [(1-r) 2^(-(2x/s)^2) + r / (1 + (2x/s)^2)] + b
template <int FAM, int PPL, int W>
__device__ __forceinline__ bool add_block(const GroupDesc& g, int b, const float* p, const Unit<PPL, W>& u,
                                          float (&acc)[PPL], float sign) {
  if (FAM == FAM_XRD) {
    if (b < g.K) {
      const float A = p[0], d2t = p[1], r = p[2], alpha = p[3], uu = p[4], vv = p[5], ww = p[6], ss = p[7],
                  tt = p[8];
      const int q1 = g.refl_off[b + 1];
      for (int q = g.refl_off[b]; q < q1; ++q) {
        const float2 rf = g.refl[q];
        const float c = rf.x + d2t;
        float sn, cs;
        sincosf(0.5f * c * 0.017453292519943295f, &sn, &cs);
        const float tn = sn / cs;
        const float disc = fmaf(fmaf(uu, tn, -vv), tn, ww);
        if (!(disc > 0.f)) return false;
        const float om0 = ss / cs + tt * tn;
        if (!(om0 > 0.f)) return false;
        const float ig_lo = 2.f / sqrtf(disc), ig_hi = ig_lo / alpha;
        const float il_lo = 2.f / om0, il_hi = il_lo / alpha;
        const float amp = sign * A * rf.y;
        const float ag = amp * (1.f - r), al = amp * r;
#pragma unroll
        for (int k = 0; k < PPL; ++k) {
          const float dx = u.x(k) - c;
          const bool pos = dx >= 0.f;
          const float tg = dx * (pos ? ig_hi : ig_lo);
          const float tl = dx * (pos ? il_hi : il_lo);
          acc[k] += fmaf(ag, ex2f(tg * -tg), al * rcpf(fmaf(tl, tl, 1.f)));
        }
      }
      return true;
    }
    if (!(p[1] > 0.f)) return false;
    const float is = 2.f / p[1];
    const float ag = sign * p[0] * (1.f - p[2]), al = sign * p[0] * p[2], off = sign * p[3];
#pragma unroll
    for (int k = 0; k < PPL; ++k) {
      const float t = u.x(k) * is;
      acc[k] += fmaf(ag, ex2f(t * -t), fmaf(al, rcpf(fmaf(t, t, 1.f)), off));
    }
    return true;
  } else {
    BlockC c = block_consts<FAM>(p);
    if (!c.ok) return false;
    c.c1 *= sign;                      // amplitudes: gm c1; xps c1, 1/c2 (gm c2 is the exponent)
    if (FAM == FAM_XPS) c.c2 *= sign;
#pragma unroll
    for (int k = 0; k < PPL; ++k) acc[k] += shape<FAM>(c, u.x(k));
    return true;
  }
}

// P_k = sum over non-faulty blocks of g_b(x_k), in layout order (combine,
// model.cpp:287-288).  Returns the bit mask of faulty blocks (eval_block
// returning false, model.cpp:272-275): any set bit means E = +inf.
template <int FAM, int PPL, int W>
__device__ __forceinline__ unsigned long long full_signal(const GroupDesc& g, const float* th,
                                                          const Unit<PPL, W>& u, float (&P)[PPL]) {
#pragma unroll
  for (int k = 0; k < PPL; ++k) P[k] = 0.f;
  const int nb = n_blocks<FAM>(g);
  unsigned long long fmask = 0ull;
  for (int b = 0; b < nb; ++b)
    if (!add_block<FAM, PPL, W>(g, b, th + block_off<FAM>(g, b), u, P, 1.f)) fmask |= 1ull << b;
  return fmask;
}

// Reduction of the lane partials over the unit, exact and order-independent:
// each lane's fp32 partial becomes a 2^-24 fixed-point int64 split into three
// 26-bit limbs, each summed with redux.sync (integer warp reduction, one
// instruction instead of five dependent shuffle rounds) and then across the
// unit's warps in int64.  Every warp obtains the identical value.  A
// non-finite partial (the fault sentinel) or one beyond 2^38 (a state whose
// likelihood underflows any weight) yields NaN, i.e. E = +inf.
template <int PPL, int W>
__device__ __forceinline__ double unit_sum(Unit<PPL, W>& u, float acc) {
  const bool bad = __any_sync(0xffffffffu, !(fabsf(acc) < 2.7e11f));
  const long long q = bad ? 0ll : __double2ll_rn((double)acc * 16777216.0);
  const unsigned a0 = (unsigned)(q & 0x3ffffff), a1 = (unsigned)((q >> 26) & 0x3ffffff);
  const int a2 = (int)(q >> 52);
  long long s0 = __reduce_add_sync(0xffffffffu, a0);
  long long s1 = __reduce_add_sync(0xffffffffu, a1);
  long long s2 = __reduce_add_sync(0xffffffffu, a2);
  bool any = bad;
  if (W > 1) {
    if (u.lane == 0) {
      u.xc->lim[u.par][u.wiu] = make_int4((int)s0, (int)s1, (int)s2, bad ? 1 : 0);
    }
    u.sync();
    s0 = s1 = s2 = 0;
    any = false;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const int4 v = u.xc->lim[u.par][w];
      s0 += (unsigned)v.x;
      s1 += (unsigned)v.y;
      s2 += v.z;
      any = any || v.w;
    }
  }
  u.par ^= 1;
  const long long tot = s0 + (s1 << 26) + (s2 << 52);
  return any ? nan("") : (double)tot * 5.9604644775390625e-08;
}

// per-point centred NLL term, in units of 1/2 ln 2 for the hetero model:
//   gauss:   r^2                                        E = a0 + a1 * sum
//   hetero:  lg2(var/s) + q' r^2/var, q' = q / (ln2/2)  E = a0 + a1 (ln2/2) sum
//            (hlin: the same with var linear in f)
//   poisson: f - y - y ln(f/y)                          E = a0 + a1 * sum
template <int NZ>
__device__ __forceinline__ float noise_term(const GroupDesc& g, float f, float2 yq) {
  const float r = yq.x - f;
  if (NZ == NZ_GAUSS) {
    return r * r;
  } else if (NZ == NZ_HETERO) {
    const float var = fmaf(fmaf(g.nz_a1, f, g.nz_a0), f, g.nz_a2);
    return fmaf(g.nz_q, (r * r) * rcpf(var), lg2f(var * yq.y));
  } else if (NZ == NZ_HLIN) {  // s1 = 0: var = s0^2 f + s2^2
    const float var = fmaf(g.nz_a0, f, g.nz_a2);
    return fmaf(g.nz_q, (r * r) * rcpf(var), lg2f(var * yq.y));
  } else if (NZ == NZ_HPROP) {  // s1 = s2 = 0: var = s0^2 f (GaussApprox-Poisson when s0 = 1);
                                // 1/s_k and q carry the s0^2 factor (host)
    return fmaf(g.nz_q, (r * r) * rcpf(f), lg2f(f * yq.y));
  } else {
    // y = 0 contributes f alone (no 0 * log f: a model value that underflowed in
    // fp32 must not turn the term into NaN); f < 0 stays the sentinel
    const float lt = yq.x > 0.f ? yq.x * (kLn2 * lg2f(f * yq.y)) : 0.f;
    return f < 0.f ? __int_as_float(0x7fc00000) : (f - yq.x) - lt;
  }
}

// Hetero terms of two points share one rcp and one lg2 (3 instead of 4 MUFU
// ops per point with the peak shape):
//   lg2(va/sa) + lg2(vb/sb) = lg2((va/sa)(vb/sb)),
//   ra^2/va + rb^2/vb = (ra^2 vb + rb^2 va) / (va vb).
// The var <= 0 sentinel survives: the lg2 argument takes the sign of min(va, vb)
// (NaN for a negative variance, energy.cpp:20), va vb = 0 gives inf.  Products
// leave the fp32 range only for states whose per-point fp32 terms already
// overflow (E >~ 1e19): those read as +inf as before.
template <int NZ>
__host__ __device__ constexpr bool nz_pairs() { return NZ == NZ_HETERO || NZ == NZ_HLIN || NZ == NZ_HPROP; }
template <int NZ>
__device__ __forceinline__ float nz_var(const GroupDesc& g, float f) {
  if (NZ == NZ_HETERO) return fmaf(fmaf(g.nz_a1, f, g.nz_a0), f, g.nz_a2);
  if (NZ == NZ_HLIN) return fmaf(g.nz_a0, f, g.nz_a2);
  return f;  // NZ_HPROP
}
// (ya, yb) = the pair's observations (host, paired layout).  The lane keeps
// three partials: quad += (ra^2 vb + rb^2 va) / (va vb), lg += lg2(va vb),
// mn = min over the variances; its noise sum is q' quad + lg, and NaN
// (E = +inf) unless every variance is > 0.  The lg2 terms are not centred
// (~25 each at C2 counts; the host moves the per-point scales into e_a0): a
// lane's fp32 sum of 16 of them carries ~1e-4 of rounding, ~1e-4 nats in N E.
struct PairAcc {
  float quad, lg, mn;
};
template <int NZ>
__device__ __forceinline__ void noise_pair(const GroupDesc& g, float fa, float fb, float2 yab, PairAcc& a) {
  const float ra = yab.x - fa, rb = yab.y - fb;
  const float va = nz_var<NZ>(g, fa), vb = nz_var<NZ>(g, fb);
  const float num = fmaf(ra * ra, vb, (rb * rb) * va);
  const float vv = va * vb;
  a.quad = fmaf(num, rcpf(vv), a.quad);
  a.lg += lg2f(vv);
  a.mn = fminf(a.mn, fminf(va, vb));  // one FMNMX3
}
template <int NZ>
__device__ __forceinline__ float pair_total(const GroupDesc& g, const PairAcc& a) {
  const float t = fmaf(g.nz_q, a.quad, a.lg);
  return a.mn > 0.f ? t : __int_as_float(0x7fc00000);
}
// f(k) -> sum of the noise terms of this lane's PPL points, and (CORR) the
// padding correction: padding points (k >= nv) replicate the lane's last point,
// so npad copies of its term are removed at once.  Without CORR the caller
// removes the padding terms (uniform xps layout, eval_shirley_nz).
template <int NZ, int PPL, int W, bool CORR = true, class F>
__device__ __forceinline__ float lane_noise_sum(const GroupDesc& g, const Unit<PPL, W>& u, F&& fk) {
  float acc = 0.f, tl = 0.f, fprev = 0.f, flast = 0.f;
  PairAcc pa{0.f, 0.f, FLT_MAX};
#pragma unroll
  for (int k = 0; k < PPL; ++k) {
    const float f = fk(k);
    if (nz_pairs<NZ>()) {
      if (k & 1)
        noise_pair<NZ>(g, fprev, f, u.y2(k >> 1), pa);
      else
        fprev = f;
      flast = f;
    } else {
      tl = noise_term<NZ>(g, f, u.y(k));
      acc += tl;
    }
  }
  if (nz_pairs<NZ>()) acc = pair_total<NZ>(g, pa);
  if (!CORR) return acc;
  if (!nz_pairs<NZ>()) return fmaf(-u.npad, tl, acc);
  if (u.npad > 0.f) acc = fmaf(-u.npad, noise_term<NZ>(g, flast, make_float2(g.y_last, g.s_last)), acc);
  return acc;
}

template <int NZ>
__device__ __forceinline__ double finish_energy(const GroupDesc& g, double s) {
  if (!isfinite(s)) return dinf();  // var <= 0 / f <= 0 sentinel (energy.cpp:16, :20, :25)
  return g.e_a0 + g.e_a1 * s;
}

template <int PPL, int W, int NZ>
__device__ __forceinline__ double eval_plain_nz(const GroupDesc& g, Unit<PPL, W>& u, const float (&Pn)[PPL]) {
  const float acc = lane_noise_sum<NZ>(g, u, [&](int k) { return Pn[k]; });
  return finish_energy<NZ>(g, unit_sum(u, acc));
}

// Shirley background + energy (lineshapes.hpp:65-83, model.cpp:289-292).
// amp_bound >= max_k |P_k| (sum of |amplitudes|) decides the degenerate-signal
// test without a max reduction unless it is inconclusive.
// scan of the lane values v over the unit: exclusive prefix and total (every
// lane of every warp gets the same total)
template <int PPL, int W>
__device__ __forceinline__ void unit_scan(Unit<PPL, W>& u, float v, float& prefix, float& total) {
  const float incl = warp_incl_scan_f(v, u.lane);
  prefix = incl - v;
  total = __shfl_sync(0xffffffffu, incl, 31);
  if (W > 1) {
    if (u.lane == 0) u.xc->scan[u.par][u.wiu] = total;
    u.sync();
    float pre = 0.f, tot = 0.f;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const float s = u.xc->scan[u.par][w];
      if (w < u.wiu) pre += s;
      tot += s;
    }
    prefix += pre;
    total = tot;
  }
}

// inconclusive degenerate-signal bound: exact max of Pn over the real points
// of the unit (rare)
template <int PPL, int W>
__device__ __forceinline__ float unit_max_real(Unit<PPL, W>& u, const float (&Pn)[PPL]) {
  float mx = -FLT_MAX;
#pragma unroll
  for (int k = 0; k < PPL; ++k)
    if (k < u.nv) mx = fmaxf(mx, Pn[k]);
  if (u.tail) mx = fmaxf(mx, Pn[PPL - 1]);
  mx = warp_max_f(mx);
  if (W > 1) {
    u.sync();  // everyone has consumed scan[par] above
    if (u.lane == 0) u.xc->scan[u.par][u.wiu] = mx;
    u.sync();
    for (int w = 0; w < W; ++w) mx = fmaxf(mx, u.xc->scan[u.par][w]);
    u.sync();
  }
  return mx;
}

// Shirley background on a uniform grid (GroupDesc::sh_uniform).  With spacing
// D the trapezoid integral is C_k = D (R_k - P_0/2 - P_k/2), R_k = sum_{j<=k} P_j,
// and D cancels in C/C_{N-1}: the scan sums Pn alone, with -P_0/2 seeded on
// lane 0 and -P_{N-1}/2 taken off the last lane's contribution (the layout
// keeps both endpoints at fixed slots; padding has Pn = 0, so it adds nothing
// and all padding points of a lane share one f).  Per point: one FADD in each
// pass and two FFMA for f, no weight loads.
template <int PPL, int W, int NZ>
__device__ __forceinline__ double eval_shirley_uniform(const GroupDesc& g, Unit<PPL, W>& u, const float (&Pn)[PPL],
                                                       float bga, float bgb, float amp_bound) {
  const float init = u.lg == 0 ? -0.5f * Pn[0] : 0.f;
  float run = init;
#pragma unroll
  for (int k = 0; k < PPL; ++k) run += Pn[k];
  const float v = u.tail ? fmaf(-0.5f, Pn[PPL - 1], run) : run;
  float prefix, total;
  unit_scan(u, v, prefix, total);
  const float ba = bgb - bga;
  const float rng = (float)(g.N - 1);  // range / D
  bool degen = !(total > 1e-12f * amp_bound * rng);
  if (degen) degen = !(total > 1e-12f * unit_max_real(u, Pn) * rng);
  float acc, fpad;
  if (!degen) {
    const float scale = ba * rcpf(total);
    const float m = fmaf(-0.5f, scale, 1.f);
    // f_k = Pn_k + a + scale (R_k - P_0/2 - Pn_k/2) = B_k + m Pn_k with the
    // running background B_k = a + scale (R_k - P_0/2): two FFMA per point
    float B = fmaf(scale, prefix + init, bga);
    acc = lane_noise_sum<NZ, PPL, W, false>(g, u, [&](int k) {
      B = fmaf(scale, Pn[k], B);
      return fmaf(m, Pn[k], B);
    });
    fpad = u.tail ? fmaf(-scale, Pn[PPL - 1], B) : B;
  } else {  // linear ramp a -> b (padding sits at x = 1e30: clamp to the last point)
    const float sl = ba * g.inv_range;
    acc = lane_noise_sum<NZ, PPL, W, false>(g, u, [&](int k) {
      return Pn[k] + fmaf(sl, fminf(u.x(k), g.x1s) - g.x0s, bga);
    });
    fpad = fmaf(sl, g.x1s - g.x0s, bga);
  }
  if (u.npad > 0.f) acc = fmaf(-u.npad, noise_term<NZ>(g, fpad, make_float2(g.y_last, g.s_last)), acc);
  return finish_energy<NZ>(g, unit_sum(u, acc));
}

template <int PPL, int W, int NZ>
__device__ __forceinline__ double eval_shirley_nz(const GroupDesc& g, Unit<PPL, W>& u, const float (&Pn)[PPL],
                                                  float bga, float bgb, float amp_bound) {
  if (g.sh_uniform) return eval_shirley_uniform<PPL, W, NZ>(g, u, Pn, bga, bgb, amp_bound);
  // pass 1: lane-local inclusive scan of c_k Pn_k; C_k is kept for PPL <= 16 and
  // recomputed in pass 2 for longer lanes (register budget)
  constexpr bool kKeepC = PPL <= 16;
  float Cn[kKeepC ? PPL : 1];
  float run = 0.f;
#pragma unroll
  for (int k = 0; k < PPL; ++k) {
    const float2 c = u.c(k);
    run = fmaf(c.x, Pn[k], run);
    if (kKeepC) Cn[k] = fmaf(-c.y, Pn[k], run);
  }
  float prefix, total;
  unit_scan(u, run, prefix, total);
  const float ba = bgb - bga;
  bool degen = !(total > 1e-12f * amp_bound * g.range);
  if (degen) degen = !(total > 1e-12f * unit_max_real(u, Pn) * g.range);  // inconclusive bound
  float acc;
  if (!degen) {
    const float scale = ba * rcpf(total);
    const float base = fmaf(scale, prefix, bga);
    float run2 = 0.f;
    acc = lane_noise_sum<NZ>(g, u, [&](int k) {
      float Ck;  // C_k = sum_{j<=k} c_j Pn_j - h_{k+1} Pn_k (lane-local part)
      if (kKeepC) {
        Ck = Cn[kKeepC ? k : 0];
      } else {
        const float2 c = u.c(k);
        run2 = fmaf(c.x, Pn[k], run2);
        Ck = fmaf(-c.y, Pn[k], run2);
      }
      return Pn[k] + fmaf(scale, Ck, base);
    });
  } else {  // linear ramp a -> b
    acc = lane_noise_sum<NZ>(g, u, [&](int k) { return Pn[k] + fmaf(ba, (u.x(k) - g.x0s) * g.inv_range, bga); });
  }
  // padding points (k >= nv, c = h = 0) replicate the lane's last point exactly
  return finish_energy<NZ>(g, unit_sum(u, acc));
}

// NZ is the device noise model, or NZ_DYN to switch on g.noise per evaluation
// (energy kernels and the offset test family: one instantiation for all noises)
template <int FAM, int PPL, int W, int NZ>
__device__ __forceinline__ double evaluate_nz(const GroupDesc& g, Unit<PPL, W>& u, const float (&Pn)[PPL], float bga,
                                              float bgb, float amp_bound) {
  if (NZ == NZ_DYN) {
    switch (g.noise) {
      case NZ_GAUSS: return evaluate_nz<FAM, PPL, W, NZ_GAUSS>(g, u, Pn, bga, bgb, amp_bound);
      case NZ_HETERO: return evaluate_nz<FAM, PPL, W, NZ_HETERO>(g, u, Pn, bga, bgb, amp_bound);
      case NZ_HLIN: return evaluate_nz<FAM, PPL, W, NZ_HLIN>(g, u, Pn, bga, bgb, amp_bound);
      case NZ_HPROP: return evaluate_nz<FAM, PPL, W, NZ_HPROP>(g, u, Pn, bga, bgb, amp_bound);
      default: return evaluate_nz<FAM, PPL, W, NZ_POISSON>(g, u, Pn, bga, bgb, amp_bound);
    }
  }
  constexpr int nz = NZ == NZ_DYN ? NZ_GAUSS : NZ;  // (the NZ_DYN branch above returned)
  if (FAM == FAM_XPS) return eval_shirley_nz<PPL, W, nz>(g, u, Pn, bga, bgb, amp_bound);
  return eval_plain_nz<PPL, W, nz>(g, u, Pn);
}

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

template <int FAM>
__device__ __forceinline__ float amp_sum(const GroupDesc& g, const float* thf) {
  if (FAM != FAM_XPS) return 0.f;
  float s = 0.f;
  for (int b = 0; b < g.K; ++b) s += fabsf(thf[4 * b]);
  return s;
}

// registers: PPL <= 8 -> 3 CTAs of 256 threads per SM (<= 85 regs), else 2 (<= 128)
template <int W, int PPL>
struct Bounds {
  static constexpr int threads = chain_threads(W);
  static constexpr int min_blocks = (65536 / threads) / (PPL <= 8 ? 85 : 128) > 0 ? (65536 / threads) / (PPL <= 8 ? 85 : 128) : 1;
  // (PPL = 32: 2 x 256 threads at <= 128 registers as well)
};

// The level's work for one chain unit (initial energy, then the move kernel's
// n sweeps), with the noise model NZ fixed at compile time for the move
// kernels: the sweep loop holds a single evaluation variant.
template <int FAM, int PPL, int W, bool ENERGY, int NZ>
__device__ __forceinline__ void chain_body(const GroupDesc& g, Unit<PPL, W>& u, const int c, const int unit,
                                           const int wiu, const int lane, const GroupState* st, const int cur,
                                           const int d, const int T, double* th, double* lsv, int* acc, double* nvb,
                                           double* dlpb, float* lub, int* flg, float* thf, float* nvf,
                                           float* gcache, float* pcache) {
  using SM = Smem<PPL, W>;
  constexpr int stride = block_stride<FAM>();
  const int ibg = 4 * g.K;  // xps Shirley endpoints (a, b) at ibg, ibg + 1
  float P[PPL];
  unsigned long long fmask = full_signal<FAM, PPL, W>(g, thf, u, P);
  float asum = amp_sum<FAM>(g, thf);
  double e = fmask ? dinf()
                   : evaluate_nz<FAM, PPL, W, NZ>(g, u, P, FAM == FAM_XPS ? thf[ibg] : 0.f,
                                           FAM == FAM_XPS ? thf[ibg + 1] : 0.f, asum);
  if (ENERGY) {
    if (wiu == 0 && lane == 0) g.E[cur][c] = e;
    return;
  }

  // ---- waste-free chain: n sweeps at beta_next, every post-sweep state kept
  const int n = g.n, S = g.S;
  const int level = st->level;
  const double beta = st->beta;
  const double nd = g.n_data;
  const int adapt_sweeps = (n + 1) / 2;  // smc.cpp:136
  const uint32_t cg = g.chain_base + (uint32_t)(st->chain_lo + c);  // global chain id
  double* thn = g.theta[cur ^ 1];
  double* En = g.E[cur ^ 1];
  // components inside a block (everything but the xps Shirley endpoints and the offset family)
  const int npeak = FAM == FAM_OFFSET ? 0 : (FAM == FAM_XRD ? g.d : stride * g.K);
  unsigned trials = 0;
  // Q[k] at Qs[k * L]: signal of every block except the one being swept (P - g_b)
  float* Qs = gcache + (size_t)unit * SM::NPT + u.lg;
  // committed peak signal: registers, or shared memory (Ps[k * L]) when p_in_smem<W>()
  constexpr bool kPsm = p_in_smem<W, PPL>();
  float* Ps = pcache + (size_t)unit * SM::NPT + u.lg;
  constexpr int L = SM::L;
  if (kPsm) {
#pragma unroll
    for (int k = 0; k < PPL; ++k) Ps[k * L] = P[k];
  }
#define SMC_P(k) (kPsm ? Ps[(k) * L] : P[k])

  const double bnd = beta * nd;
  const bool beta0 = beta == 0.0;
  for (int t = 1; t <= n; ++t) {
    u.sync();  // every warp of the unit is done with the previous sweep's shared arrays
    // ---- sweep prologue, lane-parallel over components.  Component i's value
    // and step only change at its own proposal, so the proposal, its prior
    // check (mcmc.cpp:61-68) and the Philox draws are all fixed at sweep start.
    for (int i = lane; i < d; i += 32) {
      // counter (t-1) d + i < n d <= 2^32 (make_runspec rejects larger n d): unsigned, no wrap
      const u32x4 o = philox(u32x4{cg, (uint32_t)level, (uint32_t)(t - 1) * (uint32_t)d + (uint32_t)i, ROLE_CHAIN},
                             g.key0, g.key1);
      const double old_i = th[i];
      const double nv = old_i + (double)__expf((float)lsv[i]) * (double)normal_f32(o.x, o.y);
      double dlp = 0.0;
      const bool ok = prior_delta(g.pkind[i], g.pa[i], g.pb[i], old_i, nv, dlp);
      nvb[i] = nv;
      nvf[i] = (float)nv;
      thf[i] = (float)old_i;
      dlpb[i] = dlp;
      lub[i] = __logf(u01_open_lo(o.z));
      flg[i] = ok ? 1 : 0;
      trials += ok ? 1 : 0;
    }
    __syncwarp();
    asum = amp_sum<FAM>(g, thf);
    for (int i = 0; i < d; ++i) {
      const BlockIdx<FAM> bi = block_of<FAM>(g, i);
      const int b = bi.b, j = bi.j;
      const bool peak = i < npeak;
      if (FAM != FAM_OFFSET && peak && j == 0) {  // entering block b: Q = P - g_b(x)
        float Qn[PPL];
#pragma unroll
        for (int k = 0; k < PPL; ++k) Qn[k] = SMC_P(k);
        if (!((fmask >> b) & 1ull)) add_block<FAM, PPL, W>(g, b, thf + bi.off, u, Qn, -1.f);
#pragma unroll
        for (int k = 0; k < PPL; ++k) Qs[k * L] = Qn[k];
      }
      if (!(flg[i] & 1)) continue;  // outside the prior support: no trial (mcmc.cpp:68)
      const float oldf = thf[i], newf = nvf[i];
      // ---- trial signal Pn = P + (g_new - G) (the reference's BlockEvaluator::trial, energy.cpp:57-84)
      float Pn[PPL];
      unsigned long long fnew = fmask;
      float dA = 0.f;
      // Shirley endpoint: enters combine() only (block -1), the peak signal is
      // unchanged and (registers) evaluated in place: no copy, no commit
      const bool endpoint = FAM == FAM_XPS && !peak;  // (gm, xrd: every component is in a block)
      if (FAM == FAM_OFFSET) {
        const float dv = newf - oldf;
#pragma unroll
        for (int k = 0; k < PPL; ++k) Pn[k] = SMC_P(k) + dv;
      } else if (endpoint) {
        if (kPsm) {
#pragma unroll
          for (int k = 0; k < PPL; ++k) Pn[k] = SMC_P(k);
        }
      } else if (j == 0 && oldf != 0.f && !((fmask >> b) & 1ull) &&
                 (FAM != FAM_XRD || b < g.K)) {  // amplitude: g' = (A'/A) g
        const float r = (newf - oldf) * rcpf(oldf);
#pragma unroll
        for (int k = 0; k < PPL; ++k) {
          const float pk = SMC_P(k);
          Pn[k] = fmaf(r, pk - Qs[k * L], pk);
        }
        dA = fabsf(newf) - fabsf(oldf);
      } else {
        constexpr int kMaxNp = FAM == FAM_XRD ? 9 : block_stride<FAM>();
        float pn[kMaxNp];
#pragma unroll
        for (int q = 0; q < kMaxNp; ++q) pn[q] = (q == j) ? newf : (q < bi.np ? thf[bi.off + q] : 0.f);
#pragma unroll
        for (int k = 0; k < PPL; ++k) Pn[k] = Qs[k * L];
        if (add_block<FAM, PPL, W>(g, b, pn, u, Pn, 1.f))
          fnew &= ~(1ull << b);
        else
          fnew |= 1ull << b;
        if (j == 0) dA = fabsf(newf) - fabsf(oldf);
      }
      float bga = 0.f, bgb = 0.f;
      if (FAM == FAM_XPS) {
        bga = i == ibg ? newf : thf[ibg];
        bgb = i == ibg + 1 ? newf : thf[ibg + 1];
      }
      double e_new;
      if (fnew)
        e_new = dinf();
      else if (!kPsm && endpoint)
        e_new = evaluate_nz<FAM, PPL, W, NZ>(g, u, P, bga, bgb, asum);
      else
        e_new = evaluate_nz<FAM, PPL, W, NZ>(g, u, Pn, bga, bgb, asum + dA);
      // mcmc.cpp:72-80
      const double dlp = dlpb[i];
      double lr;
      if (e_new < dinf() && e < dinf() && !beta0) {
        lr = fma(-bnd, e_new - e, dlp);
      } else {
        const bool inf_new = e_new == dinf(), inf_old = e == dinf();
        if (beta0 || (inf_new && inf_old))
          lr = dlp;
        else if (inf_new)
          lr = -dinf();
        else
          lr = dinf();
      }
      const bool accept = lr >= 0.0 || (double)lub[i] < lr;
      // commit: Q (other blocks) is unchanged; P updated in place (select) or in shared memory
      if (!kPsm && !endpoint) {
#pragma unroll
        for (int k = 0; k < PPL; ++k) P[k] = accept ? Pn[k] : P[k];
      }
      if (accept) {
        if (kPsm && !endpoint) {
#pragma unroll
          for (int k = 0; k < PPL; ++k) Ps[k * L] = Pn[k];
        }
        fmask = fnew;
        asum += dA;
        e = e_new;
        if (lane == 0) {
          th[i] = nvb[i];
          thf[i] = newf;
          flg[i] = 3;
        }
        __syncwarp();
      }
    }
    __syncwarp();
    // ---- sweep epilogue: tallies and Robbins-Monro in log space (mcmc.cpp:14-18, :89-93);
    // step i is only read by component i's next proposal, so the update can wait until here.
    // These are read-modify-writes of the unit's shared state: warp 0 alone does them
    // (the other warps read lsv after the unit barrier that opens the next sweep).
    if (wiu == 0) {
      const float gam = (t <= adapt_sweeps) ? exp2f(-0.6f * log2f((float)t)) : 0.f;  // t^-0.6
      for (int i = lane; i < d; i += 32) {
        const int a = flg[i] >> 1;
        acc[i] += a;
        if (t <= adapt_sweeps) {
          const double ls = lsv[i] + (double)gam * ((double)a - 0.5);
          lsv[i] = fmin(fmax(ls, kLogStepMin), kLogStepMax);
        }
      }
    }
    __syncwarp();
    const size_t slot = (size_t)c * n + (t - 1);  // smc.cpp:151
    if (wiu == 0) {
      for (int i = lane; i < d; i += 32) thn[(size_t)i * g.tp + slot] = th[i];
      if (lane == 0) En[slot] = e;
    }
  }
  if (wiu == 0) {
    for (int i = lane; i < d; i += 32) {
      g.chain_acc[(size_t)i * g.sp + c] = acc[i];
      g.chain_ls[(size_t)i * g.sp + c] = lsv[i];
    }
  }
#undef SMC_P
  trials = __reduce_add_sync(0xffffffffu, trials);
  if (wiu == 0 && lane == 0) atomicAdd(&g.st->trials, (unsigned long long)trials);
}

template <int FAM, int PPL, int W, bool ENERGY, int NZ>
__global__ void __launch_bounds__(Bounds<W, PPL>::threads, Bounds<W, PPL>::min_blocks)
    k_chain(const GroupDesc* __restrict__ gds, const int* __restrict__ list, const int* __restrict__ cta_prefix,
            int n_list, int U, int dpad) {
  using SM = Smem<PPL, W>;
  // W >= 4: the launch's spectrum layout rides in the high half of dpad
  // (W <= 2 kernels keep their parameter list and compile-time layout)
  int lay = kLayFull;
  if (chain_dyn_layout(W)) {
    lay = dpad >> 16;
    dpad &= 0xffff;
  }
  extern __shared__ __align__(16) unsigned char smem[];
  const int gi = find_group(cta_prefix, n_list, blockIdx.x);
  const GroupDesc& g = gds[list[gi]];
  const int cta_in_group = blockIdx.x - cta_prefix[gi];

  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  float* sx = reinterpret_cast<float*>(smem + SM::off_x);
  float2* sc = reinterpret_cast<float2*>(smem + SM::off_c);
  float2* sy = reinterpret_cast<float2*>(smem + SM::off_y(lay));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int unit = warp / W, wiu = warp - unit * W;
  unsigned char* wb = smem + SM::off_w(lay) + (size_t)unit * SM::per_unit(dpad);
  double* th = reinterpret_cast<double*>(wb);
  double* lsv = th + dpad;
  int* acc = reinterpret_cast<int*>(lsv + dpad);
  double* nvb = reinterpret_cast<double*>(acc + dpad);  // dpad is even: 8-byte aligned
  double* dlpb = nvb + dpad;
  float* lub = reinterpret_cast<float*>(dlpb + dpad);
  int* flg = reinterpret_cast<int*>(lub + dpad);
  float* thf = reinterpret_cast<float*>(flg + dpad);  // fp32 shadow of th (block constants)
  float* nvf = thf + dpad;                            // fp32 shadow of the proposals
  const size_t xoff = ((SM::off_w(lay) + (size_t)U * SM::per_unit(dpad)) + 15) & ~(size_t)15;
  Xch* xcs = reinterpret_cast<Xch*>(smem + xoff);
  float* gcache = reinterpret_cast<float*>(smem + xoff + (size_t)U * sizeof(Xch));
  float* pcache = gcache + (size_t)U * SM::NPT;

  // ---- stage the spectrum: cp.async.bulk (UBLKCP) completing on an mbarrier
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    const uint32_t bx = SM::NPT * 4u, bc = SM::NPT * 8u, by = SM::NPT * (uint32_t)SM::y_bytes(lay);
    // trapezoid weights: non-uniform grids only (the launch layout stages them then)
    const bool wc = FAM == FAM_XPS && !g.sh_uniform && (SM::layout(lay) & kLayWeights);
    mbar_expect_tx(bar, bx + (wc ? bc : 0u) + by);
    bulk_g2s(sx, g.spec_x, bx, bar);
    if (wc) bulk_g2s(sc, g.spec_c, bc, bar);
    bulk_g2s(sy, g.spec_y, by, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);

  const int c = cta_in_group * U + unit;
  const int units = ENERGY ? g.st->T_loc : g.st->S_loc;  // == T, S unless the run is particle-sharded
  if (c >= units) return;  // the whole unit leaves; no CTA-wide barrier follows

  Unit<PPL, W> u;
  u.sx = sx;
  u.sc = sc;
  u.sy = sy;
  u.xc = xcs + unit;
  u.lg = wiu * 32 + lane;
  u.wiu = wiu;
  u.lane = lane;
  u.bar_id = 1 + unit;
  u.par = 0;
  if (FAM == FAM_XPS && g.sh_uniform) {  // points 0..N-2 lead, point N-1 in the last slot
    u.nv = min(max(g.N - 1 - u.lg * PPL, 0), PPL);
    u.tail = u.lg == Unit<PPL, W>::L - 1;
    u.npad = (float)(PPL - u.nv - (u.tail ? 1 : 0));
  } else {
    u.nv = min(max(g.N - u.lg * PPL, 0), PPL);
    u.tail = false;
    u.npad = (float)(PPL - u.nv);
  }

  const GroupState* st = g.st;
  const int cur = st->cur;
  const int d = g.d, T = g.T;
  const double* thc = g.theta[cur];
  const int src = ENERGY ? c : g.anc[c];
  for (int i = lane; i < d; i += 32) {
    th[i] = thc[(size_t)i * g.tp + src];
    thf[i] = (float)th[i];
    if (!ENERGY) {
      lsv[i] = g.ls0[i];
      acc[i] = 0;
    }
  }
  __syncwarp();

  chain_body<FAM, PPL, W, ENERGY, NZ>(g, u, c, unit, wiu, lane, st, cur, d, T, th, lsv, acc, nvb, dlpb, lub, flg, thf,
                                      nvf, gcache, pcache);
}

// ------------------------------------------------------------------ launch
template <int FAM, int PPL, int W, bool ENERGY, int NZ>
cudaError_t launch_chain_t(int U, int lay, int dmax, const GroupDesc* gds, const int* list, const int* prefix,
                           int n_list, int total_ctas, cudaStream_t st) {
  const int dpad = (dmax + 1) & ~1;
  const size_t smem = Smem<PPL, W>::bytes(U, dpad, lay);
  auto kern = k_chain<FAM, PPL, W, ENERGY, NZ>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  if (total_ctas <= 0) return cudaSuccess;  // prime only (module load + attributes, see prime_level_kernels)
  const int dpad_lay = chain_dyn_layout(W) ? (dpad | (lay << 16)) : dpad;
  kern<<<total_ctas, Bounds<W, PPL>::threads, smem, st>>>(gds, list, prefix, n_list, U, dpad_lay);
  return cudaGetLastError();
}

// (W, PPL) pairs compiled (see pick_shape in kernels.cu): W = 1 for N <= 512,
// W = 2 for N <= 2048, W = 4 for N <= 4096, W = 8 for N <= 8192
#define SMC_FOR_EACH_SHAPE(X)                                                                          \
  X(1, 2) X(1, 4) X(1, 6) X(1, 8) X(1, 10) X(1, 12) X(1, 14) X(1, 16) X(1, 20) X(1, 24) X(1, 28) X(1, 32) \
  X(2, 10) X(2, 12) X(2, 14) X(2, 16) X(2, 20) X(2, 24) X(2, 28) X(2, 32)                             \
  X(4, 20) X(4, 24) X(4, 28) X(4, 32) X(8, 20) X(8, 24) X(8, 28) X(8, 32)

template <int FAM, bool ENERGY, int NZ>
cudaError_t launch_chain_fam(const Shape& s, int dmax, const GroupDesc* gds, const int* list, const int* prefix,
                             int n_list, int total_ctas, cudaStream_t st) {
#define SMC_CASE(WW, PP) \
  if (s.W == WW && s.PPL == PP) return launch_chain_t<FAM, PP, WW, ENERGY, NZ>(s.U, s.lay, dmax, gds, list, prefix, n_list, total_ctas, st);
  SMC_FOR_EACH_SHAPE(SMC_CASE)
#undef SMC_CASE
  return cudaErrorInvalidValue;
}

}  // namespace smc
