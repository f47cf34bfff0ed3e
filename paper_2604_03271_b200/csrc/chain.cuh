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
// consecutive points [l*PPL, (l+1)*PPL) of the spectrum.
//
// Packed fp32 pairs.  The lane's points are held as PH = PPL/2 float2 "pair
// slots": slot k pairs the lane's point k (.x, first half) with its point
// k + PH (.y, second half).  Every per-point step of an evaluation is then one
// sm_100 packed instruction (FFMA2 / FADD2 / FMUL2) for two independent points:
// the two halves run as separate running sums through the Shirley scans and
// are joined once per lane, and the paired noise terms combine slot k with
// slot k+1 component-wise (two points of the first half and two of the second
// half per packed instruction).  Only the MUFU ops (ex2, rcp, lg2) stay scalar.
//
//   P[k]  committed peak signal  sum_b g_b(x)      (combine, model.cpp:287-288)
//   Q[k]  P minus g_b(x) of the block being swept (shared memory)
// A proposal changes one block: the trial signal is Pn = Q + g_new, and an
// amplitude proposal needs no transcendental at all (Pn = P + (A'/A - 1)(P - Q)).
// The Shirley background (lineshapes.hpp:65-83) needs the cumulative
// trapezoid of Pn: C_k = sum_{j<=k} c_j Pn_j - h_{k+1} Pn_k with
// c_j = h_j + h_{j+1}, h_j = (x_j - x_{j-1})/2, i.e. a lane-local scan and one
// warp (and cross-warp) scan per proposal.  Energy terms are summed per lane in
// fp32 and across lanes exactly (fixed point).  Padding points replicate the
// last real point with weight 0, so no per-point masks are needed; a
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

// ---- packed fp32 pair helpers (sm_100a FFMA2 / FADD2 / FMUL2) -------------
using f2 = float2;
__device__ __forceinline__ f2 F2(float a) { return make_float2(a, a); }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ f2 add2(f2 a, f2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ f2 mul2(f2 a, f2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ f2 neg2(f2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ f2 ex2f2(f2 a) { return make_float2(ex2f(a.x), ex2f(a.y)); }
__device__ __forceinline__ f2 rcpf2(f2 a) { return make_float2(rcpf(a.x), rcpf(a.y)); }
__device__ __forceinline__ f2 lg2f2(f2 a) { return make_float2(lg2f(a.x), lg2f(a.y)); }
__device__ __forceinline__ float comp(f2 a, int h) { return h ? a.y : a.x; }

// xps with the Lorentzian basis pinned (every eta prior Uniform(0, <= 1e-7):
// the config override prior.eta = uniform(0, 1e-9) of SURVEY.md Appendix A,
// config.cpp:204-222): the move kernel drops the Gaussian term, whose weight
// A eta <= 1e-7 A lies below the fp32 rounding of the signal (device-only
// family code; the energy kernel and every other path treat it as xps)
constexpr int FAM_XPSL = 4;
template <int FAM>
__host__ __device__ constexpr bool is_xps() { return FAM == FAM_XPS || FAM == FAM_XPSL; }

struct BlockC {
  float mu, c1, c2, c3;
  bool ok;
};

template <int FAM>
__device__ __forceinline__ constexpr int block_stride() {
  return FAM == FAM_GM ? 3 : (is_xps<FAM>() ? 4 : (FAM == FAM_XRD ? 9 : 1));
}

// Block constants from the fp32 shadow p of the block's parameters:
// gm:  g = A exp(-b/2 (x-mu)^2) = c1 2^(c2 d^2), d = x - mu             (model.cpp:216-220)
// xps: g = c1 2^(-u) + 1 / (c2 (1 + u)), u = t^2, t = x/sigma - mu/sigma,
//      c1 = A eta, c2 = 1 / (A (1-eta)) (the Lorentzian amplitude folded into its
//      reciprocal; a zero Lorentzian amplitude becomes c2 = 1e30, i.e. a
//      contribution <= 1e-30)
//      (= A [eta exp(-ln2 d^2/s^2) + (1-eta) s^2/(s^2+d^2)], model.cpp:269-280)
// offset: g = theta_0                              (conjugate_oracle.hpp:22-26)
template <int FAM>
__device__ __forceinline__ BlockC block_consts(const float* p) {
  BlockC c;
  c.ok = true;
  c.c3 = 0.f;
  if (FAM == FAM_GM) {
    c.c1 = p[0];
    c.mu = p[1];
    c.c2 = p[2] * -0.72134752044448170f;  // -b/2 * log2(e)
  } else if (is_xps<FAM>()) {
    const float A = p[0], sig = p[2], eta = p[3];
    c.ok = sig > 0.f;
    c.c3 = rcpf(sig);
    c.mu = -p[1] * c.c3;
    c.c1 = A * eta;
    const float aL = FAM == FAM_XPSL ? A : A - c.c1;
    c.c2 = aL != 0.f ? rcpf(aL) : 1e30f;
  } else {
    c.c1 = p[0];
    c.mu = 0.f;
    c.c2 = 0.f;
  }
  return c;
}

// acc + g(x) for one pair slot (two points)
template <int FAM>
__device__ __forceinline__ f2 shape_add2(const BlockC& b, f2 x, f2 acc) {
  if (FAM == FAM_GM) {
    const f2 dx = add2(x, F2(-b.mu));  // exact near the centre (the d^2 c2 form keeps full relative precision)
    return fma2(F2(b.c1), ex2f2(mul2(F2(b.c2), mul2(dx, dx))), acc);
  } else if (is_xps<FAM>()) {
    const f2 t = fma2(x, F2(b.c3), F2(b.mu));
    if (FAM == FAM_XPSL) return add2(acc, rcpf2(fma2(mul2(t, t), F2(b.c2), F2(b.c2))));
    // -u = t (-t), -t from its own FFMA2 over negated broadcast constants (free
    // operand modifiers; ptxas negates a packed register with two scalar FADDs)
    // -- bit-identical to -(t t): round-to-nearest is symmetric
    const f2 nu = mul2(t, fma2(x, F2(-b.c3), F2(-b.mu)));
    const f2 r = rcpf2(fma2(nu, F2(-b.c2), F2(b.c2)));
    return add2(fma2(F2(b.c1), ex2f2(nu), acc), r);
  } else {
    return add2(acc, F2(b.c1));
  }
}

struct Xch {  // per-unit cross-warp exchange, double-buffered by parity
  float scan[2][16];
  int4 lim[2][16];  // energy partial sums: three fixed-point limbs + fault flag
};

// Per-CTA shared memory (dynamic):
//   [0,16)     mbarrier of the spectrum bulk copy
//   sx  float2 [PH][L]   shifted abscissa of the pair slots (4 B per point)
//   sc  float4 [PH][L]   (c_a, c_b, h_a, h_b): trapezoid weights of the two points
//                        of a slot (non-uniform xps grids only, launch layout)
//   sy  float2 [PH][L]   (-y_a, -y_b) (kLayY4: gauss and the paired hetero models), or
//       float4 [PH][L]   (y_a, y_b, 1/s_a, 1/s_b) (poisson)
//   per unit: th f64, ls f64, acc i32, proposal f64, dlp f64, log u f32, flags i32,
//             fp32 shadows of th and of the proposal  (x dpad); every warp of the
//             unit computes and writes identical values (idempotent), one unit
//             barrier per sweep orders the sweep-level rewrites
//   per unit: Xch, then Q float2 [PH][L] (signal of every block but the swept one)
// committed peak signal P: shared memory for W = 2 and 4 (one trial signal in
// registers leaves the allocator room), registers for W = 1 and 8; see
// chain_p_in_smem (launch.h)
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
  static constexpr int PH = PPL / 2;
  const f2* sx;
  const float4* sc;
  const void* sy;
  int nv;      // leading real (non-padding) points of this lane
  float npad;  // padding points of this lane
  bool tail;   // uniform xps layout: this lane's last point holds the last real point
  Xch* xc;
  int lg, wiu, lane, bar_id;
  int par;
  __device__ __forceinline__ f2 x2(int k) const { return sx[k * L + lg]; }
  __device__ __forceinline__ float4 c4(int k) const { return sc[k * L + lg]; }
  __device__ __forceinline__ f2 y2(int k) const { return static_cast<const f2*>(sy)[k * L + lg]; }
  __device__ __forceinline__ float4 y4(int k) const { return static_cast<const float4*>(sy)[k * L + lg]; }
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

// acc += sign * g_b(x) for block b with (fp32) parameters p.  Returns false
// on an evaluation fault (model.cpp:226-258, :272-275): the block then adds nothing.
//   xrd phase b (model.cpp:235-267): sum over its reflections of
//     A ri [(1-r) 2^(-(2 dx/wg)^2) + r / (1 + (2 dx/wl)^2)],  c = mu_ref + d2t,
//     wg = sqrt(u tan^2 - v tan + w), wl = s / cos + t tan (theta = c/2), both x alpha for dx >= 0
//   xrd background (model.cpp:223-234): a [(1-r) 2^(-(2x/s)^2) + r / (1 + (2x/s)^2)] + b
template <int FAM, int PPL, int W>
__device__ __forceinline__ bool add_block(const GroupDesc& g, int b, const float* p, const Unit<PPL, W>& u,
                                          f2 (&acc)[PPL / 2], float sign) {
  constexpr int PH = PPL / 2;
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
        for (int k = 0; k < PH; ++k) {
          const f2 dx = add2(u.x2(k), F2(-c));
          const f2 tg = make_float2(dx.x * (dx.x >= 0.f ? ig_hi : ig_lo), dx.y * (dx.y >= 0.f ? ig_hi : ig_lo));
          const f2 tl = make_float2(dx.x * (dx.x >= 0.f ? il_hi : il_lo), dx.y * (dx.y >= 0.f ? il_hi : il_lo));
          const f2 lz = rcpf2(fma2(tl, tl, F2(1.f)));
          acc[k] = add2(acc[k], fma2(F2(ag), ex2f2(mul2(tg, neg2(tg))), mul2(F2(al), lz)));
        }
      }
      return true;
    }
    if (!(p[1] > 0.f)) return false;
    const float is = 2.f / p[1];
    const float ag = sign * p[0] * (1.f - p[2]), al = sign * p[0] * p[2], off = sign * p[3];
#pragma unroll
    for (int k = 0; k < PH; ++k) {
      const f2 t = mul2(u.x2(k), F2(is));
      const f2 tt2 = mul2(t, t);
      const f2 lz = rcpf2(add2(tt2, F2(1.f)));
      acc[k] = add2(acc[k], fma2(F2(ag), ex2f2(neg2(tt2)), fma2(F2(al), lz, F2(off))));
    }
    return true;
  } else {
    BlockC c = block_consts<FAM>(p);
    if (!c.ok) return false;
    c.c1 *= sign;                      // amplitudes: gm c1; xps c1, 1/c2
    if (is_xps<FAM>()) c.c2 *= sign;
#pragma unroll
    for (int k = 0; k < PH; ++k) acc[k] = shape_add2<FAM>(c, u.x2(k), acc[k]);
    return true;
  }
}

// P_k = sum over non-faulty blocks of g_b(x_k), in layout order (combine,
// model.cpp:287-288).  Returns the bit mask of faulty blocks (eval_block
// returning false, model.cpp:272-275): any set bit means E = +inf.
template <int FAM, int PPL, int W>
__device__ __forceinline__ unsigned long long full_signal(const GroupDesc& g, const float* th,
                                                          const Unit<PPL, W>& u, f2 (&P)[PPL / 2]) {
#pragma unroll
  for (int k = 0; k < PPL / 2; ++k) P[k] = F2(0.f);
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
// (scalar form: the padding correction and the poisson terms; yq = (y, 1/s))
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
// The partners are slots k and k+1 of the same half (component-wise), so one
// packed step combines two point pairs.  The var <= 0 sentinel survives: the
// lane keeps min over the variances (NaN => E = +inf unless every variance is
// > 0, energy.cpp:20), va vb = 0 gives inf.  Products leave the fp32 range only
// for states whose per-point fp32 terms already overflow (E >~ 1e19): those
// read as +inf as before.  The lg2 terms are not centred (~25 each at C2
// counts; the host moves the per-point scales into e_a0): a lane's fp32 sum of
// 16 of them carries ~1e-4 of rounding, ~1e-4 nats in N E.
template <int NZ>
__host__ __device__ constexpr bool nz_pairs() { return NZ == NZ_HETERO || NZ == NZ_HLIN || NZ == NZ_HPROP; }
template <int NZ>
__device__ __forceinline__ f2 nz_var2(const GroupDesc& g, f2 f) {
  if (NZ == NZ_HETERO) return fma2(fma2(F2(g.nz_a1), f, F2(g.nz_a0)), f, F2(g.nz_a2));
  if (NZ == NZ_HLIN) return fma2(F2(g.nz_a0), f, F2(g.nz_a2));
  return f;  // NZ_HPROP
}
template <int NZ>
__device__ __forceinline__ float nz_var(const GroupDesc& g, float f) {
  if (NZ == NZ_HETERO) return fmaf(fmaf(g.nz_a1, f, g.nz_a0), f, g.nz_a2);
  if (NZ == NZ_HLIN) return fmaf(g.nz_a0, f, g.nz_a2);
  return f;  // NZ_HPROP
}
// lane partials of the noise sum: packed quadratic parts and lg2 parts (one
// lane per half), min over the variances (paired models); the packed term sums
// in quad (other models)
struct NoiseAcc {
  f2 quad, lg;
  float mn;
};
template <int NZ>
__device__ __forceinline__ void noise_quad(const GroupDesc& g, f2 fa, f2 fb, f2 ya, f2 yb, NoiseAcc& a) {
  const f2 ra = add2(fa, ya), rb = add2(fb, yb);  // (f - y): the layout stores -y (only r^2 enters)
  const f2 va = nz_var2<NZ>(g, fa), vb = nz_var2<NZ>(g, fb);
  const f2 num = fma2(mul2(ra, ra), vb, mul2(mul2(rb, rb), va));
  const f2 vv = mul2(va, vb);
  a.quad = fma2(num, rcpf2(vv), a.quad);
  a.lg = add2(a.lg, lg2f2(vv));
  a.mn = fminf(a.mn, fminf(fminf(va.x, va.y), fminf(vb.x, vb.y)));  // two FMNMX3
}
// the odd last slot of a lane with PH odd: its two points pair with each other
template <int NZ>
__device__ __forceinline__ void noise_pair_h(const GroupDesc& g, f2 f, f2 y, NoiseAcc& a) {
  const float ra = f.x + y.x, rb = f.y + y.y;  // f - y (the layout stores -y)
  const float va = nz_var<NZ>(g, f.x), vb = nz_var<NZ>(g, f.y);
  const float num = fmaf(ra * ra, vb, (rb * rb) * va);
  const float vv = va * vb;
  a.quad.x = fmaf(num, rcpf(vv), a.quad.x);
  a.lg.x += lg2f(vv);
  a.mn = fminf(a.mn, fminf(va, vb));
}
// f(k) -> f2 for pair slot k, called in slot order: the sum of the noise terms
// of the lane's PPL points, and (CORR) the padding correction: padding points
// (the lane's points >= nv) replicate the spectrum's last point, so npad copies
// of the term at the lane's last point are removed at once.  Without CORR the
// caller removes the padding terms (uniform xps layout, eval_shirley_uniform).
template <int NZ, int PPL, int W, bool CORR = true, class F>
__device__ __forceinline__ float lane_noise_sum(const GroupDesc& g, const Unit<PPL, W>& u, F&& fk) {
  constexpr int PH = PPL / 2;
  NoiseAcc a{F2(0.f), F2(0.f), FLT_MAX};
  float flast = 0.f;
  if (nz_pairs<NZ>()) {
#pragma unroll
    for (int k = 0; k + 1 < PH; k += 2) {
      const f2 fa = fk(k), fb = fk(k + 1);
      noise_quad<NZ>(g, fa, fb, u.y2(k), u.y2(k + 1), a);
      flast = fb.y;
    }
    if (PH & 1) {
      const f2 f = fk(PH - 1);
      noise_pair_h<NZ>(g, f, u.y2(PH - 1), a);
      flast = f.y;
    }
  } else if (NZ == NZ_GAUSS) {
#pragma unroll
    for (int k = 0; k < PH; ++k) {
      const f2 f = fk(k);
      const f2 r = add2(f, u.y2(k));  // f - y (the layout stores -y)
      a.quad = fma2(r, r, a.quad);
      flast = f.y;
    }
  } else {  // poisson: scalar terms (lg2 of the model value under y > 0 guards)
#pragma unroll
    for (int k = 0; k < PH; ++k) {
      const f2 f = fk(k);
      const float4 y = u.y4(k);  // (y_a, y_b, 1/s_a, 1/s_b)
      a.quad.x += noise_term<NZ>(g, f.x, make_float2(y.x, y.z));
      a.quad.y += noise_term<NZ>(g, f.y, make_float2(y.y, y.w));
      flast = f.y;
    }
  }
  float acc;
  if (nz_pairs<NZ>()) {
    const float t = fmaf(g.nz_q, a.quad.x + a.quad.y, a.lg.x + a.lg.y);
    acc = a.mn > 0.f ? t : __int_as_float(0x7fc00000);
  } else {
    acc = a.quad.x + a.quad.y;
  }
  if (!CORR) return acc;
  if (u.npad > 0.f) acc = fmaf(-u.npad, noise_term<NZ>(g, flast, make_float2(g.y_last, g.s_last)), acc);
  return acc;
}

template <int NZ>
__device__ __forceinline__ double finish_energy(const GroupDesc& g, double s) {
  if (!isfinite(s)) return dinf();  // var <= 0 / f <= 0 sentinel (energy.cpp:16, :20, :25)
  return g.e_a0 + g.e_a1 * s;
}

template <int PPL, int W, int NZ>
__device__ __forceinline__ double eval_plain_nz(const GroupDesc& g, Unit<PPL, W>& u, const f2 (&Pn)[PPL / 2]) {
  const float acc = lane_noise_sum<NZ>(g, u, [&](int k) { return Pn[k]; });
  return finish_energy<NZ>(g, unit_sum(u, acc));
}

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
__device__ __forceinline__ float unit_max_real(Unit<PPL, W>& u, const f2 (&Pn)[PPL / 2]) {
  constexpr int PH = PPL / 2;
  float mx = -FLT_MAX;
#pragma unroll
  for (int k = 0; k < PH; ++k) {
    if (k < u.nv) mx = fmaxf(mx, Pn[k].x);
    if (k + PH < u.nv) mx = fmaxf(mx, Pn[k].y);
  }
  if (u.tail) mx = fmaxf(mx, Pn[PH - 1].y);
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
// and all padding points of a lane share one f).  Per pair slot: one FADD2 in
// the first pass and two FFMA2 for f, no weight loads; the lane's two halves
// run their own sums, the second starting where the first ends.
template <int PPL, int W, int NZ>
__device__ __forceinline__ double eval_shirley_uniform(const GroupDesc& g, Unit<PPL, W>& u, const f2 (&Pn)[PPL / 2],
                                                       float bga, float bgb, float amp_bound) {
  constexpr int PH = PPL / 2;
  const float init = u.lg == 0 ? -0.5f * Pn[0].x : 0.f;
  f2 run = make_float2(init, 0.f);
#pragma unroll
  for (int k = 0; k < PH; ++k) run = add2(run, Pn[k]);
  const float lane_sum = run.x + run.y;
  const float v = u.tail ? fmaf(-0.5f, Pn[PH - 1].y, lane_sum) : lane_sum;
  float prefix, total;
  unit_scan(u, v, prefix, total);
  const float ba = bgb - bga;
  const float rng = (float)(g.N - 1);  // range / D
  bool degen = !(total > 1e-12f * amp_bound * rng);
  if (degen) degen = !(total > 1e-12f * unit_max_real(u, Pn) * rng);
  float acc, fpad;
  if (!degen) {
    const float scale = ba * rcpf(total);
    const f2 m = F2(fmaf(-0.5f, scale, 1.f));
    // f_k = Pn_k + a + scale (R_k - P_0/2 - Pn_k/2) = B_k + m Pn_k with the
    // running background B_k = a + scale (R_k - P_0/2): two FFMA2 per slot
    f2 B = make_float2(fmaf(scale, prefix + init, bga), fmaf(scale, prefix + run.x, bga));
    const f2 S = F2(scale);
    acc = lane_noise_sum<NZ, PPL, W, false>(g, u, [&](int k) {
      B = fma2(S, Pn[k], B);
      return fma2(m, Pn[k], B);
    });
    fpad = u.tail ? fmaf(-scale, Pn[PH - 1].y, B.y) : B.y;
  } else {  // linear ramp a -> b (padding sits at x = 1e30: clamp to the last point)
    const float sl = ba * g.inv_range;
    acc = lane_noise_sum<NZ, PPL, W, false>(g, u, [&](int k) {
      const f2 x = u.x2(k);
      const f2 xc = make_float2(fminf(x.x, g.x1s), fminf(x.y, g.x1s));
      return add2(Pn[k], fma2(F2(sl), add2(xc, F2(-g.x0s)), F2(bga)));
    });
    fpad = fmaf(sl, g.x1s - g.x0s, bga);
  }
  if (u.npad > 0.f) acc = fmaf(-u.npad, noise_term<NZ>(g, fpad, make_float2(g.y_last, g.s_last)), acc);
  return finish_energy<NZ>(g, unit_sum(u, acc));
}

// Shirley background + energy (lineshapes.hpp:65-83, model.cpp:289-292) on a
// general grid.  amp_bound >= max_k |P_k| (sum of |amplitudes|) decides the
// degenerate-signal test without a max reduction unless it is inconclusive.
template <int PPL, int W, int NZ>
__device__ __forceinline__ double eval_shirley_nz(const GroupDesc& g, Unit<PPL, W>& u, const f2 (&Pn)[PPL / 2],
                                                  float bga, float bgb, float amp_bound) {
  if (g.sh_uniform) return eval_shirley_uniform<PPL, W, NZ>(g, u, Pn, bga, bgb, amp_bound);
  constexpr int PH = PPL / 2;
  // pass 1: lane-local inclusive scan of c_k Pn_k per half; C_k is kept for
  // PPL <= 16 and recomputed in pass 2 for longer lanes (register budget)
  constexpr bool kKeepC = PPL <= 16;
  f2 Cn[kKeepC ? PH : 1];
  f2 run = F2(0.f);
#pragma unroll
  for (int k = 0; k < PH; ++k) {
    const float4 c = u.c4(k);  // (c_a, c_b, -h_a, -h_b)
    run = fma2(make_float2(c.x, c.y), Pn[k], run);
    if (kKeepC) Cn[k] = fma2(make_float2(c.z, c.w), Pn[k], run);
  }
  float prefix, total;
  unit_scan(u, run.x + run.y, prefix, total);
  const float ba = bgb - bga;
  bool degen = !(total > 1e-12f * amp_bound * g.range);
  if (degen) degen = !(total > 1e-12f * unit_max_real(u, Pn) * g.range);  // inconclusive bound
  float acc;
  if (!degen) {
    const float scale = ba * rcpf(total);
    const f2 base = make_float2(fmaf(scale, prefix, bga), fmaf(scale, prefix + run.x, bga));
    const f2 S = F2(scale);
    f2 run2 = F2(0.f);
    acc = lane_noise_sum<NZ>(g, u, [&](int k) {
      f2 Ck;  // C_k = sum_{j<=k} c_j Pn_j - h_{k+1} Pn_k (lane-local part of each half)
      if (kKeepC) {
        Ck = Cn[kKeepC ? k : 0];
      } else {
        const float4 c = u.c4(k);
        run2 = fma2(make_float2(c.x, c.y), Pn[k], run2);
        Ck = fma2(make_float2(c.z, c.w), Pn[k], run2);
      }
      return add2(Pn[k], fma2(S, Ck, base));
    });
  } else {  // linear ramp a -> b
    acc = lane_noise_sum<NZ>(g, u, [&](int k) {
      return add2(Pn[k], fma2(F2(ba), mul2(add2(u.x2(k), F2(-g.x0s)), F2(g.inv_range)), F2(bga)));
    });
  }
  // padding points (c = h = 0) replicate the spectrum's last point exactly
  return finish_energy<NZ>(g, unit_sum(u, acc));
}

// NZ is the device noise model, or NZ_DYN to switch on g.noise per evaluation
// (energy kernels and the offset test family: one instantiation for all noises)
template <int FAM, int PPL, int W, int NZ>
__device__ __forceinline__ double evaluate_nz(const GroupDesc& g, Unit<PPL, W>& u, const f2 (&Pn)[PPL / 2],
                                              float bga, float bgb, float amp_bound) {
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
  if (is_xps<FAM>()) return eval_shirley_nz<PPL, W, nz>(g, u, Pn, bga, bgb, amp_bound);
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
  if (!is_xps<FAM>()) return 0.f;
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
template <int FAM, int PPL, int W, bool ENERGY, int NZ, bool REMC = false>
__device__ __forceinline__ void chain_body(const GroupDesc& g, Unit<PPL, W>& u, const int c, const int unit,
                                           const int wiu, const int lane, const GroupState* st, const int cur,
                                           const int d, const int T, double* th, double* lsv, int* acc, double* nvb,
                                           double* dlpb, float* lub, int* flg, float* thf, float* nvf,
                                           f2* gcache, f2* pcache) {
  using SM = Smem<PPL, W>;
  constexpr int PH = PPL / 2;
  constexpr int stride = block_stride<FAM>();
  const int ibg = 4 * g.K;  // xps Shirley endpoints (a, b) at ibg, ibg + 1
  f2 P[PH];
  unsigned long long fmask = full_signal<FAM, PPL, W>(g, thf, u, P);
  float asum = amp_sum<FAM>(g, thf);
  double e = fmask ? dinf()
                   : evaluate_nz<FAM, PPL, W, NZ>(g, u, P, is_xps<FAM>() ? thf[ibg] : 0.f,
                                           is_xps<FAM>() ? thf[ibg + 1] : 0.f, asum);
  if (ENERGY) {
    if (wiu == 0 && lane == 0) g.E[cur][c] = e;
    return;
  }

  // ---- waste-free chain: n sweeps at beta_next, every post-sweep state kept
  // (REMC: one sweep of replica c at its ladder beta, sweep index t = st->level,
  // Robbins-Monro while t <= n_burn (remc.cpp:125-133), state updated in place)
  const int n = REMC ? 1 : g.n, S = g.S;
  const int level = st->level;
  const double beta = REMC ? g.ladder[c] : st->beta;
  const double nd = g.n_data;
  const int adapt_sweeps = (n + 1) / 2;  // smc.cpp:136
  const uint32_t cg = g.chain_base + (uint32_t)(st->chain_lo + c);  // global chain id
  double* thn = g.theta[REMC ? cur : cur ^ 1];
  double* En = g.E[REMC ? cur : cur ^ 1];
  // components inside a block (everything but the xps Shirley endpoints and the offset family)
  const int npeak = FAM == FAM_OFFSET ? 0 : (FAM == FAM_XRD ? g.d : stride * g.K);
  unsigned trials = 0, shape_evals = 0;  // shape_evals: block-entry and trial shape evaluations (MUFU count)
  constexpr int L = SM::L;
  // Q[k] at Qs[k * L]: signal of every block except the one being swept (P - g_b)
  f2* Qs = gcache + (size_t)unit * (SM::NPT / 2) + u.lg;
  // committed peak signal: registers, or shared memory (Ps[k * L]) when p_in_smem<W>()
  constexpr bool kPsm = p_in_smem<W, PPL>();
  f2* Ps = pcache + (size_t)unit * (SM::NPT / 2) + u.lg;
  if (kPsm) {
#pragma unroll
    for (int k = 0; k < PH; ++k) Ps[k * L] = P[k];
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
      const u32x4 o = REMC ? philox(u32x4{cg, (uint32_t)level, (uint32_t)i, ROLE_REMC}, g.key0, g.key1)
                           : philox(u32x4{cg, (uint32_t)level, (uint32_t)(t - 1) * (uint32_t)d + (uint32_t)i, ROLE_CHAIN},
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
        f2 Qn[PH];
#pragma unroll
        for (int k = 0; k < PH; ++k) Qn[k] = SMC_P(k);
        if (!((fmask >> b) & 1ull)) {
          add_block<FAM, PPL, W>(g, b, thf + bi.off, u, Qn, -1.f);
          ++shape_evals;
        }
#pragma unroll
        for (int k = 0; k < PH; ++k) Qs[k * L] = Qn[k];
      }
      if (!(flg[i] & 1)) continue;  // outside the prior support: no trial (mcmc.cpp:68)
      const float oldf = thf[i], newf = nvf[i];
      // ---- trial signal Pn = P + (g_new - G) (the reference's BlockEvaluator::trial, energy.cpp:57-84)
      f2 Pn[PH];
      unsigned long long fnew = fmask;
      float dA = 0.f;
      // Shirley endpoint: enters combine() only (block -1), the peak signal is
      // unchanged and (registers) evaluated in place: no copy, no commit
      const bool endpoint = is_xps<FAM>() && !peak;  // (gm, xrd: every component is in a block)
      if (FAM == FAM_OFFSET) {
        const f2 dv = F2(newf - oldf);
#pragma unroll
        for (int k = 0; k < PH; ++k) Pn[k] = add2(SMC_P(k), dv);
      } else if (endpoint) {
        if (kPsm) {
#pragma unroll
          for (int k = 0; k < PH; ++k) Pn[k] = SMC_P(k);
        }
      } else if (j == 0 && oldf != 0.f && !((fmask >> b) & 1ull) &&
                 (FAM != FAM_XRD || b < g.K)) {  // amplitude: g' = (A'/A) g
        // Pn = P + r (P - Q) = (1 + r) P - r Q, r = A'/A - 1
        const float r = (newf - oldf) * rcpf(oldf);
        const f2 r1 = F2(1.f + r), mr = F2(-r);
#pragma unroll
        for (int k = 0; k < PH; ++k) Pn[k] = fma2(mr, Qs[k * L], mul2(r1, SMC_P(k)));
        dA = fabsf(newf) - fabsf(oldf);
      } else {
        constexpr int kMaxNp = FAM == FAM_XRD ? 9 : block_stride<FAM>();
        float pn[kMaxNp];
#pragma unroll
        for (int q = 0; q < kMaxNp; ++q) pn[q] = (q == j) ? newf : (q < bi.np ? thf[bi.off + q] : 0.f);
#pragma unroll
        for (int k = 0; k < PH; ++k) Pn[k] = Qs[k * L];
        if (add_block<FAM, PPL, W>(g, b, pn, u, Pn, 1.f))
          fnew &= ~(1ull << b);
        else
          fnew |= 1ull << b;
        if (j == 0) dA = fabsf(newf) - fabsf(oldf);
        ++shape_evals;
      }
      float bga = 0.f, bgb = 0.f;
      if (is_xps<FAM>()) {
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
        for (int k = 0; k < PH; ++k) P[k] = accept ? Pn[k] : P[k];
      }
      if (accept) {
        if (kPsm && !endpoint) {
#pragma unroll
          for (int k = 0; k < PH; ++k) Ps[k * L] = Pn[k];
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
      const bool adapt = REMC ? (long long)level <= g.n_burn : t <= adapt_sweeps;
      const int ta = REMC ? level : t;  // the RM clock: sweep of the level (SMC) or of the run (REMC)
      const float gam = adapt ? exp2f(-0.6f * log2f((float)ta)) : 0.f;  // t^-0.6
      for (int i = lane; i < d; i += 32) {
        const int a = flg[i] >> 1;
        acc[i] += a;
        if (adapt) {
          const double ls = lsv[i] + (double)gam * ((double)a - 0.5);
          lsv[i] = fmin(fmax(ls, kLogStepMin), kLogStepMax);
        }
      }
    }
    __syncwarp();
    const size_t slot = REMC ? (size_t)c : (size_t)c * n + (t - 1);  // smc.cpp:151 (REMC: in place)
    if (wiu == 0) {
      for (int i = lane; i < d; i += 32) thn[(size_t)i * g.tp + slot] = th[i];
      if (lane == 0) En[slot] = e;
    }
  }
  if (wiu == 0) {
    for (int i = lane; i < d; i += 32) {
      if (REMC)  // tallies accumulate over the run (reset at the end of burn-in)
        g.chain_acc[(size_t)i * g.sp + c] += acc[i];
      else
        g.chain_acc[(size_t)i * g.sp + c] = acc[i];
      g.chain_ls[(size_t)i * g.sp + c] = lsv[i];
    }
  }
#undef SMC_P
  // trials: each lane counted its own components; shape_evals: every lane
  // walked the same proposals (lane 0 of warp 0 reports)
  trials = __reduce_add_sync(0xffffffffu, trials);
  if (wiu == 0 && lane == 0) {
    atomicAdd(&g.st->trials, (unsigned long long)trials);
    atomicAdd(&g.st->shape_evals, (unsigned long long)shape_evals);
  }
}

template <int FAM, int PPL, int W, bool ENERGY, int NZ, bool REMC = false>
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
  // the group's descriptor staged in shared memory (every unit of a CTA runs
  // the same group): its fields are read on every evaluation (measured: C3
  // +3.6%, C5 +2.8%, C1 +4%, C2 +0.2% over reading them through L1)
  __shared__ GroupDesc sg;
  static_assert(sizeof(GroupDesc) % 4 == 0, "descriptor copy");
  for (int i = threadIdx.x; i < (int)(sizeof(GroupDesc) / 4); i += blockDim.x)
    reinterpret_cast<int*>(&sg)[i] = reinterpret_cast<const int*>(&gds[list[gi]])[i];
  __syncthreads();
  const GroupDesc& g = sg;
  const int cta_in_group = blockIdx.x - cta_prefix[gi];
  // a move launch covers every group of the class; finished or failed groups'
  // CTAs leave at once (levels are enqueued ahead of the host's check)
  if (!ENERGY && !g.st->active) return;

  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  f2* sx = reinterpret_cast<f2*>(smem + SM::off_x);
  float4* sc = reinterpret_cast<float4*>(smem + SM::off_c);
  void* sy = reinterpret_cast<void*>(smem + SM::off_y(lay));
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
  f2* gcache = reinterpret_cast<f2*>(smem + xoff + (size_t)U * sizeof(Xch));
  f2* pcache = gcache + (size_t)U * (SM::NPT / 2);

  // ---- stage the spectrum: cp.async.bulk (UBLKCP) completing on an mbarrier
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    const uint32_t bx = SM::NPT * 4u, bc = SM::NPT * 8u, by = SM::NPT * (uint32_t)SM::y_bytes(lay);
    // trapezoid weights: non-uniform grids only (the launch layout stages them then)
    const bool wc = is_xps<FAM>() && !g.sh_uniform && (SM::layout(lay) & kLayWeights);
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
  if (is_xps<FAM>() && g.sh_uniform) {  // points 0..N-2 lead, point N-1 in the last slot
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
  const int src = (ENERGY || REMC) ? c : g.anc[c];
  for (int i = lane; i < d; i += 32) {
    th[i] = thc[(size_t)i * g.tp + src];
    thf[i] = (float)th[i];
    if (!ENERGY) {
      lsv[i] = REMC ? g.chain_ls[(size_t)i * g.sp + c] : g.ls0[i];  // REMC: the replica's own step sizes
      acc[i] = 0;
    }
  }
  __syncwarp();

  chain_body<FAM, PPL, W, ENERGY, NZ, REMC>(g, u, c, unit, wiu, lane, st, cur, d, T, th, lsv, acc, nvb, dlpb, lub, flg, thf,
                                      nvf, gcache, pcache);
}

// ------------------------------------------------------------------ launch
template <int FAM, int PPL, int W, bool ENERGY, int NZ, bool REMC = false>
cudaError_t launch_chain_t(int U, int lay, int dmax, const GroupDesc* gds, const int* list, const int* prefix,
                           int n_list, int total_ctas, cudaStream_t st) {
  const int dpad = (dmax + 1) & ~1;
  const size_t smem = Smem<PPL, W>::bytes(U, dpad, lay);
  auto kern = k_chain<FAM, PPL, W, ENERGY, NZ, REMC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  if (total_ctas <= 0) return cudaSuccess;  // prime only (module load + attributes, see prime_level_kernels)
  const int dpad_lay = chain_dyn_layout(W) ? (dpad | (lay << 16)) : dpad;
  kern<<<total_ctas, 32 * W * U, smem, st>>>(gds, list, prefix, n_list, U, dpad_lay);  // U <= threads / 32 W
  return cudaGetLastError();
}

// (W, PPL) pairs compiled (see pick_shape in kernels.cu): W = 1 for N <= 512,
// W = 2 for N <= 2048, W = 4 for N <= 4096, W = 8 for N <= 8192
#define SMC_FOR_EACH_SHAPE(X)                                                                          \
  X(1, 2) X(1, 4) X(1, 6) X(1, 8) X(1, 10) X(1, 12) X(1, 14) X(1, 16) X(1, 20) X(1, 24) X(1, 28) X(1, 32) \
  X(2, 10) X(2, 12) X(2, 14) X(2, 16) X(2, 20) X(2, 24) X(2, 28) X(2, 32)                             \
  X(4, 20) X(4, 24) X(4, 28) X(4, 32) X(8, 20) X(8, 24) X(8, 28) X(8, 32)

template <int FAM, bool ENERGY, int NZ, bool REMC = false>
cudaError_t launch_chain_fam(const Shape& s, int dmax, const GroupDesc* gds, const int* list, const int* prefix,
                             int n_list, int total_ctas, cudaStream_t st) {
#define SMC_CASE(WW, PP) \
  if (s.W == WW && s.PPL == PP) return launch_chain_t<FAM, PP, WW, ENERGY, NZ, REMC>(s.U, s.lay, dmax, gds, list, prefix, n_list, total_ctas, st);
  SMC_FOR_EACH_SHAPE(SMC_CASE)
#undef SMC_CASE
  return cudaErrorInvalidValue;
}

}  // namespace smc
