/*
 * specmc_oracle.c -- CPU restatement of the reference SMC hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the
 * B200 product path (paper_2604_03271_b200/csrc).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it.  The product never links, imports or falls back to it.
 *
 * Every function restates the reference (arxiv/paper_2604_03271, "specmc",
 * C++20 + Eigen) operation for operation, so that -- compiled with
 * -ffp-contract=off and sequential sums -- it reproduces the reference built
 * against oracle/eigen_shim bit for bit (tests/test_oracle_vs_ref.py pins
 * that).  Paths below are relative to the reference root.
 *
 *   RNG            proj/include/specmc/rng.hpp:11-92
 *   log-sum-exp    proj/include/specmc/math.hpp:20-30, cumtrapz :63-71
 *   lineshapes     proj/include/specmc/lineshapes.hpp:46-83
 *   priors         proj/src/priors.cpp:22-49, :95-110
 *   forward model  proj/src/model.cpp:191-294  (gm, xps; "offset" = the
 *                  conjugate test problem of proj/tests/conjugate_oracle.hpp:19-28)
 *   data energy    proj/src/energy.cpp:7-28
 *   MH sweep       proj/src/mcmc.cpp:7-96
 *   SMC            proj/src/smc.cpp:23-211
 *   model select   proj/src/posterior.cpp:68-104 (restated in python, tests/)
 *
 * The evaluator here always recomputes the full energy: the reference's
 * BlockEvaluator contract is that trial()/full() agree bit for bit
 * (proj/include/specmc/energy.hpp:27-29), so the numbers are identical.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_INF (1.0 / 0.0)
#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

enum { ORC_GM = 0, ORC_XPS = 1, ORC_XRD = 2, ORC_OFFSET = 3 };
enum { ORC_NOISE_GAUSS = 0, ORC_NOISE_POISSON = 1, ORC_NOISE_GAPPROX = 2, ORC_NOISE_HETERO = 3 };
enum { ORC_PRIOR_NORMAL = 0, ORC_PRIOR_GAMMA = 1, ORC_PRIOR_UNIFORM = 2 };
enum { ORC_OK = 0, ORC_EINVAL = 2, ORC_ERUNTIME = 3 };

/* ------------------------------------------------------------------ RNG */
/* rng.hpp:11-14 */
uint64_t orc_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
/* rng.hpp:16-19 */
static uint64_t splitmix64_next(uint64_t* x) {
  *x += 0x9E3779B97F4A7C15ULL;
  return orc_mix64(*x);
}
/* rng.hpp:21-23 */
uint64_t orc_hash_combine(uint64_t h, uint64_t v) {
  return orc_mix64(h ^ (0x9E3779B97F4A7C15ULL + v + (h << 6) + (h >> 2)));
}

typedef struct {
  uint64_t s[4];
  uint64_t key;
  double spare;
  int has_spare;
} orc_rng;

/* rng.hpp:31-34 */
void orc_rng_seed(orc_rng* r, uint64_t seed) {
  uint64_t sm = seed;
  r->key = seed;
  for (int i = 0; i < 4; ++i) r->s[i] = splitmix64_next(&sm);
  r->spare = 0.0;
  r->has_spare = 0;
}
/* rng.hpp:37-41 */
void orc_rng_substream(const orc_rng* base, const uint64_t* ids, int n, orc_rng* out) {
  uint64_t h = base->key;
  for (int i = 0; i < n; ++i) h = orc_hash_combine(h, ids[i]);
  orc_rng_seed(out, h);
}
static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
/* rng.hpp:44-54 (xoshiro256++) */
uint64_t orc_next_u64(orc_rng* r) {
  uint64_t* s = r->s;
  const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return result;
}
/* rng.hpp:57 */
double orc_uniform01(orc_rng* r) { return (double)(orc_next_u64(r) >> 11) * 0x1.0p-53; }
/* rng.hpp:62-74 (Box-Muller, spare cached) */
double orc_normal(orc_rng* r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  double u1 = orc_uniform01(r);
  double u2 = orc_uniform01(r);
  double rr = sqrt(-2.0 * log1p(-u1));
  double a = 6.283185307179586476925286766559 * u2;
  r->spare = rr * sin(a);
  r->has_spare = 1;
  return rr * cos(a);
}
/* rng.hpp:77-92 (Marsaglia-Tsang) */
double orc_gamma(orc_rng* r, double shape, double rate) {
  if (shape < 1.0) {
    double u = 1.0 - orc_uniform01(r);
    return orc_gamma(r, shape + 1.0, rate) * pow(u, 1.0 / shape);
  }
  const double d = shape - 1.0 / 3.0;
  const double c = 1.0 / sqrt(9.0 * d);
  for (;;) {
    double x = orc_normal(r);
    double t = 1.0 + c * x;
    if (t <= 0.0) continue;
    double v = t * t * t;
    double u = 1.0 - orc_uniform01(r);
    if (log(u) < 0.5 * x * x + d - d * v + d * log(v)) return d * v / rate;
  }
}

/* ------------------------------------------------------------ math.hpp */
/* math.hpp:20-26 */
double orc_log_sum_exp(const double* v, int64_t n) {
  if (n == 0) return -ORC_INF;
  double m = v[0];
  for (int64_t i = 1; i < n; ++i)
    if (v[i] > m) m = v[i]; /* Eigen maxCoeff */
  if (!isfinite(m)) return m;
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += exp(v[i] - m);
  return m + log(s);
}
/* math.hpp:28-30 */
double orc_log_mean_exp(const double* v, int64_t n) {
  return orc_log_sum_exp(v, n) - log((double)n);
}
/* math.hpp:63-71 */
void orc_cumtrapz(const double* xs, const double* ys, int64_t n, double* out) {
  if (n == 0) return;
  out[0] = 0.0;
  for (int64_t i = 1; i < n; ++i) out[i] = out[i - 1] + 0.5 * (xs[i] - xs[i - 1]) * (ys[i] + ys[i - 1]);
}

/* -------------------------------------------------------------- priors */
/* priors.cpp:22-35 */
double orc_prior_logpdf1(int kind, double a, double b, double x) {
  if (kind == ORC_PRIOR_NORMAL) {
    double d = x - a;
    return -0.5 * log(2.0 * M_PI * b) - d * d / (2.0 * b);
  }
  if (kind == ORC_PRIOR_GAMMA) {
    if (!(x > 0.0)) return -ORC_INF;
    return a * log(b) - lgamma(a) + (a - 1.0) * log(x) - b * x;
  }
  if (x < a || x > b) return -ORC_INF;
  return -log(b - a);
}
/* priors.cpp:37-42 (uniform: rng.hpp:59) */
double orc_prior_sample1(int kind, double a, double b, orc_rng* r) {
  if (kind == ORC_PRIOR_NORMAL) return a + sqrt(b) * orc_normal(r);
  if (kind == ORC_PRIOR_GAMMA) return orc_gamma(r, a, b);
  return a + (b - a) * orc_uniform01(r);
}
/* priors.cpp:44-49 */
double orc_prior_scale(int kind, double a, double b) {
  if (kind == ORC_PRIOR_NORMAL) return sqrt(b);
  if (kind == ORC_PRIOR_GAMMA) return sqrt(a) / b;
  return (b - a) / sqrt(12.0);
}

/* --------------------------------------------------------------- model */
typedef struct {
  int family;
  int K;
  int d;
  int noise;
  double sigma, s0, s1, s2;
  int paper_literal;
  const int* prior_kind;
  const double* prior_a;
  const double* prior_b;
  const double* xs;
  const double* ys;
  int64_t n;
  /* xrd: reflections of every phase, grouped by phase in phase order */
  int n_refl;
  const int* refl_phase;
  const double* refl_mu;
  const double* refl_int;
} orc_model;

static int n_blocks(const orc_model* m) {
  if (m->family == ORC_OFFSET) return 1;
  if (m->family == ORC_XRD) return m->K + 1; /* phases + background (model.cpp:198-202) */
  return m->K;
}

static const double kFourLn2 = 2.772588722239781237668928485832706272302; /* lineshapes.hpp:11 */

/* model.cpp:213-283, gm and xps branches; lineshapes.hpp:54-59.  Returns 0 on
 * an evaluation fault (E = +inf). */
static int eval_block(const orc_model* m, int b, const double* th, double* out) {
  const int64_t n = m->n;
  const double* xs = m->xs;
  if (m->family == ORC_GM) {
    const double A = th[3 * b], mu = th[3 * b + 1], bw = th[3 * b + 2];
    const double c = -0.5 * bw; /* (-0.5 * bw) * (xs - mu).square() */
    for (int64_t i = 0; i < n; ++i) {
      double t = xs[i] - mu;
      out[i] = A * exp(c * (t * t));
    }
    return 1;
  }
  if (m->family == ORC_XPS) {
    const double A = th[4 * b], mu = th[4 * b + 1], sig = th[4 * b + 2], eta = th[4 * b + 3];
    if (!(sig > 0.0)) return 0;
    const double cg = -0.693147180559945309417232121458176568076 / (sig * sig);
    const double s2 = sig * sig;
    const double lnum = (1.0 - eta) * (sig * sig);
    for (int64_t i = 0; i < n; ++i) {
      double dx = xs[i] - mu;
      double d2 = dx * dx;
      double g = exp(cg * d2);
      out[i] = A * (eta * g + lnum / (s2 + d2));
    }
    return 1;
  }
  if (m->family == ORC_XRD) {
    if (b == m->K) { /* background block (model.cpp:223-234) */
      const int off = 9 * m->K;
      const double a = th[off], sbg = th[off + 1], rbg = th[off + 2], bg = th[off + 3];
      if (!(sbg > 0.0)) return 0;
      for (int64_t i = 0; i < n; ++i) {
        double t = xs[i] / sbg;
        double t2 = t * t;
        out[i] = a * ((1.0 - rbg) * exp((-kFourLn2) * t2) + rbg / (1.0 + 4.0 * t2)) + bg;
      }
      return 1;
    }
    /* phase block (model.cpp:235-267) */
    const int off = 9 * b;
    const double A = th[off], d2t = th[off + 1], r = th[off + 2], alpha = th[off + 3], u = th[off + 4],
                 v = th[off + 5], w = th[off + 6], s = th[off + 7], t = th[off + 8];
    const double deg2rad = M_PI / 180.0;
    for (int64_t i = 0; i < n; ++i) out[i] = 0.0;
    for (int q = 0; q < m->n_refl; ++q) {
      if (m->refl_phase[q] != b) continue;
      const double c = m->refl_mu[q] + d2t;
      const double half = 0.5 * c * deg2rad;
      const double tn = tan(half);
      const double disc = u * tn * tn - v * tn + w;
      if (!(disc > 0.0)) return 0;
      const double sig0 = sqrt(disc);
      const double om0 = s / cos(half) + t * tn;
      if (!(om0 > 0.0)) return 0;
      const double amp = A * m->refl_int[q];
      const double gh = alpha * sig0, lh = alpha * om0;
      for (int64_t i = 0; i < n; ++i) {
        const double dx = xs[i] - c;
        const double wg = dx >= 0.0 ? dx / gh : dx / sig0;
        const double wl = dx >= 0.0 ? dx / lh : dx / om0;
        out[i] += amp * ((1.0 - r) * exp((-kFourLn2) * (wg * wg)) + r / (1.0 + 4.0 * (wl * wl)));
      }
    }
    return 1;
  }
  /* offset: the conjugate-mean problem, f_i = theta_0 */
  for (int64_t i = 0; i < n; ++i) out[i] = th[0];
  return 1;
}

/* lineshapes.hpp:65-83 */
static void shirley_add(const double* xs, double* f, int64_t n, double a, double b, double* cbuf) {
  const double range = xs[n - 1] - xs[0];
  orc_cumtrapz(xs, f, n, cbuf);
  const double total = cbuf[n - 1];
  double peak_max = f[0];
  for (int64_t i = 1; i < n; ++i)
    if (f[i] > peak_max) peak_max = f[i];
  /* out computed into cbuf, then f += out (model.cpp:290) */
  if (!(total > 1e-12 * peak_max * range)) {
    for (int64_t i = 0; i < n; ++i) cbuf[i] = a + (b - a) * (xs[i] - xs[0]) / range;
  } else {
    for (int64_t i = 0; i < n; ++i) cbuf[i] = a + (b - a) * (cbuf[i] / total);
  }
  cbuf[0] = a;
  cbuf[n - 1] = b;
  for (int64_t i = 0; i < n; ++i) f[i] += cbuf[i];
}

/* model.cpp:285-294 (combine) after every block evaluated: returns 0 on fault */
int orc_forward(const orc_model* m, const double* th, double* f) {
  const int64_t n = m->n;
  const int nb = n_blocks(m);
  double* blk = (double*)malloc(sizeof(double) * (size_t)n);
  int ok = 1;
  for (int b = 0; b < nb && ok; ++b) {
    if (!eval_block(m, b, th, blk)) {
      ok = 0;
      break;
    }
    if (b == 0)
      memcpy(f, blk, sizeof(double) * (size_t)n);
    else
      for (int64_t i = 0; i < n; ++i) f[i] += blk[i];
  }
  if (ok && m->family == ORC_XPS) shirley_add(m->xs, f, n, th[4 * m->K], th[4 * m->K + 1], blk);
  free(blk);
  return ok;
}

/* energy.cpp:7-28 */
double orc_data_energy(int noise, double sigma, double s0, double s1, double s2, int lit,
                       const double* ys, const double* f, int64_t n_) {
  const double n = (double)n_;
  if (noise == ORC_NOISE_GAUSS) {
    const double sg2 = sigma * sigma;
    double s = 0.0;
    for (int64_t i = 0; i < n_; ++i) {
      double r = ys[i] - f[i];
      s += r * r;
    }
    double q = s / (2.0 * sg2 * n);
    return 0.5 * log(2.0 * M_PI * sg2) + q;
  }
  if (noise == ORC_NOISE_POISSON) {
    for (int64_t i = 0; i < n_; ++i)
      if (!(f[i] > 0.0)) return ORC_INF;
    double s = 0.0;
    for (int64_t i = 0; i < n_; ++i) s += f[i] - ys[i] * log(f[i]);
    return s / n;
  }
  if (noise == ORC_NOISE_GAPPROX) {
    for (int64_t i = 0; i < n_; ++i)
      if (!(f[i] > 0.0)) return ORC_INF;
    double s = 0.0;
    const double tp = 2.0 * M_PI;
    for (int64_t i = 0; i < n_; ++i) {
      double r = ys[i] - f[i];
      s += 0.5 * log(tp * f[i]) + (r * r) / (2.0 * f[i]);
    }
    return s / n;
  }
  {
    const double a0 = s0 * s0, a1 = s1 * s1, a2 = s2 * s2;
    double* var = (double*)malloc(sizeof(double) * (size_t)(n_ > 0 ? n_ : 1));
    for (int64_t i = 0; i < n_; ++i) var[i] = a0 * f[i] + a1 * (f[i] * f[i]) + a2;
    for (int64_t i = 0; i < n_; ++i)
      if (!(var[i] > 0.0)) {
        free(var);
        return ORC_INF;
      }
    const double q = lit ? 1.0 : 0.5;
    const double tp = 2.0 * M_PI;
    double s = 0.0;
    for (int64_t i = 0; i < n_; ++i) {
      double r = ys[i] - f[i];
      s += 0.5 * log(tp * var[i]) + q * (r * r) / var[i];
    }
    free(var);
    return s / n;
  }
}

/* energy.cpp:43-55 (BlockEvaluator::full) */
double orc_energy(const orc_model* m, const double* th) {
  double* f = (double*)malloc(sizeof(double) * (size_t)m->n);
  double e = ORC_INF;
  if (orc_forward(m, th, f))
    e = orc_data_energy(m->noise, m->sigma, m->s0, m->s1, m->s2, m->paper_literal, m->ys, f, m->n);
  free(f);
  return e;
}

/* ---------------------------------------------------------------- MCMC */
static const double kStepMin = 1e-12, kStepMax = 1e12;
static double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* mcmc.cpp:14-18 */
double orc_rm_update(double step, int accepted, long long t) {
  const double gamma = 1.0 / pow((double)t, 0.6);
  double ls = log(step) + gamma * ((accepted ? 1.0 : 0.0) - 0.5);
  return clampd(exp(ls), kStepMin, kStepMax);
}

/* mcmc.cpp:20-53.  History arrays are [H][d] row-major, oldest first. */
void orc_predict_step_size(const double* hbeta, const double* hacc, const double* hstep, int H, int d,
                           double beta_next, const int* pk, const double* pa, const double* pb,
                           double* out) {
  if (H == 0) {
    for (int i = 0; i < d; ++i) out[i] = clampd(orc_prior_scale(pk[i], pa[i], pb[i]), kStepMin, kStepMax);
    return;
  }
  const int first = H > 5 ? H - 5 : 0;
  const int m = H - first;
  const double lx = log(beta_next);
  for (int c = 0; c < d; ++c) {
    double sx = 0, sy = 0, sxx = 0, sxy = 0;
    for (int j = first; j < H; ++j) {
      double x = log(hbeta[j]);
      double y = log(hstep[(size_t)j * d + c]) + 2.0 * (hacc[(size_t)j * d + c] - 0.5);
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
      pred = icept + slope * lx;
    }
    out[c] = clampd(exp(pred), kStepMin, kStepMax);
  }
}

/* mcmc.cpp:55-96 */
int orc_cw_mh_sweep(const orc_model* m, double* theta, double* e_cache, double beta, double* step,
                    int* accepts, int* proposals, orc_rng* rng, int adapt, long long t_adapt,
                    long long* trials) {
  const int d = m->d;
  const double n = (double)m->n;
  int accepted_count = 0;
  for (int i = 0; i < d; ++i) {
    const double z = orc_normal(rng);
    const double old_i = theta[i];
    const double new_i = old_i + step[i] * z;
    const double lp_old = orc_prior_logpdf1(m->prior_kind[i], m->prior_a[i], m->prior_b[i], old_i);
    const double lp_new = orc_prior_logpdf1(m->prior_kind[i], m->prior_a[i], m->prior_b[i], new_i);
    ++proposals[i];
    int accept = 0;
    if (lp_new != -ORC_INF) {
      theta[i] = new_i;
      const double e_new = orc_energy(m, theta);
      if (trials) ++*trials;
      double log_ratio;
      if (beta == 0.0 || (e_new == ORC_INF && *e_cache == ORC_INF)) {
        log_ratio = lp_new - lp_old;
      } else if (e_new == ORC_INF) {
        log_ratio = -ORC_INF;
      } else if (*e_cache == ORC_INF) {
        log_ratio = ORC_INF;
      } else {
        log_ratio = -beta * n * (e_new - *e_cache) + (lp_new - lp_old);
      }
      if (log_ratio >= 0.0 || log(orc_uniform01(rng)) < log_ratio) {
        accept = 1;
        *e_cache = e_new;
      } else {
        theta[i] = old_i;
      }
    }
    if (accept) {
      ++accepts[i];
      ++accepted_count;
    }
    if (adapt) step[i] = orc_rm_update(step[i], accept, t_adapt);
  }
  return accepted_count;
}

/* ----------------------------------------------------------------- SMC */
/* smc.cpp:61-66; err = 3 when every weight vanishes */
double orc_ess(const double* lw, int64_t n, int* err) {
  const double l1 = orc_log_sum_exp(lw, n);
  if (l1 == -ORC_INF) {
    if (err) *err = ORC_ERUNTIME;
    return NAN;
  }
  double* w2 = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) w2[i] = 2.0 * lw[i];
  const double l2 = orc_log_sum_exp(w2, n);
  free(w2);
  return exp(2.0 * l1 - l2);
}

/* smc.cpp:55-59 */
void orc_incremental_log_weights(const double* E, int64_t T, double delta_beta, double n_data, double* out) {
  if (delta_beta == 0.0) {
    for (int64_t i = 0; i < T; ++i) out[i] = 0.0;
    return;
  }
  const double c = -delta_beta * n_data;
  for (int64_t i = 0; i < T; ++i) out[i] = c * E[i];
}

/* smc.cpp:68-93 */
double orc_next_beta(const double* E, int64_t T_, double n_data, double beta_prev, double target, int* err) {
  if (!(beta_prev < 1.0)) {
    if (err) *err = ORC_EINVAL;
    return NAN;
  }
  const double T = (double)T_;
  double emin = ORC_INF;
  for (int64_t i = 0; i < T_; ++i)
    if (E[i] < emin) emin = E[i];
  if (!isfinite(emin)) emin = 0.0;
  double* lw = (double*)malloc(sizeof(double) * (size_t)T_);
  int e2 = 0;
#define ESS_AT(db, outv)                                               \
  do {                                                                 \
    const double c_ = -(db) * n_data;                                  \
    for (int64_t i = 0; i < T_; ++i) lw[i] = c_ * (E[i] - emin);       \
    outv = orc_ess(lw, T_, &e2) / T;                                   \
  } while (0)
  const double full = 1.0 - beta_prev;
  double r;
  ESS_AT(full, r);
  if (e2) goto fail;
  if (r >= target) {
    free(lw);
    return 1.0;
  }
  {
    double lo = 0.0, hi = full, mid = 0.5 * full;
    for (int it = 0; it < 60; ++it) {
      mid = 0.5 * (lo + hi);
      ESS_AT(mid, r);
      if (e2) goto fail;
      if (fabs(r - target) <= 1e-6) break;
      if (r > target)
        lo = mid;
      else
        hi = mid;
    }
    free(lw);
    return beta_prev + mid;
  }
#undef ESS_AT
fail:
  free(lw);
  if (err) *err = ORC_ERUNTIME;
  return NAN;
}

/* smc.cpp:95-112, with the uniform passed in (drawn from substream {3, level}) */
int orc_systematic_resample(const double* lw, int64_t T, int64_t S, double u, int64_t* out) {
  const double lse = orc_log_sum_exp(lw, T);
  if (lse == -ORC_INF) return ORC_ERUNTIME;
  int64_t i = 0;
  double c = exp(lw[0] - lse);
  for (int64_t j = 0; j < S; ++j) {
    const double target = ((double)j + u) / (double)S;
    while (c < target && i < T - 1) {
      ++i;
      c += exp(lw[i] - lse);
    }
    out[j] = i;
  }
  return ORC_OK;
}

/* smc.cpp:23-32 */
int orc_validate_smc_config(int64_t T, int n, double ess_target, int max_levels, int workers) {
  if (T < 2) return ORC_EINVAL;
  if (n < 1) return ORC_EINVAL;
  if (T % n != 0) return ORC_EINVAL;
  if (T / n < 2) return ORC_EINVAL;
  if (!(ess_target > 0.0 && ess_target < 1.0)) return ORC_EINVAL;
  if (max_levels < 1) return ORC_EINVAL;
  if (workers < 0) return ORC_EINVAL;
  return ORC_OK;
}

typedef struct {
  double F;
  int diverged;
  int levels;
  /* caller-provided, capacity max_levels (+1 for ladder) */
  double* ladder;
  double* ess_ratio;
  double* log_mean_w;
  double* acc_rate;
  /* caller-provided: d*T (column c at c*d), T; may be NULL */
  double* thetas;
  double* energies;
  long long proposals; /* sum over levels of T*d (smc.cpp:182) */
  long long trials;    /* finite-prior proposals = Evaluator::trial calls */
} orc_smc_result;

/* smc.cpp:34-53 (init_ensemble), :114-184 (wastefree_level), :186-211 (smc_run) */
int orc_smc_run(const orc_model* m, int64_t T, int n, double ess_target, int max_levels, uint64_t seed,
                orc_smc_result* res) {
  int rc = orc_validate_smc_config(T, n, ess_target, max_levels, 0);
  if (rc) return rc;
  const int d = m->d;
  const int64_t S = T / n;
  const double n_data = (double)m->n;
  double* th = (double*)malloc(sizeof(double) * (size_t)d * (size_t)T);
  double* th2 = (double*)malloc(sizeof(double) * (size_t)d * (size_t)T);
  double* E = (double*)malloc(sizeof(double) * (size_t)T);
  double* E2 = (double*)malloc(sizeof(double) * (size_t)T);
  double* lw = (double*)malloc(sizeof(double) * (size_t)T);
  int64_t* anc = (int64_t*)malloc(sizeof(int64_t) * (size_t)S);
  double* step0 = (double*)malloc(sizeof(double) * (size_t)d);
  double* step = (double*)malloc(sizeof(double) * (size_t)d);
  double* cur = (double*)malloc(sizeof(double) * (size_t)d);
  int* acc = (int*)malloc(sizeof(int) * (size_t)d);
  int* prop = (int*)malloc(sizeof(int) * (size_t)d);
  double* sacc = (double*)malloc(sizeof(double) * (size_t)d);
  double* sprop = (double*)malloc(sizeof(double) * (size_t)d);
  double* slog = (double*)malloc(sizeof(double) * (size_t)d);
  double* hbeta = (double*)malloc(sizeof(double) * (size_t)max_levels);
  double* hacc = (double*)malloc(sizeof(double) * (size_t)max_levels * (size_t)d);
  double* hstep = (double*)malloc(sizeof(double) * (size_t)max_levels * (size_t)d);
  orc_rng base;
  orc_rng_seed(&base, seed);
  res->proposals = 0;
  res->trials = 0;

  /* init_ensemble */
  for (int64_t i = 0; i < T; ++i) {
    orc_rng r;
    uint64_t ids[2] = {1, (uint64_t)i};
    orc_rng_substream(&base, ids, 2, &r);
    for (int k = 0; k < d; ++k) th[(size_t)i * d + k] = orc_prior_sample1(m->prior_kind[k], m->prior_a[k], m->prior_b[k], &r);
    E[i] = orc_energy(m, th + (size_t)i * d);
  }

  double beta = 0.0, neg_log_z = 0.0;
  int level = 0, H = 0;
  res->ladder[0] = 0.0;
  while (beta < 1.0) {
    if (level >= max_levels) {
      rc = ORC_ERUNTIME;
      goto done;
    }
    ++level;
    int err = 0;
    const double beta_next = orc_next_beta(E, T, n_data, beta, ess_target, &err);
    if (err) {
      rc = err;
      goto done;
    }
    /* wastefree_level */
    orc_incremental_log_weights(E, T, beta_next - beta, n_data, lw);
    const double ess_v = orc_ess(lw, T, &err);
    if (err) {
      rc = err;
      goto done;
    }
    res->ess_ratio[level - 1] = ess_v / (double)T;
    const double lmw = orc_log_mean_exp(lw, T);
    res->log_mean_w[level - 1] = lmw;
    orc_rng rs;
    uint64_t rids[2] = {3, (uint64_t)level};
    orc_rng_substream(&base, rids, 2, &rs);
    const double u = orc_uniform01(&rs);
    rc = orc_systematic_resample(lw, T, S, u, anc);
    if (rc) goto done;
    orc_predict_step_size(hbeta, hacc, hstep, H, d, beta_next, m->prior_kind, m->prior_a, m->prior_b, step0);
    const long long adapt_sweeps = (n + 1) / 2;
    for (int k = 0; k < d; ++k) sacc[k] = sprop[k] = slog[k] = 0.0;
    for (int64_t c = 0; c < S; ++c) {
      orc_rng rc_;
      uint64_t cids[3] = {2, (uint64_t)level, (uint64_t)c};
      orc_rng_substream(&base, cids, 3, &rc_);
      memcpy(cur, th + (size_t)anc[c] * d, sizeof(double) * (size_t)d);
      double e = orc_energy(m, cur);
      memcpy(step, step0, sizeof(double) * (size_t)d);
      memset(acc, 0, sizeof(int) * (size_t)d);
      memset(prop, 0, sizeof(int) * (size_t)d);
      for (int t = 1; t <= n; ++t) {
        orc_cw_mh_sweep(m, cur, &e, beta_next, step, acc, prop, &rc_, t <= adapt_sweeps, t, &res->trials);
        const int64_t slot = c * n + (t - 1);
        memcpy(th2 + (size_t)slot * d, cur, sizeof(double) * (size_t)d);
        E2[slot] = e;
      }
      /* smc.cpp:168-173: chain-order accumulation */
      for (int k = 0; k < d; ++k) {
        sacc[k] += (double)acc[k];
        sprop[k] += (double)prop[k];
        slog[k] += log(step[k]);
      }
    }
    { double* t = th; th = th2; th2 = t; }
    { double* t = E; E = E2; E2 = t; }
    hbeta[H] = beta_next;
    for (int k = 0; k < d; ++k) {
      hacc[(size_t)H * d + k] = sprop[k] > 0 ? sacc[k] / sprop[k] : 0.0;
      hstep[(size_t)H * d + k] = exp(slog[k] / (double)S);
    }
    ++H;
    double asum = 0.0, psum = 0.0;
    for (int k = 0; k < d; ++k) asum += sacc[k];
    for (int k = 0; k < d; ++k) psum += sprop[k];
    res->acc_rate[level - 1] = psum > 0 ? asum / psum : 0.0;
    res->proposals += (long long)T * d;
    res->ladder[level] = beta_next;
    neg_log_z -= lmw;
    beta = beta_next;
  }
  res->F = neg_log_z;
  res->diverged = !isfinite(neg_log_z);
  res->levels = level;
  if (res->thetas) memcpy(res->thetas, th, sizeof(double) * (size_t)d * (size_t)T);
  if (res->energies) memcpy(res->energies, E, sizeof(double) * (size_t)T);
done:
  res->levels = level;
  free(th); free(th2); free(E); free(E2); free(lw); free(anc); free(step0); free(step); free(cur);
  free(acc); free(prop); free(sacc); free(sprop); free(slog); free(hbeta); free(hacc); free(hstep);
  return rc;
}

/* init_ensemble only (smc.cpp:34-53): draws and energies, for IS identities */
void orc_init_ensemble(const orc_model* m, int64_t T, uint64_t seed, double* th, double* E) {
  orc_rng base;
  orc_rng_seed(&base, seed);
  const int d = m->d;
  for (int64_t i = 0; i < T; ++i) {
    orc_rng r;
    uint64_t ids[2] = {1, (uint64_t)i};
    orc_rng_substream(&base, ids, 2, &r);
    for (int k = 0; k < d; ++k) th[(size_t)i * d + k] = orc_prior_sample1(m->prior_kind[k], m->prior_a[k], m->prior_b[k], &r);
    E[i] = orc_energy(m, th + (size_t)i * d);
  }
}

/* uniform01 of the resample substream {3, level} of seed (smc.cpp:132) */
double orc_resample_uniform(uint64_t seed, int level) {
  orc_rng base, rs;
  orc_rng_seed(&base, seed);
  uint64_t rids[2] = {3, (uint64_t)level};
  orc_rng_substream(&base, rids, 2, &rs);
  return orc_uniform01(&rs);
}

/* n normals from Rng(seed) (for synthetic-data cross checks) */
void orc_normals(uint64_t seed, int64_t n, double* out) {
  orc_rng r;
  orc_rng_seed(&r, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = orc_normal(&r);
}
