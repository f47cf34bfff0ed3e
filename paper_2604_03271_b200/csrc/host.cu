// host.cu -- C++ host driver and C ABI of the B200 SMC sampler.
//
// Mirrors the reference's host-side semantics (paths relative to the
// reference root):
//   validate_smc_config        proj/src/smc.cpp:23-32
//   validate_model / _prior    proj/src/model.cpp:97-113, proj/src/priors.cpp:9-20
//   validate_spectrum          proj/src/spectrum.cpp:12-23
//   smc_run (level loop)       proj/src/smc.cpp:186-211, report fields :218-249
// The level loop runs every group (one SMC run = one (spectrum, K, seed)) of
// a batch in lock-step: per round the tempering (k_temper, one CTA per group,
// or the k_tp_* grid phases for T > 2^15), one k_chain move launch covering
// every chain of every active group (longest d first), and k_stats_grid +
// k_stats_final.  The host reads back the small GroupState of every group per
// round to retire groups that reached beta = 1.  Particle-sharded runs
// (run_sharded) add the cross-shard exchanges between the tempering phases.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include <dlfcn.h>
#include <unistd.h>
#include <nccl.h>  // types only: the library is resolved at run time (dlopen), see NcclApi

#include "../../include/specmc_b200.h"
#include "launch.h"

namespace smc {
namespace {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(SPECMC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------ instrumentation
std::mutex g_stats_mu;
specmc_stats g_stats{0, 0.0, 0, 0.0, 0.0};

void count_launch(int64_t n = 1) {
  std::lock_guard<std::mutex> lk(g_stats_mu);
  g_stats.kernel_launches += n;
}

// ------------------------------------------------------------------ validation
void validate_config(const specmc_smc_config& c) {  // smc.cpp:23-32
  if (c.T < 2) throw Error(SPECMC_EINVAL, "smc: T must be >= 2");
  if (c.n < 1) throw Error(SPECMC_EINVAL, "smc: n must be >= 1");
  if (c.T % c.n != 0) throw Error(SPECMC_EINVAL, "smc: T must be divisible by n");
  if (c.T / c.n < 2) throw Error(SPECMC_EINVAL, "smc: S = T/n must be >= 2");
  if (!(c.ess_target > 0.0 && c.ess_target < 1.0)) throw Error(SPECMC_EINVAL, "smc: ess_target must lie in (0, 1)");
  if (c.max_levels < 1) throw Error(SPECMC_EINVAL, "smc: max_levels must be >= 1");
  if (c.workers < 0) throw Error(SPECMC_EINVAL, "smc: workers must be >= 0");
  if (c.T > (int64_t)1 << 30) throw Error(SPECMC_EINVAL, "smc: T above 2^30 is not supported by the device path");
}

int model_dim(const specmc_model_desc& m) {  // model.cpp:86-93
  switch (m.family) {
    case SPECMC_FAMILY_GM: return 3 * m.K;
    case SPECMC_FAMILY_XPS: return 4 * m.K + 2;
    case SPECMC_FAMILY_XRD: return 9 * m.K + 4;
    case SPECMC_FAMILY_OFFSET: return 1;
  }
  return -1;
}

void validate_model(const specmc_model_desc& m) {
  if (m.family != SPECMC_FAMILY_GM && m.family != SPECMC_FAMILY_XPS && m.family != SPECMC_FAMILY_OFFSET &&
      m.family != SPECMC_FAMILY_XRD)
    throw Error(SPECMC_EINVAL, "unknown model family");
  if (m.K < 1) throw Error(SPECMC_EINVAL, "model needs K >= 1");
  if (m.family == SPECMC_FAMILY_XRD) {  // model.cpp:99-105, :62-72
    if (m.n_refl < 1 || !m.refl_phase || !m.refl_mu || !m.refl_int)
      throw Error(SPECMC_EINVAL, "xrd model: phases count must equal K");
    std::vector<int> cnt(m.K, 0);
    for (int q = 0; q < m.n_refl; ++q) {
      const int ph = m.refl_phase[q];
      if (ph < 0 || ph >= m.K) throw Error(SPECMC_EINVAL, "xrd model: phases count must equal K");
      if (q > 0 && ph < m.refl_phase[q - 1]) throw Error(SPECMC_EINVAL, "xrd model: reflections must be grouped by phase");
      if (m.refl_int[q] < 0.0) throw Error(SPECMC_EINVAL, "negative reflection intensity");
      ++cnt[ph];
    }
    for (int b = 0; b < m.K; ++b)
      if (!cnt[b]) throw Error(SPECMC_EINVAL, "xrd phase has no reflections");
  }
  // the move kernel tracks faulty blocks in a 64-bit mask: K peaks, or K phases + the xrd background block
  if (m.family != SPECMC_FAMILY_OFFSET && m.K + (m.family == SPECMC_FAMILY_XRD ? 1 : 0) > 64)
    throw Error(SPECMC_EINVAL, "device path supports at most 64 blocks (K <= 64; xrd K <= 63)");
  if (m.d != model_dim(m)) throw Error(SPECMC_EINVAL, "model layout length mismatch");
  if (!m.prior_kind || !m.prior_a || !m.prior_b) throw Error(SPECMC_EINVAL, "model priors missing");
  for (int i = 0; i < m.d; ++i) {  // priors.cpp:9-20
    const double a = m.prior_a[i], b = m.prior_b[i];
    switch (m.prior_kind[i]) {
      case SPECMC_PRIOR_NORMAL:
        if (!(b > 0.0) || !std::isfinite(b) || !std::isfinite(a))
          throw Error(SPECMC_EINVAL, "normal prior needs finite mean and var > 0");
        break;
      case SPECMC_PRIOR_GAMMA:
        if (!(a > 0.0) || !(b > 0.0)) throw Error(SPECMC_EINVAL, "gamma prior needs shape > 0 and rate > 0");
        break;
      case SPECMC_PRIOR_UNIFORM:
        if (!(a < b)) throw Error(SPECMC_EINVAL, "uniform prior needs lo < hi");
        break;
      default: throw Error(SPECMC_EINVAL, "unknown prior kind");
    }
  }
  switch (m.noise) {  // model.cpp:14-21
    case SPECMC_NOISE_GAUSSIAN:
      if (!(m.noise_sigma > 0.0)) throw Error(SPECMC_EINVAL, "gaussian noise needs sigma > 0");
      break;
    case SPECMC_NOISE_XPS_HETERO:
      if (m.s0 < 0.0 || m.s1 < 0.0 || m.s2 < 0.0 || (m.s0 == 0.0 && m.s1 == 0.0 && m.s2 == 0.0))
        throw Error(SPECMC_EINVAL, "hetero noise needs sigma0,1,2 >= 0, not all zero");
      break;
    case SPECMC_NOISE_POISSON:
    case SPECMC_NOISE_GAUSS_APPROX: break;
    default: throw Error(SPECMC_EINVAL, "unknown noise kind");
  }
}

void validate_spectrum(const double* xs, const double* ys, int64_t n, bool nonneg) {  // spectrum.cpp:12-23
  if (!xs || !ys) throw Error(SPECMC_EINVAL, "spectrum: null data");
  if (n < 2) throw Error(SPECMC_EINVAL, "spectrum: needs at least 2 points");
  for (int64_t i = 0; i < n; ++i) {
    if (!std::isfinite(xs[i]) || !std::isfinite(ys[i]))
      throw Error(SPECMC_EINVAL, "spectrum: non-finite value at row " + std::to_string(i));
    if (i > 0 && !(xs[i] > xs[i - 1]))
      throw Error(SPECMC_EINVAL, "spectrum: xs not strictly increasing at row " + std::to_string(i));
    if (nonneg && ys[i] < 0.0) throw Error(SPECMC_EINVAL, "spectrum: negative intensity at row " + std::to_string(i));
  }
}

// location parameters (peak centres mu_k) are shifted by x_shift on the device
// populations above this use the grid-level (multi-CTA) tempering kernels
// grid-level tempering above 2^15 particles, slices of >= 4096: at T = 65536 (C2)
// 16 CTAs per run instead of one cut the level's tempering time (C2 step
// 1.512 -> 1.490 s); small populations keep the single-CTA kernel
constexpr size_t kGridTemperT = (size_t)1 << 15;
constexpr size_t kMinSliceLen = 4096;
// tuning overrides (experiments): SPECMC_GRID_T = population above which the
// tempering runs grid-level, SPECMC_SLICE = minimum slice length
size_t grid_temper_t() {
  static const size_t v = std::getenv("SPECMC_GRID_T") ? std::strtoull(std::getenv("SPECMC_GRID_T"), nullptr, 10)
                                                        : kGridTemperT;
  return v;
}
size_t min_slice_len() {
  static const size_t v =
      std::getenv("SPECMC_SLICE") ? std::strtoull(std::getenv("SPECMC_SLICE"), nullptr, 10) : kMinSliceLen;
  return v;
}

bool is_location(int family, int K, int i) {
  if (family == SPECMC_FAMILY_GM) return i % 3 == 1;
  if (family == SPECMC_FAMILY_XPS) return i < 4 * K && i % 4 == 1;
  return false;
}

uint64_t mix64(uint64_t z) {  // rng.hpp:11-14
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// ----------------------------------------------------------- device memory
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  explicit DevBuf(size_t b) : bytes(b) {
    if (b) cuda_check(cudaMalloc(&p, b), "cudaMalloc");
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) {
    o.p = nullptr;
    o.bytes = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    std::swap(p, o.p);
    std::swap(bytes, o.bytes);
    return *this;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// bump allocator over one cudaMalloc (256-byte aligned slices)
// Process-wide cache of session arenas.  Large cudaMalloc/cudaFree pairs cost
// up to ~1 s per call at C2 sizes (cudaFree synchronises and unmaps), and
// stream-ordered pool memory measured ~16% slower in the move kernel than
// cudaMalloc'd memory, so freed arenas are kept (per device, up to kMaxCached
// bytes) and handed to later sessions of similar size.
struct ArenaCache {
  static constexpr size_t kMaxCached = size_t(16) << 30;
  std::mutex mu;
  std::multimap<size_t, std::pair<int, void*>> free_;  // bytes -> (device, ptr)
  size_t cached = 0;
  void* get(int dev, size_t b, size_t& got) {
    {
      std::lock_guard<std::mutex> lk(mu);
      for (auto it = free_.lower_bound(b); it != free_.end() && it->first <= 2 * b + (size_t(64) << 20); ++it)
        if (it->second.first == dev) {
          void* p = it->second.second;
          got = it->first;
          cached -= it->first;
          free_.erase(it);
          return p;
        }
    }
    void* p = nullptr;
    if (cudaMalloc(&p, b) != cudaSuccess) {  // retry once with the cache released
      cudaGetLastError();
      release(dev);
      cuda_check(cudaMalloc(&p, b), "cudaMalloc");
    }
    got = b;
    return p;
  }
  void put(int dev, void* p, size_t b) {
    std::lock_guard<std::mutex> lk(mu);
    free_.emplace(b, std::make_pair(dev, p));
    cached += b;
    while (cached > kMaxCached && !free_.empty()) {  // drop the smallest
      auto it = free_.begin();
      free_on(it->second.first, it->second.second);
      cached -= it->first;
      free_.erase(it);
    }
  }
  void release(int dev) {
    std::lock_guard<std::mutex> lk(mu);
    for (auto it = free_.begin(); it != free_.end();)
      if (it->second.first == dev) {
        free_on(dev, it->second.second);
        cached -= it->first;
        it = free_.erase(it);
      } else {
        ++it;
      }
  }
  static void free_on(int dev, void* p) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(dev);
    cudaFree(p);
    cudaSetDevice(cur);
  }
};
ArenaCache& arena_cache() {
  static ArenaCache* c = new ArenaCache();  // never destroyed: the CUDA context may be gone at exit
  return *c;
}

// Process-wide cache of pinned host staging buffers (results of run_batch are
// copied D2H into pinned memory while the remaining runs still step; pinning
// 100+ MB costs tens of ms, so buffers are kept for later calls).
struct PinnedCache {
  // keep up to a quarter of the host's memory pinned between calls (at most
  // 32 GB): re-pinning a large result staging buffer per call costs seconds
  // (C4: 12.9 GB, cudaHostAlloc + cudaFreeHost ~3-4 s per call)
  const size_t kMaxCached = [] {
    const long pages = sysconf(_SC_PHYS_PAGES), psz = sysconf(_SC_PAGE_SIZE);
    const size_t quarter = pages > 0 && psz > 0 ? (size_t)pages * (size_t)psz / 4 : (size_t(4) << 30);
    return std::min(quarter, size_t(32) << 30);
  }();
  std::mutex mu;
  std::multimap<size_t, void*> free_;
  size_t cached = 0;
  void* get(size_t b, size_t& got) {
    b = std::max<size_t>(b, size_t(64) << 10);  // small buffers share a 64 KB size class
    const size_t cap = b <= (size_t(64) << 10) ? b : 2 * b + (size_t(64) << 20);
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = free_.lower_bound(b);
      if (it != free_.end() && it->first <= cap) {
        void* p = it->second;
        got = it->first;
        cached -= it->first;
        free_.erase(it);
        return p;
      }
    }
    void* p = nullptr;
    cuda_check(cudaHostAlloc(&p, b, cudaHostAllocPortable), "cudaHostAlloc");
    got = b;
    return p;
  }
  void put(void* p, size_t b) {
    std::lock_guard<std::mutex> lk(mu);
    free_.emplace(b, p);
    cached += b;
    while (cached > kMaxCached && !free_.empty()) {
      auto it = free_.begin();
      cudaFreeHost(it->second);
      cached -= it->first;
      free_.erase(it);
    }
  }
};
PinnedCache& pinned_cache() {
  static PinnedCache* c = new PinnedCache();
  return *c;
}

// copy of a large block on up to 4 host threads (fresh result arrays fault
// their pages in; one thread does ~5 GB/s)
void par_memcpy(void* dst, const void* src, size_t n) {
  constexpr size_t kChunk = size_t(8) << 20;
  const int nt = (int)std::min<size_t>(4, (n + kChunk - 1) / kChunk);
  if (nt <= 1) {
    std::memcpy(dst, src, n);
    return;
  }
  std::vector<std::thread> th;
  const size_t per = (n + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    const size_t a = std::min(n, per * t), b = std::min(n, per * (t + 1));
    th.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a); });
  }
  for (auto& x : th) x.join();
}

// Row pitch (elements) of the [d][n] device arrays: a multiple of 32 doubles
// with pitch / 32 odd (GroupDesc::tp, device.cuh)
inline size_t row_pitch(size_t n) {
  size_t p = (n + 31) & ~(size_t)31;
  if (((p / 32) & 1) == 0) p += 32;
  return p;
}

// One device allocation per class of runs, carved by take().
struct Arena {
  void* p = nullptr;
  size_t bytes = 0, off = 0;
  int dev = 0;
  cudaStream_t st = nullptr;
  static size_t al(size_t b) { return (b + 255) & ~(size_t)255; }
  void reserve(size_t b, int device, cudaStream_t s) {
    dev = device;
    st = s;
    if (b) p = arena_cache().get(dev, b, bytes);
    if (const char* poison = std::getenv("SPECMC_POISON"))  // debug: fill with a byte pattern (uninitialised-read hunt)
      if (p) cuda_check(cudaMemsetAsync(p, std::atoi(poison), bytes, st), "poison");
  }
  Arena() = default;
  Arena(const Arena&) = delete;
  ~Arena() {
    if (!p) return;
    static const bool trace = std::getenv("SPECMC_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    if (cudaStreamSynchronize(st) == cudaSuccess)
      arena_cache().put(dev, p, bytes);
    else
      cudaFree(p);  // the context is in an error state: do not recycle
    if (trace)
      std::fprintf(stderr, "[specmc]   ~Arena %.1f MB %.4f s (cached %.1f MB)\n", bytes / 1e6,
                   std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(),
                   arena_cache().cached / 1e6);
  }
  template <typename T>
  T* take(size_t count) {
    const size_t b = al(sizeof(T) * std::max<size_t>(count, 1));
    if (off + b > bytes) throw Error(SPECMC_ECUDA, "arena overflow");
    T* q = reinterpret_cast<T*>(static_cast<char*>(p) + off);
    off += b;
    return q;
  }
};

// --------------------------------------------------------- host-side prep
struct PreparedSpectrum {
  std::vector<float> x;
  std::vector<float> c;  // (c_k, h_{k+1}) pairs
  std::vector<float> y;  // (y_k, 1/s_k) pairs
  double x_shift = 0.0;
  float x0s = 0.f, inv_range = 0.f, range = 0.f, x1s = 0.f;
  bool uniform = false;  // xps on a uniform grid (GroupDesc::sh_uniform)
  float y_last = 0.f, s_last = 1.f;
  double e_a0 = 0.0, e_a1 = 0.0;
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, q = 0.5f;
  int nz = NZ_GAUSS;
};

// Lane-transposed spectrum arrays for one launch shape (see device.cuh) and the
// noise constants of E = e_a0 + e_a1 * sum_k l_k (kernels.cu noise_term).
// device noise model of a model description (NoiseDev, device.cuh); the move
// kernel is instantiated per model
int dev_noise(const specmc_model_desc& m) {
  switch (m.noise) {
    case SPECMC_NOISE_GAUSSIAN: return NZ_GAUSS;
    case SPECMC_NOISE_POISSON: return NZ_POISSON;
    case SPECMC_NOISE_XPS_HETERO:
      if (m.s1 == 0.0 && m.s2 == 0.0) return NZ_HPROP;
      return m.s1 == 0.0 ? NZ_HLIN : NZ_HETERO;
    default: return NZ_HPROP;  // GaussianApproxPoisson: var = f
  }
}

struct RunSpec;
// MUFU lane-ops per point slot of one block shape evaluation (move kernel):
// gm ex2, xps ex2 + rcp, Lorentzian rcp, xrd (ex2 + rcp) per reflection
double mufu_per_shape(int kfam, const RunSpec& R);
// ... and of one evaluation's noise terms per point slot
// (paired hetero models: two points share one rcp and one lg2)
double mufu_per_noise(int nz, int /*ppl*/) { return nz == NZ_GAUSS ? 0.0 : 1.0; }

PreparedSpectrum prepare_spectrum(const specmc_model_desc& m, const double* xs, const double* ys, int64_t N,
                                  const Shape& s, double x_shift) {
  PreparedSpectrum ps;
  const int L = 32 * s.W;
  const size_t npt = (size_t)s.PPL * L;
  ps.x.assign(npt, 0.f);
  ps.c.assign(2 * npt, 0.f);
  ps.y.assign(2 * npt, 0.f);
  ps.x_shift = x_shift;
  const double range = xs[N - 1] - xs[0];
  ps.range = (float)range;
  ps.inv_range = (float)(1.0 / range);
  ps.x0s = (float)(xs[0] - x_shift);
  ps.x1s = (float)(xs[N - 1] - x_shift);
  // noise
  std::vector<double> inv_s(N, 1.0);
  double a0 = 0.0;
  switch (m.noise) {
    case SPECMC_NOISE_GAUSSIAN: {
      const double s2 = m.noise_sigma * m.noise_sigma;
      ps.nz = NZ_GAUSS;
      ps.e_a0 = 0.5 * std::log(2.0 * M_PI * s2);
      ps.e_a1 = 1.0 / (2.0 * s2 * (double)N);
      break;
    }
    case SPECMC_NOISE_POISSON: {
      ps.nz = NZ_POISSON;
      for (int64_t i = 0; i < N; ++i)
        if (ys[i] > 0.0) {
          inv_s[i] = 1.0 / ys[i];
          a0 += ys[i] - ys[i] * std::log(ys[i]);
        }
      ps.e_a0 = a0 / (double)N;
      ps.e_a1 = 1.0 / (double)N;
      break;
    }
    default: {
      double h0 = 1.0, h1 = 0.0, h2 = 0.0, q = 0.5;
      if (m.noise == SPECMC_NOISE_XPS_HETERO) {
        h0 = m.s0 * m.s0;
        h1 = m.s1 * m.s1;
        h2 = m.s2 * m.s2;
        q = m.paper_literal ? 1.0 : 0.5;
      }
      // device terms are lg2(var/s) + q' r^2/var with q' = q / (ln2/2); with
      // s1 = s2 = 0 (var = s0^2 f) the s0^2 factor moves into 1/s and q'
      const bool prop = h1 == 0.0 && h2 == 0.0;
      ps.nz = prop ? NZ_HPROP : (h1 == 0.0 ? NZ_HLIN : NZ_HETERO);
      if (ps.nz != dev_noise(m)) throw Error(SPECMC_ERUNTIME, "internal: noise model code mismatch");
      ps.a0 = (float)h0;
      ps.a1 = (float)h1;
      ps.a2 = (float)h2;
      ps.q = (float)(q / (0.5 * M_LN2) / (prop ? h0 : 1.0));
      for (int64_t i = 0; i < N; ++i) {
        const double y = std::fabs(ys[i]);
        double sc = h0 * y + h1 * y * y + h2;
        if (!(sc > 0.0)) sc = 1.0;
        inv_s[i] = (prop ? h0 : 1.0) / sc;
        a0 += 0.5 * std::log(2.0 * M_PI * sc);
      }
      ps.e_a0 = a0 / (double)N;
      ps.e_a1 = 0.5 * M_LN2 / (double)N;
      break;
    }
  }
  // xps on a uniform ascending grid: constant trapezoid weights (chain.cuh
  // eval_shirley_nz).  Uniform = every spacing within 2e-7 (relative) of the
  // mean, below the fp32 rounding of the per-point weights it replaces.
  if (m.family == SPECMC_FAMILY_XPS && N >= 3 && range > 0.0) {
    const double dx = range / (double)(N - 1);
    bool uni = true;
    for (int64_t i = 1; i < N && uni; ++i) uni = std::fabs((xs[i] - xs[i - 1]) - dx) <= 2e-7 * dx;
    ps.uniform = uni;
  }
  // noise models whose terms the kernel evaluates two points at a time
  // (chain.cuh nz_pairs): (y_2p, y_2p+1) per pair, 4 B per point.  Their lg2
  // terms are not centred by 1/s_k: e_a0 takes sum_k ln(1/s_k) / 2N instead
  const bool paired = ps.nz == NZ_HETERO || ps.nz == NZ_HLIN || ps.nz == NZ_HPROP;
  if (paired) {
    double ls = 0.0;
    for (int64_t i = 0; i < N; ++i) ls += std::log(inv_s[i]);
    ps.e_a0 += 0.5 * ls / (double)N;
  }
  // padding points replicate the last real point (the kernel removes their
  // terms by lane count); uniform xps: points 0..N-2 first, point N-1 in the
  // last slot, padding between at x = 1e30 (peak signal exactly 0)
  auto src = [&](size_t p) -> int64_t {  // spectrum point stored at slot p
    if (ps.uniform) return p + 1 < (size_t)N ? (int64_t)p : N - 1;
    return p < (size_t)N ? (int64_t)p : N - 1;
  };
  // pair-slot layout (chain.cuh): lane point k of lane l sits in slot
  // k mod PH, component k / PH; x float2, weights float4 (c_a, c_b, -h_a, -h_b),
  // y float2 (-y_a, -y_b) or, for poisson, float4 (y_a, y_b, 1/s_a, 1/s_b)
  const int PH = s.PPL / 2;
  const bool y4 = ps.nz != NZ_POISSON;
  for (size_t p = 0; p < npt; ++p) {
    const int64_t q = src(p);
    const bool real = ps.uniform ? (p + 1 < (size_t)N || p + 1 == npt) : p < (size_t)N;
    const int lane = (int)(p / s.PPL), k = (int)(p % s.PPL);
    const int slot = k % PH, h = k / PH;
    const size_t sidx = (size_t)slot * L + lane;
    const double hk = q > 0 ? 0.5 * (xs[q] - xs[q - 1]) : 0.0;
    const double hk1 = q + 1 < N ? 0.5 * (xs[q + 1] - xs[q]) : 0.0;
    ps.x[2 * sidx + h] = (ps.uniform && !real) ? 1e30f : (float)(xs[q] - x_shift);
    ps.c[4 * sidx + h] = real ? (float)(hk + hk1) : 0.f;
    ps.c[4 * sidx + 2 + h] = real ? (float)-hk1 : 0.f;  // negated: folded into the kernel's FFMA2
    if (y4) {  // negated: the kernel forms f - y with one FADD2 (only (f - y)^2 enters)
      ps.y[2 * sidx + h] = (float)-ys[q];
    } else {
      ps.y[4 * sidx + h] = (float)ys[q];
      ps.y[4 * sidx + 2 + h] = (float)inv_s[q];
    }
  }
  ps.y_last = (float)ys[N - 1];
  ps.s_last = paired ? 1.f : (float)inv_s[N - 1];
  return ps;
}

// shared-memory spectrum layout of a class (launch.h kLay*): the trapezoid
// weights only when an xps spectrum of the class is on a non-uniform grid, y
// at 4 B/point for every noise model but poisson
template <class M>
int spectrum_layout(int family, int noise, const M& prep) {
  bool weights = false;
  for (const auto& kv : prep) weights = weights || (family == SPECMC_FAMILY_XPS && !kv.second.uniform);
  return (weights ? kLayWeights : 0) | (noise != NZ_POISSON ? kLayY4 : 0);
}

double pick_shift(const specmc_model_desc& m, const double* xs, int64_t N) {
  if (m.family != SPECMC_FAMILY_GM && m.family != SPECMC_FAMILY_XPS) return 0.0;
  for (int i = 0; i < m.d; ++i)
    if (is_location(m.family, m.K, i) && m.prior_kind[i] == SPECMC_PRIOR_GAMMA) return 0.0;  // not translation-safe
  return 0.5 * (xs[0] + xs[N - 1]);
}

// fewer chains per CTA when the launch's spectrum layout leaves no room for
// the default count's caches (W = 8 on a non-uniform grid: launch.h)
void fit_units(Shape& s, int dmax) {
  while (s.U > 1 && chain_smem_bytes(s, dmax) > kChainSmemMax) --s.U;
}

// ------------------------------------------------------------------ batch
struct RunSpec {
  specmc_model_desc m;
  std::vector<int32_t> pk;
  std::vector<double> pa, pb;  // shifted
  std::vector<float> refl;     // xrd: (mu_ref, rel_intensity) pairs grouped by phase
  std::vector<int> refl_off;   // xrd: K + 1 phase offsets
  int spectrum;
  specmc_smc_config cfg;
  double x_shift;
  int64_t N;
  // particle sharding (shard.cu): shard `shard` of `nshards` holds T_loc0 of the
  // T level-0 particles, global ids [pbase, pbase + T_loc0)
  int shard = 0, nshards = 1;
  int64_t T_loc0 = 0, pbase = 0;
  int problem = 0;  // index of the run in the caller's batch
};

// kernel family of a run: the model family, or kFamXpsLorentz for an xps
// model whose every eta prior is Uniform(lo >= 0, hi <= 1e-7) -- the Lorentzian
// basis of SURVEY.md Appendix A (prior.eta = uniform(0, 1e-9), config.cpp:204-222)
int kernel_family(const RunSpec& R) {
  const auto& m = R.m;
  if (m.family != SPECMC_FAMILY_XPS || m.K < 1) return m.family;
  for (int k = 0; k < m.K; ++k) {
    const int i = 4 * k + 3;
    if (R.pk[i] != SPECMC_PRIOR_UNIFORM || !(R.pa[i] >= 0.0) || !(R.pb[i] <= 1e-7)) return m.family;
  }
  return kFamXpsLorentz;
}

double mufu_per_shape(int kfam, const RunSpec& R) {
  switch (kfam) {
    case SPECMC_FAMILY_GM: return 1.0;
    case SPECMC_FAMILY_XPS: return 2.0;
    case kFamXpsLorentz: return 1.0;
    case SPECMC_FAMILY_XRD: return R.m.K > 0 ? 2.0 * (double)(R.refl.size() / 2) / (double)R.m.K : 2.0;
    default: return 0.0;
  }
}

using SpecKey = std::tuple<int, double, int, int, double, double, double, double, int>;
SpecKey spec_key(const RunSpec& R) {
  const auto& m = R.m;
  return SpecKey(R.spectrum, R.x_shift, m.family, m.noise, m.s0, m.s1, m.s2, m.noise_sigma, m.paper_literal);
}

struct Device {
  int ordinal;
  cudaStream_t stream = nullptr;
  explicit Device(int o) : ordinal(o) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
      throw Error(SPECMC_ECUDA, "no CUDA device available (the B200 path has no CPU fallback)");
    if (o < 0 || o >= count) throw Error(SPECMC_ECUDA, "invalid CUDA device ordinal " + std::to_string(o));
    cuda_check(cudaSetDevice(o), "cudaSetDevice");
    cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
  }
  ~Device() {
    if (stream) cudaStreamDestroy(stream);
  }
  void sync() { cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize"); }
};

template <typename T>
void h2d(T* dst, const T* src, size_t n, cudaStream_t st) {
  if (n) cuda_check(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, st), "H2D");
}
template <typename T>
void d2h(T* dst, const T* src, size_t n, cudaStream_t st) {
  if (n) cuda_check(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost, st), "D2H");
}

struct Timer {
  cudaEvent_t a = nullptr, b = nullptr;
  Timer() {
    cuda_check(cudaEventCreate(&a), "event");
    cuda_check(cudaEventCreate(&b), "event");
  }
  ~Timer() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
  float ms() {
    float t = 0.f;
    cuda_check(cudaEventElapsedTime(&t, a, b), "cudaEventElapsedTime");
    return t;
  }
};

// One homogeneous class of problems (same family, same launch shape, same
// device): device buffers, descriptors and the lock-step level loop.
struct ClassRun {
  std::vector<int> idx;  // indices into the session's runs
  Shape shape{};
  int dmax = 1, Tmax = 0, family = 0, noise = 0, G = 0;
  int kfam = 0;                     // kernel family of the move kernel (kernel_family)
  std::vector<double> mufu_shape;   // per group: MUFU lane-ops per slot of one shape evaluation
  Arena ar;
  GroupDesc* d_gds = nullptr;
  GroupState* d_st = nullptr;
  int *d_list = nullptr, *d_prefix = nullptr, *d_list_all = nullptr, *d_prefix_all = nullptr;
  int *d_list_small = nullptr, *d_list_big = nullptr;
  int max_slices = 0;
  Exchange* xch = nullptr;  // non-null: the groups are shards of particle-sharded runs
  bool init_only = false;   // stop after init_ensemble (parity unit specmc_init_ensemble)
  int* d_xlist = nullptr;   // sharded: every run's shards, run-major (idx order), for the exchanges
  int nshards = 1;
  std::vector<GroupDesc> gds;
  std::vector<int64_t> runs_T0;  // level-0 particles per group
  std::vector<double*> out_shift;  // per group [d] device: posterior = theta + shift
  std::vector<int> order;
  GroupState* h_st = nullptr;
  int* h_list = nullptr;
  size_t h_st_bytes = 0, h_list_bytes = 0;
  double device_seconds = 0.0;
  // early staging (run_batch): as soon as a run reaches beta = 1 its posterior,
  // energies and diagnostics go D2H into pinned memory on a copy stream while
  // the other runs of the class still step; fetch() then only copies host-side
  bool stage_early = false;
  cudaStream_t cst = nullptr;
  cudaEvent_t cev = nullptr;
  double* stage = nullptr;
  size_t stage_bytes = 0;
  std::vector<size_t> stage_off;  // per group: [diag (4 max_levels) | posterior (d T) | energies (T)]
  std::vector<char> staged;       // 1: copy enqueued, 2: copied into hres
  std::vector<cudaEvent_t> gev;   // per group: its staging copy is done
  struct HostRes {
    double* post = nullptr;
    double* ener = nullptr;
    std::vector<double> diag;
  };
  std::vector<HostRes> hres;  // results copied out of the staging buffer (owned until fetch)

  ClassRun() = default;
  ClassRun(const ClassRun&) = delete;
  ~ClassRun() {
    static const bool trace = std::getenv("SPECMC_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    auto tick = [&](const char* what) {
      if (trace)
        std::fprintf(stderr, "[specmc]   ~ClassRun %s %.4f s\n", what,
                     std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    };
    if (cst) {
      const bool ok = cudaStreamSynchronize(cst) == cudaSuccess;
      tick("sync");
      if (stage) {
        if (ok)
          pinned_cache().put(stage, stage_bytes);
        else
          cudaFreeHost(stage);
      }
      tick("pinned");
      cudaStreamDestroy(cst);
      tick("stream");
    }
    if (cev) cudaEventDestroy(cev);
    for (cudaEvent_t e : gev) cudaEventDestroy(e);
    for (auto& r : hres) {
      std::free(r.post);
      std::free(r.ener);
    }
    if (h_st) pinned_cache().put(h_st, h_st_bytes);
    if (h_list) pinned_cache().put(h_list, h_list_bytes);
    tick("host");
  }

  void init_staging() {
    if (!stage_early || xch || init_only) {
      stage_early = false;
      return;
    }
    stage_off.assign(G + 1, 0);
    for (int gi = 0; gi < G; ++gi) {
      const size_t T = (size_t)runs_T0[gi], d = (size_t)gds[gi].d;
      stage_off[gi + 1] = stage_off[gi] + 4 * (size_t)gds[gi].max_levels + d * T + T;
    }
    stage = static_cast<double*>(pinned_cache().get(stage_off[G] * sizeof(double), stage_bytes));
    staged.assign(G, 0);
    cuda_check(cudaStreamCreateWithFlags(&cst, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaEventCreateWithFlags(&cev, cudaEventDisableTiming), "cudaEventCreate");
    gev.assign(G, nullptr);
    for (auto& e : gev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    hres.resize(G);
  }

  // host side of the staging: copy finished runs out of pinned memory into
  // their result arrays -- between level launches (wait = false: only copies
  // that are complete; the host would otherwise idle in the level sync) and in
  // fetch (wait = true)
  void drain(bool wait) {
    for (int gi = 0; gi < G; ++gi) {
      if (staged[gi] != 1) continue;
      const GroupState& s = h_st[gi];
      if (s.error != GE_NONE) {
        staged[gi] = 2;
        continue;
      }
      if (wait)
        cuda_check(cudaEventSynchronize(gev[gi]), "cudaEventSynchronize");
      else if (cudaEventQuery(gev[gi]) != cudaSuccess)
        continue;
      const size_t T = (size_t)s.T_loc, d = (size_t)gds[gi].d, L4 = 4 * (size_t)gds[gi].max_levels;
      const double* h = stage + stage_off[gi];
      HostRes& r = hres[gi];
      r.diag.assign(h, h + (size_t)s.level * 4);
      r.post = static_cast<double*>(std::malloc(sizeof(double) * std::max<size_t>(d * T, 1)));
      par_memcpy(r.post, h + L4, d * T * sizeof(double));
      r.ener = static_cast<double*>(std::malloc(sizeof(double) * std::max<size_t>(T, 1)));
      std::memcpy(r.ener, h + L4 + d * T, T * sizeof(double));
      staged[gi] = 2;
    }
  }

  // enqueue the result copy of a run that just finished (h_st is current)
  void stage_group(int gi, cudaStream_t st) {
    const GroupState& s = h_st[gi];
    staged[gi] = 1;
    if (s.error != GE_NONE) return;
    const size_t T = (size_t)s.T_loc, d = (size_t)gds[gi].d;
    double* h = stage + stage_off[gi];
    cuda_check(cudaEventRecord(cev, st), "event");
    cuda_check(cudaStreamWaitEvent(cst, cev, 0), "cudaStreamWaitEvent");
    double* pout = gds[gi].theta[s.cur ^ 1];  // idle once the run is done
    cuda_check(launch_posterior_out(gds[gi].theta[s.cur], gds[gi].tp, (int)d, (int)T, out_shift[gi], pout, cst),
               "k_posterior_out");
    d2h(h, gds[gi].diag, (size_t)s.level * 4, cst);
    d2h(h + 4 * (size_t)gds[gi].max_levels, pout, d * T, cst);
    d2h(h + 4 * (size_t)gds[gi].max_levels + d * T, gds[gi].E[s.cur], T, cst);
    cuda_check(cudaEventRecord(gev[gi], cst), "event");
  }

  // allocation + H2D of spectra, priors and descriptors
  void prepare(Device& dev, const std::vector<RunSpec>& runs, const std::vector<specmc_spectrum>& spectra) {
    G = (int)idx.size();
    family = runs[idx[0]].m.family;
    kfam = kernel_family(runs[idx[0]]);
    noise = dev_noise(runs[idx[0]].m);
    int64_t Nmax = 0;
    for (int r : idx) {
      Nmax = std::max(Nmax, runs[r].N);
      dmax = std::max(dmax, runs[r].m.d);
      Tmax = std::max<int>(Tmax, (int)runs[r].cfg.T);
    }
    shape = pick_shape(Nmax, dmax);
    if ((int64_t)32 * shape.W * shape.PPL < Nmax)
      throw Error(SPECMC_EINVAL, "spectrum has more points than the device path supports (8192)");

    // one prepared copy per (spectrum, shift, noise parameters): the inverse
    // noise scales and the centring constants depend on the noise model
    std::map<SpecKey, PreparedSpectrum> prep;
    for (int r : idx) {
      const auto key = spec_key(runs[r]);
      if (!prep.count(key)) {
        const auto& sp = spectra[runs[r].spectrum];
        prep.emplace(key, prepare_spectrum(runs[r].m, sp.xs, sp.ys, sp.n, shape, runs[r].x_shift));
      }
    }
    shape.lay = spectrum_layout(family, noise, prep);
    fit_units(shape, dmax);
    {  // few chains per level (a shard of a particle-sharded run, small populations):
       // fewer chains per CTA, so that the chains spread over every SM
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev.ordinal);
      double chains = 0.0;
      for (int r : idx) chains += (double)(runs[r].cfg.T / runs[r].cfg.n) / (double)runs[r].nshards;
      while (shape.U > 1 && shape.U % 2 == 0 && chains / (shape.U / 2) <= 2.0 * sms && chains / shape.U < sms)
        shape.U /= 2;
    }
    if (chain_smem_bytes(shape, dmax) > kChainSmemMax)  // (with the launch's spectrum layout)
      throw Error(SPECMC_EINVAL, "model too large for the device path (shared memory)");
    // module load of this class's kernels happens here, outside the timed level loop
    cuda_check(prime_level_kernels(kfam, noise, shape, dmax), "loading the level kernels");
    const size_t npt = (size_t)shape.PPL * 32 * shape.W;
    size_t bytes = Arena::al(sizeof(GroupDesc) * G) + Arena::al(sizeof(GroupState) * G) + 7 * Arena::al(4 * (G + 1));
    bytes += prep.size() * (Arena::al(npt * 4) + 2 * Arena::al(npt * 8));
    for (int r : idx) {
      const auto& R = runs[r];
      const size_t T = R.cfg.T, d = R.m.d, S = T / R.cfg.n;
      const size_t tp = row_pitch(T), sp = row_pitch(S);
      bytes += 3 * Arena::al(d * 8) + Arena::al(d * 4);
      bytes += 2 * Arena::al(d * tp * 8) + 2 * Arena::al(T * 8);
      bytes += Arena::al(S * 4) + Arena::al(d * sp * 4) + Arena::al(d * sp * 8);
      bytes += Arena::al(T * 8) + Arena::al(kHist * (1 + 2 * d) * 8);
      bytes += Arena::al((size_t)R.cfg.max_levels * 4 * 8);
      bytes += Arena::al(2 * d * 8) + Arena::al(d * 8);                         // stat_acc, out_shift
      bytes += Arena::al(2 * kEssSlots * 8) + Arena::al(2 * 8 * (size_t)R.nshards);  // xbuf, xgat
      bytes += Arena::al(R.refl.size() * 4 + 8) + Arena::al(R.refl_off.size() * 4 + 4);  // xrd reflections
      if (T > grid_temper_t() || xch) bytes += Arena::al(sizeof(TemperScratch));  // grid tempering
    }
    ar.reserve(bytes, dev.ordinal, dev.stream);
    d_gds = ar.take<GroupDesc>(G);
    d_st = ar.take<GroupState>(G);
    d_list = ar.take<int>(G + 1);
    d_prefix = ar.take<int>(G + 1);
    d_list_all = ar.take<int>(G + 1);
    d_prefix_all = ar.take<int>(G + 1);
    d_list_small = ar.take<int>(G + 1);
    d_list_big = ar.take<int>(G + 1);
    cudaStream_t st = dev.stream;
    if (xch) {  // idx is run-major, shard order: the exchange list is the identity
      nshards = runs[idx[0]].nshards;
      std::vector<int> xl(G);
      std::iota(xl.begin(), xl.end(), 0);
      d_xlist = ar.take<int>(G);
      h2d(d_xlist, xl.data(), G, st);
    }

    std::map<SpecKey, std::tuple<float*, float2*, float2*>> dspec;
    for (auto& kv : prep) {
      float* x = ar.take<float>(npt);
      float2* c = ar.take<float2>(npt);
      float2* y = ar.take<float2>(npt);
      h2d(x, kv.second.x.data(), npt, st);
      h2d(reinterpret_cast<float*>(c), kv.second.c.data(), 2 * npt, st);
      h2d(reinterpret_cast<float*>(y), kv.second.y.data(), 2 * npt, st);
      dspec[kv.first] = std::make_tuple(x, c, y);
    }
    gds.resize(G);
    runs_T0.resize(G);
    mufu_shape.resize(G);
    for (int gi = 0; gi < G; ++gi) mufu_shape[gi] = mufu_per_shape(kfam, runs[idx[gi]]);
    out_shift.resize(G);
    for (int gi = 0; gi < G; ++gi) {
      const RunSpec& R = runs[idx[gi]];
      runs_T0[gi] = R.nshards > 1 || xch ? R.T_loc0 : (int64_t)R.cfg.T;
      const auto key = spec_key(R);
      const PreparedSpectrum& ps = prep.at(key);
      GroupDesc& g = gds[gi];
      std::memset(&g, 0, sizeof(g));
      g.family = R.m.family;
      g.K = R.m.K;
      g.d = R.m.d;
      g.noise = ps.nz;
      g.T = (int)R.cfg.T;
      g.n = R.cfg.n;
      g.S = (int)(R.cfg.T / R.cfg.n);
      g.max_levels = R.cfg.max_levels;
      g.ess_target = R.cfg.ess_target;
      g.n_data = (double)R.N;
      const uint64_t k = mix64(R.cfg.seed);
      g.key0 = (uint32_t)k;
      g.key1 = (uint32_t)(k >> 32);
      g.chain_base = 0;
      g.N = (int)R.N;
      g.e_a0 = ps.e_a0;
      g.e_a1 = ps.e_a1;
      g.nz_a0 = ps.a0;
      g.nz_a1 = ps.a1;
      g.nz_a2 = ps.a2;
      g.nz_q = ps.q;
      g.x0s = ps.x0s;
      g.inv_range = ps.inv_range;
      g.range = ps.range;
      g.sh_uniform = ps.uniform ? 1 : 0;
      g.x1s = ps.x1s;
      g.y_last = ps.y_last;
      g.s_last = ps.s_last;
      auto t = dspec.at(key);
      g.spec_x = std::get<0>(t);
      g.spec_c = std::get<1>(t);
      g.spec_y = std::get<2>(t);
      const size_t T = R.cfg.T, d = R.m.d, S = g.S;
      int* pk = ar.take<int>(d);
      double* pa = ar.take<double>(d);
      double* pb = ar.take<double>(d);
      h2d(pk, R.pk.data(), d, st);
      h2d(pa, R.pa.data(), d, st);
      h2d(pb, R.pb.data(), d, st);
      g.pkind = pk;
      g.pa = pa;
      g.pb = pb;
      g.tp = (int)row_pitch(T);
      g.sp = (int)row_pitch(S);
      g.theta[0] = ar.take<double>(d * g.tp);
      g.theta[1] = ar.take<double>(d * g.tp);
      g.E[0] = ar.take<double>(T);
      g.E[1] = ar.take<double>(T);
      g.anc = ar.take<int>(S);
      g.ls0 = ar.take<double>(d);
      g.chain_acc = ar.take<int>(d * g.sp);
      g.chain_ls = ar.take<double>(d * g.sp);
      g.wbuf = ar.take<double>(T);
      g.hist = ar.take<double>(kHist * (1 + 2 * d));
      g.diag = ar.take<double>((size_t)R.cfg.max_levels * 4);
      g.st = d_st + gi;
      g.stat_acc = ar.take<double>(2 * d);
      {  // location shift undone on output (posterior = theta + shift)
        std::vector<double> sh(d, 0.0);
        for (size_t i = 0; i < d; ++i)
          if (is_location(R.m.family, R.m.K, (int)i)) sh[i] = R.x_shift;
        out_shift[gi] = ar.take<double>(d);
        h2d(out_shift[gi], sh.data(), d, st);
      }
      g.sharded = xch ? 1 : 0;
      g.shard = R.shard;
      g.nshards = R.nshards;
      g.pbase = (int)R.pbase;
      g.xbuf = ar.take<double>(2 * kEssSlots);
      g.xgat = ar.take<double>(2 * (size_t)R.nshards);
      if (!R.refl.empty()) {
        float2* rf = ar.take<float2>(R.refl.size() / 2);
        int* ro = ar.take<int>(R.refl_off.size());
        h2d(reinterpret_cast<float*>(rf), R.refl.data(), R.refl.size(), st);
        h2d(ro, R.refl_off.data(), R.refl_off.size(), st);
        g.refl = rf;
        g.refl_off = ro;
      }
      if (T > grid_temper_t() || xch) {  // grid-level tempering: slices of <= 512 x slice_len particles
        g.ts = ar.take<TemperScratch>(1);
        size_t sl = std::max<size_t>(min_slice_len(), (T + kMaxSlices - 1) / kMaxSlices);
        sl = (sl + 1023) & ~(size_t)1023;
        g.slice_len = (int)sl;
        g.nslices = (int)((T + sl - 1) / sl);
        max_slices = std::max(max_slices, g.nslices);
        cuda_check(cudaMemsetAsync(g.ts, 0, sizeof(TemperScratch), st), "memset");
      }
    }
    h2d(d_gds, gds.data(), G, st);
    // longest chains first (d descending) so the move grid drains in LPT order
    order.resize(G);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return gds[a].d > gds[b].d; });
    // pinned host mirrors from the process cache (cudaMallocHost/cudaFreeHost
    // per call measured up to 0.1 s / 0.7 s)
    h_st = static_cast<GroupState*>(pinned_cache().get(sizeof(GroupState) * G, h_st_bytes));
    h_list = static_cast<int*>(pinned_cache().get(sizeof(int) * 4 * (G + 1), h_list_bytes));
    init_staging();
    dev.sync();
  }

  // all_chains: size for every chain of the run (a shard may resolve up to S
  // of them; the kernels stop at the shard's own count)
  int build_list(const std::vector<int>& groups, bool energy, std::vector<int>& list, std::vector<int>& prefix,
                 bool all_chains = false) {
    list.clear();
    prefix.clear();
    int total = 0;
    for (int gi : groups) {
      list.push_back(gi);
      prefix.push_back(total);
      const int units = energy ? (int)runs_T0[gi] : (all_chains ? gds[gi].S : h_st[gi].S_loc);
      total += (units + shape.U - 1) / shape.U;
    }
    prefix.push_back(total);
    return total;
  }

  // init_ensemble + the level loop of smc_run (smc.cpp:186-211), all groups in lock-step
  void run(Device& dev) {
    cudaStream_t st = dev.stream;
    if (stage_early) staged.assign(G, 0);
    std::vector<GroupState> sts(G);
    for (int gi = 0; gi < G; ++gi) {
      GroupState& s = sts[gi];
      std::memset(&s, 0, sizeof(s));
      s.active = 1;
      s.T_loc = (int)runs_T0[gi];
      s.S_loc = gds[gi].S;
      s.chain_lo = 0;
      h_st[gi] = s;
    }
    Timer whole, mv;
    cuda_check(cudaEventRecord(whole.a, st), "event");
    h2d(d_st, sts.data(), G, st);
    std::vector<int> list, prefix;
    int total = build_list(order, true, list, prefix);
    std::memcpy(h_list, list.data(), sizeof(int) * G);
    std::memcpy(h_list + (G + 1), prefix.data(), sizeof(int) * (G + 1));
    h2d(d_list_all, h_list, G, st);
    h2d(d_prefix_all, h_list + (G + 1), G + 1, st);
    cuda_check(launch_init_draw(d_gds, d_list_all, G, Tmax, st), "k_init_draw");
    cuda_check(launch_energy(family, shape, dmax, d_gds, d_list_all, d_prefix_all, G, total, st), "k_chain<energy>");
    count_launch(2);
    std::vector<int> active = init_only ? std::vector<int>() : order;
    if (init_only) d2h(h_st, d_st, G, st);
    double move_ms = 0.0;
    int64_t move_launches = 0;
    if (!active.empty()) {
      // Every level is the same launch sequence over every group of the class
      // (the kernels skip finished or failed groups), so the host enqueues
      // levels ahead without waiting for them: after each level the small
      // GroupState array is copied into a pinned ring slot and an event
      // recorded; the host keeps up to kAhead levels in flight and retires /
      // stages runs as their levels' copies land.  Once every run is seen
      // inactive no further level is enqueued (at most kAhead levels of empty
      // launches run past the end).  Particle-sharded classes (xch) run the
      // sharded tempering and statistics with their exchanges (stream-ordered
      // NCCL collectives or device kernels) and size the move grid for all S
      // chains of each run (a shard resolves its own share after the
      // tempering; the other CTAs leave at once): no host round trip per level.
      constexpr int kAhead = 3, kRing = kAhead + 1;
      total = build_list(order, false, list, prefix, /*all_chains=*/xch != nullptr);  // static
      const int na = (int)list.size();
      dev.sync();  // h_list's pinned bytes of the init launches may still be in flight
      std::vector<int> small, big;
      for (int gi : order) (gds[gi].nslices > 0 || xch ? big : small).push_back(gi);
      std::memcpy(h_list, list.data(), sizeof(int) * na);
      std::memcpy(h_list + (G + 1), prefix.data(), sizeof(int) * (na + 1));
      std::copy(small.begin(), small.end(), h_list + 2 * (G + 1));
      std::copy(big.begin(), big.end(), h_list + 3 * (G + 1));
      h2d(d_list, h_list, na, st);
      h2d(d_prefix, h_list + (G + 1), na + 1, st);
      if (!small.empty()) h2d(d_list_small, h_list + 2 * (G + 1), small.size(), st);
      if (!big.empty()) h2d(d_list_big, h_list + 3 * (G + 1), big.size(), st);
      size_t ring_bytes = 0;
      GroupState* ring = static_cast<GroupState*>(pinned_cache().get(sizeof(GroupState) * G * kRing, ring_bytes));
      std::vector<cudaEvent_t> lev(kRing), ma(kRing), mb(kRing);
      for (int k = 0; k < kRing; ++k) {
        cuda_check(cudaEventCreateWithFlags(&lev[k], cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventCreate(&ma[k]), "cudaEventCreate");
        cuda_check(cudaEventCreate(&mb[k]), "cudaEventCreate");
      }
      std::vector<char> seen_done(G, 0);
      int n_live = (int)active.size();
      int64_t enq = 0, obs = 0;
      bool live_before = true;  // some run was active when the observed level started
      while (true) {
        while (n_live > 0 && enq - obs < kAhead) {  // enqueue one level
          const int k = (int)(enq % kRing);
          if (!small.empty()) {
            cuda_check(launch_temper(d_gds, d_list_small, (int)small.size(), st), "k_temper");
            count_launch(1);
          }
          if (!big.empty() && xch) {
            cuda_check(launch_temper_sharded(d_gds, d_list_big, (int)big.size(), max_slices, *xch, st),
                       "k_tp_* (sharded)");
            count_launch(temper_sharded_launches());
          } else if (!big.empty()) {
            cuda_check(launch_temper_grid(d_gds, d_list_big, (int)big.size(), max_slices, st), "k_tp_*");
            count_launch(temper_grid_launches());
          }
          cuda_check(cudaEventRecord(ma[k], st), "event");
          cuda_check(launch_move(kfam, noise, shape, dmax, d_gds, d_list, d_prefix, na, total, st), "k_chain<move>");
          cuda_check(cudaEventRecord(mb[k], st), "event");
          if (xch)
            cuda_check(launch_stats_sharded(d_gds, d_list, na, dmax, *xch, st), "k_stats (sharded)");
          else
            cuda_check(launch_stats_grid(d_gds, d_list, na, dmax, st), "k_stats_grid");
          count_launch(3);
          d2h(ring + (size_t)k * G, d_st, G, st);
          cuda_check(cudaEventRecord(lev[k], st), "event");
          ++enq;
        }
        if (obs == enq) break;
        const int k = (int)(obs % kRing);
        if (stage_early) drain(false);  // host copies of finished runs while the levels run
        cuda_check(cudaEventSynchronize(lev[k]), "cudaEventSynchronize");
        const GroupState* hs = ring + (size_t)k * G;
        if (live_before) {  // (a level past the end of every run moves nothing: not counted)
          float ms = 0.f;
          cuda_check(cudaEventElapsedTime(&ms, ma[k], mb[k]), "cudaEventElapsedTime");
          move_ms += ms;
          ++move_launches;
        }
        live_before = false;
        for (int gi = 0; gi < G; ++gi) live_before = live_before || hs[gi].active;
        std::memcpy(h_st, hs, sizeof(GroupState) * G);
        for (int gi = 0; gi < G; ++gi)
          if (!h_st[gi].active && !seen_done[gi]) {
            seen_done[gi] = 1;
            --n_live;
            if (stage_early) stage_group(gi, st);
          }
        ++obs;
      }
      for (int k = 0; k < kRing; ++k) {
        cudaEventDestroy(lev[k]);
        cudaEventDestroy(ma[k]);
        cudaEventDestroy(mb[k]);
      }
      pinned_cache().put(ring, ring_bytes);
    }
    cuda_check(cudaEventRecord(whole.b, st), "event");
    dev.sync();
    device_seconds = whole.ms() * 1e-3;
    std::lock_guard<std::mutex> lk(g_stats_mu);
    g_stats.move_kernel_ms += move_ms;
    g_stats.move_launches += move_launches;
    double pe = 0.0, mo = 0.0;
    const double slots = (double)shape.PPL * 32.0 * shape.W;  // every lane evaluates its padded slots
    for (int gi = 0; gi < G; ++gi) {
      pe += (double)h_st[gi].trials * (double)gds[gi].N;
      mo += slots * ((double)h_st[gi].shape_evals * mufu_shape[gi] + (double)h_st[gi].trials * mufu_per_noise(noise, shape.PPL));
    }
    g_stats.point_evals += pe;
    g_stats.move_mufu_ops += mo;
  }

  // D2H of diagnostics, posterior and energies (report fields of smc.cpp:221-247)
  void fetch(Device& dev, const std::vector<RunSpec>& runs, specmc_smc_result* out) {
    cudaStream_t st = dev.stream;
    bool synced = false;
    for (int gi = 0; gi < G; ++gi) {
      const RunSpec& R = runs[idx[gi]];
      specmc_smc_result& o = out[idx[gi]];
      const GroupState& s = h_st[gi];
      const size_t T = (size_t)s.T_loc, d = R.m.d;  // T_loc == T unless sharded
      o.d = (int)d;
      o.T = (int64_t)T;
      o.levels = s.level;
      o.trials = (int64_t)s.trials;
      o.proposals = (int64_t)R.cfg.T * (int64_t)d * s.level;
      o.device_seconds = device_seconds;
      if (s.error != GE_NONE) {
        o.status = SPECMC_ERUNTIME;
        continue;
      }
      o.status = SPECMC_OK;
      o.F = s.neg_log_z;
      o.diverged = !std::isfinite(o.F);
      const int Lv = s.level;
      std::vector<double> diag((size_t)Lv * 4);
      if (stage_early && staged[gi]) {  // copied out during the run (or now): hand the arrays over
        if (!synced) {
          drain(true);
          synced = true;
        }
        HostRes& r = hres[gi];
        diag = r.diag;
        o.posterior = r.post;
        o.energies = r.ener;
        r.post = r.ener = nullptr;
      } else {
        d2h(diag.data(), gds[gi].diag, diag.size(), st);
        // posterior: transposed to [T][d] on the device into the idle theta buffer, one D2H
        double* pout = gds[gi].theta[s.cur ^ 1];
        cuda_check(launch_posterior_out(gds[gi].theta[s.cur], gds[gi].tp, (int)d, (int)T, out_shift[gi], pout, st),
                   "k_posterior_out");
        o.posterior = static_cast<double*>(std::malloc(sizeof(double) * std::max<size_t>(d * T, 1)));
        d2h(o.posterior, pout, d * T, st);
        o.energies = static_cast<double*>(std::malloc(sizeof(double) * std::max<size_t>(T, 1)));
        d2h(o.energies, gds[gi].E[s.cur], T, st);
        dev.sync();
      }
      o.ladder = static_cast<double*>(std::malloc(sizeof(double) * (Lv + 1)));
      o.level_ess_ratio = static_cast<double*>(std::malloc(sizeof(double) * std::max(Lv, 1)));
      o.level_log_mean_w = static_cast<double*>(std::malloc(sizeof(double) * std::max(Lv, 1)));
      o.level_acc_rate = static_cast<double*>(std::malloc(sizeof(double) * std::max(Lv, 1)));
      o.ladder[0] = 0.0;
      for (int l = 0; l < Lv; ++l) {
        o.ladder[l + 1] = diag[4 * l];
        o.level_ess_ratio[l] = diag[4 * l + 1];
        o.level_log_mean_w[l] = diag[4 * l + 2];
        o.level_acc_rate[l] = diag[4 * l + 3];
      }
    }
  }
};

void copy_err(char* err, size_t errlen, const std::string& m) {
  if (err && errlen) {
    std::strncpy(err, m.c_str(), errlen - 1);
    err[errlen - 1] = 0;
  }
}

RunSpec make_runspec(const specmc_model_desc& m, int spectrum, const specmc_smc_config& cfg,
                     const specmc_spectrum& sp) {
  validate_config(cfg);
  validate_model(m);
  validate_spectrum(sp.xs, sp.ys, sp.n, m.noise == SPECMC_NOISE_POISSON);
  // the chain kernel's Philox counter (sweep - 1) d + component is 32-bit
  if ((uint64_t)cfg.n * (uint64_t)m.d > ((uint64_t)1 << 32))
    throw Error(SPECMC_EINVAL, "SmcConfig: n * d must not exceed 2^32 (device RNG counter range)");
  RunSpec R;
  R.m = m;
  R.spectrum = spectrum;
  R.cfg = cfg;
  R.N = sp.n;
  R.x_shift = pick_shift(m, sp.xs, sp.n);
  R.pk.assign(m.prior_kind, m.prior_kind + m.d);
  R.pa.assign(m.prior_a, m.prior_a + m.d);
  R.pb.assign(m.prior_b, m.prior_b + m.d);
  for (int i = 0; i < m.d; ++i)
    if (is_location(m.family, m.K, i) && R.x_shift != 0.0) {
      if (R.pk[i] == SPECMC_PRIOR_NORMAL) R.pa[i] -= R.x_shift;
      if (R.pk[i] == SPECMC_PRIOR_UNIFORM) {
        R.pa[i] -= R.x_shift;
        R.pb[i] -= R.x_shift;
      }
    }
  if (m.family == SPECMC_FAMILY_XRD) {
    R.refl_off.assign(m.K + 1, 0);
    for (int q = 0; q < m.n_refl; ++q) {
      R.refl.push_back((float)m.refl_mu[q]);
      R.refl.push_back((float)m.refl_int[q]);
      ++R.refl_off[m.refl_phase[q] + 1];
    }
    for (int b = 0; b < m.K; ++b) R.refl_off[b + 1] += R.refl_off[b];
  }
  R.m.prior_kind = nullptr;  // owned copies live in R
  R.m.prior_a = nullptr;
  R.m.prior_b = nullptr;
  R.m.refl_phase = nullptr;
  R.m.refl_mu = nullptr;
  R.m.refl_int = nullptr;
  return R;
}

// A batch of SMC runs resident on one device: create (validate, allocate,
// upload) -> run (device only) -> fetch (D2H).  specmc_smc_run_batch is
// create + run + fetch.
struct Session {
  std::vector<specmc_spectrum> spectra;
  std::vector<RunSpec> runs;
  std::unique_ptr<Device> dev;
  std::vector<std::unique_ptr<ClassRun>> classes;
  double device_seconds = 0.0;

  Session(int n_problems, const specmc_problem* problems, int n_spectra, const specmc_spectrum* sps,
          bool stage_early = false) {
    if (n_problems < 1 || !problems) throw Error(SPECMC_EINVAL, "batch: no problems");
    if (n_spectra < 1 || !sps) throw Error(SPECMC_EINVAL, "batch: no spectra");
    spectra.assign(sps, sps + n_spectra);
    for (int i = 0; i < n_problems; ++i) {
      const auto& p = problems[i];
      if (p.spectrum < 0 || p.spectrum >= n_spectra) throw Error(SPECMC_EINVAL, "batch: spectrum index out of range");
      runs.push_back(make_runspec(p.model, p.spectrum, p.cfg, spectra[p.spectrum]));
    }
    const int device = runs[0].cfg.device;
    for (auto& r : runs)
      if (r.cfg.device != device) throw Error(SPECMC_EINVAL, "batch: all problems must target the same device");
    dev = std::make_unique<Device>(device);
    // one class per (family, noise model, launch shape): each has its own move kernel
    std::map<std::tuple<int, int, int>, std::vector<int>> cls;
    for (int i = 0; i < n_problems; ++i) {
      const Shape s = pick_shape(runs[i].N, runs[i].m.d);
      cls[{kernel_family(runs[i]), dev_noise(runs[i].m), s.W * 100 + s.PPL}].push_back(i);
    }
    for (auto& kv : cls) {
      classes.push_back(std::make_unique<ClassRun>());
      classes.back()->idx = kv.second;
      classes.back()->stage_early = stage_early;
      classes.back()->prepare(*dev, runs, spectra);
    }
    spectra.clear();  // host inputs are borrowed only for the call
  }

  void run() {
    cuda_check(cudaSetDevice(dev->ordinal), "cudaSetDevice");
    device_seconds = 0.0;
    for (auto& c : classes) {
      c->run(*dev);
      device_seconds += c->device_seconds;
    }
  }

  int fetch(specmc_smc_result* out) {
    cuda_check(cudaSetDevice(dev->ordinal), "cudaSetDevice");
    for (size_t i = 0; i < runs.size(); ++i) std::memset(&out[i], 0, sizeof(specmc_smc_result));
    for (auto& c : classes) c->fetch(*dev, runs, out);
    int first = SPECMC_OK;
    for (size_t i = 0; i < runs.size(); ++i) {
      out[i].device_seconds = device_seconds;
      if (out[i].status != SPECMC_OK && first == SPECMC_OK) first = out[i].status;
    }
    return first;
  }
};

int run_batch(int n_problems, const specmc_problem* problems, int n_spectra, const specmc_spectrum* spectra,
              specmc_smc_result* out, char* err, size_t errlen) {
  const auto t0 = std::chrono::steady_clock::now();
  if (!out) throw Error(SPECMC_EINVAL, "batch: null results");
  static const bool trace = std::getenv("SPECMC_TRACE") != nullptr;  // phase timings on stderr
  auto since = [&](std::chrono::steady_clock::time_point a) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
  };
  int first;
  double t_create, t_run, t_fetch;
  {
    Session s(n_problems, problems, n_spectra, spectra, /*stage_early=*/true);
    t_create = since(t0);
    s.run();
    t_run = since(t0);
    first = s.fetch(out);
    t_fetch = since(t0);
  }
  const double wall = since(t0);
  if (trace)
    std::fprintf(stderr, "[specmc] run_batch create %.4f run %.4f fetch %.4f destroy %.4f s\n", t_create,
                 t_run - t_create, t_fetch - t_run, wall - t_fetch);
  for (int i = 0; i < n_problems; ++i) out[i].wall_seconds = wall;
  if (first != SPECMC_OK)
    copy_err(err, errlen, "smc: max_levels exceeded before reaching beta = 1 (or total weight is zero)");
  return first;
}

// ------------------------------------------------------ particle sharding
// Shards resident on this device: the exchanges are kernels over their descriptors.
struct VirtualExchange : Exchange {
  const ClassRun* cr;
  explicit VirtualExchange(const ClassRun* c) : cr(c) {}
  cudaError_t reduce(int buf, int count, int op, cudaStream_t st) override {
    return launch_xreduce(cr->d_gds, cr->d_xlist, cr->G / cr->nshards, cr->nshards, buf, count, op, st);
  }
  cudaError_t gather(cudaStream_t st) override {
    return launch_xgather(cr->d_gds, cr->d_xlist, cr->G / cr->nshards, cr->nshards, st);
  }
};

// NCCL, resolved with dlopen so that the library has no link-time NCCL
// dependency and shares the copy a host process (e.g. torch) already loaded
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;  // NCCL >= 2.18
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*ErrorString)(ncclResult_t) = nullptr;
  static NcclApi& get() {
    static NcclApi api = [] {
      NcclApi a;
      a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
      if (!a.h) a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!a.h) a.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
      if (!a.h) return a;
      a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(a.h, "ncclGetUniqueId"));
      a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(a.h, "ncclCommInitRank"));
      a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(a.h, "ncclAllReduce"));
      a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(a.h, "ncclAllGather"));
      a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(a.h, "ncclCommDestroy"));
      a.CommSplit = reinterpret_cast<decltype(a.CommSplit)>(dlsym(a.h, "ncclCommSplit"));
      a.ErrorString = reinterpret_cast<decltype(a.ErrorString)>(dlsym(a.h, "ncclGetErrorString"));
      a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(a.h, "ncclGroupStart"));
      a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(a.h, "ncclGroupEnd"));
      return a;
    }();
    if (!api.h || !api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.AllGather || !api.CommDestroy ||
        !api.GroupStart || !api.GroupEnd)
      throw Error(SPECMC_ECOMM, "NCCL (libnccl.so.2) is not available");
    return api;
  }
  void check(ncclResult_t r, const char* what) const {
    if (r != ncclSuccess)
      throw Error(SPECMC_ECOMM, std::string(what) + ": " + (ErrorString ? ErrorString(r) : "nccl error"));
  }
};

struct CommImpl {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1, device = 0;
  // sub-communicators of the distributed entry (one per rank block that shares
  // a particle-sharded run), split once from comm and kept for later calls
  std::map<std::pair<int, int>, ncclComm_t> subs;
};

// One shard of every run per rank: the exchanges are NCCL collectives on the
// shards' buffers, one per run, aggregated in an NCCL group and enqueued on the
// level stream (no host round trip inside a level)
struct NcclExchange : Exchange {
  const ClassRun* cr;
  CommImpl* c;
  NcclExchange(const ClassRun* r, CommImpl* cc) : cr(r), c(cc) {}
  cudaError_t reduce(int buf, int count, int op, cudaStream_t st) override {
    NcclApi& api = NcclApi::get();
    const ncclRedOp_t o = op == XOP_SUM ? ncclSum : (op == XOP_MIN ? ncclMin : ncclMax);
    api.check(api.GroupStart(), "ncclGroupStart");
    for (const GroupDesc& g : cr->gds) {
      double* p = buf == 0 ? g.xbuf : g.stat_acc;
      const size_t n = count < 0 ? (size_t)2 * g.d : (size_t)count;
      api.check(api.AllReduce(p, p, n, ncclFloat64, o, c->comm, st), "ncclAllReduce");
    }
    api.check(api.GroupEnd(), "ncclGroupEnd");
    return cudaSuccess;
  }
  cudaError_t gather(cudaStream_t st) override {
    NcclApi& api = NcclApi::get();
    api.check(api.GroupStart(), "ncclGroupStart");
    for (const GroupDesc& g : cr->gds)
      api.check(api.AllGather(g.xbuf, g.xgat, 2, ncclFloat64, c->comm, st), "ncclAllGather");
    api.check(api.GroupEnd(), "ncclGroupEnd");
    return cudaSuccess;
  }
};

// Particle-sharded runs: the T particles of every problem are
// split over nshards shards; comm == nullptr runs all of them on this device.
// Problems of one (family, noise, launch shape) advance together in one class.
// Results: F, ladder and diagnostics are global (identical on every shard);
// the posterior holds this process's particles (all of them for virtual shards).
int run_sharded_batch(int n_problems, const specmc_problem* problems, int n_spectra, const specmc_spectrum* sps,
                      int n_virtual, CommImpl* comm, specmc_smc_result* out) {
  const auto t0 = std::chrono::steady_clock::now();
  if (n_problems < 1 || !problems) throw Error(SPECMC_EINVAL, "sharded batch: no problems");
  if (n_spectra < 1 || !sps) throw Error(SPECMC_EINVAL, "sharded batch: no spectra");
  const int nsh = comm ? comm->world : n_virtual;
  if (nsh < 1) throw Error(SPECMC_EINVAL, "sharded run: shard count must be >= 1");
  const int device = problems[0].cfg.device;
  std::vector<RunSpec> runs;
  const int first = comm ? comm->rank : 0, count = comm ? 1 : nsh;
  for (int p = 0; p < n_problems; ++p) {
    const specmc_problem& pr = problems[p];
    if (pr.spectrum < 0 || pr.spectrum >= n_spectra) throw Error(SPECMC_EINVAL, "batch: spectrum index out of range");
    if (pr.cfg.T % nsh != 0) throw Error(SPECMC_EINVAL, "sharded run: T must be divisible by the shard count");
    if (pr.cfg.device != device) throw Error(SPECMC_EINVAL, "batch: all problems must target the same device");
    if (comm && pr.cfg.device != comm->device)
      throw Error(SPECMC_EINVAL, "sharded run: cfg.device differs from the communicator's device");
    for (int r = first; r < first + count; ++r) {
      RunSpec R = make_runspec(pr.model, pr.spectrum, pr.cfg, sps[pr.spectrum]);
      R.shard = r;
      R.nshards = nsh;
      R.T_loc0 = pr.cfg.T / nsh;
      R.pbase = (int64_t)r * (pr.cfg.T / nsh);
      R.problem = p;
      runs.push_back(std::move(R));
    }
  }
  Device dev(device);
  std::vector<specmc_spectrum> spectra(sps, sps + n_spectra);
  // one class per (family, noise model, launch shape); runs stay run-major, shard order
  std::map<std::tuple<int, int, int>, std::vector<int>> cls;
  for (int i = 0; i < (int)runs.size(); ++i) {
    const Shape s = pick_shape(runs[i].N, runs[i].m.d);
    cls[{kernel_family(runs[i]), dev_noise(runs[i].m), s.W * 100 + s.PPL}].push_back(i);
  }
  std::vector<specmc_smc_result> res(runs.size());
  for (auto& r : res) std::memset(&r, 0, sizeof(r));
  for (auto& kv : cls) {  // same order on every rank (map order)
    ClassRun cr;
    cr.idx = kv.second;
    std::unique_ptr<Exchange> x;
    if (comm)
      x = std::make_unique<NcclExchange>(&cr, comm);
    else
      x = std::make_unique<VirtualExchange>(&cr);
    cr.xch = x.get();
    cr.prepare(dev, runs, spectra);
    cr.run(dev);
    cr.fetch(dev, runs, res.data());
  }
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  // merge each problem's local shards into one result (shard order)
  int first_bad = SPECMC_OK;
  for (int p = 0; p < n_problems; ++p) {
    specmc_smc_result& o = out[p];
    const int i0 = p * count;
    o = res[i0];
    int64_t Ttot = 0, trials = 0;
    for (int r = 0; r < count; ++r) {
      Ttot += res[i0 + r].T;
      trials += res[i0 + r].trials;
      if (res[i0 + r].status != SPECMC_OK) o.status = res[i0 + r].status;
    }
    o.trials = trials;
    o.T = Ttot;
    o.proposals = (int64_t)problems[p].cfg.T * problems[p].model.d * o.levels * count / nsh;
    o.wall_seconds = wall;
    if (count > 1) {
      if (o.status == SPECMC_OK) {
        const size_t d = problems[p].model.d;
        o.posterior = static_cast<double*>(std::malloc(sizeof(double) * d * std::max<int64_t>(Ttot, 1)));
        o.energies = static_cast<double*>(std::malloc(sizeof(double) * std::max<int64_t>(Ttot, 1)));
        size_t at = 0;
        for (int r = 0; r < count; ++r) {
          const specmc_smc_result& q = res[i0 + r];
          std::memcpy(o.posterior + at * d, q.posterior, sizeof(double) * d * q.T);
          std::memcpy(o.energies + at, q.energies, sizeof(double) * q.T);
          at += q.T;
        }
        std::free(res[i0].posterior);
        std::free(res[i0].energies);
      }
      for (int r = 1; r < count; ++r) specmc_result_free(&res[i0 + r]);
    }
    if (o.status != SPECMC_OK && first_bad == SPECMC_OK) first_bad = o.status;
  }
  return first_bad;
}

// ----------------------------------------------------- replica exchange MC
// The paper's comparator (remc.cpp:78-163) on the device: every run of the
// batch is a group whose T = S = R replicas are chain units; per sweep one
// launch of k_chain in REMC mode over every replica of every run, then
// k_remc_exchange (swaps, accumulators, draws, sweep counter).  Runs are
// classed like SMC runs (family, noise, launch shape); the host enqueues all
// sweeps without waiting and reads the accumulators once at the end.
std::vector<double> remc_ladder(const specmc_remc_config& c) {  // remc.cpp:22-41
  std::vector<double> b;
  if (c.n_ladder > 0) {
    if (!c.ladder) throw Error(SPECMC_EINVAL, "remc: null ladder");
    b.assign(c.ladder, c.ladder + c.n_ladder);
    if (b.size() < 2) throw Error(SPECMC_EINVAL, "remc: explicit ladder needs >= 2 entries");
    if (b[0] != 0.0) throw Error(SPECMC_EINVAL, "remc: ladder must start at beta = 0");
    if (b.back() != 1.0) throw Error(SPECMC_EINVAL, "remc: ladder must end at beta = 1");
    for (size_t i = 1; i < b.size(); ++i)
      if (!(b[i] > b[i - 1])) throw Error(SPECMC_EINVAL, "remc: ladder must be strictly increasing");
    return b;
  }
  if (c.L < 1) throw Error(SPECMC_EINVAL, "remc: L must be >= 1");
  b.assign(c.L + 1, 0.0);
  for (int j = 1; j <= c.L; ++j)
    b[j] = c.L == 1 ? 1.0 : std::pow(10.0, -5.0 * (double)(c.L - j) / (double)(c.L - 1));
  b[c.L] = 1.0;
  return b;
}

void validate_remc(const specmc_remc_config& c) {  // remc.cpp:43-51
  remc_ladder(c);
  if (c.total_sweeps < 1) throw Error(SPECMC_EINVAL, "remc: total_sweeps must be >= 1");
  if (!(c.burn_in_fraction > 0.0 && c.burn_in_fraction < 1.0))
    throw Error(SPECMC_EINVAL, "remc: burn_in_fraction must lie in (0, 1)");
  if (c.swap_period < 1) throw Error(SPECMC_EINVAL, "remc: swap_period must be >= 1");
  if (c.workers < 0) throw Error(SPECMC_EINVAL, "remc: workers must be >= 0");
  if (c.total_sweeps > ((int64_t)1 << 31) - 2) throw Error(SPECMC_EINVAL, "remc: total_sweeps above 2^31");
}

int run_remc_batch(int n, const specmc_remc_problem* problems, int n_spectra, const specmc_spectrum* sps,
                   specmc_remc_result* out) {
  const auto t0 = std::chrono::steady_clock::now();
  if (n < 1 || !problems) throw Error(SPECMC_EINVAL, "remc batch: no problems");
  if (n_spectra < 1 || !sps) throw Error(SPECMC_EINVAL, "remc batch: no spectra");
  std::vector<RunSpec> runs;
  std::vector<std::vector<double>> ladders;
  const int device = problems[0].cfg.device;
  for (int i = 0; i < n; ++i) {
    const auto& p = problems[i];
    if (p.spectrum < 0 || p.spectrum >= n_spectra) throw Error(SPECMC_EINVAL, "batch: spectrum index out of range");
    if (p.cfg.device != device) throw Error(SPECMC_EINVAL, "batch: all problems must target the same device");
    validate_remc(p.cfg);
    ladders.push_back(remc_ladder(p.cfg));
    const int R = (int)ladders.back().size();
    specmc_smc_config sc{R, 1, 0.5, 1, p.cfg.seed, p.cfg.workers, device};  // T = S = R replicas
    runs.push_back(make_runspec(p.model, p.spectrum, sc, sps[p.spectrum]));
  }
  Device dev(device);
  cudaStream_t st = dev.stream;
  std::map<std::tuple<int, int, int>, std::vector<int>> cls;
  for (int i = 0; i < n; ++i) {
    const Shape s = pick_shape(runs[i].N, runs[i].m.d);
    cls[{runs[i].m.family, dev_noise(runs[i].m), s.W * 100 + s.PPL}].push_back(i);
  }
  Timer whole;
  cuda_check(cudaEventRecord(whole.a, st), "event");
  struct Done {
    GroupDesc g;
    GroupState* d_st;
    int64_t draws;
  };
  std::vector<Done> done(n);
  std::vector<std::unique_ptr<Arena>> arenas;
  for (auto& kv : cls) {
    const std::vector<int>& idx = kv.second;
    const int G = (int)idx.size();
    int64_t Nmax = 0;
    int dmax = 1;
    for (int r : idx) {
      Nmax = std::max(Nmax, runs[r].N);
      dmax = std::max(dmax, runs[r].m.d);
    }
    Shape shape = pick_shape(Nmax, dmax);
    if ((int64_t)32 * shape.W * shape.PPL < Nmax)
      throw Error(SPECMC_EINVAL, "spectrum has more points than the device path supports (8192)");
    const int family = runs[idx[0]].m.family, noise = dev_noise(runs[idx[0]].m);
    std::map<SpecKey, PreparedSpectrum> prep;
    for (int r : idx) {
      const auto key = spec_key(runs[r]);
      if (!prep.count(key)) {
        const auto& sp = sps[runs[r].spectrum];
        prep.emplace(key, prepare_spectrum(runs[r].m, sp.xs, sp.ys, sp.n, shape, runs[r].x_shift));
      }
    }
    shape.lay = spectrum_layout(family, noise, prep);
    fit_units(shape, dmax);
    if (chain_smem_bytes(shape, dmax) > kChainSmemMax)
      throw Error(SPECMC_EINVAL, "model too large for the device path (shared memory)");
    const size_t npt = (size_t)shape.PPL * 32 * shape.W;
    size_t bytes = Arena::al(sizeof(GroupDesc) * G) + Arena::al(sizeof(GroupState) * G) + 2 * Arena::al(4 * (G + 1));
    bytes += prep.size() * (Arena::al(npt * 4) + 2 * Arena::al(npt * 8));
    for (int gi = 0; gi < G; ++gi) {
      const RunSpec& R = runs[idx[gi]];
      const size_t Rn = ladders[idx[gi]].size(), d = R.m.d, tp = row_pitch(Rn);
      const int64_t nb = std::min<int64_t>(std::max<int64_t>(std::llround(problems[idx[gi]].cfg.burn_in_fraction *
                                                                          (double)problems[idx[gi]].cfg.total_sweeps), 0),
                                           problems[idx[gi]].cfg.total_sweeps - 1);
      const size_t draws = (size_t)(problems[idx[gi]].cfg.total_sweeps - nb);
      bytes += 3 * Arena::al(d * 8) + Arena::al(d * 4) + Arena::al(d * tp * 8) + Arena::al(Rn * 8);
      bytes += Arena::al(d * tp * 4) + Arena::al(d * tp * 8) + Arena::al(Rn * 8) + Arena::al(2 * Rn * 8);
      bytes += Arena::al(2 * Rn * 4) + Arena::al(d * draws * 8) + Arena::al(R.refl.size() * 4 + 8) +
               Arena::al(R.refl_off.size() * 4 + 4);
    }
    arenas.push_back(std::make_unique<Arena>());
    Arena& ar = *arenas.back();
    ar.reserve(bytes, dev.ordinal, st);
    cuda_check(prime_level_kernels(family, noise, shape, dmax), "loading the level kernels");
    GroupDesc* d_gds = ar.take<GroupDesc>(G);
    GroupState* d_st = ar.take<GroupState>(G);
    int* d_list = ar.take<int>(G + 1);
    int* d_prefix = ar.take<int>(G + 1);
    std::map<SpecKey, std::tuple<float*, float2*, float2*>> dspec;
    for (auto& p : prep) {
      float* x = ar.take<float>(npt);
      float2* c = ar.take<float2>(npt);
      float2* y = ar.take<float2>(npt);
      h2d(x, p.second.x.data(), npt, st);
      h2d(reinterpret_cast<float*>(c), p.second.c.data(), 2 * npt, st);
      h2d(reinterpret_cast<float*>(y), p.second.y.data(), 2 * npt, st);
      dspec[p.first] = std::make_tuple(x, c, y);
    }
    std::vector<GroupDesc> gds(G);
    std::vector<GroupState> sts(G);
    std::vector<int> list(G), prefix(G + 1);
    int total = 0;
    for (int gi = 0; gi < G; ++gi) {
      const int ri = idx[gi];
      const RunSpec& R = runs[ri];
      const auto& lad = ladders[ri];
      const int Rn = (int)lad.size(), d = R.m.d;
      const PreparedSpectrum& ps = prep.at(spec_key(R));
      GroupDesc& g = gds[gi];
      std::memset(&g, 0, sizeof(g));
      g.family = R.m.family;
      g.K = R.m.K;
      g.d = d;
      g.noise = ps.nz;
      g.T = g.S = Rn;
      g.n = 1;
      g.max_levels = 1;
      g.n_data = (double)R.N;
      const uint64_t k = mix64(R.cfg.seed);
      g.key0 = (uint32_t)k;
      g.key1 = (uint32_t)(k >> 32);
      g.N = (int)R.N;
      g.e_a0 = ps.e_a0;
      g.e_a1 = ps.e_a1;
      g.nz_a0 = ps.a0;
      g.nz_a1 = ps.a1;
      g.nz_a2 = ps.a2;
      g.nz_q = ps.q;
      g.x0s = ps.x0s;
      g.inv_range = ps.inv_range;
      g.range = ps.range;
      g.sh_uniform = ps.uniform ? 1 : 0;
      g.x1s = ps.x1s;
      g.y_last = ps.y_last;
      g.s_last = ps.s_last;
      auto t = dspec.at(spec_key(R));
      g.spec_x = std::get<0>(t);
      g.spec_c = std::get<1>(t);
      g.spec_y = std::get<2>(t);
      int* pk = ar.take<int>(d);
      double* pa = ar.take<double>(d);
      double* pb = ar.take<double>(d);
      h2d(pk, R.pk.data(), d, st);
      h2d(pa, R.pa.data(), d, st);
      h2d(pb, R.pb.data(), d, st);
      g.pkind = pk;
      g.pa = pa;
      g.pb = pb;
      g.tp = g.sp = (int)row_pitch(Rn);
      g.theta[0] = g.theta[1] = ar.take<double>((size_t)d * g.tp);
      g.E[0] = g.E[1] = ar.take<double>(Rn);
      g.chain_acc = ar.take<int>((size_t)d * g.sp);
      g.chain_ls = ar.take<double>((size_t)d * g.sp);
      double* lad_d = ar.take<double>(Rn);
      h2d(lad_d, lad.data(), Rn, st);
      g.ladder = lad_d;
      g.pair_acc = ar.take<double>(2 * (size_t)Rn);
      g.swaps = ar.take<int>(2 * (size_t)Rn);
      const auto& c = problems[ri].cfg;
      g.total_sweeps = c.total_sweeps;
      g.n_burn = std::min<int64_t>(std::max<int64_t>(std::llround(c.burn_in_fraction * (double)c.total_sweeps), 0),
                                   c.total_sweeps - 1);
      g.swap_period = c.swap_period;
      const int64_t draws = c.total_sweeps - g.n_burn;
      g.post = ar.take<double>((size_t)d * draws);
      if (!R.refl.empty()) {
        float2* rf = ar.take<float2>(R.refl.size() / 2);
        int* ro = ar.take<int>(R.refl_off.size());
        h2d(reinterpret_cast<float*>(rf), R.refl.data(), R.refl.size(), st);
        h2d(ro, R.refl_off.data(), R.refl_off.size(), st);
        g.refl = rf;
        g.refl_off = ro;
      }
      g.st = d_st + gi;
      // initial step sizes clamp(prior_scale) (mcmc.cpp:7-12) for every replica; tallies 0;
      // accumulators (max, sum) = (-inf, 0); swap tallies 0
      std::vector<double> ls((size_t)d * g.sp, 0.0);
      for (int i = 0; i < d; ++i) {
        const int kd = R.pk[i];
        const double a = R.pa[i], b = R.pb[i];
        double sc = kd == SPECMC_PRIOR_NORMAL ? std::sqrt(b) : (kd == SPECMC_PRIOR_GAMMA ? std::sqrt(a) / b : (b - a) / std::sqrt(12.0));
        sc = std::min(std::max(sc, 1e-12), 1e12);
        for (int r = 0; r < Rn; ++r) ls[(size_t)i * g.sp + r] = std::log(sc);
      }
      h2d(g.chain_ls, ls.data(), ls.size(), st);
      cuda_check(cudaMemsetAsync(g.chain_acc, 0, sizeof(int) * (size_t)d * g.sp, st), "memset");
      std::vector<double> pa0(2 * (size_t)Rn, 0.0);
      for (int l = 0; l < Rn; ++l) pa0[2 * l] = -INFINITY;
      h2d(g.pair_acc, pa0.data(), pa0.size(), st);
      cuda_check(cudaMemsetAsync(g.swaps, 0, sizeof(int) * 2 * (size_t)Rn, st), "memset");
      GroupState& s = sts[gi];
      std::memset(&s, 0, sizeof(s));
      s.active = 1;
      s.level = 1;
      s.T_loc = s.S_loc = Rn;
      list[gi] = gi;
      prefix[gi] = total;
      total += (Rn + shape.U - 1) / shape.U;
      done[ri] = Done{g, d_st + gi, draws};
    }
    prefix[G] = total;
    h2d(d_gds, gds.data(), G, st);
    h2d(d_st, sts.data(), G, st);
    h2d(d_list, list.data(), G, st);
    h2d(d_prefix, prefix.data(), G + 1, st);
    dev.sync();  // (host vectors above go out of scope)
    int64_t sweeps = 0;
    for (int r : idx) sweeps = std::max<int64_t>(sweeps, problems[r].cfg.total_sweeps);
    // init: prior draws and energies of every replica (remc.cpp:113-119)
    int rmax = 0;
    for (int r : idx) rmax = std::max<int>(rmax, (int)ladders[r].size());
    cuda_check(launch_init_draw(d_gds, d_list, G, rmax, st), "k_init_draw");
    cuda_check(launch_energy(family, shape, dmax, d_gds, d_list, d_prefix, G, total, st), "k_chain<energy>");
    count_launch(2);
    for (int64_t t = 1; t <= sweeps; ++t) {  // (a run with fewer sweeps turns inactive after its last one)
      cuda_check(launch_remc_sweep(family, shape, dmax, d_gds, d_list, d_prefix, G, total, st), "k_chain<remc>");
      cuda_check(launch_remc_exchange(d_gds, d_list, G, st), "k_remc_exchange");
      count_launch(2);
    }
  }
  cuda_check(cudaEventRecord(whole.b, st), "event");
  dev.sync();
  const double dsec = whole.ms() * 1e-3;
  int first = SPECMC_OK;
  for (int i = 0; i < n; ++i) {
    const Done& dn = done[i];
    const GroupDesc& g = dn.g;
    specmc_remc_result& o = out[i];
    const int Rn = g.S, d = g.d;
    o.status = SPECMC_OK;
    o.R = Rn;
    o.d = d;
    o.draws = dn.draws;
    std::vector<double> acc(2 * (size_t)Rn), post((size_t)d * dn.draws);
    std::vector<int> swaps(2 * (size_t)Rn), tall((size_t)d * g.sp);
    d2h(acc.data(), g.pair_acc, acc.size(), st);
    d2h(swaps.data(), g.swaps, swaps.size(), st);
    d2h(tall.data(), g.chain_acc, tall.size(), st);
    d2h(post.data(), g.post, post.size(), st);
    dev.sync();
    double F = 0.0;  // free_energy_remc (remc.cpp:75-79), LogMeanAcc::log_mean (math.hpp:48-54)
    for (int l = 0; l + 1 < Rn; ++l) {
      const double mx = acc[2 * l], sm = acc[2 * l + 1];
      const double lm = std::isnan(mx) ? NAN : (mx == -INFINITY ? -INFINITY : mx + std::log(sm) - std::log((double)dn.draws));
      F -= lm;
    }
    o.diverged = !std::isfinite(F);
    o.F = std::isfinite(F) ? F : NAN;
    o.ladder = static_cast<double*>(std::malloc(sizeof(double) * Rn));
    std::memcpy(o.ladder, ladders[i].data(), sizeof(double) * Rn);
    o.swap_rate = static_cast<double*>(std::malloc(sizeof(double) * std::max(Rn - 1, 1)));
    for (int l = 0; l + 1 < Rn; ++l)
      o.swap_rate[l] = swaps[2 * l + 1] > 0 ? (double)swaps[2 * l] / swaps[2 * l + 1] : 0.0;
    o.replica_acc = static_cast<double*>(std::malloc(sizeof(double) * Rn));
    for (int r = 0; r < Rn; ++r) {
      double a = 0.0;
      for (int c = 0; c < d; ++c) a += tall[(size_t)c * g.sp + r];
      const double prop = (double)dn.draws * d;  // proposals after the burn-in reset (mcmc.cpp:64)
      o.replica_acc[r] = prop > 0 ? a / prop : 0.0;
    }
    o.posterior = static_cast<double*>(std::malloc(sizeof(double) * std::max<int64_t>((int64_t)d * dn.draws, 1)));
    const RunSpec& R = runs[i];
    for (int64_t k = 0; k < dn.draws; ++k)
      for (int c = 0; c < d; ++c) {
        double v = post[(size_t)c * dn.draws + k];
        if (is_location(R.m.family, R.m.K, c)) v += R.x_shift;
        o.posterior[(size_t)k * d + c] = v;
      }
    o.device_seconds = dsec;
    o.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  return first;
}

// ------------------------------------------------- multi-GPU model selection
// Placement of a batch of runs (the K range of a model selection, SURVEY.md
// 8e-1/8e-3) on `world` ranks, by cost (run_cost: T d^1.5 N).  A run costing more
// than alpha x a rank's share (sum / world) is particle-sharded over s ranks
// (the smallest power of two >= cost / (alpha share) whose shards keep whole
// chains), placed on the contiguous block of s ranks with the least load; every
// other run goes to the least loaded rank, longest first (LPT).  The loads
// charge a sharded run 3% per doubling for its exchanges; the plan with the
// least makespan over alpha in {1, 0.85, 0.7, 0.55, 0.4} wins.  Deterministic:
// every rank computes the same plan from the same inputs.
struct Plan {
  std::vector<int> rank0, shards;
  std::vector<double> load;
  double makespan = 0.0;
};
// one placement with the sharding threshold alpha * share
Plan place(int n, const double* cost, const int64_t* T, const int32_t* n_sweeps, int world, double alpha) {
  Plan p;
  p.rank0.assign(n, 0);
  p.shards.assign(n, 1);
  p.load.assign(world, 0.0);
  double total = 0.0;
  for (int i = 0; i < n; ++i) total += cost[i];
  const double cut = alpha * total / world;
  int wpow = 1;
  while (wpow * 2 <= world) wpow *= 2;
  std::vector<int> sh(n, 1);
  std::vector<double> piece(n);
  for (int i = 0; i < n; ++i) {
    int s = 1;
    if (world > 1 && cost[i] > cut * (1.0 + 1e-9)) {
      while (s < wpow && s * cut < cost[i]) s *= 2;
      // every shard keeps whole chains: T / s divisible by n with >= 2 chains
      while (s > 1 && (T[i] % s != 0 || (T[i] / s) % n_sweeps[i] != 0 || T[i] / s / n_sweeps[i] < 2)) s /= 2;
    }
    sh[i] = s;
    // a sharded run pays its per-level exchanges: 3% per doubling of the shard count
    piece[i] = cost[i] / s * (1.0 + 0.03 * std::log2((double)s));
  }
  // largest pieces first (LPT over the pieces; ties: more shards first)
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return piece[a] != piece[b] ? piece[a] > piece[b] : sh[a] > sh[b];
  });
  for (int i : order) {
    const int s = sh[i];
    int best = 0;
    if (s > 1) {
      double bl = 1e300;
      for (int b = 0; b + s <= world; ++b) {  // any contiguous block of s ranks
        double m = 0.0;
        for (int r = b; r < b + s; ++r) m = std::max(m, p.load[r]);
        if (m < bl) {
          bl = m;
          best = b;
        }
      }
      for (int r = best; r < best + s; ++r) p.load[r] += piece[i];
    } else {
      for (int r = 1; r < world; ++r)
        if (p.load[r] < p.load[best]) best = r;
      p.load[best] += piece[i];
    }
    p.rank0[i] = best;
    p.shards[i] = s;
  }
  p.makespan = *std::max_element(p.load.begin(), p.load.end());
  return p;
}

// the placement with the least makespan over a few sharding thresholds (runs
// above alpha x a rank's share are split; ties keep the larger alpha, i.e.
// fewer shards)
Plan make_plan(int n, const double* cost, const int64_t* T, const int32_t* n_sweeps, int world) {
  Plan best;
  bool have = false;
  for (double alpha : {1.0, 0.85, 0.7, 0.55, 0.4}) {
    Plan p = place(n, cost, T, n_sweeps, world, alpha);
    if (!have || p.makespan < best.makespan * (1.0 - 1e-12)) {
      best = std::move(p);
      have = true;
    }
  }
  return best;
}

// T d N per level times the level count, which grows about as sqrt(d) (the
// reference's own C2 run, profiles/r02_cpu_c2_full.json: 20 levels at d = 6,
// 57 at d = 42)
double run_cost(const specmc_problem& pr, const specmc_spectrum* sps) {
  return (double)pr.cfg.T * (double)pr.model.d * std::sqrt((double)pr.model.d) * (double)sps[pr.spectrum].n;
}

// The batch split over the ranks of `world` by make_plan: first the sharded
// runs, block by block in (first rank, shards) order on sub-communicators split
// from world (every rank takes part in every split, in the same order), then
// this rank's own runs in one batch, then one all-reduce of the per-run
// scalars (F, levels, status, ... from the run's first rank; trials summed over
// its shards) so that every rank can select K.  Arrays (posterior, energies,
// ladder, diagnostics) stay with the ranks that ran the run.
int run_distributed(int n_problems, const specmc_problem* problems, int n_spectra, const specmc_spectrum* sps,
                    CommImpl* world, int32_t* plan_rank0, int32_t* plan_shards, specmc_smc_result* out) {
  if (n_problems < 1 || !problems) throw Error(SPECMC_EINVAL, "distributed: no problems");
  if (n_spectra < 1 || !sps) throw Error(SPECMC_EINVAL, "distributed: no spectra");
  if (!world) throw Error(SPECMC_EINVAL, "distributed: null communicator");
  for (int i = 0; i < n_problems; ++i) {
    if (problems[i].spectrum < 0 || problems[i].spectrum >= n_spectra)
      throw Error(SPECMC_EINVAL, "batch: spectrum index out of range");
    validate_config(problems[i].cfg);
  }
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<double> cost(n_problems);
  std::vector<int64_t> Ts(n_problems);
  std::vector<int32_t> ns(n_problems);
  for (int i = 0; i < n_problems; ++i) {
    cost[i] = run_cost(problems[i], sps);
    Ts[i] = problems[i].cfg.T;
    ns[i] = problems[i].cfg.n;
  }
  const Plan plan = make_plan(n_problems, cost.data(), Ts.data(), ns.data(), world->world);
  if (plan_rank0) std::copy(plan.rank0.begin(), plan.rank0.end(), plan_rank0);
  if (plan_shards) std::copy(plan.shards.begin(), plan.shards.end(), plan_shards);
  const int me = world->rank;
  Device dev(world->device);
  Timer whole;
  cuda_check(cudaEventRecord(whole.a, dev.stream), "event");
  NcclApi& api = NcclApi::get();
  std::vector<specmc_problem> probs(problems, problems + n_problems);
  for (auto& p : probs) p.cfg.device = world->device;
  // 1) particle-sharded runs, one rank block at a time
  // SPECMC_DIST_SHARD_ALL=1 (tests): every run takes the sharded path, even on
  // a one-rank block -- the sub-communicator split and the NCCL exchanges then
  // run on one GPU without any rank waiting on another
  const bool shard_all = std::getenv("SPECMC_DIST_SHARD_ALL") && std::atoi(std::getenv("SPECMC_DIST_SHARD_ALL")) == 1;
  auto sharded = [&](int i) { return plan.shards[i] > 1 || shard_all; };
  std::map<std::pair<int, int>, std::vector<int>> blocks;
  for (int i = 0; i < n_problems; ++i)
    if (sharded(i)) blocks[{plan.rank0[i], plan.shards[i]}].push_back(i);
  int first_bad = SPECMC_OK;
  // every split first (collective over the world, in block order), so that
  // disjoint blocks then run concurrently instead of waiting in the next split
  for (auto& kv : blocks) {
    const int b0 = kv.first.first, s = kv.first.second;
    if (world->subs.count(kv.first)) continue;
    if (!api.CommSplit) throw Error(SPECMC_ECOMM, "NCCL without ncclCommSplit (needs >= 2.18)");
    const bool in = me >= b0 && me < b0 + s;
    ncclComm_t sub = nullptr;
    api.check(api.CommSplit(world->comm, in ? b0 * 4096 + s : NCCL_SPLIT_NOCOLOR, me, &sub, nullptr),
              "ncclCommSplit");
    world->subs.emplace(kv.first, sub);
  }
  for (auto& kv : blocks) {
    const int b0 = kv.first.first, s = kv.first.second;
    const bool in = me >= b0 && me < b0 + s;
    if (!in) continue;
    auto it = world->subs.find(kv.first);
    CommImpl sc;
    sc.comm = it->second;
    sc.rank = me - b0;
    sc.world = s;
    sc.device = world->device;
    std::vector<specmc_problem> bp;
    for (int i : kv.second) bp.push_back(probs[i]);
    std::vector<specmc_smc_result> br(bp.size());
    for (auto& r : br) std::memset(&r, 0, sizeof(r));
    const int rc = run_sharded_batch((int)bp.size(), bp.data(), n_spectra, sps, 1, &sc, br.data());
    if (rc != SPECMC_OK && first_bad == SPECMC_OK) first_bad = rc;
    for (size_t j = 0; j < kv.second.size(); ++j) out[kv.second[j]] = br[j];
  }
  // 2) this rank's own runs
  std::vector<int> mine;
  for (int i = 0; i < n_problems; ++i)
    if (!sharded(i) && plan.rank0[i] == me) mine.push_back(i);
  if (!mine.empty()) {
    std::vector<specmc_problem> bp;
    for (int i : mine) bp.push_back(probs[i]);
    std::vector<specmc_smc_result> br(bp.size());
    for (auto& r : br) std::memset(&r, 0, sizeof(r));
    char e2[256];
    const int rc = run_batch((int)bp.size(), bp.data(), n_spectra, sps, br.data(), e2, sizeof(e2));
    if (rc != SPECMC_OK && first_bad == SPECMC_OK) first_bad = rc;
    for (size_t j = 0; j < mine.size(); ++j) out[mine[j]] = br[j];
  }
  // 3) every run's scalars on every rank (one all-reduce, sum; zeros from non-owners)
  constexpr int kF = 7;
  std::vector<double> h((size_t)kF * n_problems, 0.0);
  for (int i = 0; i < n_problems; ++i) {
    const bool ran = sharded(i) ? (me >= plan.rank0[i] && me < plan.rank0[i] + plan.shards[i]) : me == plan.rank0[i];
    if (!ran) continue;
    double* r = h.data() + (size_t)kF * i;
    r[5] = (double)out[i].trials;  // local share of a sharded run
    if (me != plan.rank0[i]) continue;
    r[0] = out[i].F;
    r[1] = out[i].diverged;
    r[2] = out[i].levels;
    r[3] = out[i].status;
    r[4] = (double)((int64_t)problems[i].cfg.T * problems[i].model.d * out[i].levels);
    r[6] = out[i].d;
  }
  double* dbuf = nullptr;
  cuda_check(cudaMalloc(&dbuf, sizeof(double) * h.size()), "cudaMalloc");
  h2d(dbuf, h.data(), h.size(), dev.stream);
  api.check(api.AllReduce(dbuf, dbuf, h.size(), ncclFloat64, ncclSum, world->comm, dev.stream), "ncclAllReduce");
  d2h(h.data(), dbuf, h.size(), dev.stream);
  cuda_check(cudaEventRecord(whole.b, dev.stream), "event");
  dev.sync();
  cudaFree(dbuf);
  const double dsec = whole.ms() * 1e-3;
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  for (int i = 0; i < n_problems; ++i) {
    const double* r = h.data() + (size_t)kF * i;
    specmc_smc_result& o = out[i];
    o.F = r[0];
    o.diverged = (int32_t)r[1];
    o.levels = (int32_t)r[2];
    o.status = (int32_t)r[3];
    o.proposals = (int64_t)r[4];
    o.trials = (int64_t)r[5];
    o.d = (int32_t)r[6];
    o.device_seconds = dsec;
    o.wall_seconds = wall;
    if (o.status != SPECMC_OK && first_bad == SPECMC_OK) first_bad = o.status;
  }
  return first_bad;
}

template <typename F>
int guarded(char* err, size_t errlen, F&& f) {
  try {
    return f();
  } catch (const Error& e) {
    copy_err(err, errlen, e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    copy_err(err, errlen, "host allocation failed");
    return SPECMC_ERUNTIME;
  } catch (const std::exception& e) {
    copy_err(err, errlen, e.what());
    return SPECMC_ERUNTIME;
  }
}

// device scratch for the unit entry points
struct Scratch {
  std::vector<DevBuf> bufs;
  template <typename T>
  T* alloc(size_t n) {
    bufs.emplace_back(sizeof(T) * std::max<size_t>(n, 1));
    return bufs.back().as<T>();
  }
};

// One unsharded group holding a caller's array as its current energies, for
// the parity units of the grid-level tempering (T > 2^15): the same slices and
// k_tp_* launches as ClassRun::prepare / run give a production group.
struct GridUnit {
  Scratch sc;
  GroupDesc* d_g = nullptr;
  GroupState* d_st = nullptr;
  TemperScratch* d_ts = nullptr;
  int* d_list = nullptr;
  int nslices = 0;
  GroupDesc g;
  GridUnit(const double* host_e, int64_t T, double n_data, double beta, double ess_target, int64_t S,
           cudaStream_t st) {
    std::memset(&g, 0, sizeof(g));
    d_g = sc.alloc<GroupDesc>(1);
    d_st = sc.alloc<GroupState>(1);
    d_ts = sc.alloc<TemperScratch>(1);
    d_list = sc.alloc<int>(1);
    double* dE = sc.alloc<double>(T);
    h2d(dE, host_e, T, st);
    g.T = (int)T;
    g.n = 1;
    g.S = (int)S;
    g.max_levels = 1;
    g.ess_target = ess_target;
    g.n_data = n_data;
    g.E[0] = g.E[1] = dE;
    g.wbuf = sc.alloc<double>(T);
    g.anc = sc.alloc<int>(S);
    g.diag = sc.alloc<double>(4);
    g.st = d_st;
    g.ts = d_ts;
    size_t sl = std::max<size_t>(min_slice_len(), (T + kMaxSlices - 1) / kMaxSlices);
    sl = (sl + 1023) & ~(size_t)1023;
    g.slice_len = (int)sl;
    g.nslices = nslices = (int)((T + sl - 1) / sl);
    GroupState s;
    std::memset(&s, 0, sizeof(s));
    s.beta = beta;
    s.active = 1;
    s.T_loc = (int)T;
    s.S_loc = (int)S;
    h2d(d_st, &s, 1, st);
    h2d(d_g, &g, 1, st);
    const int zero = 0;
    h2d(d_list, &zero, 1, st);
    cuda_check(cudaMemsetAsync(d_ts, 0, sizeof(TemperScratch), st), "memset");
  }
};

}  // namespace
}  // namespace smc

using namespace smc;

extern "C" {

int specmc_smc_run(const specmc_model_desc* model, const double* xs, const double* ys, int64_t n_points,
                   const specmc_smc_config* cfg, specmc_smc_result* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> int {
    if (!model || !cfg || !out) throw Error(SPECMC_EINVAL, "null argument");
    std::memset(out, 0, sizeof(*out));
    specmc_problem p;
    p.model = *model;
    p.spectrum = 0;
    p.cfg = *cfg;
    specmc_spectrum sp{xs, ys, n_points};
    const int rc = run_batch(1, &p, 1, &sp, out, err, errlen);
    return rc;
  });
}

int specmc_smc_run_batch(int32_t n_problems, const specmc_problem* problems, int32_t n_spectra,
                         const specmc_spectrum* spectra, specmc_smc_result* out, char* err, size_t errlen) {
  if (out && n_problems > 0) std::memset(out, 0, sizeof(specmc_smc_result) * (size_t)n_problems);
  const int rc = guarded(err, errlen, [&]() -> int { return run_batch(n_problems, problems, n_spectra, spectra, out, err, errlen); });
  if (rc != SPECMC_OK && out)  // an ABI-level failure leaves every run with that status
    for (int i = 0; i < n_problems; ++i)
      if (out[i].status == SPECMC_OK && !out[i].posterior) out[i].status = rc;
  return rc;
}

int specmc_session_create(int32_t n_problems, const specmc_problem* problems, int32_t n_spectra,
                          const specmc_spectrum* spectra, specmc_session** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> int {
    if (!out) throw Error(SPECMC_EINVAL, "null session pointer");
    *out = reinterpret_cast<specmc_session*>(new Session(n_problems, problems, n_spectra, spectra));
    return SPECMC_OK;
  });
}

int specmc_session_run(specmc_session* s, double* device_seconds, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> int {
    if (!s) throw Error(SPECMC_EINVAL, "null session");
    auto* S = reinterpret_cast<Session*>(s);
    S->run();
    if (device_seconds) *device_seconds = S->device_seconds;
    return SPECMC_OK;
  });
}

int specmc_session_fetch(specmc_session* s, specmc_smc_result* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> int {
    if (!s || !out) throw Error(SPECMC_EINVAL, "null argument");
    const int rc = reinterpret_cast<Session*>(s)->fetch(out);
    if (rc != SPECMC_OK)
      copy_err(err, errlen, "smc: max_levels exceeded before reaching beta = 1 (or total weight is zero)");
    return rc;
  });
}

void specmc_session_destroy(specmc_session* s) { delete reinterpret_cast<Session*>(s); }

int specmc_init_ensemble(const specmc_model_desc* model, const double* xs, const double* ys, int64_t n_points,
                         const specmc_smc_config* cfg, specmc_smc_result* out, char* err, size_t errlen) {
  if (out) std::memset(out, 0, sizeof(*out));
  return guarded(err, errlen, [&]() -> int {
    if (!model || !cfg || !out) throw Error(SPECMC_EINVAL, "null argument");
    specmc_spectrum sp{xs, ys, n_points};
    std::vector<RunSpec> runs{make_runspec(*model, 0, *cfg, sp)};
    Device dev(cfg->device);
    std::vector<specmc_spectrum> spectra{sp};
    ClassRun cr;
    cr.idx = {0};
    cr.init_only = true;
    cr.prepare(dev, runs, spectra);
    cr.run(dev);
    cr.fetch(dev, runs, out);
    return out->status;
  });
}

int specmc_smc_run_sharded_batch(int32_t n_problems, const specmc_problem* problems, int32_t n_spectra,
                                 const specmc_spectrum* spectra, int32_t n_virtual, specmc_comm* comm,
                                 specmc_smc_result* out, char* err, size_t errlen) {
  if (out && n_problems > 0) std::memset(out, 0, sizeof(specmc_smc_result) * (size_t)n_problems);
  const int rc = guarded(err, errlen, [&]() -> int {
    if (!out) throw Error(SPECMC_EINVAL, "null results");
    const int r = run_sharded_batch(n_problems, problems, n_spectra, spectra, n_virtual,
                                    reinterpret_cast<CommImpl*>(comm), out);
    if (r != SPECMC_OK)
      copy_err(err, errlen, "smc: max_levels exceeded before reaching beta = 1 (or total weight is zero)");
    return r;
  });
  if (rc != SPECMC_OK && out)
    for (int i = 0; i < n_problems; ++i)
      if (out[i].status == SPECMC_OK && !out[i].posterior) out[i].status = rc;
  return rc;
}

int specmc_smc_run_sharded(const specmc_model_desc* model, const double* xs, const double* ys, int64_t n_points,
                           const specmc_smc_config* cfg, int32_t n_virtual, specmc_comm* comm,
                           specmc_smc_result* out, char* err, size_t errlen) {
  if (out) std::memset(out, 0, sizeof(*out));
  if (!model || !cfg || !out) {
    copy_err(err, errlen, "null argument");
    return SPECMC_EINVAL;
  }
  const specmc_problem p{*model, 0, *cfg};
  const specmc_spectrum sp{xs, ys, n_points};
  return specmc_smc_run_sharded_batch(1, &p, 1, &sp, n_virtual, comm, out, err, errlen);
}

int specmc_nccl_unique_id(uint8_t* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> int {
    if (!out) throw Error(SPECMC_EINVAL, "null argument");
    NcclApi& api = NcclApi::get();
    ncclUniqueId id;
    api.check(api.GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == SPECMC_COMM_ID_BYTES, "ncclUniqueId size");
    std::memcpy(out, &id, sizeof(id));
    return SPECMC_OK;
  });
}

int specmc_comm_init_nccl(int32_t rank, int32_t world, const uint8_t* id, int32_t device, specmc_comm** out,
                          char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> int {
    if (!id || !out) throw Error(SPECMC_EINVAL, "null argument");
    if (world < 1 || rank < 0 || rank >= world) throw Error(SPECMC_EINVAL, "comm: bad rank / world size");
    Device dev(device);
    NcclApi& api = NcclApi::get();
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    auto c = std::make_unique<CommImpl>();
    c->rank = rank;
    c->world = world;
    c->device = device;
    api.check(api.CommInitRank(&c->comm, world, uid, rank), "ncclCommInitRank");
    *out = reinterpret_cast<specmc_comm*>(c.release());
    return SPECMC_OK;
  });
}

void specmc_comm_destroy(specmc_comm* c) {
  auto* p = reinterpret_cast<CommImpl*>(c);
  if (!p) return;
  for (auto& kv : p->subs) {
    try {
      if (kv.second) NcclApi::get().CommDestroy(kv.second);
    } catch (...) {
    }
  }
  if (p->comm) {
    try {
      NcclApi::get().CommDestroy(p->comm);
    } catch (...) {
    }
  }
  delete p;
}

int specmc_plan(int32_t n_runs, const double* costs, const int64_t* T, const int32_t* n_sweeps, int32_t world,
                int32_t* rank0, int32_t* shards, double* rank_load, double* makespan) {
  if (n_runs < 1 || !costs || !T || !n_sweeps || world < 1 || !rank0 || !shards) return SPECMC_EINVAL;
  for (int i = 0; i < n_runs; ++i)
    if (!(costs[i] >= 0.0) || T[i] < 2 || n_sweeps[i] < 1) return SPECMC_EINVAL;
  const Plan p = make_plan(n_runs, costs, T, n_sweeps, world);
  std::copy(p.rank0.begin(), p.rank0.end(), rank0);
  std::copy(p.shards.begin(), p.shards.end(), shards);
  if (rank_load) std::copy(p.load.begin(), p.load.end(), rank_load);
  if (makespan) *makespan = p.makespan;
  return SPECMC_OK;
}

int specmc_smc_run_distributed(int32_t n_problems, const specmc_problem* problems, int32_t n_spectra,
                               const specmc_spectrum* spectra, specmc_comm* comm, int32_t* plan_rank0,
                               int32_t* plan_shards, specmc_smc_result* out, char* err, size_t errlen) {
  if (out && n_problems > 0) std::memset(out, 0, sizeof(specmc_smc_result) * (size_t)n_problems);
  return guarded(err, errlen, [&]() -> int {
    if (!out) throw Error(SPECMC_EINVAL, "null results");
    const int r = run_distributed(n_problems, problems, n_spectra, spectra, reinterpret_cast<CommImpl*>(comm),
                                  plan_rank0, plan_shards, out);
    if (r != SPECMC_OK)
      copy_err(err, errlen, "smc: max_levels exceeded before reaching beta = 1 (or total weight is zero)");
    return r;
  });
}

int specmc_remc_run_batch(int32_t n_problems, const specmc_remc_problem* problems, int32_t n_spectra,
                          const specmc_spectrum* spectra, specmc_remc_result* out, char* err, size_t errlen) {
  if (out && n_problems > 0) std::memset(out, 0, sizeof(specmc_remc_result) * (size_t)n_problems);
  return guarded(err, errlen, [&]() -> int {
    if (!out) throw Error(SPECMC_EINVAL, "null results");
    return run_remc_batch(n_problems, problems, n_spectra, spectra, out);
  });
}

void specmc_remc_result_free(specmc_remc_result* r) {
  if (!r) return;
  std::free(r->ladder);
  std::free(r->swap_rate);
  std::free(r->replica_acc);
  std::free(r->posterior);
  r->ladder = r->swap_rate = r->replica_acc = r->posterior = nullptr;
}

void specmc_free(void* p) { std::free(p); }

void specmc_result_free(specmc_smc_result* r) {
  if (!r) return;
  std::free(r->ladder);
  std::free(r->level_ess_ratio);
  std::free(r->level_log_mean_w);
  std::free(r->level_acc_rate);
  std::free(r->posterior);
  std::free(r->energies);
  r->ladder = r->level_ess_ratio = r->level_log_mean_w = r->level_acc_rate = r->posterior = r->energies = nullptr;
}

int specmc_validate_config(const specmc_smc_config* cfg, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> int {
    if (!cfg) throw Error(SPECMC_EINVAL, "null config");
    validate_config(*cfg);
    return SPECMC_OK;
  });
}

int specmc_validate_problem(const specmc_model_desc* model, const double* xs, const double* ys, int64_t n_points,
                            char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> int {
    if (!model) throw Error(SPECMC_EINVAL, "null model");
    validate_model(*model);
    validate_spectrum(xs, ys, n_points, model->noise == SPECMC_NOISE_POISSON);
    return SPECMC_OK;
  });
}

int specmc_energy_batch(const specmc_model_desc* model, const double* xs, const double* ys, int64_t n_points,
                        const double* thetas, int64_t n_thetas, int32_t device, double* energies_out, char* err,
                        size_t errlen) {
  return guarded(err, errlen, [&]() -> int {
    if (!model || !thetas || !energies_out) throw Error(SPECMC_EINVAL, "null argument");
    if (n_thetas < 1) throw Error(SPECMC_EINVAL, "energy_batch: no parameter vectors");
    specmc_smc_config cfg{std::max<int64_t>(n_thetas, 2), 1, 0.5, 1, 0, 1, device};
    specmc_spectrum sp{xs, ys, n_points};
    RunSpec R = make_runspec(*model, 0, cfg, sp);
    Device dev(device);
    Shape shape = pick_shape(n_points, model->d);
    if ((int64_t)32 * shape.W * shape.PPL < n_points)
      throw Error(SPECMC_EINVAL, "spectrum has more points than the device path supports (8192)");
    const PreparedSpectrum ps = prepare_spectrum(*model, xs, ys, n_points, shape, R.x_shift);
    shape.lay = spectrum_layout(model->family, ps.nz, std::map<int, PreparedSpectrum>{{0, ps}});
    fit_units(shape, model->d);
    const int d = model->d;
    const int64_t T = n_thetas;
    Scratch sc;
    const size_t npt = ps.x.size();
    float* dx = sc.alloc<float>(npt);
    float2* dc = sc.alloc<float2>(npt);
    float2* dy = sc.alloc<float2>(npt);
    int* pk = sc.alloc<int>(d);
    double* pa = sc.alloc<double>(d);
    double* pb = sc.alloc<double>(d);
    double* th = sc.alloc<double>((size_t)d * T);
    double* E = sc.alloc<double>(T);
    float2* rf = sc.alloc<float2>(std::max<size_t>(R.refl.size() / 2, 1));
    int* ro = sc.alloc<int>(std::max<size_t>(R.refl_off.size(), 1));
    GroupState* gst = sc.alloc<GroupState>(1);
    GroupDesc* gd = sc.alloc<GroupDesc>(1);
    int* lst = sc.alloc<int>(2);
    int* pre = sc.alloc<int>(2);
    cudaStream_t st = dev.stream;
    h2d(dx, ps.x.data(), npt, st);
    h2d(reinterpret_cast<float*>(dc), ps.c.data(), 2 * npt, st);
    h2d(reinterpret_cast<float*>(dy), ps.y.data(), 2 * npt, st);
    h2d(pk, R.pk.data(), d, st);
    h2d(pa, R.pa.data(), d, st);
    h2d(pb, R.pb.data(), d, st);
    h2d(reinterpret_cast<float*>(rf), R.refl.data(), R.refl.size(), st);
    h2d(ro, R.refl_off.data(), R.refl_off.size(), st);
    std::vector<double> soa((size_t)d * T);
    for (int64_t c = 0; c < T; ++c)
      for (int i = 0; i < d; ++i) {
        double v = thetas[c * d + i];
        if (is_location(model->family, model->K, i)) v -= R.x_shift;
        soa[(size_t)i * T + c] = v;
      }
    h2d(th, soa.data(), soa.size(), st);
    GroupDesc g;
    std::memset(&g, 0, sizeof(g));
    g.family = model->family;
    g.K = model->K;
    g.d = d;
    g.noise = ps.nz;
    g.T = (int)T;
    g.n = 1;
    g.S = (int)T;
    g.tp = (int)T;  // SoA uploaded with pitch T
    g.sp = (int)T;
    g.max_levels = 1;
    g.n_data = (double)n_points;
    g.N = (int)n_points;
    g.e_a0 = ps.e_a0;
    g.e_a1 = ps.e_a1;
    g.nz_a0 = ps.a0;
    g.nz_a1 = ps.a1;
    g.nz_a2 = ps.a2;
    g.nz_q = ps.q;
    g.x0s = ps.x0s;
    g.inv_range = ps.inv_range;
    g.range = ps.range;
    g.sh_uniform = ps.uniform ? 1 : 0;
    g.x1s = ps.x1s;
    g.y_last = ps.y_last;
    g.s_last = ps.s_last;
    g.spec_x = dx;
    g.spec_c = dc;
    g.spec_y = dy;
    g.pkind = pk;
    g.pa = pa;
    g.pb = pb;
    g.theta[0] = g.theta[1] = th;
    g.E[0] = g.E[1] = E;
    g.st = gst;
    g.refl = rf;
    g.refl_off = ro;
    GroupState s;
    std::memset(&s, 0, sizeof(s));
    s.T_loc = (int)T;
    s.S_loc = (int)T;
    h2d(gd, &g, 1, st);
    h2d(gst, &s, 1, st);
    const int total = (int)((T + shape.U - 1) / shape.U);
    const int hl[2] = {0, 0}, hp[2] = {0, total};
    h2d(lst, hl, 2, st);
    h2d(pre, hp, 2, st);
    cuda_check(launch_energy(model->family, shape, d, gd, lst, pre, 1, total, st), "k_chain<energy>");
    count_launch();
    d2h(energies_out, E, T, st);
    dev.sync();
    return SPECMC_OK;
  });
}

int specmc_ess(const double* lw, int64_t n, int32_t device, double* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> int {
    if (!lw || !out || n < 1) throw Error(SPECMC_EINVAL, "ess: empty input");
    Device dev(device);
    Scratch sc;
    double* d_lw = sc.alloc<double>(n);
    double* d_out = sc.alloc<double>(1);
    int* d_err = sc.alloc<int>(1);
    h2d(d_lw, lw, n, dev.stream);
    cuda_check(launch_unit_ess(d_lw, n, d_out, d_err, dev.stream), "k_unit_ess");
    count_launch();
    int e = 0;
    d2h(out, d_out, 1, dev.stream);
    d2h(&e, d_err, 1, dev.stream);
    dev.sync();
    if (e) throw Error(SPECMC_ERUNTIME, "ess: total weight is zero");
    return SPECMC_OK;
  });
}

int specmc_log_mean_exp(const double* v, int64_t n, int32_t device, double* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> int {
    if (!v || !out || n < 1) throw Error(SPECMC_EINVAL, "log_mean_exp: empty input");
    Device dev(device);
    Scratch sc;
    double* d_v = sc.alloc<double>(n);
    double* d_out = sc.alloc<double>(1);
    h2d(d_v, v, n, dev.stream);
    cuda_check(launch_unit_log_mean_exp(d_v, n, d_out, dev.stream), "k_unit_lme");
    count_launch();
    d2h(out, d_out, 1, dev.stream);
    dev.sync();
    return SPECMC_OK;
  });
}

int specmc_next_beta(const double* E, int64_t n, double n_data, double beta_prev, double ess_target, int32_t device,
                     double* beta_out, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> int {
    if (!E || !beta_out || n < 1) throw Error(SPECMC_EINVAL, "next_beta: empty input");
    if (!(beta_prev < 1.0)) throw Error(SPECMC_EINVAL, "next_beta: beta_prev must be < 1");
    Device dev(device);
    if ((size_t)n > grid_temper_t()) {  // the production grid path (k_tp_emin + k_tp_ess_tree passes)
      if (n > ((int64_t)1 << 31) - 1) throw Error(SPECMC_EINVAL, "next_beta: too many particles");
      GridUnit gu(E, n, n_data, beta_prev, ess_target, 1, dev.stream);
      cuda_check(launch_tp_next_beta(gu.d_g, gu.d_list, 1, gu.nslices, dev.stream), "k_tp_ess_tree");
      count_launch(temper_grid_launches() - 4);
      TemperScratch ts;
      d2h(&ts, gu.d_ts, 1, dev.stream);
      dev.sync();
      if (ts.err) throw Error(SPECMC_ERUNTIME, "ess: total weight is zero");
      *beta_out = ts.beta_next;
      return SPECMC_OK;
    }
    Scratch sc;
    double* d_E = sc.alloc<double>(n);
    double* d_out = sc.alloc<double>(1);
    int* d_err = sc.alloc<int>(1);
    h2d(d_E, E, n, dev.stream);
    cuda_check(launch_unit_next_beta(d_E, n, n_data, beta_prev, ess_target, d_out, d_err, dev.stream),
               "k_unit_next_beta");
    count_launch();
    int e = 0;
    d2h(beta_out, d_out, 1, dev.stream);
    d2h(&e, d_err, 1, dev.stream);
    dev.sync();
    if (e) throw Error(SPECMC_ERUNTIME, "ess: total weight is zero");
    return SPECMC_OK;
  });
}

int specmc_systematic_resample(const double* lw, int64_t n, int64_t S, double u, int32_t device, int64_t* anc_out,
                               char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> int {
    if (!lw || !anc_out || n < 1 || S < 1) throw Error(SPECMC_EINVAL, "systematic_resample: empty input");
    if (n > ((int64_t)1 << 31) - 1) throw Error(SPECMC_EINVAL, "systematic_resample: too many weights");
    Device dev(device);
    if ((size_t)n > grid_temper_t()) {
      // the production grid path (k_tp_wmax, k_tp_wsum, k_tp_offsets, k_tp_resample) with the
      // log-weights as energies: beta 0 -> -1 at n_data 1 gives lw_i = 1.0 * E_i exactly
      if (S > ((int64_t)1 << 31) - 1) throw Error(SPECMC_EINVAL, "systematic_resample: too many targets");
      GridUnit gu(lw, n, 1.0, 0.0, 0.5, S, dev.stream);
      TemperScratch ts;
      std::memset(&ts, 0, sizeof(ts));
      ts.beta_next = -1.0;
      ts.full = 1.0;
      h2d(gu.d_ts, &ts, 1, dev.stream);
      cuda_check(launch_tp_resample(gu.d_g, gu.d_list, 1, gu.nslices, &u, dev.stream), "k_tp_resample");
      count_launch(5);
      std::vector<int> a(S);
      d2h(a.data(), gu.g.anc, S, dev.stream);
      d2h(&ts, gu.d_ts, 1, dev.stream);
      dev.sync();
      if (ts.err) throw Error(SPECMC_ERUNTIME, "systematic_resample: total weight is zero");
      for (int64_t j = 0; j < S; ++j) anc_out[j] = a[j];
      return SPECMC_OK;
    }
    Scratch sc;
    double* d_lw = sc.alloc<double>(n);
    double* d_w = sc.alloc<double>(n);
    int* d_anc = sc.alloc<int>(S);
    int* d_err = sc.alloc<int>(1);
    h2d(d_lw, lw, n, dev.stream);
    cuda_check(launch_unit_resample(d_lw, n, S, u, d_w, d_anc, d_err, dev.stream), "k_unit_resample");
    count_launch();
    std::vector<int> a(S);
    int e = 0;
    d2h(a.data(), d_anc, S, dev.stream);
    d2h(&e, d_err, 1, dev.stream);
    dev.sync();
    if (e) throw Error(SPECMC_ERUNTIME, "systematic_resample: total weight is zero");
    for (int64_t j = 0; j < S; ++j) anc_out[j] = a[j];
    return SPECMC_OK;
  });
}

int specmc_predict_step_size(const double* hist_beta, const double* hist_acc, const double* hist_step, int32_t H,
                             const specmc_model_desc* model, double beta_next, int32_t device, double* out, char* err,
                             size_t errlen) {
  return guarded(err, errlen, [&]() -> int {
    if (!model || !out || H < 0) throw Error(SPECMC_EINVAL, "predict_step_size: bad arguments");
    const int d = model->d;
    // ring layout of the device: entry j at slot j % 5
    std::vector<double> ring((size_t)kHist * (1 + 2 * d), 0.0);
    for (int j = std::max(0, H - kHist); j < H; ++j) {
      double* e = ring.data() + (size_t)(j % kHist) * (1 + 2 * d);
      e[0] = hist_beta[j];
      for (int i = 0; i < d; ++i) {
        e[1 + i] = hist_acc[(size_t)j * d + i];
        e[1 + d + i] = hist_step[(size_t)j * d + i];
      }
    }
    Device dev(device);
    Scratch sc;
    double* d_ring = sc.alloc<double>(ring.size());
    int* d_pk = sc.alloc<int>(d);
    double* d_pa = sc.alloc<double>(d);
    double* d_pb = sc.alloc<double>(d);
    double* d_out = sc.alloc<double>(d);
    h2d(d_ring, ring.data(), ring.size(), dev.stream);
    h2d(d_pk, model->prior_kind, d, dev.stream);
    h2d(d_pa, model->prior_a, d, dev.stream);
    h2d(d_pb, model->prior_b, d, dev.stream);
    cuda_check(launch_unit_predict(d_ring, H, d, beta_next, d_pk, d_pa, d_pb, d_out, dev.stream), "k_unit_predict");
    count_launch();
    d2h(out, d_out, d, dev.stream);
    dev.sync();
    return SPECMC_OK;
  });
}

int specmc_stats_get(specmc_stats* out) {
  if (!out) return SPECMC_EINVAL;
  std::lock_guard<std::mutex> lk(g_stats_mu);
  *out = g_stats;
  return SPECMC_OK;
}

void specmc_stats_reset(void) {
  std::lock_guard<std::mutex> lk(g_stats_mu);
  g_stats = specmc_stats{0, 0.0, 0, 0.0, 0.0};
}

int specmc_launch_shape(int64_t n_points, int32_t* W, int32_t* PPL, int32_t* U) {
  if (n_points < 1) return SPECMC_EINVAL;
  const Shape s = pick_shape(n_points, 0);  // shape for a model that fits any W
  if (W) *W = s.W;
  if (PPL) *PPL = s.PPL;
  if (U) *U = s.U;
  return (int64_t)32 * s.W * s.PPL >= n_points ? SPECMC_OK : SPECMC_EINVAL;
}

int specmc_probe_mufu(int32_t device, double* ops, char* err, size_t errlen) {
  return guarded(err, errlen, [&]() -> int {
    if (!ops) throw Error(SPECMC_EINVAL, "null output");
    Device dev(device);
    int sms = 0;
    cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "attr");
    const int blocks = sms * 8, iters = 4096;
    Scratch sc;
    float* d = sc.alloc<float>(blocks);
    Timer t;
    cuda_check(launch_probe_mufu(d, blocks, 64, dev.stream), "probe warmup");
    cuda_check(cudaEventRecord(t.a, dev.stream), "event");
    cuda_check(launch_probe_mufu(d, blocks, iters, dev.stream), "probe");
    cuda_check(cudaEventRecord(t.b, dev.stream), "event");
    dev.sync();
    count_launch(2);
    *ops = (double)blocks * 256.0 * iters * 8.0 / (t.ms() * 1e-3);
    return SPECMC_OK;
  });
}

int specmc_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

const char* specmc_version(void) { return "specmc_b200 0.1 (sm_100a)"; }

}  // extern "C"
