// dtwgpu.cu -- native host side of the C-ABI (include/dtwgpu.h).
//
// Mirrors the reference's host logic around the hot path and drives the sm_100a
// kernels:
//   * build_matrix's validation order and errors (pairwise.hpp:62-79,
//     time_series.hpp:24-45, distance_matrix.hpp:27-41);
//   * the per-pair window (pair_window, pairwise.hpp:29-33) and a cost-model planner
//     that assigns each pair shape to a kernel family / (G, R) instantiation;
//   * kmedoids' restart loop, RNG, seeding draws, empty-cluster repair, dedupe and
//     refill, convergence test and ordered cost sums, line for line with
//     kmedoids.hpp:33-189 and cluster_result.hpp:40-72, with the O(p k) and
//     O(sum |C|^2) distance reads on the GPU (kmedoids.cu).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <functional>
#include <map>
#include <string>
#include <thread>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "../../include/dtwgpu.h"
#include "dtw_fill.cuh"

using dtwgpu::Family;
using dtwgpu::FillArgs;
using dtwgpu::KernelCfg;

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();
// Zero-filled guard elements before and after the packed series: wavefront lanes that
// run past a series' ends (rows < 1 or > n, band columns outside [1, m]) read valid
// memory and never branch; their cells are masked or unused (dtw_kernels.cuh).
constexpr int64_t kGuard = 4096;

template <class T>
struct DevBuf {
  T* ptr = nullptr;
  size_t cap = 0;  // elements
  cudaError_t reserve(size_t n) {
    if (n <= cap && ptr) return cudaSuccess;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&ptr, std::max<size_t>(n, 1) * sizeof(T));
    if (e == cudaSuccess) cap = std::max<size_t>(n, 1);
    return e;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
  }
};

// SplitMix64 / restart_stream, rng.hpp:10-41.
struct SplitMix64 {
  uint64_t state;
  explicit SplitMix64(uint64_t s) : state(s) {}
  uint64_t next() {
    uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double next_double() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  uint64_t next_below(uint64_t n) {
    return static_cast<uint64_t>((static_cast<unsigned __int128>(next()) *
                                  static_cast<unsigned __int128>(n)) >> 64);
  }
};
SplitMix64 restart_stream(uint64_t seed, uint64_t restart) {
  SplitMix64 mixer(seed);
  const uint64_t base = mixer.next();
  return SplitMix64(base + (restart + 1) * 0xD1B54A32D192ED03ULL);
}

struct Shape {
  int64_t n, m, hw;  // n >= m; hw effective (unlimited -> n)
  bool operator<(const Shape& o) const {
    return std::tie(n, m, hw) < std::tie(o.n, o.m, o.hw);
  }
};

struct PlanClass {
  KernelCfg cfg;
  std::vector<int64_t> slots;  // empty + range mode when uniform
  double cost = 0;
  int64_t max_n = 0;
  double cells = 0;  // in-band cells of the class (diagnostics: dtwg_last_plan)
  // Strip family: strips per pair (uniform) or prefix sums over `slots` (ragged)
  int strips_per_pair = 0;
  std::vector<int64_t> strip_base;
};

int64_t row_off(int64_t i, int64_t p) { return i * p - i * (i + 1) / 2; }

// In-band cells of one pair.
int64_t pair_cells(int64_t n, int64_t m, int64_t hw) {
  if (hw >= n) return n * m;
  const int64_t T = std::max<int64_t>(n - hw - 1, 0);
  const int64_t a = std::min(T, m);
  const int64_t left = a * (a + 1) / 2 + std::max<int64_t>(T - m, 0) * m;
  const int64_t S = std::max<int64_t>(m - hw - 1, 0);
  return n * m - left - S * (S + 1) / 2;
}

// ---- planner ------------------------------------------------------------------------
// Candidate instantiations with their measured throughput in computed lane-cells per
// ns on one B200 (tools/sweep.py, profiles/round1_sweep.md): the cost of a shape is
// the lane-cells a configuration computes (band waste, wavefront fill/drain, padding
// columns, masked rows all included) divided by that rate. Multi-pass Full fills with
// few lanes pay an extra per-pass boundary-column cost (measured on c4).
struct Cand {
  int G, R;
  double rate;  // computed lane-cells / ns
  int P = 1;    // band family: pairs per lane group
  int TR = 2;   // full family: rows per step
  bool ring = false;  // band family: shared-memory y ring
  int U = 1;          // ring variant: units per lane
};
const Cand kFull[] = {{2, 23, 1913},         {2, 23, 2141, 1, 4},  {4, 12, 2026},
                      {4, 12, 1956, 1, 4},   {8, 8, 1804},         {8, 8, 1700, 1, 4},
                      {16, 8, 1800},         {16, 16, 1850},       {16, 16, 1850, 1, 4},
                      {32, 4, 1300},         {32, 8, 1650},        {32, 12, 1950},
                      {32, 15, 2000},        {32, 15, 2150, 1, 4}, {32, 16, 2100},
                      {32, 16, 2050, 1, 4}};
const Cand kBand[] = {{16, 7, 1500},    {16, 9, 1600},    {16, 11, 1700},  {16, 13, 1800},
                      {32, 3, 1000},    {32, 5, 1250},    {32, 7, 1490},   {32, 9, 1500},
                      {32, 13, 1450},   {32, 3, 600, 2},  {32, 5, 600, 2},  {32, 7, 700, 2},
                      {8, 16, 1900, 1, 2, true},  {8, 26, 2221, 1, 2, true},
                      {16, 8, 1500, 1, 2, true},  {16, 14, 2105, 1, 2, true},
                      {32, 6, 1300, 1, 2, true},
                      // ring with U units per lane (c2 sweep, round 1)
                      {8, 26, 2286, 1, 2, true, 3}, {8, 26, 2198, 1, 2, true, 5},
                      {16, 14, 2166, 1, 2, true, 3}, {16, 13, 2128, 1, 2, true, 2},
                      // wide bands (512-slot ring)
                      {16, 20, 2186, 1, 2, true, 3}, {16, 26, 2220, 1, 2, true, 3},
                      {32, 20, 2150, 1, 2, true, 3}, {32, 26, 2170, 1, 2, true, 3}};

// fp32 mode: the cell is FADD FMUL FMNMX3 FADD, so the Full family runs ~2.15x the fp64
// rate while the Band family (shuffle-heavy per step) gains ~1.45x (measured on c2 after the warp-uniform renormalisation).
constexpr double kFp32Full = 2.15, kFp32Band = 1.45;

// Masked Full fills: rows where the strip lies entirely inside the band run the plain
// cell; rows crossing a band edge run the masked cell at 1.79x the cost (least-squares fit
// over hw = 101..400 at n = m = 1000, tools: exp/band_rates.py, profiles/round1_sweep.md).
constexpr double kMaskedRowCost = 1.79;

double full_cost(const Shape& s, const Cand& c, bool mask, bool fp32) {
  const int64_t W = (int64_t)c.G * c.R;
  const int64_t npass = (s.m + W - 1) / W;
  double cells = 0;
  for (int64_t p = 0; p < npass; ++p) {
    const int64_t c0 = p * W;
    int64_t rs = 1, re = s.n;
    if (mask) {
      rs = std::max<int64_t>(1, c0 + 1 - s.hw);
      re = std::min<int64_t>(s.n, c0 + W + s.hw);
    }
    // TR rows per step, G-1 steps of wavefront fill/drain
    const int64_t rows = ((re - rs + c.TR) / c.TR) * c.TR;
    double eff_rows = double(rows);
    if (mask) {
      const int64_t fast = std::max<int64_t>(
          0, std::min<int64_t>(re, c0 + 1 + s.hw) - std::max<int64_t>(rs, c0 + W - s.hw) + 1);
      const int64_t masked = std::max<int64_t>(0, rows - fast);
      eff_rows = double(rows - masked) + kMaskedRowCost * double(masked);
    }
    cells += (eff_rows + c.TR * (c.G - 1)) * double(W);
  }
  double rate = c.rate * (fp32 ? kFp32Full : 1.0);
  if (npass > 1) {  // boundary-column round trips per pass (measured on c4)
    // The per-group boundary columns stay in L2 up to ~n = 1500 (c5, L = 1000 sweeps);
    // the c4-measured penalties apply beyond.
    const bool l2_resident = s.n <= 1500;
    if (c.G == 2) rate *= c.TR == 4 ? 0.68 : 0.59;
    else if (c.G == 4) rate *= (c.TR == 4 && l2_resident) ? 1.05 : (c.TR == 4 ? 0.92 : 0.78);
    else if (c.G == 8) rate *= c.TR == 4 ? 1.0 : 0.95;
  }
  return cells / rate;
}

double band_cost(const Shape& s, const Cand& c, bool fp32) {
  // fp32 / fp64 throughput ratios measured on c2 (G=8 R=26: 1.69 ring, 2.06 units;
  // G=16 R=14: 1.52 ring, 1.72 units; register-rotation band 1.45)
  const double f32 = c.ring ? (c.U > 1 ? 1.9 : 1.6) : kFp32Band;
  // wavefront fill/drain: one step per unit of the group
  return double(s.n + c.G * c.U - 1) * double(c.G * c.R) / (c.rate * (fp32 ? f32 : 1.0));
}

KernelCfg choose_cfg_model(const Shape& s, bool fp32, double* cost_out, int64_t count, int sms);

// Planner entry: a forced (family, G, R) wins when it can legally run the shape.
KernelCfg choose_cfg(const dtwg_ctx* ctx, const Shape& s, bool fp32, double* cost_out,
                     int64_t count = 0);

// Fraction of the GPU a class of `count` pairs can keep busy with G lanes per pair: about
// 8 warps per SM are needed to cover the cell chain (c1: 4950 pairs fill it with G = 32,
// not with G = 4 -- 1765 against 946 GCUPS). count = 0: unknown (ragged classes).
double fill_factor(int64_t count, int G, int sms) {
  if (count <= 0) return 1.0;
  const double warps = double(count) * G / 32.0;
  return std::min(1.0, warps / (8.0 * sms));
}

KernelCfg choose_cfg_model(const Shape& s, bool fp32, double* cost_out, int64_t count = 0,
                           int sms = 148) {
  KernelCfg best{Family::Full, 32, 16, true, fp32};
  double bc = 1e300;
  const bool mask = s.hw < s.n - 1;  // a band that excludes some cell
  for (const Cand& c : kFull) {
    const double cst = full_cost(s, c, mask, fp32) / fill_factor(count, c.G, sms);
    if (cst < bc) {
      bc = cst;
      best = KernelCfg{Family::Full, c.G, c.R, mask, fp32, -1, 1, c.TR};
    }
  }
  if (mask) {
    const int64_t K = 2 * s.hw + 1;
    for (const Cand& c : kBand) {
      if ((int64_t)c.G * c.R < K) continue;
      const double cst = band_cost(s, c, fp32) / fill_factor(count, c.G, sms);
      if (cst < bc) {
        bc = cst;
        // static kill position: fp64 everywhere, fp32 for the unit-ring variant
        const bool static_kr = !fp32 || (c.ring && c.U > 1);
        best = KernelCfg{Family::Band, c.G, c.R, false, fp32, static_kr ? (int)(K % c.R) : -1,
                         c.P, 2, c.ring, c.U};
      }
    }
  }
  if (cost_out) *cost_out = bc;
  return best;
}

const char* family_name(Family f) {
  return f == Family::Full ? "full" : (f == Family::Band ? "band" : "strip");
}

}  // namespace

struct dtwg_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // Side streams: the kernel classes of a ragged fill run concurrently so one class's
  // tail wave overlaps the next class's work.
  static constexpr int kAux = 4;
  cudaStream_t aux[kAux] = {};
  cudaEvent_t aux_done[kAux] = {};
  cudaEvent_t fork = nullptr;
  float last_fill_ms = 0.f;
  uint64_t launches = 0;
  std::string last_error;
  std::string last_plan;
  int64_t err_i = -1, err_j = -1;
  int force_family = -1, force_G = 0, force_R = 0;  // dtwg_force_kernel (tests/diagnostics)

  // cached plan of the last ragged fill (planning 12.5M pairs costs ~1 s of host time)
  struct PlanKey {
    int64_t hw, sb, se;
    int auto_widen;
    bool fp32;
    int force_family, force_G, force_R;
    bool operator==(const PlanKey& o) const {
      return hw == o.hw && sb == o.sb && se == o.se && auto_widen == o.auto_widen &&
             fp32 == o.fp32 && force_family == o.force_family && force_G == o.force_G &&
             force_R == o.force_R;
    }
  };
  bool plan_valid = false;
  PlanKey plan_key{};
  std::vector<int64_t> plan_lens;
  std::vector<PlanClass> plan_cache;
  bool list_uploaded = false;

  // series
  int64_t p = 0;
  std::vector<int64_t> h_offsets;
  std::vector<int64_t> h_len;
  bool uniform = true;
  DevBuf<double> d_samples;
  DevBuf<float> d_samples32;
  bool have32 = false;
  DevBuf<int64_t> d_offsets;
  DevBuf<double> d_scratch;
  DevBuf<int64_t> d_list;
  // Strip family: strip prefix sums, progress counters, item counters, boundary columns
  DevBuf<int64_t> d_strip_base;
  DevBuf<int> d_prog;
  DevBuf<unsigned long long> d_work;
  DevBuf<double> d_cols;
  // multi-device context (dtwg_create_multi): one child context per further device;
  // this context drives the first
  std::vector<dtwg_ctx*> devs;
  // fused fill + all-gather over peer memory (dtwg_exchange_*): other ranks' resident
  // matrices opened through CUDA IPC
  std::vector<double*> peers;
  bool exchange_open = false;
  // streamed build (large outputs): copy stream, two pinned staging buffers
  cudaStream_t copy_stream = nullptr;
  double* h_stage[2] = {nullptr, nullptr};
  size_t stage_elems = 0;
  // +inf-padded copies of the series for the band family (kBandPad each side)
  DevBuf<double> d_bsamples;
  DevBuf<float> d_bsamples32;
  DevBuf<int64_t> d_boffsets;
  bool have_band64 = false, have_band32 = false;

  // resident matrix
  int64_t mat_p = 0;
  DevBuf<double> d_cond;
  bool cond_valid = false;
  DevBuf<double> d_square;
  bool square_valid = false;  // the sweep view is ready (square expanded, or condensed mode)
  bool km_condensed = false;  // sweeps read the condensed matrix (square does not fit)
  // k-medoids restart workers: contexts on the same device (own stream and sweep buffers)
  // that read this context's matrix (km_src), so independent restarts run concurrently
  std::vector<dtwg_ctx*> kmw;
  const dtwg_ctx* km_src = nullptr;
  DevBuf<int> d_flag;

  // k-medoids sweep statistics (dtwg_km_stats): device time and algorithmic bytes of the
  // assignment and candidate-sum kernels (8 bytes per distance read).
  cudaEvent_t km0 = nullptr, km1 = nullptr;
  double km_assign_ms = 0, km_update_ms = 0, km_assign_bytes = 0, km_update_bytes = 0;
  int64_t km_sweeps = 0;

  // k-medoids scratch
  DevBuf<int64_t> d_medoids, d_assign, d_best_member, d_cb;
  DevBuf<double> d_dist, d_nearest, d_best_sum;
  DevBuf<uint8_t> d_chosen;
  DevBuf<int32_t> d_members;
  DevBuf<int32_t> d_sil_cls;

  int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    last_error = buf;
    return code;
  }
  int cuda_fail(cudaError_t e, const char* what) {
    return fail(DTWG_CUDA_ERROR, "%s: %s", what, cudaGetErrorString(e));
  }
};

#define CU(call, what)                                   \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return ctx->cuda_fail(e_, what); \
  } while (0)

namespace {

KernelCfg choose_cfg(const dtwg_ctx* ctx, const Shape& s, bool fp32, double* cost_out,
                     int64_t count) {
  const bool mask = s.hw < s.n - 1;
  if (ctx->force_family >= 0) {
    // 0: full (2 rows/step), 1: band P=1, 2: band P=2, 3: full (4 rows/step), 4: band ring,
    // 10 + U: band ring with U units per lane
    const int ff = ctx->force_family;
    if (ff == 5) {  // strip family (long pairs spread over warps), G = 32, 4 rows per step
      KernelCfg f{Family::Strip, 32, ctx->force_R, mask, fp32, -1, 1, 4};
      if (dtwgpu::fill_cfg_supported(f)) {
        if (cost_out) *cost_out = 1.0;
        return f;
      }
    }
    const bool band = ff == 1 || ff == 2 || ff == 4 || ff > 10;
    KernelCfg f{band ? Family::Band : Family::Full, ctx->force_G, ctx->force_R,
                band ? false : mask, fp32,
                (band && (!fp32 || ff > 10) && ctx->force_R > 0) ? (int)((2 * s.hw + 1) % ctx->force_R)
                                                                  : -1,
                ff == 2 ? 2 : 1, ff == 3 ? 4 : 2, ff == 4 || ff > 10, ff > 10 ? ff - 10 : 1};
    const bool ok = dtwgpu::fill_cfg_supported(f) &&
                    (f.family == Family::Full ||
                     (mask && f.R >= 2 && (int64_t)f.G * f.R >= 2 * s.hw + 1));
    if (ok) {
      if (cost_out) *cost_out = 1.0;
      return f;
    }
  }
  return choose_cfg_model(s, fp32, cost_out, count, ctx->num_sms);
}

// time_series.hpp:24-33 per-series checks (ids are the caller's; see dtwgpu.hpp).
int validate_series(dtwg_ctx* ctx, const double* samples, const int64_t* offsets, int64_t p) {
  for (int64_t i = 0; i < p; ++i) {
    const int64_t b = offsets[i], e = offsets[i + 1];
    if (e < b) return ctx->fail(DTWG_INVALID_ARGUMENTS, "offsets must be non-decreasing");
    if (e == b) return ctx->fail(DTWG_INVALID_SERIES, "series #%lld: series is empty", (long long)i);
    for (int64_t t = b; t < e; ++t) {
      if (!std::isfinite(samples[t]))
        return ctx->fail(DTWG_INVALID_SERIES, "series #%lld: series contains a non-finite sample",
                         (long long)i);
    }
  }
  return DTWG_OK;
}

// pairwise.hpp:70-79: first infeasible pair in row-major order.
int check_band(dtwg_ctx* ctx, int64_t hw, int auto_widen) {
  ctx->err_i = ctx->err_j = -1;
  if (auto_widen || hw < 0 || ctx->p < 2) return DTWG_OK;
  const auto mm = std::minmax_element(ctx->h_len.begin(), ctx->h_len.end());
  if (*mm.second - *mm.first <= hw) return DTWG_OK;  // every gap fits
  const int64_t p = ctx->p;
  for (int64_t i = 0; i < p; ++i) {
    for (int64_t j = i + 1; j < p; ++j) {
      const int64_t a = ctx->h_len[i], b = ctx->h_len[j];
      const int64_t gap = a > b ? a - b : b - a;
      if (gap > hw) {
        ctx->err_i = i;
        ctx->err_j = j;
        return ctx->fail(DTWG_BAND_INFEASIBLE,
                         "pair (%lld, %lld): half-width %lld is narrower than the length gap of "
                         "%lld (lengths %lld and %lld)",
                         (long long)i, (long long)j, (long long)hw, (long long)gap, (long long)a,
                         (long long)b);
      }
    }
  }
  return DTWG_OK;
}

Shape shape_of(const dtwg_ctx* ctx, int64_t a, int64_t b, int64_t hw, int auto_widen) {
  int64_t la = ctx->h_len[a], lb = ctx->h_len[b];
  Shape s;
  s.n = std::max(la, lb);
  s.m = std::min(la, lb);
  if (hw < 0) {
    s.hw = s.n;
  } else {
    const int64_t gap = s.n - s.m;
    s.hw = (auto_widen && gap > hw) ? gap : hw;
  }
  if (s.hw > s.n) s.hw = s.n;  // a band at least max(n,m) wide is the unlimited window
  return s;
}

// A Full-family class of few, long pairs leaves most of the GPU idle (one lane group per
// pair, passes in sequence). Such classes become Strip classes: every column strip of
// every pair is a work item for a full warp, pipelined along the pair (dtw_strip_kernel).
// Rule: at most 4 pairs per SM with >= 2 strips per pair, or at most 16 pairs per SM with
// >= 8 strips per pair (c1's 4950 pairs of 2 strips stay Full: 1763 against 776 GCUPS).
// m_uniform < 0: ragged class (lengths per slot).
constexpr int kStripR = 15;
void maybe_strip(dtwg_ctx* ctx, PlanClass& pc, int64_t count, int64_t m_uniform) {
  if (count <= 0) return;
  const bool forced = pc.cfg.family == Family::Strip;  // dtwg_force_kernel(5, ., R)
  KernelCfg sc = pc.cfg;
  if (!forced) {
    if (pc.cfg.family != Family::Full || ctx->force_family >= 0) return;
    if (count > 16 * (int64_t)ctx->num_sms) return;  // enough pairs to fill the GPU already
    sc = KernelCfg{Family::Strip, 32, kStripR, pc.cfg.mask, pc.cfg.fp32, -1, 1, 4};
    if (!dtwgpu::fill_cfg_supported(sc)) return;
  }
  const int64_t W = 32 * (int64_t)sc.R;
  const int64_t min_strips = count <= 4 * (int64_t)ctx->num_sms ? 2 : 8;  // strips per pair
  if (m_uniform >= 0) {
    const int64_t S = (m_uniform + W - 1) / W;
    if (S < min_strips && !forced) return;
    pc.strips_per_pair = (int)S;
  } else {
    std::vector<int64_t> base(count + 1, 0);
    const int64_t p = ctx->p;
    for (int64_t q = 0; q < count; ++q) {
      const int64_t slot = pc.slots[q];
      int64_t lo = 0, hi = p - 1;
      while (lo < hi) {
        const int64_t mid = (lo + hi + 1) / 2;
        if (row_off(mid, p) <= slot) lo = mid;
        else hi = mid - 1;
      }
      const int64_t i = lo, j = i + 1 + (slot - row_off(i, p));
      const int64_t m = std::min(ctx->h_len[i], ctx->h_len[j]);
      base[q + 1] = base[q] + (m + W - 1) / W;
    }
    if (base[count] < min_strips * count && !forced) return;
    pc.strip_base = std::move(base);
  }
  pc.cfg = sc;
}

std::vector<PlanClass> make_plan(dtwg_ctx* ctx, int64_t hw, int auto_widen, bool fp32,
                                 int64_t sb, int64_t se) {
  std::vector<PlanClass> plan;
  if (se <= sb) return plan;
  const int64_t p = ctx->p;
  if (ctx->uniform) {
    PlanClass pc;
    const Shape s = shape_of(ctx, 0, 1, hw, auto_widen);
    pc.cfg = choose_cfg(ctx, s, fp32, &pc.cost, se - sb);
    pc.max_n = s.n;
    plan.push_back(pc);
    maybe_strip(ctx, plan[0], se - sb, s.m);
    return plan;
  }
  // Ragged dataset: classify every pair by shape (memoised on (n, m)), then bucket the
  // slots of each class by (passes, rows) with a counting sort -- longest first (LPT),
  // and pairs of equal pass count and row count adjacent, so the lane groups of one warp
  // run in lockstep. O(pairs); no comparison sort.
  int64_t maxlen = 0;
  for (int64_t t = 0; t < p; ++t) maxlen = std::max(maxlen, ctx->h_len[t]);
  const int64_t L1 = maxlen + 1;
  std::vector<int> cls_tab;
  const bool use_tab = L1 * L1 <= (int64_t)1 << 26;
  if (use_tab) cls_tab.assign((size_t)(L1 * L1), -1);
  std::map<Shape, int> cls_of_shape;
  std::map<std::tuple<int, int, int, bool, int, int, int>, int> cls_of_cfg;
  auto class_of = [&](int64_t a, int64_t b, Shape& s) -> int {
    s = shape_of(ctx, a, b, hw, auto_widen);
    int* slotp = use_tab ? &cls_tab[(size_t)(s.n * L1 + s.m)] : nullptr;
    if (slotp && *slotp >= 0) return *slotp;
    if (!slotp) {
      auto it = cls_of_shape.find(s);
      if (it != cls_of_shape.end()) return it->second;
    }
    double cst = 0;
    const KernelCfg cfg = choose_cfg(ctx, s, fp32, &cst);
    const auto key = std::make_tuple((int)cfg.family * 2 + (int)cfg.ring + 4 * cfg.U, cfg.G, cfg.R, cfg.mask,
                                     cfg.kr, cfg.P, cfg.TR);
    int cls;
    auto ic = cls_of_cfg.find(key);
    if (ic == cls_of_cfg.end()) {
      PlanClass pc;
      pc.cfg = cfg;
      plan.push_back(pc);
      cls = (int)plan.size() - 1;
      cls_of_cfg[key] = cls;
    } else {
      cls = ic->second;
    }
    if (slotp) *slotp = cls;
    else cls_of_shape[s] = cls;
    return cls;
  };
  auto bucket_of = [&](int cls, const Shape& s) -> int64_t {
    const KernelCfg& cc = plan[cls].cfg;
    const int64_t W = (int64_t)cc.G * cc.R;
    const int64_t npass = cc.family == Family::Full ? (s.m + W - 1) / W : 1;
    return npass * L1 + s.n;  // larger = earlier
  };
  int64_t i0;
  {
    int64_t lo = 0, hi = p - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) / 2;
      if (row_off(mid, p) <= sb) lo = mid;
      else hi = mid - 1;
    }
    i0 = lo;
  }
  const int64_t j0 = i0 + 1 + (sb - row_off(i0, p));
  // pass 1: classes, bucket counts
  std::vector<std::vector<int64_t>> counts;
  {
    int64_t i = i0, j = j0;
    Shape s;
    for (int64_t slot = sb; slot < se; ++slot) {
      const int cls = class_of(i, j, s);
      if ((int)counts.size() <= cls) counts.resize(cls + 1);
      const int64_t bk = bucket_of(cls, s);
      if ((int64_t)counts[cls].size() <= bk) counts[cls].resize(bk + 1, 0);
      counts[cls][bk]++;
      plan[cls].max_n = std::max(plan[cls].max_n, s.n);
      plan[cls].cost += double(s.n) * double(s.m);
      plan[cls].cells += double(pair_cells(s.n, s.m, s.hw));
      if (++j == p) {
        ++i;
        j = i + 1;
      }
    }
  }
  // descending bucket order -> start offsets
  std::vector<std::vector<int64_t>> start(plan.size());
  for (size_t c = 0; c < plan.size(); ++c) {
    auto& cn = counts[c];
    start[c].assign(cn.size(), 0);
    int64_t acc = 0;
    for (int64_t b = (int64_t)cn.size() - 1; b >= 0; --b) {
      start[c][b] = acc;
      acc += cn[b];
    }
    plan[c].slots.resize(acc);
  }
  // pass 2: place slots (and remember each one's shorter length)
  std::vector<std::vector<int32_t>> mkey(plan.size());
  for (size_t c = 0; c < plan.size(); ++c) mkey[c].resize(plan[c].slots.size());
  {
    int64_t i = i0, j = j0;
    Shape s;
    for (int64_t slot = sb; slot < se; ++slot) {
      const int cls = class_of(i, j, s);
      const int64_t at = start[cls][bucket_of(cls, s)]++;
      plan[cls].slots[at] = slot;
      mkey[cls][at] = (int32_t)s.m;
      if (++j == p) {
        ++i;
        j = i + 1;
      }
    }
  }
  // pass 3: inside each (passes, rows) bucket, order by the shorter length too, so the
  // lane groups of a warp mostly share one (n, m) -- same band geometry, same masked
  // steps, same trip counts. Counting sort per bucket (start[c][b] now marks its end).
  {
    std::vector<int64_t> cnt(L1 + 1);
    std::vector<int64_t> tmp;
    for (size_t c = 0; c < plan.size(); ++c) {
      auto& cn = counts[c];
      auto& sl = plan[c].slots;
      auto& mk = mkey[c];
      for (int64_t b = 0; b < (int64_t)cn.size(); ++b) {
        const int64_t e = start[c][b], a = e - cn[b];
        if (e - a < 2) continue;
        std::fill(cnt.begin(), cnt.end(), 0);
        for (int64_t t = a; t < e; ++t) cnt[mk[t]]++;
        int64_t acc = a;
        for (int64_t v = L1; v >= 0; --v) {  // descending m
          const int64_t k = cnt[v];
          cnt[v] = acc;
          acc += k;
        }
        tmp.assign(sl.begin() + a, sl.begin() + e);
        for (int64_t t = a; t < e; ++t) sl[cnt[mk[t]]++] = tmp[t - a];
      }
    }
  }
  for (auto& pc : plan) maybe_strip(ctx, pc, (int64_t)pc.slots.size(), -1);
  return plan;
}

int ensure_fp32(dtwg_ctx* ctx) {
  if (ctx->have32) return DTWG_OK;
  // the whole guarded buffer, guards included (zeros stay zeros)
  const int64_t total = ctx->h_offsets[ctx->p] + 2 * kGuard;
  CU(ctx->d_samples32.reserve(total), "cudaMalloc samples32");
  CU(dtwgpu::launch_to_f32(ctx->d_samples.ptr, total, ctx->d_samples32.ptr, ctx->stream),
     "to f32");
  ctx->launches++;
  ctx->have32 = true;
  return DTWG_OK;
}

// Band-family copy of the series: each series surrounded by kBandPad +inf samples,
// scattered on the device from the packed (guarded) series.
int ensure_band(dtwg_ctx* ctx, bool fp32) {
  if (fp32 ? ctx->have_band32 : ctx->have_band64) return DTWG_OK;
  const int64_t p = ctx->p;
  const int64_t pad = dtwgpu::kBandPad;
  std::vector<int64_t> boff(p + 1);
  int64_t pos = pad;
  for (int64_t i = 0; i < p; ++i) {
    boff[i] = pos;
    pos += ctx->h_len[i] + 2 * pad;
  }
  boff[p] = pos;
  const int64_t total = pos + pad;
  CU(ctx->d_boffsets.reserve(p + 1), "cudaMalloc boffsets");
  CU(cudaMemcpyAsync(ctx->d_boffsets.ptr, boff.data(), (p + 1) * 8, cudaMemcpyHostToDevice,
                     ctx->stream),
     "H2D boffsets");
  void* out;
  if (fp32) {
    CU(ctx->d_bsamples32.reserve(total), "cudaMalloc bsamples32");
    out = ctx->d_bsamples32.ptr;
  } else {
    CU(ctx->d_bsamples.reserve(total), "cudaMalloc bsamples");
    out = ctx->d_bsamples.ptr;
  }
  CU(dtwgpu::launch_band_pad(ctx->d_samples.ptr + kGuard, ctx->d_offsets.ptr, ctx->d_boffsets.ptr,
                             p, pad, out, fp32, ctx->stream),
     "band pad");
  ctx->launches++;
  (fp32 ? ctx->have_band32 : ctx->have_band64) = true;
  return DTWG_OK;
}

int run_fill(dtwg_ctx* ctx, int64_t hw, int auto_widen, int precision, int64_t sb, int64_t se,
             double* d_out, int64_t out_base, bool sync = true) {
  const bool fp32 = precision == DTWG_FP32;
  if (fp32) {
    const int rc = ensure_fp32(ctx);
    if (rc) return rc;
  }
  const dtwg_ctx::PlanKey key{hw, sb, se, auto_widen, fp32, ctx->force_family, ctx->force_G,
                              ctx->force_R};
  if (!(ctx->plan_valid && ctx->plan_key == key)) {
    ctx->plan_cache = make_plan(ctx, hw, auto_widen, fp32, sb, se);
    ctx->plan_key = key;
    ctx->plan_valid = true;
    ctx->list_uploaded = false;
  }
  std::vector<PlanClass>& plan = ctx->plan_cache;
  ctx->last_plan.clear();
  for (auto& pc : plan) {
    if (pc.cfg.family == Family::Band) {
      const int rc = ensure_band(ctx, fp32);
      if (rc) return rc;
      break;
    }
  }
  CU(cudaEventRecord(ctx->ev0, ctx->stream), "event");
  // Upload all class lists in one buffer.
  size_t total_list = 0;
  for (auto& pc : plan) total_list += pc.slots.size();
  if (total_list && !ctx->list_uploaded) {
    ctx->list_uploaded = true;
    CU(ctx->d_list.reserve(total_list), "cudaMalloc list");
    size_t pos = 0;
    for (auto& pc : plan) {
      if (!pc.slots.empty())
        CU(cudaMemcpyAsync(ctx->d_list.ptr + pos, pc.slots.data(), pc.slots.size() * 8,
                           cudaMemcpyHostToDevice, ctx->stream),
           "H2D list");
      pos += pc.slots.size();
    }
  }
  // Per-class scratch (multi-pass Full classes may run concurrently).
  const bool concurrent = plan.size() > 1;
  if (concurrent && !ctx->aux[0]) {
    for (int a = 0; a < dtwg_ctx::kAux; ++a) {
      CU(cudaStreamCreateWithFlags(&ctx->aux[a], cudaStreamNonBlocking), "aux stream");
      CU(cudaEventCreateWithFlags(&ctx->aux_done[a], cudaEventDisableTiming), "aux event");
    }
    CU(cudaEventCreateWithFlags(&ctx->fork, cudaEventDisableTiming), "fork event");
  }
  std::vector<int64_t> blocks_of(plan.size()), scratch_off(plan.size(), -1);
  int64_t scratch_total = 0;
  // Strip classes: offsets into the strip buffers
  std::vector<int64_t> sb_off(plan.size(), -1), prog_off(plan.size(), 0), cols_off(plan.size(), 0);
  int64_t sb_total = 0, prog_total = 0, cols_total = 0;
  int n_strip_cls = 0;
  for (size_t c = 0; c < plan.size(); ++c) {
    const PlanClass& pc = plan[c];
    const int64_t count = ctx->uniform ? (se - sb) : (int64_t)pc.slots.size();
    const int bps = dtwgpu::fill_blocks_per_sm(pc.cfg);
    const int64_t groups_per_block = dtwgpu::kThreads / pc.cfg.G;
    const int64_t items_per_block =
        groups_per_block * (pc.cfg.family == Family::Band ? pc.cfg.P : 1);
    int64_t blocks = (int64_t)ctx->num_sms * bps;
    blocks = std::min<int64_t>(blocks, (count + items_per_block - 1) / items_per_block);
    blocks_of[c] = std::max<int64_t>(blocks, 1);
    if (pc.cfg.family == Family::Strip && count > 0) {
      blocks_of[c] = (int64_t)ctx->num_sms * bps;  // persistent: items are strips
      const int64_t strips =
          pc.strip_base.empty() ? count * pc.strips_per_pair : pc.strip_base[count];
      if (!pc.strip_base.empty()) {
        sb_off[c] = sb_total;
        sb_total += count + 1;
      }
      prog_off[c] = prog_total;
      prog_total += strips;
      cols_off[c] = cols_total;
      cols_total += count * 2 * (pc.max_n + 2);
      ++n_strip_cls;
      continue;
    }
    const int64_t W = (int64_t)pc.cfg.G * pc.cfg.R;
    const bool multipass = pc.cfg.family == Family::Full &&
                           (ctx->uniform ? (ctx->h_len[0] > W) : true);
    if (multipass && count > 0) {
      scratch_off[c] = scratch_total;
      scratch_total += (pc.max_n + 2) * blocks_of[c] * groups_per_block;
    }
  }
  if (scratch_total) CU(ctx->d_scratch.reserve((size_t)scratch_total), "cudaMalloc scratch");
  if (n_strip_cls) {
    CU(ctx->d_prog.reserve((size_t)prog_total), "cudaMalloc prog");
    CU(ctx->d_cols.reserve((size_t)cols_total), "cudaMalloc cols");
    CU(ctx->d_work.reserve((size_t)plan.size()), "cudaMalloc work");
    CU(cudaMemsetAsync(ctx->d_prog.ptr, 0, prog_total * sizeof(int), ctx->stream), "memset prog");
    CU(cudaMemsetAsync(ctx->d_work.ptr, 0, plan.size() * sizeof(unsigned long long), ctx->stream),
       "memset work");
    if (sb_total) {
      CU(ctx->d_strip_base.reserve((size_t)sb_total), "cudaMalloc strip_base");
      for (size_t c = 0; c < plan.size(); ++c)
        if (sb_off[c] >= 0)
          CU(cudaMemcpyAsync(ctx->d_strip_base.ptr + sb_off[c], plan[c].strip_base.data(),
                             plan[c].strip_base.size() * 8, cudaMemcpyHostToDevice, ctx->stream),
             "H2D strip_base");
    }
  }
  if (concurrent) {  // fork after the list upload
    CU(cudaEventRecord(ctx->fork, ctx->stream), "fork event");
    for (int a = 0; a < dtwg_ctx::kAux; ++a)
      CU(cudaStreamWaitEvent(ctx->aux[a], ctx->fork, 0), "fork");
  }
  size_t pos = 0;
  int next_aux = 0;
  for (size_t c = 0; c < plan.size(); ++c) {
    auto& pc = plan[c];
    if (!dtwgpu::fill_cfg_supported(pc.cfg))
      return ctx->fail(DTWG_INTERNAL, "no kernel for %s G=%d R=%d", family_name(pc.cfg.family),
                       pc.cfg.G, pc.cfg.R);
    const int64_t count = ctx->uniform ? (se - sb) : (int64_t)pc.slots.size();
    if (count == 0) continue;
    const int bps = dtwgpu::fill_blocks_per_sm(pc.cfg);
    const int64_t blocks = blocks_of[c];
    FillArgs a{};
    a.samples = ctx->d_samples.ptr + kGuard;
    a.samples32 = fp32 ? ctx->d_samples32.ptr + kGuard : nullptr;
    a.bsamples = ctx->have_band64 ? ctx->d_bsamples.ptr : nullptr;
    a.bsamples32 = ctx->have_band32 ? ctx->d_bsamples32.ptr : nullptr;
    a.boffsets = (ctx->have_band64 || ctx->have_band32) ? ctx->d_boffsets.ptr : nullptr;
    a.offsets = ctx->d_offsets.ptr;
    a.p = ctx->p;
    a.half_width = hw;
    a.auto_widen = auto_widen;
    a.list = ctx->uniform ? nullptr : ctx->d_list.ptr + pos;
    a.begin = ctx->uniform ? sb : 0;
    a.count = count;
    a.out_base = out_base;
    a.out = d_out;
    if (scratch_off[c] >= 0) {
      a.scratch = ctx->d_scratch.ptr + scratch_off[c];
      a.scratch_stride = pc.max_n + 2;
    }
    if (ctx->exchange_open && d_out - out_base == ctx->d_cond.ptr) {  // resident, global slots
      a.n_peer = (int)ctx->peers.size();
      for (int r = 0; r < a.n_peer; ++r) a.peer_out[r] = ctx->peers[r];
      a.peer_base = 0;
    }
    if (pc.cfg.family == Family::Strip) {
      a.strip_base = sb_off[c] >= 0 ? ctx->d_strip_base.ptr + sb_off[c] : nullptr;
      a.strips_per_pair = pc.strips_per_pair;
      a.work = ctx->d_work.ptr + c;
      a.prog = ctx->d_prog.ptr + prog_off[c];
      a.cols = ctx->d_cols.ptr + cols_off[c];
      a.col_stride = pc.max_n + 2;
    }
    cudaStream_t st = concurrent ? ctx->aux[next_aux++ % dtwg_ctx::kAux] : ctx->stream;
    CU(dtwgpu::launch_fill(pc.cfg, a, (int)blocks, st), "fill launch");
    ctx->launches++;
    char buf[200];
    char krs[32] = "";
    if (pc.cfg.family == Family::Band)
      snprintf(krs, sizeof(krs), "%s,P=%d%s%s",
               pc.cfg.kr >= 0 ? (",kr=" + std::to_string(pc.cfg.kr)).c_str() : "", pc.cfg.P,
               pc.cfg.ring ? ",ring" : "",
               pc.cfg.U > 1 ? (",U=" + std::to_string(pc.cfg.U)).c_str() : "");
    if (pc.cfg.family != Family::Band) snprintf(krs, sizeof(krs), ",T=%d", pc.cfg.TR);
    char cellsb[32] = "";
    if (pc.cells > 0) snprintf(cellsb, sizeof(cellsb), " cells=%.4g", pc.cells);
    snprintf(buf, sizeof(buf), "%s%s[G=%d,R=%d%s%s%s] pairs=%lld%s blocks=%lld(%d/SM)",
             ctx->last_plan.empty() ? "" : "; ", family_name(pc.cfg.family), pc.cfg.G, pc.cfg.R,
             pc.cfg.mask ? ",mask" : "", fp32 ? ",fp32" : "", krs, (long long)count, cellsb,
             (long long)blocks, bps);
    ctx->last_plan += buf;
    pos += pc.slots.size();
  }
  if (concurrent) {  // join
    for (int a = 0; a < dtwg_ctx::kAux; ++a) {
      CU(cudaEventRecord(ctx->aux_done[a], ctx->aux[a]), "join event");
      CU(cudaStreamWaitEvent(ctx->stream, ctx->aux_done[a], 0), "join");
    }
  }
  CU(cudaEventRecord(ctx->ev1, ctx->stream), "event");
  if (!sync) return DTWG_OK;
  CU(cudaEventSynchronize(ctx->ev1), "fill sync");
  CU(cudaEventElapsedTime(&ctx->last_fill_ms, ctx->ev0, ctx->ev1), "elapsed");
  return DTWG_OK;
}

int ensure_resident(dtwg_ctx* ctx, int64_t p) {
  const size_t total = (size_t)(p * (p - 1) / 2);
  CU(ctx->d_cond.reserve(total), "cudaMalloc condensed");
  ctx->mat_p = p;
  ctx->square_valid = false;
  return DTWG_OK;
}

// distance_matrix.hpp:34-38 over slots [sb, se) of the resident matrix (se < 0: all).
int validate_resident(dtwg_ctx* ctx, int64_t sb = 0, int64_t se = -1) {
  const int64_t total = ctx->mat_p * (ctx->mat_p - 1) / 2;
  if (se < 0) se = total;
  if (se <= sb) return DTWG_OK;
  CU(ctx->d_flag.reserve(1), "cudaMalloc flag");
  CU(cudaMemsetAsync(ctx->d_flag.ptr, 0, sizeof(int), ctx->stream), "memset");
  CU(dtwgpu::launch_validate_condensed(ctx->d_cond.ptr + sb, se - sb, ctx->d_flag.ptr,
                                       ctx->stream),
     "validate");
  ctx->launches++;
  int bad = 0;
  CU(cudaMemcpyAsync(&bad, ctx->d_flag.ptr, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream),
     "D2H flag");
  CU(cudaStreamSynchronize(ctx->stream), "sync");
  if (bad) {
    ctx->cond_valid = false;
    return ctx->fail(DTWG_DISTANCE_MATRIX_INVALID, "entries must be finite and non-negative");
  }
  ctx->cond_valid = sb == 0 && se == total;
  return DTWG_OK;
}

// The sweeps read a dense p x p square (contiguous rows) when it fits in HBM next to the
// condensed matrix -- p up to ~140 000 on a 180 GB B200 -- and the condensed matrix
// itself beyond that (or with DTWGPU_KM_CONDENSED=1); both give identical results.
const double* km_matrix(const dtwg_ctx* ctx) {
  const dtwg_ctx* m = ctx->km_src ? ctx->km_src : ctx;
  return m->km_condensed ? m->d_cond.ptr : m->d_square.ptr;
}
bool km_is_cond(const dtwg_ctx* ctx) {
  return (ctx->km_src ? ctx->km_src : ctx)->km_condensed;
}

int ensure_square(dtwg_ctx* ctx) {
  if (ctx->square_valid) return DTWG_OK;
  if (!ctx->cond_valid) return ctx->fail(DTWG_INVALID_ARGUMENTS, "no resident distance matrix");
  const int64_t p = ctx->mat_p;
  const char* force = std::getenv("DTWGPU_KM_CONDENSED");
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  const double need = double(p) * double(p) * 8.0 - double(ctx->d_square.cap) * 8.0;
  ctx->km_condensed = (force && force[0] == '1') || need > 0.85 * double(free_b);
  if (ctx->km_condensed) {
    ctx->d_square.release();
    ctx->square_valid = true;
    return DTWG_OK;
  }
  CU(ctx->d_square.reserve((size_t)(p * p)), "cudaMalloc square");
  if (p >= 2) {
    CU(dtwgpu::launch_expand_square(ctx->d_cond.ptr, p, ctx->d_square.ptr, ctx->stream),
       "expand");
    ctx->launches++;
  } else {
    CU(cudaMemsetAsync(ctx->d_square.ptr, 0, sizeof(double), ctx->stream), "memset");
  }
  ctx->square_valid = true;
  return DTWG_OK;
}

// ---- k-medoids host loop ------------------------------------------------------------
struct KmState {
  dtwg_ctx* ctx;
  int64_t p, k;
  std::vector<int64_t> assignment;
  std::vector<double> dist;
};

int km_assign(KmState& S, const std::vector<int64_t>& medoids) {
  dtwg_ctx* ctx = S.ctx;
  CU(cudaMemcpyAsync(ctx->d_medoids.ptr, medoids.data(), medoids.size() * 8,
                     cudaMemcpyHostToDevice, ctx->stream),
     "H2D medoids");
  CU(cudaEventRecord(ctx->km0, ctx->stream), "event");
  CU(dtwgpu::launch_assign(km_matrix(ctx), km_is_cond(ctx), S.p, ctx->d_medoids.ptr,
                           (int64_t)medoids.size(),
                           ctx->d_assign.ptr, ctx->d_dist.ptr, ctx->stream),
     "assign");
  CU(cudaEventRecord(ctx->km1, ctx->stream), "event");
  ctx->launches++;
  S.assignment.resize(S.p);
  S.dist.resize(S.p);
  CU(cudaMemcpyAsync(S.assignment.data(), ctx->d_assign.ptr, S.p * 8, cudaMemcpyDeviceToHost,
                     ctx->stream),
     "D2H assignment");
  CU(cudaMemcpyAsync(S.dist.data(), ctx->d_dist.ptr, S.p * 8, cudaMemcpyDeviceToHost,
                     ctx->stream),
     "D2H dist");
  CU(cudaStreamSynchronize(ctx->stream), "sync");
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, ctx->km0, ctx->km1), "elapsed");
  ctx->km_assign_ms += ms;
  ctx->km_assign_bytes += 8.0 * (double)S.p * (double)medoids.size() + 16.0 * (double)S.p;
  return DTWG_OK;
}

// cluster_result.hpp:65-72 -- ascending-j sequential sum on the host.
double km_cost(const KmState& S) {
  double total = 0.0;
  for (int64_t j = 0; j < S.p; ++j) total += S.dist[j];
  return total;
}

// kmedoids.hpp:84-139.
int km_update(KmState& S, const std::vector<int64_t>& medoids, std::vector<int64_t>& updated) {
  dtwg_ctx* ctx = S.ctx;
  const int64_t p = S.p, k = (int64_t)medoids.size();
  // Stable bucket by lower_bound slot (kmedoids.hpp:88-92).
  std::vector<int64_t> cb(k + 1, 0);
  std::vector<int64_t> slot_of(p);
  for (int64_t j = 0; j < p; ++j) {
    const int64_t c = std::lower_bound(medoids.begin(), medoids.end(), S.assignment[j]) -
                      medoids.begin();
    slot_of[j] = c;
    cb[c + 1]++;
  }
  for (int64_t c = 0; c < k; ++c) cb[c + 1] += cb[c];
  std::vector<int32_t> members(p);
  {
    std::vector<int64_t> fill(cb.begin(), cb.end() - 1);
    for (int64_t j = 0; j < p; ++j) members[fill[slot_of[j]]++] = (int32_t)j;
  }
  CU(cudaMemcpyAsync(ctx->d_members.ptr, members.data(), p * 4, cudaMemcpyHostToDevice,
                     ctx->stream),
     "H2D members");
  CU(cudaMemcpyAsync(ctx->d_cb.ptr, cb.data(), (k + 1) * 8, cudaMemcpyHostToDevice, ctx->stream),
     "H2D cb");
  CU(cudaEventRecord(ctx->km0, ctx->stream), "event");
  CU(dtwgpu::launch_update(km_matrix(ctx), km_is_cond(ctx), p, ctx->d_members.ptr, ctx->d_cb.ptr, k,
                           ctx->d_best_member.ptr, ctx->d_best_sum.ptr, ctx->stream),
     "update");
  CU(cudaEventRecord(ctx->km1, ctx->stream), "event");
  ctx->launches += 2;
  std::vector<int64_t> best(k);
  CU(cudaMemcpyAsync(best.data(), ctx->d_best_member.ptr, k * 8, cudaMemcpyDeviceToHost,
                     ctx->stream),
     "D2H best");
  CU(cudaStreamSynchronize(ctx->stream), "sync");
  {
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, ctx->km0, ctx->km1), "elapsed");
    double sq = 0;
    for (int64_t c = 0; c < k; ++c) sq += double(cb[c + 1] - cb[c]) * double(cb[c + 1] - cb[c]);
    ctx->km_update_ms += ms;
    ctx->km_update_bytes += 8.0 * sq + 12.0 * (double)p;
    ctx->km_sweeps += 1;
  }

  updated.assign(k, 0);
  for (int64_t c = 0; c < k; ++c) {
    if (cb[c] == cb[c + 1]) {  // kmedoids.hpp:97-109: worst-served non-medoid, strict >
      int64_t worst = medoids[c];
      double worst_d = -1.0;
      for (int64_t j = 0; j < p; ++j) {
        if (std::find(medoids.begin(), medoids.end(), j) != medoids.end()) continue;
        const double d = S.dist[j];  // == D(j, assignment[j])
        if (d > worst_d) {
          worst_d = d;
          worst = j;
        }
      }
      updated[c] = worst;
      continue;
    }
    updated[c] = best[c];
  }
  std::sort(updated.begin(), updated.end());
  updated.erase(std::unique(updated.begin(), updated.end()), updated.end());
  if ((int64_t)updated.size() < k) {  // kmedoids.hpp:127-137
    std::vector<char> used(p, 0);
    for (int64_t m : updated) used[m] = 1;
    for (int64_t j = 0; j < p && (int64_t)updated.size() < k; ++j) {
      if (!used[j]) {
        updated.push_back(j);
        used[j] = 1;
      }
    }
    std::sort(updated.begin(), updated.end());
  }
  return DTWG_OK;
}

// kmedoids.hpp:33-79.
int km_seeds(KmState& S, int64_t k, SplitMix64& rng, std::vector<int64_t>& medoids) {
  dtwg_ctx* ctx = S.ctx;
  const int64_t p = S.p;
  medoids.clear();
  std::vector<uint8_t> chosen(p, 0);
  std::vector<double> nearest(p, kInf);
  CU(cudaMemsetAsync(ctx->d_chosen.ptr, 0, p, ctx->stream), "memset chosen");
  CU(cudaMemcpyAsync(ctx->d_nearest.ptr, nearest.data(), p * 8, cudaMemcpyHostToDevice,
                     ctx->stream),
     "H2D nearest");
  int64_t current = (int64_t)rng.next_below((uint64_t)p);
  while ((int64_t)medoids.size() < k) {
    medoids.push_back(current);
    chosen[current] = 1;
    if ((int64_t)medoids.size() == k) break;
    CU(cudaMemcpyAsync(ctx->d_chosen.ptr + current, &chosen[current], 1, cudaMemcpyHostToDevice,
                       ctx->stream),
       "H2D chosen");
    CU(dtwgpu::launch_nearest_update(km_matrix(ctx), km_is_cond(ctx), p, current, ctx->d_chosen.ptr,
                                     ctx->d_nearest.ptr, ctx->stream),
       "nearest");
    ctx->launches++;
    CU(cudaMemcpyAsync(nearest.data(), ctx->d_nearest.ptr, p * 8, cudaMemcpyDeviceToHost,
                       ctx->stream),
       "D2H nearest");
    CU(cudaStreamSynchronize(ctx->stream), "sync");
    double total = 0.0;
    for (int64_t j = 0; j < p; ++j) {
      if (chosen[j]) continue;
      total += nearest[j];
    }
    int64_t next = p;
    if (total > 0.0) {
      const double target = rng.next_double() * total;
      double acc = 0.0;
      for (int64_t j = 0; j < p; ++j) {
        if (chosen[j]) continue;
        acc += nearest[j];
        if (acc > target) {
          next = j;
          break;
        }
      }
    }
    if (next == p) {
      for (int64_t j = 0; j < p; ++j) {
        if (!chosen[j]) {
          next = j;
          break;
        }
      }
    }
    current = next;
  }
  std::sort(medoids.begin(), medoids.end());
  return DTWG_OK;
}

int km_reserve(dtwg_ctx* ctx, int64_t p, int64_t k) {
  if (!ctx->km0) {
    CU(cudaEventCreate(&ctx->km0), "event");
    CU(cudaEventCreate(&ctx->km1), "event");
  }
  CU(ctx->d_medoids.reserve(k), "malloc");
  CU(ctx->d_assign.reserve(p), "malloc");
  CU(ctx->d_dist.reserve(p), "malloc");
  CU(ctx->d_nearest.reserve(p), "malloc");
  CU(ctx->d_chosen.reserve(p), "malloc");
  CU(ctx->d_members.reserve(p), "malloc");
  CU(ctx->d_cb.reserve(k + 1), "malloc");
  CU(ctx->d_best_member.reserve(k), "malloc");
  CU(ctx->d_best_sum.reserve(k + p), "malloc");
  return DTWG_OK;
}

}  // namespace

// =====================================================================================
// C-ABI
// =====================================================================================
extern "C" {

int dtwg_create(int device, dtwg_ctx** out) {
  if (!out) return DTWG_INVALID_ARGUMENTS;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0 || device < 0 || device >= n) {
    cudaGetLastError();
    return DTWG_NO_DEVICE;
  }
  if (cudaSetDevice(device) != cudaSuccess) return DTWG_NO_DEVICE;
  auto* ctx = new dtwg_ctx();
  ctx->device = device;
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess) {
    delete ctx;
    return DTWG_CUDA_ERROR;
  }
  ctx->own_stream = true;
  *out = ctx;
  return DTWG_OK;
}

int dtwg_create_multi(const int* devices, int n_devices, dtwg_ctx** out) {
  if (!out || !devices || n_devices < 1) return DTWG_INVALID_ARGUMENTS;
  *out = nullptr;
  dtwg_ctx* ctx = nullptr;
  int rc = dtwg_create(devices[0], &ctx);
  if (rc) return rc;
  for (int d = 1; d < n_devices; ++d) {
    dtwg_ctx* c = nullptr;
    rc = dtwg_create(devices[d], &c);
    if (rc) {
      dtwg_destroy(ctx);
      return rc;
    }
    ctx->devs.push_back(c);
  }
  *out = ctx;
  return DTWG_OK;
}

int dtwg_device_count(const dtwg_ctx* ctx) { return ctx ? 1 + (int)ctx->devs.size() : 0; }

int dtwg_visible_devices(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void dtwg_destroy(dtwg_ctx* ctx) {
  if (!ctx) return;
  for (dtwg_ctx* c : ctx->devs) dtwg_destroy(c);
  ctx->devs.clear();
  for (dtwg_ctx* c : ctx->kmw) dtwg_destroy(c);
  ctx->kmw.clear();
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  ctx->d_samples.release();
  ctx->d_samples32.release();
  ctx->d_bsamples.release();
  ctx->d_bsamples32.release();
  ctx->d_boffsets.release();
  ctx->d_offsets.release();
  ctx->d_scratch.release();
  ctx->d_list.release();
  ctx->d_cond.release();
  ctx->d_square.release();
  ctx->d_flag.release();
  ctx->d_medoids.release();
  ctx->d_assign.release();
  ctx->d_best_member.release();
  ctx->d_cb.release();
  ctx->d_dist.release();
  ctx->d_nearest.release();
  ctx->d_best_sum.release();
  ctx->d_chosen.release();
  ctx->d_members.release();
  ctx->d_sil_cls.release();
  ctx->d_strip_base.release();
  ctx->d_prog.release();
  ctx->d_work.release();
  ctx->d_cols.release();
  dtwg_exchange_close(ctx);
  for (double*& h : ctx->h_stage)
    if (h) cudaFreeHost(h);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  for (int a = 0; a < dtwg_ctx::kAux; ++a) {
    if (ctx->aux[a]) cudaStreamDestroy(ctx->aux[a]);
    if (ctx->aux_done[a]) cudaEventDestroy(ctx->aux_done[a]);
  }
  if (ctx->fork) cudaEventDestroy(ctx->fork);
  if (ctx->km0) cudaEventDestroy(ctx->km0);
  if (ctx->km1) cudaEventDestroy(ctx->km1);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* dtwg_last_error(const dtwg_ctx* ctx) { return ctx ? ctx->last_error.c_str() : ""; }

void dtwg_last_error_pair(const dtwg_ctx* ctx, int64_t* i, int64_t* j) {
  if (i) *i = ctx ? ctx->err_i : -1;
  if (j) *j = ctx ? ctx->err_j : -1;
}

int dtwg_set_stream(dtwg_ctx* ctx, void* stream) {
  if (!ctx) return DTWG_INVALID_ARGUMENTS;
  cudaSetDevice(ctx->device);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  if (stream) {
    ctx->stream = (cudaStream_t)stream;
    ctx->own_stream = false;
  } else {
    CU(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "stream");
    ctx->own_stream = true;
  }
  return DTWG_OK;
}

int dtwg_synchronize(dtwg_ctx* ctx) {
  if (!ctx) return DTWG_INVALID_ARGUMENTS;
  CU(cudaStreamSynchronize(ctx->stream), "sync");
  return DTWG_OK;
}

// Starts the upload (async H2D on the context's stream) without the per-series checks;
// dtwg_upload_series adds them, dtwg_build_matrix overlaps them with the fill.
static int upload_begin(dtwg_ctx* ctx, const double* samples, const int64_t* offsets,
                        int64_t p) {
  cudaSetDevice(ctx->device);
  if (p <= 0) return ctx->fail(DTWG_EMPTY_DATASET, "dataset contains no series");
  if (!offsets || (offsets[p] > 0 && !samples))
    return ctx->fail(DTWG_INVALID_ARGUMENTS, "null series buffers");
  for (int64_t i = 0; i < p; ++i)
    if (offsets[i + 1] < offsets[i])
      return ctx->fail(DTWG_INVALID_ARGUMENTS, "offsets must be non-decreasing");
  ctx->p = 0;  // nothing uploaded is usable until the series validate
  ctx->h_offsets.assign(offsets, offsets + p + 1);
  const int64_t base = offsets[0];
  for (auto& o : ctx->h_offsets) o -= base;
  ctx->h_len.resize(p);
  ctx->uniform = true;
  for (int64_t i = 0; i < p; ++i) {
    ctx->h_len[i] = offsets[i + 1] - offsets[i];
    if (ctx->h_len[i] != ctx->h_len[0]) ctx->uniform = false;
  }
  const int64_t n = ctx->h_offsets[p];
  ctx->have32 = false;
  ctx->have_band64 = ctx->have_band32 = false;
  // The plan depends only on the series lengths (and window/precision/range): keep it
  // when a new upload has the same lengths.
  if (ctx->plan_valid && ctx->plan_lens != ctx->h_len) ctx->plan_valid = false;
  if (!ctx->plan_valid) ctx->plan_lens = ctx->h_len;
  CU(ctx->d_samples.reserve(n + 2 * kGuard), "cudaMalloc samples");
  CU(ctx->d_offsets.reserve(p + 1), "cudaMalloc offsets");
  CU(cudaMemsetAsync(ctx->d_samples.ptr, 0, kGuard * sizeof(double), ctx->stream), "memset");
  CU(cudaMemsetAsync(ctx->d_samples.ptr + kGuard + n, 0, kGuard * sizeof(double), ctx->stream),
     "memset");
  CU(cudaMemcpyAsync(ctx->d_samples.ptr + kGuard, samples + base, n * sizeof(double),
                     cudaMemcpyHostToDevice, ctx->stream),
     "H2D samples");
  CU(cudaMemcpyAsync(ctx->d_offsets.ptr, ctx->h_offsets.data(), (p + 1) * sizeof(int64_t),
                     cudaMemcpyHostToDevice, ctx->stream),
     "H2D offsets");
  ctx->p = p;
  return DTWG_OK;
}

int dtwg_upload_series(dtwg_ctx* ctx, const double* samples, const int64_t* offsets, int64_t p) {
  if (!ctx) return DTWG_INVALID_ARGUMENTS;
  int rc = upload_begin(ctx, samples, offsets, p);
  if (rc) return rc;
  // time_series.hpp:24-33 on the host while the (pinned) copy runs
  rc = validate_series(ctx, samples, offsets, p);
  CU(cudaStreamSynchronize(ctx->stream), "sync");
  if (rc) {
    ctx->p = 0;  // nothing uploaded is usable
    return rc;
  }
  return DTWG_OK;
}

int dtwg_fill_slots(dtwg_ctx* ctx, int64_t half_width, int auto_widen, int precision,
                    int64_t slot_begin, int64_t slot_end, double* d_out) {
  if (!ctx) return DTWG_INVALID_ARGUMENTS;
  cudaSetDevice(ctx->device);
  if (ctx->p <= 0) return ctx->fail(DTWG_EMPTY_DATASET, "dataset contains no series");
  if (precision != DTWG_FP64 && precision != DTWG_FP32)
    return ctx->fail(DTWG_INVALID_ARGUMENTS, "precision must be 0 (fp64) or 1 (fp32)");
  const int64_t total = ctx->p * (ctx->p - 1) / 2;
  if (slot_begin < 0 || slot_end > total || slot_begin > slot_end)
    return ctx->fail(DTWG_INVALID_ARGUMENTS, "slot range [%lld, %lld) outside [0, %lld)",
                     (long long)slot_begin, (long long)slot_end, (long long)total);
  int rc = check_band(ctx, half_width, auto_widen);
  if (rc) return rc;
  int64_t out_base = slot_begin;
  if (!d_out) {
    rc = ensure_resident(ctx, ctx->p);
    if (rc) return rc;
    d_out = ctx->d_cond.ptr;
    out_base = 0;
    ctx->cond_valid = false;
  }
  rc = run_fill(ctx, half_width, auto_widen, precision, slot_begin, slot_end, d_out, out_base);
  if (rc) return rc;
  if (d_out == ctx->d_cond.ptr && slot_begin == 0 && slot_end == total) ctx->cond_valid = true;
  return DTWG_OK;
}

int dtwg_count_cells(dtwg_ctx* ctx, int64_t half_width, int auto_widen, int64_t sb, int64_t se,
                     uint64_t* cells) {
  if (!ctx || !cells) return DTWG_INVALID_ARGUMENTS;
  const int64_t p = ctx->p;
  uint64_t total = 0;
  if (se > sb && p >= 2) {
    if (ctx->uniform) {
      const Shape s = shape_of(ctx, 0, 1, half_width, auto_widen);
      total = (uint64_t)pair_cells(s.n, s.m, s.hw) * (uint64_t)(se - sb);
    } else {
      int64_t lo = 0, hi = p - 1;
      while (lo < hi) {
        const int64_t mid = (lo + hi + 1) / 2;
        if (row_off(mid, p) <= sb) lo = mid;
        else hi = mid - 1;
      }
      int64_t i = lo, j = lo + 1 + (sb - row_off(lo, p));
      for (int64_t s = sb; s < se; ++s) {
        const Shape sh = shape_of(ctx, i, j, half_width, auto_widen);
        total += (uint64_t)pair_cells(sh.n, sh.m, sh.hw);
        if (++j == p) {
          ++i;
          j = i + 1;
        }
      }
    }
  }
  *cells = total;
  return DTWG_OK;
}

int dtwg_last_fill_ms(dtwg_ctx* ctx, float* ms) {
  if (!ctx || !ms) return DTWG_INVALID_ARGUMENTS;
  *ms = ctx->last_fill_ms;
  return DTWG_OK;
}

int dtwg_measure_cell_peak(dtwg_ctx* ctx, int precision, double* cells_per_s) {
  if (!ctx || !cells_per_s) return DTWG_INVALID_ARGUMENTS;
  cudaSetDevice(ctx->device);
  CU(dtwgpu::measure_cell_peak(ctx->stream, ctx->num_sms, precision == DTWG_FP32, cells_per_s),
     "cell peak");
  return DTWG_OK;
}

int dtwg_silhouette(dtwg_ctx* ctx, const int64_t* medoids, int64_t k, const int64_t* assignment,
                    int64_t p_assign, double* silhouette_out, double* mean_out) {
  if (!ctx || !medoids || !assignment) return DTWG_INVALID_ARGUMENTS;
  cudaSetDevice(ctx->device);
  if (!ctx->cond_valid) return ctx->fail(DTWG_INVALID_ARGUMENTS, "no resident distance matrix");
  const int64_t p = ctx->mat_p;
  // validation.hpp:33-49, in the reference's order
  if (p_assign != p)
    return ctx->fail(DTWG_INVALID_ARGUMENTS, "clustering covers %lld series, matrix has %lld",
                     (long long)p_assign, (long long)p);
  if (k < 2)
    return ctx->fail(DTWG_SINGLE_CLUSTER_UNDEFINED, "silhouette scores are undefined for a single cluster; request k >= 2");
  std::vector<int64_t> cb(k + 1, 0);
  std::vector<int32_t> cls(p);
  for (int64_t j = 0; j < p; ++j) {
    const int64_t* it = std::lower_bound(medoids, medoids + k, assignment[j]);
    if (it == medoids + k || *it != assignment[j])
      return ctx->fail(DTWG_INVALID_ARGUMENTS, "series %lld is assigned to a non-medoid",
                       (long long)j);
    cls[j] = (int32_t)(it - medoids);
    cb[cls[j] + 1]++;
  }
  for (int64_t c = 0; c < k; ++c) cb[c + 1] += cb[c];
  std::vector<int32_t> members(p);
  {
    std::vector<int64_t> fill(cb.begin(), cb.end() - 1);
    for (int64_t j = 0; j < p; ++j) members[fill[cls[j]]++] = (int32_t)j;
  }
  int rc = ensure_square(ctx);
  if (rc) return rc;
  rc = km_reserve(ctx, p, k);
  if (rc) return rc;
  CU(ctx->d_sil_cls.reserve(p), "malloc");
  CU(cudaMemcpyAsync(ctx->d_members.ptr, members.data(), p * 4, cudaMemcpyHostToDevice, ctx->stream),
     "H2D members");
  CU(cudaMemcpyAsync(ctx->d_cb.ptr, cb.data(), (k + 1) * 8, cudaMemcpyHostToDevice, ctx->stream),
     "H2D cb");
  CU(cudaMemcpyAsync(ctx->d_sil_cls.ptr, cls.data(), p * 4, cudaMemcpyHostToDevice, ctx->stream),
     "H2D cls");
  CU(dtwgpu::launch_silhouette(km_matrix(ctx), km_is_cond(ctx), p, ctx->d_members.ptr, ctx->d_cb.ptr,
                               ctx->d_sil_cls.ptr, k, ctx->d_dist.ptr, ctx->stream),
     "silhouette");
  ctx->launches++;
  std::vector<double> sil(p);
  CU(cudaMemcpyAsync(sil.data(), ctx->d_dist.ptr, p * 8, cudaMemcpyDeviceToHost, ctx->stream),
     "D2H silhouette");
  CU(cudaStreamSynchronize(ctx->stream), "sync");
  // validation.hpp:54-77: the mean sums cluster by cluster, members ascending, singletons
  // skipped (adding their 0 would not change the bits anyway).
  double sum = 0.0;
  for (int64_t c = 0; c < k; ++c) {
    if (cb[c + 1] - cb[c] == 1) continue;
    for (int64_t q = cb[c]; q < cb[c + 1]; ++q) sum += sil[members[q]];
  }
  if (silhouette_out) std::copy(sil.begin(), sil.end(), silhouette_out);
  if (mean_out) *mean_out = sum / (double)p;
  return DTWG_OK;
}

int dtwg_km_stats(dtwg_ctx* ctx, double* out, int reset) {
  if (!ctx || !out) return DTWG_INVALID_ARGUMENTS;
  out[0] = (double)ctx->km_sweeps;
  out[1] = ctx->km_assign_ms;
  out[2] = ctx->km_assign_bytes;
  out[3] = ctx->km_update_ms;
  out[4] = ctx->km_update_bytes;
  if (reset) {
    ctx->km_sweeps = 0;
    ctx->km_assign_ms = ctx->km_update_ms = ctx->km_assign_bytes = ctx->km_update_bytes = 0;
  }
  return DTWG_OK;
}

int dtwg_force_kernel(dtwg_ctx* ctx, int family, int G, int R) {
  if (!ctx) return DTWG_INVALID_ARGUMENTS;
  ctx->force_family = family;
  ctx->force_G = G;
  ctx->force_R = R;
  return DTWG_OK;
}

uint64_t dtwg_launch_count(const dtwg_ctx* ctx) { return ctx ? ctx->launches : 0; }

const char* dtwg_last_plan(const dtwg_ctx* ctx) { return ctx ? ctx->last_plan.c_str() : ""; }

// Large outputs (c3: 2.3 GB): the fill runs in slot chunks on the compute stream while
// finished chunks go D2H on a copy stream into two pinned staging buffers, and host
// threads copy each staged chunk into the caller's (pageable) buffer -- so the transfer,
// and the page faults of a fresh output array, hide behind the remaining fill.
namespace {
constexpr int64_t kStreamMinBytes = 1ll << 20;       // staged D2H from 1 MB of output
constexpr int64_t kChunkFillMinBytes = 256ll << 20;  // chunked fill from 256 MB
constexpr int64_t kStreamChunk = 4ll << 20;  // slots per chunk (32 MB)
// Tests shrink both through the environment to exercise many chunks on small inputs.
int64_t env_or(const char* name, int64_t dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::strtoll(v, nullptr, 10) : dflt;
}

void parallel_copy(double* dst, const double* src, int64_t n) {
  const int nt = (int)std::min<int64_t>(8, std::max<int64_t>(1, n >> 18));
  if (nt == 1) {
    std::memcpy(dst, src, n * sizeof(double));
    return;
  }
  std::vector<std::thread> th;
  const int64_t per = (n + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    const int64_t b = t * per, e = std::min(n, b + per);
    if (b < e) th.emplace_back([=] { std::memcpy(dst + b, src + b, (e - b) * sizeof(double)); });
  }
  for (auto& x : th) x.join();
}
}  // namespace

// Slots [sb, se) of the matrix (all when se < 0) into out[sb, se).
static int build_streamed(dtwg_ctx* ctx, int64_t hw, int auto_widen, int precision, double* out,
                          bool chunk_fill, int64_t sb = 0, int64_t se = -1,
                          const std::function<int()>& host_work = {}) {
  const int64_t all = ctx->p * (ctx->p - 1) / 2;
  if (se < 0) se = all;
  const int64_t total = se - sb;  // slots of this range
  const int64_t chunk = std::max<int64_t>(1, env_or("DTWGPU_STREAM_CHUNK", kStreamChunk));
  int rc = check_band(ctx, hw, auto_widen);
  if (rc) return rc;
  rc = ensure_resident(ctx, ctx->p);
  if (rc) return rc;
  ctx->cond_valid = false;
  if (!ctx->copy_stream)
    CU(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking), "copy stream");
  if (ctx->stage_elems < (size_t)chunk) {
    for (double*& h : ctx->h_stage) {
      if (h) cudaFreeHost(h);
      h = nullptr;
      CU(cudaMallocHost(&h, chunk * sizeof(double)), "pinned staging");
    }
    ctx->stage_elems = chunk;
  }
  const int64_t nchunk = (total + chunk - 1) / chunk;
  if (nchunk == 0) return DTWG_OK;
  std::vector<cudaEvent_t> filled(nchunk, nullptr), copied(nchunk, nullptr);
  auto cleanup = [&] {
    for (auto& e : filled) if (e) cudaEventDestroy(e);
    for (auto& e : copied) if (e) cudaEventDestroy(e);
  };
  auto fail = [&](int code) { cleanup(); return code; };
  for (int64_t c = 0; c < nchunk; ++c) {
    if (cudaEventCreateWithFlags(&filled[c], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&copied[c], cudaEventDisableTiming) != cudaSuccess)
      return fail(ctx->fail(DTWG_CUDA_ERROR, "event create"));
  }
  float fill_ms = 0;
  cudaEvent_t t0 = nullptr;
  cudaEventCreate(&t0);
  cudaEventRecord(t0, ctx->stream);
  if (!chunk_fill) {  // one fill (its plan stays cached); the D2H is still staged
    rc = run_fill(ctx, hw, auto_widen, precision, sb, se, ctx->d_cond.ptr, 0, false);
    if (rc) return fail(rc);
  }
  for (int64_t c = 0; c < nchunk; ++c) {
    if (chunk_fill) {
      const int64_t b = sb + c * chunk, e = std::min(se, b + chunk);
      rc = run_fill(ctx, hw, auto_widen, precision, b, e, ctx->d_cond.ptr, 0, false);
      if (rc) return fail(rc);
    }
    if (cudaEventRecord(filled[c], ctx->stream) != cudaSuccess)
      return fail(ctx->fail(DTWG_CUDA_ERROR, "event record"));
  }
  cudaEventRecord(ctx->ev1, ctx->stream);
  if (host_work) {  // e.g. the per-series checks, overlapping the fill just enqueued
    rc = host_work();
    if (rc) {
      cudaStreamSynchronize(ctx->stream);
      return fail(rc);
    }
  }
  auto enqueue_copy = [&](int64_t c) -> int {
    const int64_t b = sb + c * chunk, e = std::min(se, b + chunk);
    if (cudaStreamWaitEvent(ctx->copy_stream, filled[c], 0) != cudaSuccess ||
        cudaMemcpyAsync(ctx->h_stage[c & 1], ctx->d_cond.ptr + b, (e - b) * sizeof(double),
                        cudaMemcpyDeviceToHost, ctx->copy_stream) != cudaSuccess ||
        cudaEventRecord(copied[c], ctx->copy_stream) != cudaSuccess)
      return ctx->fail(DTWG_CUDA_ERROR, "D2H chunk");
    return DTWG_OK;
  };
  for (int64_t c = 0; c < std::min<int64_t>(2, nchunk); ++c) {
    rc = enqueue_copy(c);
    if (rc) return fail(rc);
  }
  for (int64_t c = 0; c < nchunk; ++c) {
    const cudaError_t err = cudaEventSynchronize(copied[c]);
    if (err != cudaSuccess) return fail(ctx->cuda_fail(err, "D2H chunk sync"));
    const int64_t b = sb + c * chunk, e = std::min(se, b + chunk);
    parallel_copy(out + b, ctx->h_stage[c & 1], e - b);
    if (c + 2 < nchunk) {
      rc = enqueue_copy(c + 2);
      if (rc) return fail(rc);
    }
  }
  if (cudaEventElapsedTime(&fill_ms, t0, ctx->ev1) == cudaSuccess) ctx->last_fill_ms = fill_ms;
  cudaEventDestroy(t0);
  cleanup();
  return validate_resident(ctx, sb, se);  // distance_matrix.hpp:34-38
}

// ---- one context, several devices ---------------------------------------------------
extern "C++" {
// Cell-balanced contiguous slot ranges, one per device (equal pairs for same-length
// series), like the per-rank shards of the multi-process path.
std::vector<int64_t> device_bounds(dtwg_ctx* ctx, int64_t hw, int auto_widen, int nd) {
  const int64_t p = ctx->p, total = p * (p - 1) / 2;
  std::vector<int64_t> bnd(nd + 1, total);
  bnd[0] = 0;
  if (ctx->uniform) {
    for (int d = 1; d < nd; ++d) bnd[d] = total * d / nd;
    return bnd;
  }
  double all = 0;
  for (int64_t i = 0; i + 1 < p; ++i)
    for (int64_t j = i + 1; j < p; ++j) {
      const Shape sh = shape_of(ctx, i, j, hw, auto_widen);
      all += (double)pair_cells(sh.n, sh.m, sh.hw);
    }
  double acc = 0;
  int d = 1;
  int64_t slot = 0;
  for (int64_t i = 0; i + 1 < p && d < nd; ++i)
    for (int64_t j = i + 1; j < p && d < nd; ++j, ++slot) {
      const Shape sh = shape_of(ctx, i, j, hw, auto_widen);
      acc += (double)pair_cells(sh.n, sh.m, sh.hw);
      while (d < nd && acc >= all * d / nd) bnd[d++] = slot + 1;
    }
  for (int k = 1; k <= nd; ++k) bnd[k] = std::max(bnd[k], bnd[k - 1]);
  return bnd;
}

// Runs f(ctx_d, d) for every device of the context on its own host thread; returns the
// first error in device order (its message copied to the parent).
template <class F>
int for_each_device(dtwg_ctx* ctx, F&& f) {
  const int nd = 1 + (int)ctx->devs.size();
  std::vector<int> rcs(nd, DTWG_OK);
  std::vector<std::thread> th;
  for (int d = 0; d < nd; ++d) {
    dtwg_ctx* c = d == 0 ? ctx : ctx->devs[d - 1];
    th.emplace_back([&, c, d] {
      cudaSetDevice(c->device);
      rcs[d] = f(c, d);
    });
  }
  for (auto& t : th) t.join();
  for (int d = 0; d < nd; ++d) {
    if (rcs[d] != DTWG_OK) {
      dtwg_ctx* c = d == 0 ? ctx : ctx->devs[d - 1];
      if (c != ctx) {
        ctx->last_error = c->last_error;
        ctx->err_i = c->err_i;
        ctx->err_j = c->err_j;
      }
      return rcs[d];
    }
  }
  return DTWG_OK;
}
}  // extern "C++"

int dtwg_build_matrix(dtwg_ctx* ctx, const double* samples, const int64_t* offsets, int64_t p,
                      int64_t half_width, int auto_widen, unsigned workers, int precision,
                      double* out_condensed, uint64_t* evaluations) {
  if (!ctx) return DTWG_INVALID_ARGUMENTS;
  cudaSetDevice(ctx->device);
  ctx->err_i = ctx->err_j = -1;
  // pairwise.hpp:65-67: EmptyDataset, then workers, then series validation.
  if (p <= 0) return ctx->fail(DTWG_EMPTY_DATASET, "dataset contains no series");
  if (workers == 0) return ctx->fail(DTWG_INVALID_ARGUMENTS, "workers must be >= 1");
  const int64_t total = p * (p - 1) / 2;
  const int64_t out_bytes = total * (int64_t)sizeof(double);
  const bool staged = ctx->devs.empty() && out_condensed && total > 0 &&
                      out_bytes >= env_or("DTWGPU_STREAM_MIN_BYTES", kStreamMinBytes);
  if (staged) {
    // H2D, fill and D2H are enqueued first; the per-series checks (pairwise.hpp:65-67)
    // run on the host meanwhile and decide before anything is returned
    int rc = upload_begin(ctx, samples, offsets, p);
    if (rc) return rc;
    rc = check_band(ctx, half_width, auto_widen);
    if (rc) {
      cudaStreamSynchronize(ctx->stream);
      const int vr = validate_series(ctx, samples, offsets, p);  // earlier in the order
      ctx->p = vr ? 0 : ctx->p;
      return vr ? vr : rc;
    }
    const bool chunk_fill =
        ctx->uniform && out_bytes >= env_or("DTWGPU_CHUNK_FILL_MIN_BYTES", kChunkFillMinBytes);
    rc = build_streamed(ctx, half_width, auto_widen, precision, out_condensed, chunk_fill, 0, -1,
                        [&] { return validate_series(ctx, samples, offsets, p); });
    if (rc) {
      if (rc == DTWG_INVALID_SERIES || rc == DTWG_INVALID_ARGUMENTS) ctx->p = 0;
      return rc;
    }
    if (evaluations) *evaluations = (uint64_t)total;
    return DTWG_OK;
  }
  int rc = dtwg_upload_series(ctx, samples, offsets, p);
  if (rc) return rc;
  if (!ctx->devs.empty() && out_condensed && total > 0) {
    // every device fills its slot range and copies it straight into the caller's buffer
    rc = check_band(ctx, half_width, auto_widen);  // first infeasible pair, row-major
    if (rc) return rc;
    const std::vector<int64_t> bnd =
        device_bounds(ctx, half_width, auto_widen, 1 + (int)ctx->devs.size());
    rc = for_each_device(ctx, [&](dtwg_ctx* c, int d) -> int {
      if (c != ctx) {
        const int r = dtwg_upload_series(c, samples, offsets, p);
        if (r) return r;
      }
      return build_streamed(c, half_width, auto_widen, precision, out_condensed,
                            c->uniform && (bnd[d + 1] - bnd[d]) * 8 >= kChunkFillMinBytes,
                            bnd[d], bnd[d + 1]);
    });
    if (rc) return rc;
    if (evaluations) *evaluations = (uint64_t)total;
    return DTWG_OK;
  }
  rc = dtwg_fill_slots(ctx, half_width, auto_widen, precision, 0, total, nullptr);
  if (rc) return rc;
  if (total == 0) {
    ensure_resident(ctx, p);
    ctx->cond_valid = true;
  }
  rc = validate_resident(ctx);  // distance_matrix.hpp:34-38
  if (rc) return rc;
  if (total > 0 && out_condensed) {
    CU(cudaMemcpyAsync(out_condensed, ctx->d_cond.ptr, total * sizeof(double),
                       cudaMemcpyDeviceToHost, ctx->stream),
       "D2H condensed");
    CU(cudaStreamSynchronize(ctx->stream), "sync");
  }
  if (evaluations) *evaluations = (uint64_t)total;
  return DTWG_OK;
}

// ---- fused fill + all-gather over peer memory ----------------------------------------
int dtwg_exchange_export(dtwg_ctx* ctx, int64_t p, unsigned char* handle_out) {
  if (!ctx || !handle_out || p < 2) return DTWG_INVALID_ARGUMENTS;
  cudaSetDevice(ctx->device);
  int rc = ensure_resident(ctx, p);
  if (rc) return rc;
  ctx->cond_valid = false;
  cudaIpcMemHandle_t h;
  CU(cudaIpcGetMemHandle(&h, ctx->d_cond.ptr), "ipc export");
  std::memcpy(handle_out, &h, sizeof(h));
  return DTWG_OK;
}

int dtwg_exchange_open(dtwg_ctx* ctx, const unsigned char* handles, int n_ranks, int my_rank) {
  if (!ctx || !handles || n_ranks < 1 || my_rank < 0 || my_rank >= n_ranks ||
      n_ranks - 1 > dtwgpu::FillArgs::kMaxPeers)
    return ctx ? ctx->fail(DTWG_INVALID_ARGUMENTS, "bad exchange geometry (at most %d peers)",
                           dtwgpu::FillArgs::kMaxPeers)
               : DTWG_INVALID_ARGUMENTS;
  cudaSetDevice(ctx->device);
  dtwg_exchange_close(ctx);
  for (int r = 0; r < n_ranks; ++r) {
    if (r == my_rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + (size_t)r * sizeof(h), sizeof(h));
    void* ptr = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaGetLastError();
      dtwg_exchange_close(ctx);
      return ctx->cuda_fail(e, "ipc open of a peer's matrix");
    }
    ctx->peers.push_back(static_cast<double*>(ptr));
  }
  ctx->exchange_open = true;
  return DTWG_OK;
}

int dtwg_exchange_close(dtwg_ctx* ctx) {
  if (!ctx) return DTWG_INVALID_ARGUMENTS;
  for (double* ptr : ctx->peers) cudaIpcCloseMemHandle(ptr);
  ctx->peers.clear();
  ctx->exchange_open = false;
  return DTWG_OK;
}

int dtwg_exchange_fill(dtwg_ctx* ctx, int64_t half_width, int auto_widen, int precision,
                       int64_t slot_begin, int64_t slot_end) {
  if (!ctx) return DTWG_INVALID_ARGUMENTS;
  if (!ctx->exchange_open) return ctx->fail(DTWG_INVALID_ARGUMENTS, "exchange not open");
  if (ctx->mat_p != ctx->p)
    return ctx->fail(DTWG_INVALID_ARGUMENTS, "exchange buffer is for %lld series, dataset has %lld",
                     (long long)ctx->mat_p, (long long)ctx->p);
  cudaSetDevice(ctx->device);
  ctx->cond_valid = false;
  if (slot_end <= slot_begin) return DTWG_OK;
  // slots [b, e) into this rank's resident matrix at their global index, and (inside the
  // same kernels) into every peer's
  return dtwg_fill_slots(ctx, half_width, auto_widen, precision, slot_begin, slot_end,
                         ctx->d_cond.ptr + slot_begin);
}

int dtwg_exchange_complete(dtwg_ctx* ctx) {
  if (!ctx) return DTWG_INVALID_ARGUMENTS;
  cudaSetDevice(ctx->device);
  ctx->cond_valid = true;
  ctx->square_valid = false;
  return validate_resident(ctx);  // distance_matrix.hpp:34-38
}

static int adopt_one(dtwg_ctx* ctx, const double* condensed, int64_t p, int on_device) {
  cudaSetDevice(ctx->device);
  if (p <= 0) return ctx->fail(DTWG_DISTANCE_MATRIX_INVALID, "matrix needs at least one series");
  int rc = ensure_resident(ctx, p);
  if (rc) return rc;
  const int64_t total = p * (p - 1) / 2;
  if (total > 0) {
    if (!condensed) return ctx->fail(DTWG_INVALID_ARGUMENTS, "null condensed buffer");
    CU(cudaMemcpyAsync(ctx->d_cond.ptr, condensed, total * sizeof(double),
                       on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                       ctx->stream),
       "copy condensed");
  }
  return validate_resident(ctx);
}

int dtwg_adopt_condensed(dtwg_ctx* ctx, const double* condensed, int64_t p, int on_device) {
  if (!ctx) return DTWG_INVALID_ARGUMENTS;
  if (ctx->devs.empty()) return adopt_one(ctx, condensed, p, on_device);
  // every device of the context gets the matrix (device pointers may live on any device)
  return for_each_device(ctx, [&](dtwg_ctx* c, int) { return adopt_one(c, condensed, p, on_device); });
}

int dtwg_download_condensed(dtwg_ctx* ctx, double* out) {
  if (!ctx || !out) return DTWG_INVALID_ARGUMENTS;
  if (!ctx->cond_valid) return ctx->fail(DTWG_INVALID_ARGUMENTS, "no resident distance matrix");
  const int64_t total = ctx->mat_p * (ctx->mat_p - 1) / 2;
  if (total > 0) {
    CU(cudaMemcpyAsync(out, ctx->d_cond.ptr, total * 8, cudaMemcpyDeviceToHost, ctx->stream),
       "D2H");
    CU(cudaStreamSynchronize(ctx->stream), "sync");
  }
  return DTWG_OK;
}

static int km_run(dtwg_ctx* ctx, int64_t k, int64_t restarts, int64_t max_iterations,
                  uint64_t seed, int64_t restart_begin, int64_t restart_end,
                  dtwg_observer_fn observer, void* user, int64_t* medoids_out,
                  int64_t* assignment_out, double* cost_out, int64_t* best_restart_out);
static int km_loop(dtwg_ctx* ctx, int64_t p, int64_t k, int64_t max_iterations, uint64_t seed,
                   int64_t restart_begin, int64_t restart_end, dtwg_observer_fn observer,
                   void* user, int64_t* medoids_out, int64_t* assignment_out, double* cost_out,
                   int64_t* best_restart_out);

namespace {
struct KmRecord {
  int64_t r, it;
  double cost;
};
void km_record(void* user, int64_t r, int64_t it, double cost) {
  static_cast<std::vector<KmRecord>*>(user)->push_back({r, it, cost});
}
}  // namespace

int dtwg_kmedoids(dtwg_ctx* ctx, int64_t k, int64_t restarts, int64_t max_iterations,
                  uint64_t seed, int64_t restart_begin, int64_t restart_end,
                  dtwg_observer_fn observer, void* user, int64_t* medoids_out,
                  int64_t* assignment_out, double* cost_out, int64_t* best_restart_out) {
  if (!ctx) return DTWG_INVALID_ARGUMENTS;
  if (ctx->devs.empty() || !ctx->cond_valid)
    return km_run(ctx, k, restarts, max_iterations, seed, restart_begin, restart_end, observer,
                  user, medoids_out, assignment_out, cost_out, best_restart_out);
  // Several devices: contiguous blocks of restarts per device, run concurrently over a
  // copy of the matrix on each device; observer calls are replayed in restart order and
  // the best restart is reduced in restart order with strict < (kmedoids.hpp:182).
  if (restart_end > restarts) restart_end = restarts;
  const int nd = 1 + (int)ctx->devs.size();
  const int64_t p = ctx->mat_p;
  if (k < 1 || k > p || restart_begin < 0 || restart_begin >= restart_end)
    return km_run(ctx, k, restarts, max_iterations, seed, restart_begin, restart_end, observer,
                  user, medoids_out, assignment_out, cost_out, best_restart_out);  // errors
  struct Part {
    std::vector<int64_t> med, asg;
    double cost = 0;
    int64_t best_r = -1;
    std::vector<KmRecord> recs;
  };
  std::vector<Part> parts(nd);
  const int64_t nr = restart_end - restart_begin;
  int rc = for_each_device(ctx, [&](dtwg_ctx* c, int d) -> int {
    const int64_t rb = restart_begin + nr * d / nd, re = restart_begin + nr * (d + 1) / nd;
    if (re <= rb) return DTWG_OK;
    if (c != ctx) {
      const int r = adopt_one(c, ctx->d_cond.ptr, p, 1);
      if (r) return r;
    }
    Part& P = parts[d];
    P.med.resize(k);
    P.asg.resize(p);
    return km_run(c, k, restarts, max_iterations, seed, rb, re, observer ? km_record : nullptr,
                  &P.recs, P.med.data(), P.asg.data(), &P.cost, &P.best_r);
  });
  if (rc) return rc;
  bool have = false;
  double best = 0.0;
  for (const Part& P : parts) {
    for (const KmRecord& r : P.recs) observer(user, r.r, r.it, r.cost);
    if (P.best_r < 0) continue;
    if (!have || P.cost < best) {
      have = true;
      best = P.cost;
      if (cost_out) *cost_out = P.cost;
      if (medoids_out) std::copy(P.med.begin(), P.med.end(), medoids_out);
      if (assignment_out) std::copy(P.asg.begin(), P.asg.end(), assignment_out);
      if (best_restart_out) *best_restart_out = P.best_r;
    }
  }
  return DTWG_OK;
}

static int km_run(dtwg_ctx* ctx, int64_t k, int64_t restarts, int64_t max_iterations,
                  uint64_t seed, int64_t restart_begin, int64_t restart_end,
                  dtwg_observer_fn observer, void* user, int64_t* medoids_out,
                  int64_t* assignment_out, double* cost_out, int64_t* best_restart_out) {
  cudaSetDevice(ctx->device);
  if (!ctx->cond_valid) return ctx->fail(DTWG_INVALID_ARGUMENTS, "no resident distance matrix");
  const int64_t p = ctx->mat_p;
  // kmedoids.hpp:152-154
  if (k < 1 || k > p)
    return ctx->fail(DTWG_K_OUT_OF_RANGE, "k=%lld is outside [1, p] with p=%lld", (long long)k,
                     (long long)p);
  if (restarts < 1) return ctx->fail(DTWG_INVALID_ARGUMENTS, "restarts must be >= 1");
  if (max_iterations < 1) return ctx->fail(DTWG_INVALID_ARGUMENTS, "max_iterations must be >= 1");
  if (restart_end > restarts) restart_end = restarts;
  if (restart_begin < 0 || restart_begin >= restart_end)
    return ctx->fail(DTWG_INVALID_ARGUMENTS, "empty restart range");
  int rc = ensure_square(ctx);
  if (rc) return rc;
  // Independent restarts run concurrently: contiguous restart blocks on restart workers
  // (same device, own streams), observer calls replayed and the best restart reduced in
  // restart order with strict < -- the sequential loop's result, bit for bit.
  const int64_t nr = restart_end - restart_begin;
  // (small matrices: a restart is a few tens of microseconds, less than a thread hand-off)
  const int64_t cap = p >= 2048 ? 8 : 1;
  const int nw = (int)std::min<int64_t>(nr, std::max<int64_t>(1, env_or("DTWGPU_KM_WORKERS", cap)));
  if (nw <= 1)
    return km_loop(ctx, p, k, max_iterations, seed, restart_begin, restart_end, observer, user,
                   medoids_out, assignment_out, cost_out, best_restart_out);
  while ((int)ctx->kmw.size() < nw - 1) {
    dtwg_ctx* w = nullptr;
    rc = dtwg_create(ctx->device, &w);
    if (rc) return ctx->fail(rc, "cannot create a k-medoids worker context");
    w->km_src = ctx;
    ctx->kmw.push_back(w);
  }
  struct Part {
    std::vector<int64_t> med, asg;
    double cost = 0;
    int64_t best_r = -1;
    std::vector<KmRecord> recs;
    int rc = DTWG_OK;
  };
  std::vector<Part> parts(nw);
  std::vector<std::thread> th;
  for (int w = 0; w < nw; ++w) {
    dtwg_ctx* c = w == 0 ? ctx : ctx->kmw[w - 1];
    th.emplace_back([&, c, w] {
      cudaSetDevice(c->device);
      Part& P = parts[w];
      const int64_t rb = restart_begin + nr * w / nw, re = restart_begin + nr * (w + 1) / nw;
      if (re <= rb) return;
      P.med.resize(k);
      P.asg.resize(p);
      P.rc = km_loop(c, p, k, max_iterations, seed, rb, re, observer ? km_record : nullptr,
                     &P.recs, P.med.data(), P.asg.data(), &P.cost, &P.best_r);
    });
  }
  for (auto& t : th) t.join();
  for (int w = 0; w < nw; ++w) {
    dtwg_ctx* c = w == 0 ? ctx : ctx->kmw[w - 1];
    if (c != ctx) {  // fold the worker's sweep statistics into this context's
      ctx->km_assign_ms += c->km_assign_ms;
      ctx->km_assign_bytes += c->km_assign_bytes;
      ctx->km_update_ms += c->km_update_ms;
      ctx->km_update_bytes += c->km_update_bytes;
      ctx->km_sweeps += c->km_sweeps;
      ctx->launches += c->launches;
      c->km_assign_ms = c->km_assign_bytes = c->km_update_ms = c->km_update_bytes = 0;
      c->km_sweeps = 0;
      c->launches = 0;
    }
  }
  for (int w = 0; w < nw; ++w) {
    if (parts[w].rc != DTWG_OK) {
      dtwg_ctx* c = w == 0 ? ctx : ctx->kmw[w - 1];
      if (c != ctx) ctx->last_error = c->last_error;
      return parts[w].rc;
    }
  }
  bool have = false;
  double best = 0.0;
  for (const Part& P : parts) {
    for (const KmRecord& r : P.recs) observer(user, r.r, r.it, r.cost);
    if (P.best_r < 0) continue;
    if (!have || P.cost < best) {
      have = true;
      best = P.cost;
      if (cost_out) *cost_out = P.cost;
      if (medoids_out) std::copy(P.med.begin(), P.med.end(), medoids_out);
      if (assignment_out) std::copy(P.asg.begin(), P.asg.end(), assignment_out);
      if (best_restart_out) *best_restart_out = P.best_r;
    }
  }
  return DTWG_OK;
}

// The reference's restart loop (kmedoids.hpp:158-187) over restarts [restart_begin,
// restart_end) on one context's stream and sweep buffers.
static int km_loop(dtwg_ctx* ctx, int64_t p, int64_t k, int64_t max_iterations, uint64_t seed,
                   int64_t restart_begin, int64_t restart_end, dtwg_observer_fn observer,
                   void* user, int64_t* medoids_out, int64_t* assignment_out, double* cost_out,
                   int64_t* best_restart_out) {
  int rc = km_reserve(ctx, p, k);
  if (rc) return rc;
  KmState S{ctx, p, k, {}, {}};
  bool have_best = false;
  double best_cost = 0.0;
  std::vector<int64_t> medoids, updated;
  for (int64_t r = restart_begin; r < restart_end; ++r) {  // kmedoids.hpp:158-187
    SplitMix64 rng = restart_stream(seed, (uint64_t)r);
    rc = km_seeds(S, k, rng, medoids);
    if (rc) return rc;
    double cost = 0.0;
    bool converged = false;
    for (int64_t it = 0; it < max_iterations && !converged; ++it) {
      rc = km_assign(S, medoids);
      if (rc) return rc;
      cost = km_cost(S);
      if (observer) observer(user, r, it, cost);
      rc = km_update(S, medoids, updated);
      if (rc) return rc;
      if (updated == medoids) converged = true;
      else medoids = updated;
    }
    if (!converged) {
      rc = km_assign(S, medoids);
      if (rc) return rc;
      cost = km_cost(S);
    }
    if (!have_best || cost < best_cost) {
      best_cost = cost;
      have_best = true;
      if (medoids_out) std::copy(medoids.begin(), medoids.end(), medoids_out);
      if (assignment_out) std::copy(S.assignment.begin(), S.assignment.end(), assignment_out);
      if (best_restart_out) *best_restart_out = r;
    }
  }
  if (cost_out) *cost_out = best_cost;
  return DTWG_OK;
}

int dtwg_km_nearest_update(dtwg_ctx* ctx, int64_t current, const uint8_t* chosen,
                           double* nearest_inout) {
  if (!ctx || !chosen || !nearest_inout) return DTWG_INVALID_ARGUMENTS;
  cudaSetDevice(ctx->device);
  int rc = ensure_square(ctx);
  if (rc) return rc;
  const int64_t p = ctx->mat_p;
  if (current < 0 || current >= p)
    return ctx->fail(DTWG_INDEX_OUT_OF_RANGE, "index %lld is outside [0, %lld)",
                     (long long)current, (long long)p);
  rc = km_reserve(ctx, p, 1);
  if (rc) return rc;
  CU(cudaMemcpyAsync(ctx->d_chosen.ptr, chosen, p, cudaMemcpyHostToDevice, ctx->stream), "H2D");
  CU(cudaMemcpyAsync(ctx->d_nearest.ptr, nearest_inout, p * 8, cudaMemcpyHostToDevice,
                     ctx->stream),
     "H2D");
  CU(dtwgpu::launch_nearest_update(km_matrix(ctx), km_is_cond(ctx), p, current, ctx->d_chosen.ptr,
                                   ctx->d_nearest.ptr, ctx->stream),
     "nearest");
  ctx->launches++;
  CU(cudaMemcpyAsync(nearest_inout, ctx->d_nearest.ptr, p * 8, cudaMemcpyDeviceToHost,
                     ctx->stream),
     "D2H");
  CU(cudaStreamSynchronize(ctx->stream), "sync");
  return DTWG_OK;
}

int dtwg_km_assign(dtwg_ctx* ctx, const int64_t* medoids, int64_t k, int64_t* assignment_out,
                   double* dist_out) {
  if (!ctx || !medoids) return DTWG_INVALID_ARGUMENTS;
  cudaSetDevice(ctx->device);
  int rc = ensure_square(ctx);
  if (rc) return rc;
  const int64_t p = ctx->mat_p;
  if (k < 1 || k > p) return ctx->fail(DTWG_K_OUT_OF_RANGE, "k=%lld is outside [1, p]", (long long)k);
  rc = km_reserve(ctx, p, k);
  if (rc) return rc;
  KmState S{ctx, p, k, {}, {}};
  std::vector<int64_t> med(medoids, medoids + k);
  rc = km_assign(S, med);
  if (rc) return rc;
  if (assignment_out) std::copy(S.assignment.begin(), S.assignment.end(), assignment_out);
  if (dist_out) std::copy(S.dist.begin(), S.dist.end(), dist_out);
  return DTWG_OK;
}

int dtwg_km_update(dtwg_ctx* ctx, const int64_t* medoids, int64_t k, const int64_t* assignment,
                   int64_t* updated_out) {
  if (!ctx || !medoids || !assignment || !updated_out) return DTWG_INVALID_ARGUMENTS;
  cudaSetDevice(ctx->device);
  int rc = ensure_square(ctx);
  if (rc) return rc;
  const int64_t p = ctx->mat_p;
  if (k < 1 || k > p) return ctx->fail(DTWG_K_OUT_OF_RANGE, "k=%lld is outside [1, p]", (long long)k);
  rc = km_reserve(ctx, p, k);
  if (rc) return rc;
  KmState S{ctx, p, k, {}, {}};
  std::vector<int64_t> med(medoids, medoids + k);
  // Needs D(j, assignment[j]) for the empty-cluster repair: one assign-side gather.
  S.assignment.assign(assignment, assignment + p);
  S.dist.resize(p);
  {
    // dist[j] = D(j, assignment[j]) from the dense matrix rows.
    std::vector<double> row(p);
    for (int64_t j = 0; j < p; ++j) {
      const int64_t a = assignment[j];
      if (a < 0 || a >= p) return ctx->fail(DTWG_INDEX_OUT_OF_RANGE, "assignment out of range");
      if (a == j) {
        S.dist[j] = 0.0;
        continue;
      }
      CU(cudaMemcpy(&S.dist[j], ctx->d_square.ptr + a * p + j, 8, cudaMemcpyDeviceToHost),
         "D2H entry");
    }
  }
  std::vector<int64_t> upd;
  rc = km_update(S, med, upd);
  if (rc) return rc;
  std::copy(upd.begin(), upd.end(), updated_out);
  return DTWG_OK;
}

}  // extern "C"
