// host_ctx.cuh -- internals shared by the native host's translation units
// (dtwgpu.cu: context, upload, fill, build, exchange; planner.cu: kernel choice and pair
// classes; km_host.cu: the k-medoids restart loop and sweep entry points).
#pragma once
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

namespace dtwgpu {
namespace host {

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
inline SplitMix64 restart_stream(uint64_t seed, uint64_t restart) {
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
  int64_t range_begin = -1;    // uniform: this class fills [range_begin, +range_count) only
  int64_t range_count = 0;
  double cost = 0;
  int64_t max_n = 0;
  int64_t max_m = 0;  // longest shorter series: decides single- vs multi-strip Full kernels
  double cells = 0;  // in-band cells of the class (diagnostics: dtwg_last_plan)
  // Strip family: strips per pair (uniform) or prefix sums over `slots` (ragged)
  int strips_per_pair = 0;
  std::vector<int64_t> strip_base;
  // Launch on the previous class's stream, after it (a split tail round: its CTAs must not
  // take SM slots before every CTA of the full rounds is resident)
  bool after_prev = false;
};

inline int64_t row_off(int64_t i, int64_t p) { return i * p - i * (i + 1) / 2; }

// In-band cells of one pair.
inline int64_t pair_cells(int64_t n, int64_t m, int64_t hw) {
  if (hw >= n) return n * m;
  const int64_t T = std::max<int64_t>(n - hw - 1, 0);
  const int64_t a = std::min(T, m);
  const int64_t left = a * (a + 1) / 2 + std::max<int64_t>(T - m, 0) * m;
  const int64_t S = std::max<int64_t>(m - hw - 1, 0);
  return n * m - left - S * (S + 1) / 2;
}

}  // namespace host
}  // namespace dtwgpu

using dtwgpu::Family;
using dtwgpu::FillArgs;
using dtwgpu::KernelCfg;
using dtwgpu::host::DevBuf;
using dtwgpu::host::PlanClass;

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
    int64_t replan;  // DTWGPU_UNDERFILL_REPLAN, DTWGPU_PLAN_TABLE (planner.cu)
    bool operator==(const PlanKey& o) const {
      return hw == o.hw && sb == o.sb && se == o.se && auto_widen == o.auto_widen &&
             fp32 == o.fp32 && force_family == o.force_family && force_G == o.force_G &&
             force_R == o.force_R && replan == o.replan;
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
  int64_t max_len = 0;
  int64_t tail_guard = 0;  // zeros after the packed series (>= kGuard + the longest series)
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
  cudaEvent_t km0 = nullptr, km1 = nullptr, km2 = nullptr, km3 = nullptr;
  double km_assign_ms = 0, km_update_ms = 0, km_assign_bytes = 0, km_update_bytes = 0;
  double km_prep_ms = 0;
  int64_t km_sweeps = 0;

  // Cluster-ordered copy of the square (km_host.cu ensure_layout): psq[u][v] =
  // square[perm[u]][perm[v]] with series grouped by their nearest farthest-point anchor, so
  // a cluster's members occupy runs of consecutive positions and the candidate sums read
  // whole sectors. Built once per resident matrix when two squares fit in HBM.
  DevBuf<double> d_psq;
  DevBuf<int32_t> d_perm, d_pinv;
  bool layout_valid = false;  // d_psq/d_perm/d_pinv match the square
  bool layout32 = false;      // d_psq holds fp32 values (p*p floats)
  bool fp32_safe = false;     // every non-zero entry in [2^-100, 2^100] (validate_resident)
  bool layout_tried = false;  // decided for this square (built, or skipped: p small / no room)
  DevBuf<int64_t> d_anchors;
  cudaStream_t layout_stream = nullptr;  // the copy is built here, overlapping the seeding
  cudaEvent_t layout_ready = nullptr;    // sweeps reading it wait on this
  cudaEvent_t layout_t0 = nullptr;
  // the square expansion runs on `stream` without a host wait: the seeding reads the
  // condensed matrix meanwhile, sweeps and the layout wait on square_ready
  cudaEvent_t square_t0 = nullptr, square_ready = nullptr;
  bool square_timed = false;  // square_t0/square_ready bracket an expansion not yet counted
  DevBuf<int64_t> d_layout_asg;
  DevBuf<double> d_layout_dist;
  DevBuf<int32_t> d_layout_lab, d_layout_keys;
  DevBuf<uint8_t> d_layout_cub;

  // Device-side bucketing (kmedoids.hpp:86-92): slot per series, radix-sort keys, iota,
  // members in layout order, cub temporary storage.
  DevBuf<int32_t> d_lab, d_keys_a, d_keys_b, d_iota, d_members_p;
  DevBuf<uint8_t> d_cub;
  size_t cub_bytes = 0;
  int64_t iota_n = 0;
  // Pinned host staging for the per-sweep and per-seed-step copies.
  double* h_km_dist[2] = {nullptr, nullptr};
  double* h_km_nearest = nullptr;
  int64_t* h_km_best = nullptr;
  int64_t* h_km_cb = nullptr;
  int64_t* h_km_med = nullptr;
  int64_t h_km_p = 0, h_km_k = 0;

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

namespace dtwgpu {
namespace host {

// Tests shrink both through the environment to exercise many chunks on small inputs.
inline int64_t env_or(const char* name, int64_t dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::strtoll(v, nullptr, 10) : dflt;
}

// ---- planner.cu
KernelCfg choose_cfg(const dtwg_ctx* ctx, const Shape& s, bool fp32, double* cost_out,
                     int64_t count = 0);
Shape shape_of(const dtwg_ctx* ctx, int64_t a, int64_t b, int64_t hw, int auto_widen);
std::vector<PlanClass> make_plan(dtwg_ctx* ctx, int64_t hw, int auto_widen, bool fp32,
                                 int64_t sb, int64_t se);
const char* family_name(Family f);

// ---- dtwgpu.cu
int validate_series(dtwg_ctx* ctx, const double* samples, const int64_t* offsets, int64_t p);
int check_band(dtwg_ctx* ctx, int64_t hw, int auto_widen);
int ensure_fp32(dtwg_ctx* ctx);
int ensure_band(dtwg_ctx* ctx, bool fp32);
int run_fill(dtwg_ctx* ctx, int64_t hw, int auto_widen, int precision, int64_t sb, int64_t se,
             double* d_out, int64_t out_base, bool sync = true);
int ensure_resident(dtwg_ctx* ctx, int64_t p);
int validate_resident(dtwg_ctx* ctx, int64_t sb = 0, int64_t se = -1);
int adopt_one(dtwg_ctx* ctx, const double* condensed, int64_t p, int on_device);

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

}  // namespace host
}  // namespace dtwgpu
