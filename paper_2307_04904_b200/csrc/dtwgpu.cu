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
//
// This file: the context, series upload, fills, builds (staged, multi-device), the fused
// exchange and the remaining entry points; the planner lives in planner.cu and the
// k-medoids host loop in km_host.cu (shared internals: host_ctx.cuh).
#include "host_ctx.cuh"

#include <chrono>
#include <cstdio>

namespace dtwgpu {
namespace host {

// Rows of padding after each group's boundary column: lane 0 of a multi-pass Full group
// prefetches its boundary rows unconditionally, up to TR * (G + 2) rows past the pair's
// last row.
constexpr int64_t kScratchPad = 160;

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

int ensure_fp32(dtwg_ctx* ctx) {
  if (ctx->have32) return DTWG_OK;
  // the whole guarded buffer, guards included (zeros stay zeros)
  const int64_t total = ctx->h_offsets[ctx->p] + kGuard + ctx->tail_guard;
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
  // Lanes of a warp run to the warp's longest pair, so a shorter pair's lane streams past
  // its series' end by up to the longest length: the tail past the last series covers it.
  const int64_t total = pos + pad + ctx->max_len;
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
  CU(cudaMemsetAsync(static_cast<char*>(out) + (pos - pad) * (fp32 ? 4 : 8), 0,
                     (total - (pos - pad)) * (fp32 ? 4 : 8), ctx->stream),
     "memset band tail");
  CU(dtwgpu::launch_band_pad(ctx->d_samples.ptr + kGuard, ctx->d_offsets.ptr, ctx->d_boffsets.ptr,
                             p, pad, out, fp32, ctx->stream),
     "band pad");
  ctx->launches++;
  (fp32 ? ctx->have_band32 : ctx->have_band64) = true;
  return DTWG_OK;
}

int run_fill(dtwg_ctx* ctx, int64_t hw, int auto_widen, int precision, int64_t sb, int64_t se,
             double* d_out, int64_t out_base, bool sync) {
  const bool fp32 = precision == DTWG_FP32;
  if (fp32) {
    const int rc = ensure_fp32(ctx);
    if (rc) return rc;
  }
  const dtwg_ctx::PlanKey key{hw, sb, se, auto_widen, fp32, ctx->force_family, ctx->force_G,
                              ctx->force_R,
                              env_or("DTWGPU_UNDERFILL_REPLAN", 1) * 2 + env_or("DTWGPU_PLAN_TABLE", 1) +
                                  4 * env_or("DTWGPU_TAIL_SPLIT", 1) +
                                  8 * (env_or("DTWGPU_TAIL_SERIAL", -1) + 1)};
  if (!(ctx->plan_valid && ctx->plan_key == key)) {
    const auto t0 = std::chrono::steady_clock::now();
    ctx->plan_cache = make_plan(ctx, hw, auto_widen, fp32, sb, se);
    ctx->plan_key = key;
    ctx->plan_valid = true;
    ctx->list_uploaded = false;
    if (env_or("DTWGPU_VERBOSE", 0))
      fprintf(stderr, "dtwgpu: planned %lld pairs into %zu classes in %.1f ms\n",
              (long long)(se - sb), ctx->plan_cache.size(),
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                  .count());
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
    const int64_t count = ctx->uniform ? (pc.range_begin >= 0 ? pc.range_count : se - sb)
                                       : (int64_t)pc.slots.size();
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
    const bool multipass = pc.cfg.family == Family::Full && pc.cfg.mp &&
                           (ctx->uniform ? (ctx->h_len[0] > W) : true);
    if (multipass && count > 0) {
      // One boundary column per resident lane group: with one lane per pair and very long
      // series that is max_n * 8 B * 37,888 groups (30 GB at n = 1e5). Cap the class's
      // scratch at a share of free HBM by running fewer (persistent, grid-stride) blocks.
      const int64_t per_block = (pc.max_n + kScratchPad) * groups_per_block;
      size_t free_b = 0, total_b = 0;
      if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) free_b = size_t(8) << 30;
      const int64_t budget = std::min<int64_t>((int64_t)(free_b / 4 / sizeof(double)),
                                               env_or("DTWGPU_SCRATCH_MAX_MB", 16384) << 17);
      const int64_t cap = std::max<int64_t>(1, budget / std::max<int64_t>(per_block, 1));
      if (blocks_of[c] > cap) blocks_of[c] = cap;
      scratch_off[c] = scratch_total;
      scratch_total += per_block * blocks_of[c];
    }
  }
  if (scratch_total) CU(ctx->d_scratch.reserve((size_t)scratch_total), "cudaMalloc scratch");
  // One item counter per class: dynamic item scheduling in every fill kernel (take_items,
  // dtw_kernels.cuh), strip items in the Strip family. DTWGPU_DYNAMIC_ITEMS=0: static
  // grid-stride items (diagnostics).
  const bool dynamic_items = env_or("DTWGPU_DYNAMIC_ITEMS", 1) != 0;
  CU(ctx->d_work.reserve((size_t)plan.size()), "cudaMalloc work");
  CU(cudaMemsetAsync(ctx->d_work.ptr, 0, plan.size() * sizeof(unsigned long long), ctx->stream),
     "memset work");
  if (n_strip_cls) {
    CU(ctx->d_prog.reserve((size_t)prog_total), "cudaMalloc prog");
    CU(ctx->d_cols.reserve((size_t)cols_total), "cudaMalloc cols");
    CU(cudaMemsetAsync(ctx->d_prog.ptr, 0, prog_total * sizeof(int), ctx->stream), "memset prog");
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
  cudaStream_t prev_st = ctx->stream;
  for (size_t c = 0; c < plan.size(); ++c) {
    auto& pc = plan[c];
    if (!dtwgpu::fill_cfg_supported(pc.cfg))
      return ctx->fail(DTWG_INTERNAL, "no kernel for %s G=%d R=%d", family_name(pc.cfg.family),
                       pc.cfg.G, pc.cfg.R);
    const int64_t count = ctx->uniform ? (pc.range_begin >= 0 ? pc.range_count : se - sb)
                                       : (int64_t)pc.slots.size();
    if (count == 0) continue;
    const int bps = dtwgpu::fill_blocks_per_sm(pc.cfg);
    const int64_t blocks = blocks_of[c];
    FillArgs a{};
    a.samples = ctx->d_samples.ptr + kGuard;
    a.samples32 = fp32 ? ctx->d_samples32.ptr + kGuard : nullptr;
    a.guard_lo = -kGuard;
    a.guard_hi = ctx->h_offsets[ctx->p] + ctx->tail_guard;
    a.bsamples = ctx->have_band64 ? ctx->d_bsamples.ptr : nullptr;
    a.bsamples32 = ctx->have_band32 ? ctx->d_bsamples32.ptr : nullptr;
    a.boffsets = (ctx->have_band64 || ctx->have_band32) ? ctx->d_boffsets.ptr : nullptr;
    a.offsets = ctx->d_offsets.ptr;
    a.p = ctx->p;
    a.half_width = hw;
    a.auto_widen = auto_widen;
    a.list = ctx->uniform ? nullptr : ctx->d_list.ptr + pos;
    a.begin = ctx->uniform ? (pc.range_begin >= 0 ? pc.range_begin : sb) : 0;
    a.count = count;
    a.out_base = out_base;
    a.out = d_out;
    if (scratch_off[c] >= 0) {
      a.scratch = ctx->d_scratch.ptr + scratch_off[c];
      a.scratch_stride = pc.max_n + kScratchPad;
    }
    if (ctx->exchange_open && d_out - out_base == ctx->d_cond.ptr) {  // resident, global slots
      a.n_peer = (int)ctx->peers.size();
      for (int r = 0; r < a.n_peer; ++r) a.peer_out[r] = ctx->peers[r];
      a.peer_base = 0;
    }
    a.work = dynamic_items ? ctx->d_work.ptr + c : nullptr;
    if (pc.cfg.family == Family::Strip) {
      a.strip_base = sb_off[c] >= 0 ? ctx->d_strip_base.ptr + sb_off[c] : nullptr;
      a.strips_per_pair = pc.strips_per_pair;
      a.work = ctx->d_work.ptr + c;
      a.prog = ctx->d_prog.ptr + prog_off[c];
      a.cols = ctx->d_cols.ptr + cols_off[c];
      a.col_stride = pc.max_n + 2;
    }
    cudaStream_t st = concurrent ? (pc.after_prev && c > 0 ? prev_st
                                                          : ctx->aux[next_aux++ % dtwg_ctx::kAux])
                                 : ctx->stream;
    prev_st = st;
    CU(dtwgpu::launch_fill(pc.cfg, a, (int)blocks, st), "fill launch");
    ctx->launches++;
    char buf[200];
    char krs[32] = "";
    if (pc.cfg.family == Family::Band)
      snprintf(krs, sizeof(krs), "%s,P=%d%s%s",
               pc.cfg.kr >= 0 ? (",kr=" + std::to_string(pc.cfg.kr)).c_str() : "", pc.cfg.P,
               pc.cfg.ring ? ",ring" : "",
               pc.cfg.U > 1 ? (",U=" + std::to_string(pc.cfg.U)).c_str() : "");
    if (pc.cfg.family != Family::Band)
      snprintf(krs, sizeof(krs), ",T=%d%s%s", pc.cfg.TR,
               pc.cfg.family == Family::Full && !pc.cfg.mp ? ",1strip" : "",
               pc.cfg.ysm ? ",ysm" : "");
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
  ctx->layout_valid = ctx->layout_tried = false;
  return DTWG_OK;
}

// distance_matrix.hpp:34-38 over slots [sb, se) of the resident matrix (se < 0: all).
int validate_resident(dtwg_ctx* ctx, int64_t sb, int64_t se) {
  const int64_t total = ctx->mat_p * (ctx->mat_p - 1) / 2;
  if (se < 0) se = total;
  if (se <= sb) return DTWG_OK;
  CU(ctx->d_flag.reserve(2), "cudaMalloc flag");
  CU(cudaMemsetAsync(ctx->d_flag.ptr, 0, 2 * sizeof(int), ctx->stream), "memset");
  CU(dtwgpu::launch_validate_condensed(ctx->d_cond.ptr + sb, se - sb, ctx->d_flag.ptr,
                                       ctx->stream),
     "validate");
  ctx->launches++;
  int flags[2] = {0, 0};
  CU(cudaMemcpyAsync(flags, ctx->d_flag.ptr, 2 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream),
     "D2H flag");
  CU(cudaStreamSynchronize(ctx->stream), "sync");
  const int bad = flags[0];
  ctx->fp32_safe = sb == 0 && se == total && !flags[1];
  if (bad) {
    ctx->cond_valid = false;
    return ctx->fail(DTWG_DISTANCE_MATRIX_INVALID, "entries must be finite and non-negative");
  }
  ctx->cond_valid = sb == 0 && se == total;
  return DTWG_OK;
}

}  // namespace host
}  // namespace dtwgpu

using namespace dtwgpu::host;

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
  ctx->d_psq.release();
  ctx->d_perm.release();
  ctx->d_pinv.release();
  ctx->d_anchors.release();
  ctx->d_lab.release();
  ctx->d_keys_a.release();
  ctx->d_keys_b.release();
  ctx->d_iota.release();
  ctx->d_members_p.release();
  ctx->d_cub.release();
  for (double*& h : ctx->h_km_dist)
    if (h) cudaFreeHost(h);
  if (ctx->h_km_nearest) cudaFreeHost(ctx->h_km_nearest);
  if (ctx->h_km_best) cudaFreeHost(ctx->h_km_best);
  if (ctx->h_km_cb) cudaFreeHost(ctx->h_km_cb);
  if (ctx->h_km_med) cudaFreeHost(ctx->h_km_med);
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
  if (ctx->km2) cudaEventDestroy(ctx->km2);
  if (ctx->layout_ready) cudaEventDestroy(ctx->layout_ready);
  if (ctx->layout_t0) cudaEventDestroy(ctx->layout_t0);
  if (ctx->square_t0) cudaEventDestroy(ctx->square_t0);
  if (ctx->square_ready) cudaEventDestroy(ctx->square_ready);
  ctx->d_layout_asg.release();
  ctx->d_layout_dist.release();
  ctx->d_layout_lab.release();
  ctx->d_layout_keys.release();
  ctx->d_layout_cub.release();
  if (ctx->layout_stream) {
    cudaStreamSynchronize(ctx->layout_stream);
    cudaStreamDestroy(ctx->layout_stream);
  }
  if (ctx->km3) cudaEventDestroy(ctx->km3);
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
  ctx->max_len = p ? *std::max_element(ctx->h_len.begin(), ctx->h_len.end()) : 0;
  // Lanes of a warp run to the warp's longest pair and prefetch rows past their own
  // series' end (unused values): the guard after the last series covers the longest one.
  ctx->tail_guard = kGuard + ctx->max_len;
  ctx->have32 = false;
  ctx->have_band64 = ctx->have_band32 = false;
  // The plan depends only on the series lengths (and window/precision/range): keep it
  // when a new upload has the same lengths.
  if (ctx->plan_valid && ctx->plan_lens != ctx->h_len) ctx->plan_valid = false;
  if (!ctx->plan_valid) ctx->plan_lens = ctx->h_len;
  CU(ctx->d_samples.reserve(n + kGuard + ctx->tail_guard), "cudaMalloc samples");
  CU(ctx->d_offsets.reserve(p + 1), "cudaMalloc offsets");
  CU(cudaMemsetAsync(ctx->d_samples.ptr, 0, kGuard * sizeof(double), ctx->stream), "memset");
  CU(cudaMemsetAsync(ctx->d_samples.ptr + kGuard + n, 0, ctx->tail_guard * sizeof(double),
                     ctx->stream),
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
  ctx->layout_valid = ctx->layout_tried = false;
  return validate_resident(ctx);  // distance_matrix.hpp:34-38
}
int dtwg_download_range(dtwg_ctx* ctx, int64_t b, int64_t e, double* out) {
  if (!ctx || (!out && e > b)) return DTWG_INVALID_ARGUMENTS;
  if (!ctx->cond_valid && !ctx->exchange_open)
    return ctx->fail(DTWG_INVALID_ARGUMENTS, "no resident distance matrix");
  const int64_t total = ctx->mat_p * (ctx->mat_p - 1) / 2;
  if (b < 0 || e > total || b > e)
    return ctx->fail(DTWG_INVALID_ARGUMENTS, "slot range [%lld, %lld) outside [0, %lld)",
                     (long long)b, (long long)e, (long long)total);
  cudaSetDevice(ctx->device);
  if (e > b) {
    CU(cudaMemcpyAsync(out, ctx->d_cond.ptr + b, (e - b) * 8, cudaMemcpyDeviceToHost, ctx->stream),
       "D2H");
    CU(cudaStreamSynchronize(ctx->stream), "sync");
  }
  return DTWG_OK;
}

}  // extern "C"

namespace dtwgpu {
namespace host {
int adopt_one(dtwg_ctx* ctx, const double* condensed, int64_t p, int on_device) {
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
}  // namespace host
}  // namespace dtwgpu

extern "C" {

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


}  // extern "C"
