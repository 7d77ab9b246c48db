// km_host.cu -- the k-medoids host side of the C-ABI: the reference's restart loop, RNG,
// seeding draws, empty-cluster repair, dedupe/refill and ordered cost sums
// (kmedoids.hpp:33-189, cluster_result.hpp:40-72, validation.hpp:30-79), driving the
// sweep kernels of kmedoids.cu over the resident matrix; restart blocks run concurrently
// on restart-worker contexts and, for multi-device contexts, on several GPUs.
#include "host_ctx.cuh"

namespace dtwgpu {
namespace host {

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

}  // namespace host
}  // namespace dtwgpu

using namespace dtwgpu::host;

extern "C" {

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
