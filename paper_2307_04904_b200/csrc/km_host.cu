// km_host.cu -- the k-medoids host side of the C-ABI: the reference's restart loop, RNG,
// seeding draws, empty-cluster repair, dedupe/refill and ordered cost sums
// (kmedoids.hpp:33-189, cluster_result.hpp:40-72, validation.hpp:30-79), driving the
// sweep kernels of kmedoids.cu over the resident matrix; restart blocks run concurrently
// on restart-worker contexts and, for multi-device contexts, on several GPUs.
#include "host_ctx.cuh"

#include <chrono>

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
  // a cluster-ordered copy still being built from the old square must finish first
  if (ctx->layout_stream) CU(cudaStreamSynchronize(ctx->layout_stream), "sync layout");
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
  if (!ctx->square_ready) {
    CU(cudaEventCreate(&ctx->square_t0), "event");
    CU(cudaEventCreate(&ctx->square_ready), "event");
  }
  CU(cudaEventRecord(ctx->square_t0, ctx->stream), "event");
  if (p >= 2) {
    CU(dtwgpu::launch_expand_square(ctx->d_cond.ptr, p, ctx->d_square.ptr, ctx->stream),
       "expand");
    ctx->launches++;
  } else {
    CU(cudaMemsetAsync(ctx->d_square.ptr, 0, sizeof(double), ctx->stream), "memset");
  }
  // no host wait: the seeding reads the condensed matrix while the square is written;
  // the layout build and the sweeps wait on square_ready (km_wait_ready)
  CU(cudaEventRecord(ctx->square_ready, ctx->stream), "event");
  ctx->square_timed = true;
  ctx->square_valid = true;
  return DTWG_OK;
}

int ensure_iota(dtwg_ctx* ctx, int64_t p);

// ---- cluster-ordered layout --------------------------------------------------------
// The medoid update reads, for every candidate, its row at its cluster's member columns
// (sum over clusters of |C|^2 distances). Members of a cluster are scattered over the
// row, so in the plain square every 8-byte read costs a whole 32-byte sector (round 1:
// ~15x the algorithmic bytes). ensure_layout builds once per resident matrix a copy of
// the square with the series grouped by their nearest anchor -- 4k anchors drawn
// uniformly with a fixed seed (a k-medoids cluster is then mostly a union of whole anchor
// groups, i.e. runs of consecutive positions; exp. on c3 subsets: DRAM bytes of the sums
// 1.9-2.0x the algorithmic ones, against 6.7x in the plain square; farthest-point anchors
// 3.5x). It only moves data -- the candidate sums read the same doubles and the
// contenders' exact sums keep reading the plain square in ascending member order -- so
// results are bit-identical with or without it. Skipped for small p (the plain gathers
// are cheap there), in condensed mode, and when a second square does not fit in HBM.
int ensure_layout(dtwg_ctx* ctx, int64_t k) {
  if (ctx->layout_tried) return DTWG_OK;
  if (ctx->layout_stream) CU(cudaStreamSynchronize(ctx->layout_stream), "sync layout");
  ctx->layout_tried = true;
  ctx->layout_valid = false;
  const int64_t p = ctx->mat_p;
  const int64_t min_p = env_or("DTWGPU_KM_LAYOUT_MIN_P", 8192);
  if (ctx->km_condensed || p < std::max<int64_t>(min_p, 2) || env_or("DTWGPU_KM_LAYOUT", 1) == 0)
    return DTWG_OK;
  // fp32 copy when every entry keeps a 2^-24 relative rounding bound in fp32 (the
  // candidate sums only filter; cluster_select_kernel widens its threshold by 2^-24):
  // half the bytes per candidate-sum read and per copy write
  const bool f32 = ctx->fp32_safe && env_or("DTWGPU_KM_LAYOUT32", 1) != 0;
  const size_t words = f32 ? (size_t)((p * p + 1) / 2) : (size_t)(p * p);
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  const double need = double(words) * 8.0 - double(ctx->d_psq.cap) * 8.0;
  if (need > 0.8 * double(free_b)) return DTWG_OK;
  const int na = (int)std::min<int64_t>(std::max<int64_t>(4 * k, 2), std::min<int64_t>(p, 256));
  // na distinct anchors, uniformly at random (fixed seed), ascending
  std::vector<int64_t> anchors;
  {
    SplitMix64 rng(0x5EEDC0DEULL);
    std::vector<char> used(p, 0);
    while ((int)anchors.size() < na) {
      const int64_t j = (int64_t)rng.next_below((uint64_t)p);
      if (!used[j]) {
        used[j] = 1;
        anchors.push_back(j);
      }
    }
    std::sort(anchors.begin(), anchors.end());
  }
  CU(ctx->d_psq.reserve(words), "cudaMalloc layout square");
  ctx->layout32 = f32;
  CU(ctx->d_perm.reserve(p), "malloc");
  CU(ctx->d_pinv.reserve(p), "malloc");
  CU(ctx->d_anchors.reserve(na), "malloc");
  CU(ctx->d_assign.reserve(p), "malloc");
  CU(ctx->d_dist.reserve(p), "malloc");
  CU(ctx->d_lab.reserve(p), "malloc");
  CU(ctx->d_keys_a.reserve(p), "malloc");
  int rc = ensure_iota(ctx, p);
  if (rc) return rc;
  // Built on its own stream (own scratch: anchors' assignment in d_layout_*) while the
  // restarts seed from the condensed matrix; sweeps wait on layout_ready (km_wait_ready).
  if (!ctx->layout_stream) {
    CU(cudaStreamCreateWithFlags(&ctx->layout_stream, cudaStreamNonBlocking), "stream");
    CU(cudaEventCreate(&ctx->layout_ready), "event");
    CU(cudaEventCreate(&ctx->layout_t0), "event");
  }
  CU(ctx->d_layout_asg.reserve(p), "malloc");
  CU(ctx->d_layout_dist.reserve(p), "malloc");
  CU(ctx->d_layout_lab.reserve(p), "malloc");
  CU(ctx->d_layout_keys.reserve(p), "malloc");
  CU(ctx->d_layout_cub.reserve(ctx->cub_bytes), "malloc");
  cudaStream_t ls = ctx->layout_stream;
  CU(cudaMemcpyAsync(ctx->d_anchors.ptr, anchors.data(), na * 8, cudaMemcpyHostToDevice, ls),
     "H2D anchors");
  CU(cudaStreamSynchronize(ls), "sync");  // `anchors` is pageable and about to go away
  // the square (and iota) are enqueued on ctx->stream: wait for them on the device
  CU(cudaEventRecord(ctx->km3, ctx->stream), "event");
  CU(cudaStreamWaitEvent(ls, ctx->km3, 0), "wait square");
  CU(cudaEventRecord(ctx->layout_t0, ls), "event");
  CU(dtwgpu::launch_cluster_layout(ctx->d_square.ptr, p, na, ctx->d_anchors.ptr,
                                   ctx->d_layout_asg.ptr, ctx->d_layout_dist.ptr,
                                   ctx->d_layout_lab.ptr, ctx->d_layout_keys.ptr, ctx->d_iota.ptr,
                                   ctx->d_perm.ptr, ctx->d_pinv.ptr, ctx->d_psq.ptr, f32,
                                   ctx->d_layout_cub.ptr, ctx->cub_bytes, ctx->num_sms, ls),
     "cluster layout");
  CU(cudaEventRecord(ctx->layout_ready, ls), "event");
  ctx->launches += 6;
  ctx->layout_valid = true;
  return DTWG_OK;
}

// ---- k-medoids host loop ------------------------------------------------------------
// One sweep is enqueued as: H2D medoids -> assign_slots (assignment, distance, cluster
// slot) -> device bucketing (stable radix sort by slot; the cluster bounds) -> candidate
// sums and per-cluster selection -> one D2H of the distances, bounds and winners into
// pinned buffers. The host then waits once, repairs/dedupes (O(k log k); O(p) only for an
// empty cluster) and launches the next sweep before it sums the previous assignment's cost
// in ascending order, so that sequential sum overlaps the GPU.
struct KmState {
  dtwg_ctx* ctx;  // this worker's stream and sweep buffers
  int64_t p, k;
  const double* sq;      // sweep view (square or condensed)
  bool cond;             // sweep view is the condensed matrix
  const double* cmat;    // the condensed matrix (seeding reads it while the square is built)
  const dtwg_ctx* src;   // the context owning the matrix (square_ready / layout_ready)
  bool ready = false;    // this stream already waits for the square and the layout
  const void* psq;       // cluster-ordered copy (nullptr: none)
  bool psq32;            // ... holding fp32 values
  const int32_t* perm;   // its order
  const int32_t* pinv;
  int buf = 0;           // pinned distance buffer of the sweep in flight
};

// kernels of one device bucketing + update (cub's radix sort launches 3 per sort)
int km_update_launches(const KmState& S) {
  if (S.k <= 256) return 4;
  return S.psq ? 10 : 6;
}

// Before the first sweep on a stream: the square and the cluster-ordered copy are ready.
void km_wait_ready(KmState& S) {
  if (S.ready) return;
  if (S.src->square_ready) cudaStreamWaitEvent(S.ctx->stream, S.src->square_ready, 0);
  if (S.psq) cudaStreamWaitEvent(S.ctx->stream, S.src->layout_ready, 0);
  S.ready = true;
}

int km_enqueue_assign(KmState& S, const std::vector<int64_t>& medoids) {
  dtwg_ctx* ctx = S.ctx;
  km_wait_ready(S);
  std::copy(medoids.begin(), medoids.end(), ctx->h_km_med);
  CU(cudaMemcpyAsync(ctx->d_medoids.ptr, ctx->h_km_med, medoids.size() * 8,
                     cudaMemcpyHostToDevice, ctx->stream),
     "H2D medoids");
  CU(cudaEventRecord(ctx->km0, ctx->stream), "event");
  // with k <= 256 the kernel also counts the cluster sizes for the bucketing (into keys_a)
  CU(dtwgpu::launch_assign_slots(S.sq, S.cond, S.p, ctx->d_medoids.ptr, (int64_t)medoids.size(),
                                 ctx->d_assign.ptr, ctx->d_dist.ptr, ctx->d_lab.ptr, ctx->stream,
                                 ctx->d_keys_a.ptr),
     "assign");
  ctx->launches++;
  return DTWG_OK;
}

// assignment + update of one sweep, results to the pinned buffers (dist into buf)
int km_enqueue_sweep(KmState& S, const std::vector<int64_t>& medoids, int buf) {
  dtwg_ctx* ctx = S.ctx;
  const int64_t p = S.p, k = (int64_t)medoids.size();
  int rc = km_enqueue_assign(S, medoids);
  if (rc) return rc;
  CU(cudaEventRecord(ctx->km1, ctx->stream), "event");
  CU(cudaEventRecord(ctx->km2, ctx->stream), "event");
  CU(dtwgpu::launch_bucket(ctx->d_lab.ptr, S.psq ? S.perm : nullptr, ctx->d_iota.ptr, p, k,
                           ctx->d_keys_a.ptr, ctx->d_keys_b.ptr, ctx->d_members.ptr,
                           ctx->d_members_p.ptr, ctx->d_cb.ptr, ctx->d_cub.ptr, ctx->cub_bytes,
                           ctx->stream, /*counted=*/true),
     "bucket");
  CU(dtwgpu::launch_update2(S.sq, S.cond, S.psq, S.psq32, S.pinv, p, ctx->d_members.ptr,
                            ctx->d_members_p.ptr, ctx->d_cb.ptr, k, ctx->d_best_member.ptr,
                            ctx->d_best_sum.ptr, ctx->stream),
     "update");
  CU(cudaEventRecord(ctx->km3, ctx->stream), "event");
  ctx->launches += km_update_launches(S) - (S.k <= 256 ? 1 : 0);
  CU(cudaMemcpyAsync(ctx->h_km_dist[buf], ctx->d_dist.ptr, p * 8, cudaMemcpyDeviceToHost,
                     ctx->stream),
     "D2H dist");
  CU(cudaMemcpyAsync(ctx->h_km_cb, ctx->d_cb.ptr, (k + 1) * 8, cudaMemcpyDeviceToHost,
                     ctx->stream),
     "D2H cb");
  CU(cudaMemcpyAsync(ctx->h_km_best, ctx->d_best_member.ptr, k * 8, cudaMemcpyDeviceToHost,
                     ctx->stream),
     "D2H best");
  return DTWG_OK;
}

int km_wait_sweep(KmState& S) {
  dtwg_ctx* ctx = S.ctx;
  CU(cudaStreamSynchronize(ctx->stream), "sync");
  float ms = 0, ms2 = 0;
  CU(cudaEventElapsedTime(&ms, ctx->km0, ctx->km1), "elapsed");
  CU(cudaEventElapsedTime(&ms2, ctx->km2, ctx->km3), "elapsed");
  const int64_t k = S.k;
  double sq = 0;
  for (int64_t c = 0; c < k; ++c) {
    const double n = double(ctx->h_km_cb[c + 1] - ctx->h_km_cb[c]);
    sq += n * n;
  }
  ctx->km_assign_ms += ms;
  ctx->km_assign_bytes += 8.0 * (double)S.p * (double)k + 20.0 * (double)S.p;
  ctx->km_update_ms += ms2;
  ctx->km_update_bytes += 8.0 * sq + 12.0 * (double)S.p;
  ctx->km_sweeps += 1;
  return DTWG_OK;
}

// cluster_result.hpp:65-72 -- ascending-j sequential sum on the host.
double km_cost(const double* dist, int64_t p) {
  double total = 0.0;
  for (int64_t j = 0; j < p; ++j) total += dist[j];
  return total;
}

// kmedoids.hpp:94-137 from the sweep's winners: empty clusters take the worst-served
// non-medoid (strict >, from the assignment distances), then sort, unique and refill.
void km_finish_update(const KmState& S, const std::vector<int64_t>& medoids, const double* dist,
                      std::vector<int64_t>& updated) {
  const dtwg_ctx* ctx = S.ctx;
  const int64_t p = S.p, k = (int64_t)medoids.size();
  updated.assign(k, 0);
  int64_t worst = -2;  // computed once: the same for every empty cluster
  for (int64_t c = 0; c < k; ++c) {
    if (ctx->h_km_cb[c] == ctx->h_km_cb[c + 1]) {  // kmedoids.hpp:97-109
      if (worst == -2) {
        worst = medoids[c];
        double worst_d = -1.0;
        for (int64_t j = 0; j < p; ++j) {
          if (std::binary_search(medoids.begin(), medoids.end(), j)) continue;
          if (dist[j] > worst_d) {  // dist[j] == D(j, assignment[j])
            worst_d = dist[j];
            worst = j;
          }
        }
      }
      updated[c] = worst < 0 ? medoids[c] : worst;
      continue;
    }
    updated[c] = ctx->h_km_best[c];
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
}

// kmedoids.hpp:33-79. The device refreshes nearest[] (and marks the new seed chosen); the
// host keeps the reference's sequential weight sum -- stored as running prefixes, since
// the draw's accumulation repeats exactly the same additions, the draw is then the first
// prefix above the target (prefixes of non-negative terms never decrease).
int km_seeds(KmState& S, int64_t k, SplitMix64& rng, std::vector<int64_t>& medoids) {
  dtwg_ctx* ctx = S.ctx;
  const int64_t p = S.p;
  medoids.clear();
  std::vector<uint8_t> chosen(p, 0);
  std::vector<double> pre(p);
  CU(cudaMemsetAsync(ctx->d_chosen.ptr, 0, p, ctx->stream), "memset chosen");
  CU(dtwgpu::launch_fill_inf(ctx->d_nearest.ptr, p, ctx->stream), "fill nearest");
  int64_t current = (int64_t)rng.next_below((uint64_t)p);
  while ((int64_t)medoids.size() < k) {
    medoids.push_back(current);
    chosen[current] = 1;
    if ((int64_t)medoids.size() == k) break;
    // the condensed matrix: ready now, while the square expansion may still be running
    CU(dtwgpu::launch_seed_step(S.cmat, true, p, current, ctx->d_chosen.ptr, ctx->d_nearest.ptr,
                                ctx->stream),
       "nearest");
    ctx->launches++;
    CU(cudaMemcpyAsync(ctx->h_km_nearest, ctx->d_nearest.ptr, p * 8, cudaMemcpyDeviceToHost,
                       ctx->stream),
       "D2H nearest");
    CU(cudaStreamSynchronize(ctx->stream), "sync");
    const double* nearest = ctx->h_km_nearest;
    double total = 0.0;
    for (int64_t j = 0; j < p; ++j) {
      if (!chosen[j]) total += nearest[j];
      pre[j] = total;
    }
    int64_t next = p;
    if (total > 0.0) {
      const double target = rng.next_double() * total;
      next = std::upper_bound(pre.begin(), pre.end(), target) - pre.begin();
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

int ensure_iota(dtwg_ctx* ctx, int64_t p) {
  if (ctx->iota_n < p) {
    CU(ctx->d_iota.reserve(p), "malloc");
    CU(dtwgpu::launch_iota(ctx->d_iota.ptr, p, ctx->stream), "iota");
    ctx->iota_n = p;
  }
  const size_t need = dtwgpu::bucket_temp_bytes(p);
  if (ctx->cub_bytes < need) {
    CU(ctx->d_cub.reserve(need), "malloc");
    ctx->cub_bytes = need;
  }
  return DTWG_OK;
}

int km_reserve(dtwg_ctx* ctx, int64_t p, int64_t k) {
  if (!ctx->km0) {
    CU(cudaEventCreate(&ctx->km0), "event");
    CU(cudaEventCreate(&ctx->km1), "event");
    CU(cudaEventCreate(&ctx->km2), "event");
    CU(cudaEventCreate(&ctx->km3), "event");
  }
  if (ctx->h_km_p < p) {
    for (double*& h : ctx->h_km_dist) {
      if (h) cudaFreeHost(h);
      h = nullptr;
      CU(cudaMallocHost(&h, std::max<int64_t>(p, 1) * 8), "pinned");
    }
    if (ctx->h_km_nearest) cudaFreeHost(ctx->h_km_nearest);
    ctx->h_km_nearest = nullptr;
    CU(cudaMallocHost(&ctx->h_km_nearest, std::max<int64_t>(p, 1) * 8), "pinned");
    ctx->h_km_p = p;
  }
  if (ctx->h_km_k < k) {
    for (int64_t** h : {&ctx->h_km_best, &ctx->h_km_cb, &ctx->h_km_med}) {
      if (*h) cudaFreeHost(*h);
      *h = nullptr;
      CU(cudaMallocHost(h, (k + 1) * 8), "pinned");
    }
    ctx->h_km_k = k;
  }
  CU(ctx->d_lab.reserve(p), "malloc");
  CU(ctx->d_keys_a.reserve(p), "malloc");
  CU(ctx->d_keys_b.reserve(p), "malloc");
  CU(ctx->d_members_p.reserve(p), "malloc");
  int rc = ensure_iota(ctx, p);
  if (rc) return rc;
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
  if (ctx->square_timed) {
    float ms = 0.f;
    if (cudaEventSynchronize(ctx->square_ready) == cudaSuccess &&
        cudaEventElapsedTime(&ms, ctx->square_t0, ctx->square_ready) == cudaSuccess)
      ctx->km_prep_ms += ms;
    cudaGetLastError();
    ctx->square_timed = false;
  }
  out[5] = ctx->km_prep_ms;
  out[6] = ctx->layout_valid ? (ctx->layout32 ? 2.0 : 1.0) : 0.0;
  out[7] = 0.0;
  if (ctx->layout_valid) {
    float ms = 0.f;
    if (cudaEventSynchronize(ctx->layout_ready) == cudaSuccess &&
        cudaEventElapsedTime(&ms, ctx->layout_t0, ctx->layout_ready) == cudaSuccess)
      out[7] = ms;
    cudaGetLastError();
  }
  if (reset) {
    ctx->km_prep_ms = 0;
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
  rc = km_reserve(ctx, p, k);
  if (rc) return rc;
  rc = ensure_layout(ctx, k);
  if (rc) return rc;
  // Independent restarts run concurrently: contiguous restart blocks on restart workers
  // (same device, own streams), observer calls replayed and the best restart reduced in
  // restart order with strict < -- the sequential loop's result, bit for bit.
  const int64_t nr = restart_end - restart_begin;
  // (small matrices: a restart is a few tens of microseconds, less than a thread hand-off).
  // Each worker's host thread spin-waits on its stream and runs the ordered host sums: on
  // the 16-thread GPU host, 8-10 workers made whole c3 runs swing 11 -> 22 ms (and up to
  // 260 ms), 4 workers held 11.1-11.7 ms (tools/km_bench.py --workers, profiles/round2).
  const int64_t hw = (int64_t)std::max(1u, std::thread::hardware_concurrency());
  // Small matrices (c5, p = 5000: latency-bound restarts) keep up to 10 workers.
  const int64_t cap = p < 2048 ? 1
                      : p >= 16384 ? std::min<int64_t>(std::max<int64_t>(hw / 4, 1), 4)
                                   : std::min<int64_t>(std::max<int64_t>(hw - 2, 1), 10);
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

// The matrix views a context's sweeps read: its own, or (restart workers) the source's.
static KmState km_state(dtwg_ctx* ctx, int64_t p, int64_t k) {
  const dtwg_ctx* m = ctx->km_src ? ctx->km_src : ctx;
  KmState S{ctx, p, k, km_matrix(ctx), km_is_cond(ctx), m->d_cond.ptr, m};
  if (m->layout_valid) {  // the sweeps wait for it (km_wait_ready), the seeding does not
    S.psq = m->d_psq.ptr;
    S.psq32 = m->layout32;
    S.perm = m->d_perm.ptr;
    S.pinv = m->d_pinv.ptr;
  }
  return S;
}

// The reference's restart loop (kmedoids.hpp:158-187) over restarts [restart_begin,
// restart_end) on one context's stream and sweep buffers.
static int km_loop(dtwg_ctx* ctx, int64_t p, int64_t k, int64_t max_iterations, uint64_t seed,
                   int64_t restart_begin, int64_t restart_end, dtwg_observer_fn observer,
                   void* user, int64_t* medoids_out, int64_t* assignment_out, double* cost_out,
                   int64_t* best_restart_out) {
  int rc = km_reserve(ctx, p, k);
  if (rc) return rc;
  KmState S = km_state(ctx, p, k);
  bool have_best = false;
  double best_cost = 0.0;
  std::vector<int64_t> medoids, updated;
  for (int64_t r = restart_begin; r < restart_end; ++r) {  // kmedoids.hpp:158-187
    SplitMix64 rng = restart_stream(seed, (uint64_t)r);
    rc = km_seeds(S, k, rng, medoids);
    if (rc) return rc;
    double cost = 0.0;
    bool converged = false;
    int buf = 0;
    rc = km_enqueue_sweep(S, medoids, buf);
    if (rc) return rc;
    for (int64_t it = 0; it < max_iterations && !converged; ++it) {
      rc = km_wait_sweep(S);  // assignment of `medoids` and its update are on the host now
      if (rc) return rc;
      const double* dist = ctx->h_km_dist[buf];
      km_finish_update(S, medoids, dist, updated);
      converged = updated == medoids;
      // the next sweep runs while the host sums this assignment's cost
      const bool more = !converged && it + 1 < max_iterations;
      if (more) {
        rc = km_enqueue_sweep(S, updated, buf ^ 1);
        if (rc) return rc;
      }
      cost = km_cost(dist, p);  // cluster_result.hpp:65-72
      if (observer) observer(user, r, it, cost);
      if (!converged) {
        medoids = updated;
        buf ^= 1;
      }
    }
    if (!converged) {  // iteration cap hit right after an update (kmedoids.hpp:177-180)
      rc = km_enqueue_assign(S, medoids);
      if (rc) return rc;
      CU(cudaMemcpyAsync(ctx->h_km_dist[buf], ctx->d_dist.ptr, p * 8, cudaMemcpyDeviceToHost,
                         ctx->stream),
         "D2H dist");
      CU(cudaStreamSynchronize(ctx->stream), "sync");
      cost = km_cost(ctx->h_km_dist[buf], p);
    }
    if (!have_best || cost < best_cost) {
      best_cost = cost;
      have_best = true;
      if (medoids_out) std::copy(medoids.begin(), medoids.end(), medoids_out);
      if (assignment_out)
        CU(cudaMemcpy(assignment_out, ctx->d_assign.ptr, p * 8, cudaMemcpyDeviceToHost),
           "D2H assignment");
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
  KmState S = km_state(ctx, p, k);
  std::vector<int64_t> med(medoids, medoids + k);
  rc = km_enqueue_assign(S, med);
  if (rc) return rc;
  if (assignment_out)
    CU(cudaMemcpyAsync(assignment_out, ctx->d_assign.ptr, p * 8, cudaMemcpyDeviceToHost,
                       ctx->stream),
       "D2H assignment");
  if (dist_out)
    CU(cudaMemcpyAsync(dist_out, ctx->d_dist.ptr, p * 8, cudaMemcpyDeviceToHost, ctx->stream),
       "D2H dist");
  CU(cudaStreamSynchronize(ctx->stream), "sync");
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
  for (int64_t j = 0; j < p; ++j)
    if (assignment[j] < 0 || assignment[j] >= p)
      return ctx->fail(DTWG_INDEX_OUT_OF_RANGE, "assignment out of range");
  KmState S = km_state(ctx, p, k);
  km_wait_ready(S);
  std::vector<int64_t> med(medoids, medoids + k);
  // The caller's assignment (any, not necessarily nearest-medoid): cluster slots by
  // lower_bound (kmedoids.hpp:88-90) and D(j, assignment[j]) for the empty-cluster repair.
  CU(ctx->d_assign.reserve(p), "malloc");
  std::copy(med.begin(), med.end(), ctx->h_km_med);
  CU(cudaMemcpyAsync(ctx->d_medoids.ptr, ctx->h_km_med, k * 8, cudaMemcpyHostToDevice, ctx->stream),
     "H2D medoids");
  CU(cudaMemcpyAsync(ctx->d_assign.ptr, assignment, p * 8, cudaMemcpyHostToDevice, ctx->stream),
     "H2D assignment");
  CU(dtwgpu::launch_slots_of(S.sq, S.cond, p, ctx->d_medoids.ptr, k, ctx->d_assign.ptr,
                             ctx->d_dist.ptr, ctx->d_lab.ptr, ctx->stream),
     "slots");
  CU(cudaEventRecord(ctx->km2, ctx->stream), "event");
  CU(dtwgpu::launch_bucket(ctx->d_lab.ptr, S.psq ? S.perm : nullptr, ctx->d_iota.ptr, p, k,
                           ctx->d_keys_a.ptr, ctx->d_keys_b.ptr, ctx->d_members.ptr,
                           ctx->d_members_p.ptr, ctx->d_cb.ptr, ctx->d_cub.ptr, ctx->cub_bytes,
                           ctx->stream),
     "bucket");
  CU(dtwgpu::launch_update2(S.sq, S.cond, S.psq, S.psq32, S.pinv, p, ctx->d_members.ptr,
                            ctx->d_members_p.ptr, ctx->d_cb.ptr, k, ctx->d_best_member.ptr,
                            ctx->d_best_sum.ptr, ctx->stream),
     "update");
  CU(cudaEventRecord(ctx->km3, ctx->stream), "event");
  ctx->launches += 1 + km_update_launches(S);
  CU(cudaMemcpyAsync(ctx->h_km_dist[0], ctx->d_dist.ptr, p * 8, cudaMemcpyDeviceToHost, ctx->stream),
     "D2H dist");
  CU(cudaMemcpyAsync(ctx->h_km_cb, ctx->d_cb.ptr, (k + 1) * 8, cudaMemcpyDeviceToHost, ctx->stream),
     "D2H cb");
  CU(cudaMemcpyAsync(ctx->h_km_best, ctx->d_best_member.ptr, k * 8, cudaMemcpyDeviceToHost,
                     ctx->stream),
     "D2H best");
  CU(cudaStreamSynchronize(ctx->stream), "sync");
  std::vector<int64_t> upd;
  km_finish_update(S, med, ctx->h_km_dist[0], upd);
  std::copy(upd.begin(), upd.end(), updated_out);
  return DTWG_OK;
}

}  // extern "C"
