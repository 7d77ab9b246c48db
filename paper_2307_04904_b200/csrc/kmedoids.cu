// kmedoids.cu -- sm_100a sweep kernels over the device-resident distance matrix.
//
// They replace the O(p*k) and O(sum |C|^2) distance reads of the reference's
// k-medoids: the nearest-distance refresh of spread seeding
// (kmedoids.hpp:48-52), nearest-medoid assignment (cluster_result.hpp:40-61) and the
// per-candidate member sums of the medoid update (kmedoids.hpp:111-121). Every
// floating-point result that decides an outcome keeps the reference's order: the
// winning candidate's sum (and any candidate that could tie it) is one thread's
// ascending-member sequential loop; warp-tree sums only rule candidates out, with a
// rigorous error bound (see tree_sum_kernel). Comparisons are strict with the lowest
// index winning. Sequential scalar sums over p (assignment_cost, seeding weights) stay
// on the host, exactly as written in the reference.
//
// The matrix is expanded once from condensed to a dense p x p square so every sweep
// reads contiguous rows (D is symmetric and D[i][j], D[j][i] are the same stored
// double, so reading the transposed entry is bit-identical).
#include <cuda_runtime.h>

#include <algorithm>
#include <cub/device/device_radix_sort.cuh>
#include <math_constants.h>

#include <cstdint>

#include "dtw_fill.cuh"

namespace dtwgpu {
namespace {

__device__ __forceinline__ int64_t coff(int64_t i, int64_t p) { return i * p - i * (i + 1) / 2; }

// The sweeps read D(r, c) through a view: the dense square (contiguous rows, the fast
// path) or, when p x p doubles do not fit next to everything else in HBM, the condensed
// matrix itself (D(r, r) = 0; other entries at the upper-triangle slot). Both return the
// same stored double for (r, c) and (c, r), so results are identical either way.
struct SquareView {
  const double* m;
  int64_t p;
  __device__ __forceinline__ double operator()(int64_t r, int64_t c) const { return m[r * p + c]; }
};
struct CondView {
  const double* m;
  int64_t p;
  __device__ __forceinline__ double operator()(int64_t r, int64_t c) const {
    if (r == c) return 0.0;
    const int64_t i = r < c ? r : c, j = r < c ? c : r;
    return m[coff(i, p) + (j - i - 1)];
  }
};

// Dense square from condensed: 32x32 tiles; lower tiles read their transposed upper
// tile coalesced through shared memory.
__global__ void expand_square_kernel(const double* __restrict__ cond, int64_t p,
                                     double* __restrict__ sq) {
  __shared__ double tile[32][33];
  const int64_t bi = (int64_t)blockIdx.y * 32, bj = (int64_t)blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  if (bi <= bj) {
    for (int r = ty; r < 32; r += 8) {
      const int64_t i = bi + r, j = bj + tx;
      if (i < p && j < p) {
        double v;
        if (i == j) v = 0.0;
        else if (i < j) v = cond[coff(i, p) + (j - i - 1)];
        else v = cond[coff(j, p) + (i - j - 1)];
        sq[i * p + j] = v;
      }
    }
  } else {
    // tile (bi, bj) below the diagonal = transpose of upper tile (bj, bi)
    for (int r = ty; r < 32; r += 8) {
      const int64_t i = bj + r, j = bi + tx;  // upper element (i < j)
      if (i < p && j < p) tile[r][tx] = cond[coff(i, p) + (j - i - 1)];
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
      const int64_t i = bi + r, j = bj + tx;
      if (i < p && j < p) sq[i * p + j] = tile[tx][r];
    }
  }
}

// DistanceMatrix::from_condensed validation (distance_matrix.hpp:34-38). flags[0]: some
// entry is not finite or negative; flags[1]: some non-zero entry lies outside
// [2^-100, 2^100] (the fp32 copy for the k-medoids candidate-sum filter would then lose
// its relative error bound, see ensure_layout).
__global__ void validate_kernel(const double* __restrict__ cond, int64_t total, int* flags) {
  int local = 0, range = 0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const double v = cond[t];
    if (!(isfinite(v) && v >= 0.0)) local = 1;
    if (v != 0.0 && !(v >= 0x1p-100 && v <= 0x1p100)) range = 1;
  }
  if (__any_sync(0xffffffffu, local) && (threadIdx.x & 31) == 0) atomicOr(flags, 1);
  if (__any_sync(0xffffffffu, range) && (threadIdx.x & 31) == 0) atomicOr(flags + 1, 1);
}

// kmedoids.hpp:48-52: nearest[j] = std::min(nearest[j], D(j, current)) for unchosen j.
template <class V>
__global__ void nearest_update_kernel(const V D, int64_t p, int64_t current,
                                      const uint8_t* __restrict__ chosen,
                                      double* __restrict__ nearest) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p;
       j += (int64_t)gridDim.x * blockDim.x) {
    if (chosen[j]) continue;
    const double a = nearest[j], b = D(current, j);  // D(current, j) == D(j, current)
    nearest[j] = b < a ? b : a;
  }
}

// cluster_result.hpp:40-61. Medoids ascending; a medoid owns itself; otherwise the
// strictly smaller distance wins, so ties keep the lowest medoid index. Row reads
// D(medoid_t, j) are coalesced across j.
template <class V>
__global__ void assign_kernel(const V D, int64_t p, const int64_t* __restrict__ medoids, int64_t k,
                              int64_t* __restrict__ assignment, double* __restrict__ dist) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p;
       j += (int64_t)gridDim.x * blockDim.x) {
    bool is_med = false;
    for (int64_t t = 0; t < k; ++t) is_med |= (__ldg(medoids + t) == j);
    if (is_med) {
      assignment[j] = j;
      dist[j] = 0.0;
      continue;
    }
    int64_t best = __ldg(medoids);
    double bd = D(best, j);
    for (int64_t t = 1; t < k; ++t) {
      const int64_t mt = __ldg(medoids + t);
      const double d = D(mt, j);
      if (d < bd) {
        bd = d;
        best = mt;
      }
    }
    assignment[j] = best;
    dist[j] = bd;
  }
}

// kmedoids.hpp:113-120: one thread per candidate; sequential ascending-member sum.
// members: all clusters concatenated, each ascending; cluster c = [cb[c], cb[c+1]).
// ---- medoid update (kmedoids.hpp:84-139) -------------------------------------------
// The reference sums each candidate's distances to its cluster sequentially, in
// ascending member order, and keeps the first candidate with the strictly smallest sum.
// Only that argmin (and its sum) matters, so the sums are computed in two passes:
//  1. tree_sum_kernel: one warp per candidate, lanes stride over the members and the
//     warp reduces with shuffles -- full parallelism and bandwidth, any summation order.
//  2. cluster_select_kernel: one block per cluster. With n = |C| non-negative terms, any
//     order of the n-1 roundings is within gamma_{n-1} * S of the exact sum S (Higham,
//     Accuracy and Stability, sec. 4.2), for the tree sum and the reference's sequential
//     sum alike. So a candidate whose tree sum exceeds min_tree * ((1+g)/(1-g))^2 cannot
//     have the smallest sequential sum; the remaining "contenders" (normally just one)
//     get the reference's exact sequential sum, and the (sum, position) minimum over
//     them is the reference's choice, bit for bit.
template <class V>
__global__ void tree_sum_kernel(const V D, int64_t p, const int32_t* __restrict__ members,
                                const int64_t* __restrict__ cb, int64_t k,
                                double* __restrict__ tsum) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < p; q += nw) {
    int64_t lo = 0, hi = k - 1;  // cluster c with cb[c] <= q < cb[c+1]
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) / 2;
      if (__ldg(cb + mid) <= q) lo = mid;
      else hi = mid - 1;
    }
    const int64_t b = __ldg(cb + lo), e = __ldg(cb + lo + 1);
    const int64_t a = __ldg(members + q);  // D[a][.] == D[.][a]
    double acc = 0.0;
    int64_t t = b + lane;
    for (; t + 96 < e; t += 128) {  // 4 loads in flight per lane
      const double v0 = D(a, __ldg(members + t)), v1 = D(a, __ldg(members + t + 32));
      const double v2 = D(a, __ldg(members + t + 64)), v3 = D(a, __ldg(members + t + 96));
      acc = __dadd_rn(__dadd_rn(acc, v0), __dadd_rn(__dadd_rn(v1, v2), v3));
    }
    for (; t < e; t += 32) acc = __dadd_rn(acc, D(a, __ldg(members + t)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    if (lane == 0) tsum[q] = acc;
  }
}

template <class V>
__global__ void cluster_select_kernel(const V D, int64_t p, const int32_t* __restrict__ members,
                                      const int64_t* __restrict__ cb,
                                      const double* __restrict__ tsum, int64_t* best_member,
                                      double* best_sum, bool in32 = false) {
  const int64_t c = blockIdx.x;
  const int64_t b = cb[c], e = cb[c + 1];
  __shared__ double sv[256];
  __shared__ int64_t sq_[256];
  // (1) minimum tree sum
  double mn = CUDART_INF;
  for (int64_t q = b + threadIdx.x; q < e; q += blockDim.x) mn = fmin(mn, tsum[q]);
  sv[threadIdx.x] = mn;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sv[threadIdx.x] = fmin(sv[threadIdx.x], sv[threadIdx.x + w]);
    __syncthreads();
  }
  mn = sv[0];
  __syncthreads();
  // (2) contenders: exact sequential sums (ascending members, kmedoids.hpp:111-121)
  const double n = (double)(e - b);
  const double u = 1.1102230246251565e-16;  // 2^-53
  // fp32 inputs (in32): every term is also rounded once to fp32, relative 2^-24
  const double g = n * u / (1.0 - n * u) + (in32 ? 0x1p-24 : 0.0);
  const double thr = mn * (1.0 + 8.0 * g) * (1.0 + 4.0 * u);
  // Collect the contenders; the block then computes each one's sequential sum: all
  // threads gather the candidate's member distances into shared memory (parallel loads),
  // thread 0 adds them in ascending member order (the reference's order).
  constexpr int kMaxCand = 64, kChunk = 2048;
  __shared__ int ncand;
  __shared__ int64_t cand[kMaxCand];
  __shared__ double vals[kChunk];
  if (threadIdx.x == 0) ncand = 0;
  __syncthreads();
  for (int64_t q = b + threadIdx.x; q < e; q += blockDim.x) {
    if (!(tsum[q] <= thr)) continue;
    const int slot = atomicAdd(&ncand, 1);
    if (slot < kMaxCand) cand[slot] = q;
  }
  __syncthreads();
  double bv = CUDART_INF;
  int64_t bq = -1;
  if (ncand == 1) {
    // A single contender is the reference's choice whatever its exact sum (only the
    // argmin is used; best_sum then holds the tree sum).
    if (threadIdx.x == 0) {
      bv = tsum[cand[0]];
      bq = cand[0];
    }
  } else if (ncand <= kMaxCand) {
    for (int ci = 0; ci < ncand; ++ci) {
      const int64_t q = cand[ci];
      const int64_t a = members[q];
      double sum = 0.0;
      for (int64_t t0 = b; t0 < e; t0 += kChunk) {
        const int64_t len = e - t0 < kChunk ? e - t0 : kChunk;
        for (int64_t t = threadIdx.x; t < len; t += blockDim.x) vals[t] = D(a, __ldg(members + t0 + t));
        __syncthreads();
        if (threadIdx.x == 0) {
          int64_t t = 0;
          for (; t + 8 <= len; t += 8) {  // loads batched, additions in order
            double v[8];
#pragma unroll
            for (int uu = 0; uu < 8; ++uu) v[uu] = vals[t + uu];
#pragma unroll
            for (int uu = 0; uu < 8; ++uu) sum = __dadd_rn(sum, v[uu]);
          }
          for (; t < len; ++t) sum = __dadd_rn(sum, vals[t]);
        }
        __syncthreads();
      }
      // contenders arrive in any order: lexicographic (sum, position) keeps the first minimum
      if (threadIdx.x == 0 && (bq < 0 || sum < bv || (sum == bv && q < bq))) {
        bv = sum;
        bq = q;
      }
    }
  } else {  // many near-equal sums (e.g. duplicated series): one thread per contender
    for (int64_t q = b + threadIdx.x; q < e; q += blockDim.x) {
      if (!(tsum[q] <= thr)) continue;
      const int64_t a = members[q];
      double sum = 0.0;
      int64_t t = b;
      for (; t + 8 <= e; t += 8) {  // loads batched, additions kept in order
        double v[8];
#pragma unroll
        for (int uu = 0; uu < 8; ++uu) v[uu] = D(a, __ldg(members + t + uu));
#pragma unroll
        for (int uu = 0; uu < 8; ++uu) sum = __dadd_rn(sum, v[uu]);
      }
      for (; t < e; ++t) sum = __dadd_rn(sum, D(a, __ldg(members + t)));
      if (bq < 0 || sum < bv) {  // q ascending per thread: strict < keeps the first minimum
        bv = sum;
        bq = q;
      }
    }
  }
  sv[threadIdx.x] = bv;
  sq_[threadIdx.x] = bq;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const double ov = sv[threadIdx.x + w];
      const int64_t oq = sq_[threadIdx.x + w];
      const int64_t mq = sq_[threadIdx.x];
      if (oq >= 0 && (mq < 0 || ov < sv[threadIdx.x] || (ov == sv[threadIdx.x] && oq < mq))) {
        sv[threadIdx.x] = ov;
        sq_[threadIdx.x] = oq;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    best_member[c] = sq_[0] >= 0 ? (int64_t)members[sq_[0]] : -1;
    best_sum[c] = sv[0];
  }
}

// Band-family series copy: series i at bsamples[boff[i] .. + len), surrounded by pad
// +inf samples (built on the device from the packed series).
template <class T>
__global__ void band_pad_kernel(const double* __restrict__ samples, const int64_t* __restrict__ off,
                                const int64_t* __restrict__ boff, int64_t p, int64_t pad,
                                T* __restrict__ out) {
  const T inf = (T)CUDART_INF;
  for (int64_t i = blockIdx.x; i < p; i += gridDim.x) {
    const int64_t s0 = off[i], len = off[i + 1] - s0, d0 = boff[i];
    for (int64_t t = threadIdx.x; t < len + 2 * pad; t += blockDim.x) {
      const int64_t k = t - pad;
      out[d0 - pad + t] = (k >= 0 && k < len) ? (T)samples[s0 + k] : inf;
    }
  }
}

__global__ void to_f32_kernel(const double* __restrict__ in, int64_t n, float* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = (float)in[t];
}

// validation.hpp:30-79 silhouette, per series t: a = mean distance to the other members
// of its own cluster, b = smallest mean distance to another non-empty cluster, s =
// (b - a) / max(a, b) (0 when that is 0; singletons score 0). Every sum runs over the
// members in ascending order, as the reference does, reading D(m, t) = D(t, m) so a warp
// of consecutive t reads one coalesced row segment per member m.
template <class V>
__global__ void silhouette_kernel(const V D, int64_t p,
                                  const int32_t* __restrict__ members,
                                  const int64_t* __restrict__ cb, const int32_t* __restrict__ cls,
                                  int64_t k, double* __restrict__ sil) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < p;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = cls[t];
    const int64_t own_n = cb[c + 1] - cb[c];
    if (own_n == 1) {
      sil[t] = 0.0;
      continue;
    }
    double own = 0.0;
    for (int64_t q = cb[c]; q < cb[c + 1]; ++q) {
      const int64_t m = members[q];
      if (m != t) own = __dadd_rn(own, D(m, t));
    }
    const double a = __ddiv_rn(own, (double)(own_n - 1));
    double b = CUDART_INF;
    for (int64_t o = 0; o < k; ++o) {
      const int64_t n_o = cb[o + 1] - cb[o];
      if (o == c || n_o == 0) continue;
      double across = 0.0;
      for (int64_t q = cb[o]; q < cb[o + 1]; ++q) across = __dadd_rn(across, D((int64_t)members[q], t));
      const double mean = __ddiv_rn(across, (double)n_o);
      b = mean < b ? mean : b;  // std::min(b, mean)
    }
    const double denom = a < b ? b : a;  // std::max(a, b)
    sil[t] = denom > 0.0 ? __ddiv_rn(__dsub_rn(b, a), denom) : 0.0;
  }
}


// ---- sweep kernels, round 2 -----------------------------------------------------------
// cluster_result.hpp:40-61, one block per 32 consecutive series j: warp w of the block's
// 8 takes the medoids t = w, w+8, w+16, ... (4 independent row loads in flight per lane,
// every load a coalesced 256-byte row segment D(m_t, j0..j0+31)); the 8 per-warp minima
// are then merged in shared memory by (distance, t) -- the lowest t among equal
// distances, which is exactly what the reference's ascending-t scan with strict < keeps.
// A medoid owns itself. Besides the assignment and its distance, the kernel writes the
// cluster slot t (medoids ascending: slot = lower_bound(medoids, assignment[j]),
// kmedoids.hpp:88-90) for the device-side bucketing that follows.
template <class V>
__global__ void __launch_bounds__(256) assign_slots_kernel(
    const V D, int64_t p, const int64_t* __restrict__ medoids, int64_t k,
    int64_t* __restrict__ assignment, double* __restrict__ dist, int32_t* __restrict__ lab,
    int32_t* __restrict__ counts) {
  __shared__ double sd[8][32];
  __shared__ int st[8][32];
  __shared__ int sm[8][32];
  __shared__ int hist[256];  // cluster sizes (counts != nullptr: k <= 256)
  if (counts)
    for (int c = threadIdx.x; c < k; c += blockDim.x) hist[c] = 0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t j0 = (int64_t)blockIdx.x * 32; j0 < p; j0 += (int64_t)gridDim.x * 32) {
    const int64_t j = j0 + lane;
    const bool in = j < p;
    double bd = CUDART_INF;
    int bt = -1, med = -1;
    for (int64_t t = w; t < k; t += 32) {
      int64_t m[4];
      double d[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t tt = t + 8 * u;
        m[u] = tt < k ? __ldg(medoids + tt) : -1;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) d[u] = (m[u] >= 0 && in) ? D(m[u], j) : CUDART_INF;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (m[u] < 0) continue;
        if (m[u] == j) med = (int)(t + 8 * u);
        if (bt < 0 || d[u] < bd) {  // t ascending within the warp: strict < keeps the first
          bd = d[u];
          bt = (int)(t + 8 * u);
        }
      }
    }
    sd[w][lane] = bd;
    st[w][lane] = bt;
    sm[w][lane] = med;
    __syncthreads();
    if (w == 0 && in) {
      double b = CUDART_INF;
      int tb = -1, md = -1;
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        if (sm[x][lane] >= 0) md = sm[x][lane];
        const int tx = st[x][lane];
        const double vx = sd[x][lane];
        if (tx >= 0 && (tb < 0 || vx < b || (vx == b && tx < tb))) {
          b = vx;
          tb = tx;
        }
      }
      if (md >= 0) {
        assignment[j] = j;
        dist[j] = 0.0;
        lab[j] = md;
      } else {
        assignment[j] = __ldg(medoids + tb);
        dist[j] = b;
        lab[j] = tb;
      }
      if (counts) atomicAdd(&hist[md >= 0 ? md : tb], 1);
    }
    __syncthreads();
  }
  if (counts)
    for (int c = threadIdx.x; c < k; c += blockDim.x)
      if (hist[c]) atomicAdd(counts + c, hist[c]);
}

// kmedoids.hpp:88-90 for a caller-given assignment (dtwg_km_update): the cluster slot
// lower_bound(medoids, assignment[j]) and D(j, assignment[j]).
template <class V>
__global__ void slots_of_kernel(const V D, int64_t p, const int64_t* __restrict__ medoids,
                                int64_t k, const int64_t* __restrict__ assignment,
                                double* __restrict__ dist, int32_t* __restrict__ lab) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = assignment[j];
    int64_t lo = 0, hi = k;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (medoids[mid] < a) lo = mid + 1;
      else hi = mid;
    }
    lab[j] = (int32_t)lo;
    dist[j] = a == j ? 0.0 : D(a, j);
  }
}

// kmedoids.hpp:45-52 for one seeding step: `current` becomes chosen and every unchosen
// nearest[j] = std::min(nearest[j], D(j, current)) (b < a ? b : a).
template <class V>
__global__ void seed_step_kernel(const V D, int64_t p, int64_t current,
                                 uint8_t* __restrict__ chosen, double* __restrict__ nearest) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p;
       j += (int64_t)gridDim.x * blockDim.x) {
    if (j == current) {
      chosen[j] = 1;
      continue;
    }
    if (chosen[j]) continue;
    const double a = nearest[j], b = D(current, j);
    nearest[j] = b < a ? b : a;
  }
}

// Cluster boundaries from the labels sorted ascending: cb[c] = first position with
// label >= c, cb[k] = p (empty clusters get equal neighbours).
__global__ void cluster_bounds_kernel(const int32_t* __restrict__ sorted, int64_t p, int64_t k,
                                      int64_t* __restrict__ cb) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < p;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = q == 0 ? 0 : (int64_t)sorted[q - 1] + 1, hi = sorted[q];
    for (int64_t c = lo; c <= hi; ++c) cb[c] = q;
    if (q == p - 1)
      for (int64_t c = hi + 1; c <= k; ++c) cb[c] = p;
  }
}

__global__ void fill_inf_kernel(double* __restrict__ out, int64_t n) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = CUDART_INF;
}

__global__ void iota_kernel(int32_t* __restrict__ out, int64_t n) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = (int32_t)t;
}

// keys[u] = lab[perm[u]]: the cluster slot of the series stored at permuted position u.
__global__ void permuted_labels_kernel(const int32_t* __restrict__ lab,
                                       const int32_t* __restrict__ perm, int64_t p,
                                       int32_t* __restrict__ keys) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < p;
       u += (int64_t)gridDim.x * blockDim.x)
    keys[u] = lab[perm[u]];
}

__global__ void inverse_perm_kernel(const int32_t* __restrict__ perm, int64_t p,
                                    int32_t* __restrict__ pinv) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < p;
       u += (int64_t)gridDim.x * blockDim.x)
    pinv[perm[u]] = (int32_t)u;
}

// Candidate sums over the cluster-ordered copy of the square (see launch_update2): the
// candidate's row is psq row pinv[a] and its cluster's members, as positions u of that
// copy, are ascending -- runs of consecutive u, so the warp's loads are coalesced instead
// of one 32-byte sector per member. Any summation order: these sums only rule candidates
// out (cluster_select_kernel).
template <class T>
__global__ void tree_sum_perm_kernel(const T* __restrict__ psq, int64_t p,
                                     const int32_t* __restrict__ pinv,
                                     const int32_t* __restrict__ members,
                                     const int32_t* __restrict__ members_perm,
                                     const int64_t* __restrict__ cb, int64_t k,
                                     double* __restrict__ tsum) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < p; q += nw) {
    int64_t lo = 0, hi = k - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) / 2;
      if (__ldg(cb + mid) <= q) lo = mid;
      else hi = mid - 1;
    }
    const int64_t b = __ldg(cb + lo), e = __ldg(cb + lo + 1);
    const T* row = psq + (int64_t)__ldg(pinv + __ldg(members + q)) * p;
    double acc0 = 0.0, acc1 = 0.0;
    int64_t t = b + lane;
    for (; t + 224 < e; t += 256) {  // 8 loads in flight per lane
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = (double)__ldg(row + __ldg(members_perm + t + 32 * u));
      acc0 = __dadd_rn(acc0, __dadd_rn(__dadd_rn(v[0], v[1]), __dadd_rn(v[2], v[3])));
      acc1 = __dadd_rn(acc1, __dadd_rn(__dadd_rn(v[4], v[5]), __dadd_rn(v[6], v[7])));
    }
    for (; t < e; t += 32) acc0 = __dadd_rn(acc0, (double)__ldg(row + __ldg(members_perm + t)));
    double acc = __dadd_rn(acc0, acc1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    if (lane == 0) tsum[q] = acc;
  }
}

// psq[u][v] = sq[perm[u]][perm[v]]. Rows up to kPermSmemRow doubles: the source row is
// staged in shared memory by coalesced 16-byte loads and the output row is written from
// it, so DRAM reads every source row once. Longer rows gather through L2 with few rows in
// flight (a grid sized so the rows being gathered stay L2-resident).
constexpr int kPermSmemRow = 26624;  // 208 KB
template <class T>
__global__ void __launch_bounds__(1024) permute_square_smem_kernel(const double* __restrict__ sq,
                                                                   int64_t p,
                                                                   const int32_t* __restrict__ perm,
                                                                   T* __restrict__ psq) {
  // the row is staged already converted to T: an fp32 copy stages half the bytes, so two
  // blocks (two rows in flight) fit per SM
  extern __shared__ __align__(16) unsigned char row_raw[];
  T* row = reinterpret_cast<T*>(row_raw);
  for (int64_t u = blockIdx.x; u < p; u += gridDim.x) {
    const double* src = sq + (int64_t)__ldg(perm + u) * p;
    if ((p & 1) == 0) {
      const double2* s2 = reinterpret_cast<const double2*>(src);
      for (int64_t v = threadIdx.x; v < p / 2; v += blockDim.x) {
        const double2 d = __ldcs(s2 + v);
        row[2 * v] = (T)d.x;
        row[2 * v + 1] = (T)d.y;
      }
    } else {
      for (int64_t v = threadIdx.x; v < p; v += blockDim.x) row[v] = (T)__ldcs(src + v);
    }
    __syncthreads();
    T* dst = psq + u * p;
    for (int64_t v = threadIdx.x; v < p; v += blockDim.x) __stcs(dst + v, row[__ldg(perm + v)]);
    __syncthreads();
  }
}

template <class T>
__global__ void __launch_bounds__(512) permute_square_l2_kernel(const double* __restrict__ sq,
                                                                int64_t p,
                                                                const int32_t* __restrict__ perm,
                                                                T* __restrict__ psq) {
  for (int64_t u = blockIdx.x; u < p; u += gridDim.x) {
    const double* src = sq + (int64_t)__ldg(perm + u) * p;
    T* dst = psq + u * p;
    for (int64_t v = threadIdx.x; v < p; v += 512)
      __stcs(dst + v, (T)__ldg(src + __ldg(perm + v)));
  }
}


// Device bucketing for k <= kBucketSmallK (kmedoids.hpp:86-92): counts per cluster slot,
// then one block per (cluster, order) compacts the series of that cluster in ascending
// order -- series index order (members) or, for the cluster-ordered copy, position order
// (members_perm) -- with warp ballots/scans; each block derives its cluster's start from
// the counts, so the bounds cb come out of the same pass. Integer-only and deterministic.
constexpr int kBucketSmallK = 256;
__global__ void cluster_count_kernel(const int32_t* __restrict__ lab, int64_t p, int64_t k,
                                     int32_t* __restrict__ counts) {
  __shared__ int h[kBucketSmallK];
  for (int c = threadIdx.x; c < k; c += blockDim.x) h[c] = 0;
  __syncthreads();
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p;
       j += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&h[lab[j]], 1);
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x)
    if (h[c]) atomicAdd(counts + c, h[c]);
}

__global__ void __launch_bounds__(1024) cluster_compact_kernel(
    const int32_t* __restrict__ lab, const int32_t* __restrict__ perm, int64_t p, int64_t k,
    const int32_t* __restrict__ counts, int32_t* __restrict__ members,
    int32_t* __restrict__ members_perm, int64_t* __restrict__ cb) {
  __shared__ int wsum[32];
  __shared__ int64_t sbase;
  const int c = blockIdx.x % k;
  const bool by_pos = blockIdx.x >= k;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (w == 0) {
    int64_t b = 0;
    for (int x = lane; x < c; x += 32) b += counts[x];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
    if (lane == 0) {
      sbase = b;
      if (!by_pos) {
        cb[c] = b;
        if (c == k - 1) cb[k] = p;
      }
    }
  }
  __syncthreads();
  int32_t* out = by_pos ? members_perm : members;
  int64_t running = sbase;
  for (int64_t c0 = 0; c0 < p; c0 += 8 * 1024) {
    const int64_t u0 = c0 + 8 * (int64_t)tid;
    bool f[8];
    int cnt = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t u = u0 + i;
      f[i] = u < p && (by_pos ? __ldg(lab + __ldg(perm + u)) : __ldg(lab + u)) == c;
      cnt += f[i];
    }
    int x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      int v = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      wsum[lane] = v;
    }
    __syncthreads();
    int64_t off = running + (w ? wsum[w - 1] : 0) + x - cnt;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (f[i]) out[off++] = (int32_t)(u0 + i);
    running += wsum[31];
    __syncthreads();
  }
}

int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 32) g = 148 * 32;
  return (int)(g > 0 ? g : 1);
}

}  // namespace

cudaError_t launch_band_pad(const double* samples, const int64_t* off, const int64_t* boff,
                            int64_t p, int64_t pad, void* out, bool fp32, cudaStream_t s) {
  const unsigned blocks = (unsigned)(p < 148 * 16 ? p : 148 * 16);
  if (fp32)
    band_pad_kernel<float><<<blocks, 256, 0, s>>>(samples, off, boff, p, pad, (float*)out);
  else
    band_pad_kernel<double><<<blocks, 256, 0, s>>>(samples, off, boff, p, pad, (double*)out);
  return cudaGetLastError();
}

cudaError_t launch_to_f32(const double* in, int64_t n, float* out, cudaStream_t s) {
  to_f32_kernel<<<grid_for(n, 256), 256, 0, s>>>(in, n, out);
  return cudaGetLastError();
}

cudaError_t launch_silhouette(const double* matrix, bool condensed, int64_t p,
                              const int32_t* members, const int64_t* cluster_begin,
                              const int32_t* cls, int64_t k, double* sil, cudaStream_t s) {
  if (condensed)
    silhouette_kernel<<<grid_for(p, 128), 128, 0, s>>>(CondView{matrix, p}, p, members,
                                                        cluster_begin, cls, k, sil);
  else
    silhouette_kernel<<<grid_for(p, 128), 128, 0, s>>>(SquareView{matrix, p}, p, members,
                                                        cluster_begin, cls, k, sil);
  return cudaGetLastError();
}

cudaError_t launch_expand_square(const double* condensed, int64_t p, double* square,
                                 cudaStream_t s) {
  const unsigned nb = (unsigned)((p + 31) / 32);
  expand_square_kernel<<<dim3(nb, nb), dim3(32, 8), 0, s>>>(condensed, p, square);
  return cudaGetLastError();
}

cudaError_t launch_validate_condensed(const double* condensed, int64_t total, int* flags,
                                      cudaStream_t s) {
  validate_kernel<<<grid_for(total, 256), 256, 0, s>>>(condensed, total, flags);
  return cudaGetLastError();
}

cudaError_t launch_nearest_update(const double* matrix, bool condensed, int64_t p,
                                  int64_t current, const uint8_t* chosen, double* nearest,
                                  cudaStream_t s) {
  if (condensed)
    nearest_update_kernel<<<grid_for(p, 256), 256, 0, s>>>(CondView{matrix, p}, p, current,
                                                           chosen, nearest);
  else
    nearest_update_kernel<<<grid_for(p, 256), 256, 0, s>>>(SquareView{matrix, p}, p, current,
                                                           chosen, nearest);
  return cudaGetLastError();
}

cudaError_t launch_assign(const double* matrix, bool condensed, int64_t p,
                          const int64_t* medoids, int64_t k, int64_t* assignment, double* dist,
                          cudaStream_t s) {
  if (condensed)
    assign_kernel<<<grid_for(p, 256), 256, 0, s>>>(CondView{matrix, p}, p, medoids, k,
                                                   assignment, dist);
  else
    assign_kernel<<<grid_for(p, 256), 256, 0, s>>>(SquareView{matrix, p}, p, medoids, k,
                                                   assignment, dist);
  return cudaGetLastError();
}

cudaError_t launch_update(const double* matrix, bool condensed, int64_t p,
                          const int32_t* members, const int64_t* cluster_begin, int64_t k,
                          int64_t* best_member, double* best_sum, cudaStream_t s) {
  // sums scratch lives right after best_sum (k doubles) -- caller allocates p more.
  double* sums = best_sum + k;
  const int64_t warps = std::min<int64_t>(p, 148 * 64);
  const unsigned tb = (unsigned)((warps + 7) / 8);
  if (condensed)
    tree_sum_kernel<<<tb, 256, 0, s>>>(CondView{matrix, p}, p, members, cluster_begin, k, sums);
  else
    tree_sum_kernel<<<tb, 256, 0, s>>>(SquareView{matrix, p}, p, members, cluster_begin, k, sums);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (condensed)
    cluster_select_kernel<<<(unsigned)k, 256, 0, s>>>(CondView{matrix, p}, p, members,
                                                      cluster_begin, sums, best_member, best_sum);
  else
    cluster_select_kernel<<<(unsigned)k, 256, 0, s>>>(SquareView{matrix, p}, p, members,
                                                      cluster_begin, sums, best_member, best_sum);
  return cudaGetLastError();
}


// ---- round-2 sweep launchers ----------------------------------------------------------
cudaError_t launch_assign_slots(const double* matrix, bool condensed, int64_t p,
                                const int64_t* medoids, int64_t k, int64_t* assignment,
                                double* dist, int32_t* lab, cudaStream_t s, int32_t* counts) {
  if (counts && k > 256) counts = nullptr;
  if (counts) {
    const cudaError_t e = cudaMemsetAsync(counts, 0, k * sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
  }
  const unsigned blocks = (unsigned)std::min<int64_t>((p + 31) / 32, 148 * 8);
  if (condensed)
    assign_slots_kernel<<<blocks, 256, 0, s>>>(CondView{matrix, p}, p, medoids, k, assignment,
                                                dist, lab, counts);
  else
    assign_slots_kernel<<<blocks, 256, 0, s>>>(SquareView{matrix, p}, p, medoids, k, assignment,
                                                dist, lab, counts);
  return cudaGetLastError();
}

cudaError_t launch_slots_of(const double* matrix, bool condensed, int64_t p,
                            const int64_t* medoids, int64_t k, const int64_t* assignment,
                            double* dist, int32_t* lab, cudaStream_t s) {
  if (condensed)
    slots_of_kernel<<<grid_for(p, 256), 256, 0, s>>>(CondView{matrix, p}, p, medoids, k,
                                                     assignment, dist, lab);
  else
    slots_of_kernel<<<grid_for(p, 256), 256, 0, s>>>(SquareView{matrix, p}, p, medoids, k,
                                                     assignment, dist, lab);
  return cudaGetLastError();
}

cudaError_t launch_seed_step(const double* matrix, bool condensed, int64_t p, int64_t current,
                             uint8_t* chosen, double* nearest, cudaStream_t s) {
  if (condensed)
    seed_step_kernel<<<grid_for(p, 256), 256, 0, s>>>(CondView{matrix, p}, p, current, chosen,
                                                      nearest);
  else
    seed_step_kernel<<<grid_for(p, 256), 256, 0, s>>>(SquareView{matrix, p}, p, current, chosen,
                                                      nearest);
  return cudaGetLastError();
}

static int key_bits(int64_t k) {
  int b = 1;
  while (b < 31 && (int64_t(1) << b) < k) ++b;
  return b;
}

size_t bucket_temp_bytes(int64_t p) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)p, 0, 31);
  return bytes;
}

cudaError_t launch_fill_inf(double* out, int64_t n, cudaStream_t s) {
  fill_inf_kernel<<<grid_for(n, 256), 256, 0, s>>>(out, n);
  return cudaGetLastError();
}

cudaError_t launch_iota(int32_t* out, int64_t n, cudaStream_t s) {
  iota_kernel<<<grid_for(n, 256), 256, 0, s>>>(out, n);
  return cudaGetLastError();
}

// kmedoids.hpp:86-92 on the device: members of each cluster in ascending series order (a
// stable radix sort of the iota by cluster slot) and the cluster bounds; with a
// cluster-ordered copy of the square (perm != nullptr) also each cluster's members as
// ascending positions of that copy.
cudaError_t launch_bucket(const int32_t* lab, const int32_t* perm, const int32_t* iota, int64_t p,
                          int64_t k, int32_t* keys_a, int32_t* keys_b, int32_t* members,
                          int32_t* members_perm, int64_t* cb, void* tmp, size_t tmp_bytes,
                          cudaStream_t s, bool counted) {
  cudaError_t e;
  if (k <= kBucketSmallK) {
    // keys_a holds the int32 cluster sizes (counted: already by assign_slots)
    if (!counted) {
      if ((e = cudaMemsetAsync(keys_a, 0, k * sizeof(int32_t), s)) != cudaSuccess) return e;
      cluster_count_kernel<<<(unsigned)std::min<int64_t>((p + 255) / 256, 148), 256, 0, s>>>(
          lab, p, k, keys_a);
    }
    cluster_compact_kernel<<<(unsigned)(perm ? 2 * k : k), 1024, 0, s>>>(
        lab, perm, p, k, keys_a, members, members_perm, cb);
    return cudaGetLastError();
  }
  const int bits = key_bits(k);
  size_t bytes = tmp_bytes;
  e = cub::DeviceRadixSort::SortPairs(tmp, bytes, lab, keys_a, iota, members, (int)p, 0, bits, s);
  if (e != cudaSuccess) return e;
  cluster_bounds_kernel<<<grid_for(p, 256), 256, 0, s>>>(keys_a, p, k, cb);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (!perm) return cudaSuccess;
  permuted_labels_kernel<<<grid_for(p, 256), 256, 0, s>>>(lab, perm, p, keys_b);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  bytes = tmp_bytes;
  return cub::DeviceRadixSort::SortPairs(tmp, bytes, keys_b, keys_a, iota, members_perm, (int)p,
                                         0, bits, s);
}

// Candidate sums + per-cluster selection (kmedoids.hpp:111-121). With psq (the
// cluster-ordered copy) the sums read contiguous runs; the contenders' exact sequential
// sums always read the square in ascending member order (cluster_select_kernel).
cudaError_t launch_update2(const double* matrix, bool condensed, const void* psq, bool psq32,
                           const int32_t* pinv, int64_t p, const int32_t* members,
                           const int32_t* members_perm, const int64_t* cluster_begin,
                           int64_t k, int64_t* best_member, double* best_sum,
                           cudaStream_t s) {
  if (!psq)
    return launch_update(matrix, condensed, p, members, cluster_begin, k, best_member, best_sum,
                         s);
  double* sums = best_sum + k;
  const int64_t warps = std::min<int64_t>(p, 148 * 64);
  const unsigned tb = (unsigned)((warps + 7) / 8);
  if (psq32)
    tree_sum_perm_kernel<float><<<tb, 256, 0, s>>>((const float*)psq, p, pinv, members,
                                                   members_perm, cluster_begin, k, sums);
  else
    tree_sum_perm_kernel<double><<<tb, 256, 0, s>>>((const double*)psq, p, pinv, members,
                                                    members_perm, cluster_begin, k, sums);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  cluster_select_kernel<<<(unsigned)k, 256, 0, s>>>(SquareView{matrix, p}, p, members,
                                                    cluster_begin, sums, best_member, best_sum,
                                                    psq32);
  return cudaGetLastError();
}

// The cluster-ordered copy of the square: each series' nearest anchor (anchors given,
// ascending), a stable sort by anchor -> perm, its inverse, and the copy.
cudaError_t launch_cluster_layout(const double* sq, int64_t p, int n_anchor, const int64_t* anchors,
                                  int64_t* asg_tmp, double* dist_tmp, int32_t* lab,
                                  int32_t* keys_tmp, const int32_t* iota, int32_t* perm,
                                  int32_t* pinv, void* psq, bool psq32, void* tmp,
                                  size_t tmp_bytes, int num_sms, cudaStream_t s) {
  cudaError_t e = launch_assign_slots(sq, false, p, anchors, n_anchor, asg_tmp, dist_tmp, lab, s,
                                      nullptr);
  if (e != cudaSuccess) return e;
  size_t bytes = tmp_bytes;
  e = cub::DeviceRadixSort::SortPairs(tmp, bytes, lab, keys_tmp, iota, perm, (int)p, 0,
                                      key_bits(n_anchor), s);
  if (e != cudaSuccess) return e;
  inverse_perm_kernel<<<grid_for(p, 256), 256, 0, s>>>(perm, p, pinv);
  if (p <= kPermSmemRow) {
    const int smem = (int)(p * (psq32 ? sizeof(float) : sizeof(double)));
    // fp32 rows: 2 blocks per SM (<= 104 KB of staging each)
    const int per_sm = (psq32 && 2 * smem <= (int)(220 << 10)) ? 2 : 1;
    const unsigned g = (unsigned)std::min<int64_t>(p, (int64_t)num_sms * per_sm);
    if (psq32) {
      e = cudaFuncSetAttribute(permute_square_smem_kernel<float>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      permute_square_smem_kernel<float><<<g, 1024, smem, s>>>(sq, p, perm, (float*)psq);
    } else {
      e = cudaFuncSetAttribute(permute_square_smem_kernel<double>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      permute_square_smem_kernel<double><<<g, 1024, smem, s>>>(sq, p, perm, (double*)psq);
    }
  } else {
    // ~48 MB of source rows in flight
    const int64_t rows = std::max<int64_t>(1, (int64_t)(48 << 20) / (p * 8));
    const unsigned g = (unsigned)std::min<int64_t>(p, rows);
    if (psq32)
      permute_square_l2_kernel<float><<<g, 512, 0, s>>>(sq, p, perm, (float*)psq);
    else
      permute_square_l2_kernel<double><<<g, 512, 0, s>>>(sq, p, perm, (double*)psq);
  }
  return cudaGetLastError();
}

}  // namespace dtwgpu
