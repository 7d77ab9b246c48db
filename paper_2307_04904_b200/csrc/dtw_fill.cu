// dtw_fill.cu -- sm_100a kernels for the all-pairs banded DTW distance-matrix fill.
//
// Replaces the inside of dtwclust::build_matrix (pairwise.hpp:81-126), whose per-pair
// work is dtw_distance (dtw.hpp:40-75, hot loop :59-73):
//     cur[j] = (x_i - y_j)^2 + min(prev[j-1], prev[j], cur[j-1])
// Two kernel families, both "one group of G lanes per pair, R DP cells per lane per
// row, anti-diagonal wavefront across lanes, rolling rows in registers":
//
//  * Full  (column strips).  Lane l owns R consecutive columns of the shorter series
//    (y held in registers) and runs one row behind lane l-1; the cell left of its
//    strip arrives from lane l-1 by __shfl_up_sync. Series longer than G*R columns are
//    done in passes; the strip's last column is handed to the next pass through a
//    per-group boundary column in global memory (L2-resident). Used for unlimited and
//    wide (auto-widened) bands; `MASK` adds warp-uniform band masking.
//  * Band  (sheared coordinates k = j - i + hw).  For narrow Sakoe-Chiba bands: lane l
//    owns band offsets [lR, lR+R), so the 2hw+1-wide band is covered by one group and
//    no out-of-band cell is ever touched. Dependencies become left (k-1, same row),
//    diag (k, prev row) and up (k+1, prev row): the left cell arrives from lane l-1
//    (shfl_up, previous step), the up cell of the strip's last column from lane l+1's
//    first cell of the previous row (shfl_down, same step). The y window slides one
//    sample per row; it is rotated through registers by unrolling R steps and fed
//    from lane l+1 (shfl_down), so no shared memory and no per-cell loads.
//
// Arithmetic (fp64): __dsub_rn / __dmul_rn / __dadd_rn (no FMA contraction) and a
// plain compare-select min -- bit-identical to the reference built without -march
// (SURVEY.md finding 4, hard part H1). Out-of-band and padding cells are +inf, as in
// dtw.hpp:61-71. Orientation (longer series on rows) follows dtw.hpp:45-47; the
// recurrence is bitwise transposable anyway.
//
// fp32 mode (precision == DTWG_FP32): samples rounded to fp32, squared differences
// and the running sums in fp32, with a per-lane fp64 renormalisation offset every
// kRenorm rows so the fp32 magnitudes stay small.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>

#include "dtw_fill.cuh"

namespace dtwgpu {
namespace {

constexpr int kRenorm = 16;  // fp32 mode: rows between per-lane offset renormalisations

__device__ __forceinline__ int64_t row_off(int64_t i, int64_t p) { return i * p - i * (i + 1) / 2; }

// Condensed slot -> (i, j), i < j (pairwise.hpp:41-53), closed form + fix-up.
__device__ __forceinline__ void decode_slot(int64_t s, int64_t p, int64_t& i, int64_t& j) {
  const double tp = 2.0 * (double)p - 1.0;
  const double disc = tp * tp - 8.0 * (double)s;
  int64_t r = (int64_t)((tp - sqrt(disc > 0.0 ? disc : 0.0)) * 0.5);
  if (r < 0) r = 0;
  if (r > p - 2) r = p - 2;
  while (r > 0 && row_off(r, p) > s) --r;
  while (r + 1 <= p - 2 && row_off(r + 1, p) <= s) ++r;
  i = r;
  j = r + 1 + (s - row_off(r, p));
}

// ---- arithmetic policies ----------------------------------------------------------
struct F64 {
  using T = double;
  static __device__ __forceinline__ T inf() { return CUDART_INF; }
  static __device__ __forceinline__ T mn(T a, T b) { return b < a ? b : a; }
  // (x - y)^2 + best, each op rounded separately (dtw.hpp:16-19, :69).
  static __device__ __forceinline__ T cell(T x, T y, T best) {
    const T d = __dsub_rn(x, y);
    return __dadd_rn(__dmul_rn(d, d), best);
  }
  static __device__ __forceinline__ T load(const FillArgs& A, int64_t idx) {
    return __ldg(A.samples + idx);
  }
};

struct F32 {
  using T = float;
  static __device__ __forceinline__ T inf() { return CUDART_INF_F; }
  static __device__ __forceinline__ T mn(T a, T b) { return fminf(a, b); }
  static __device__ __forceinline__ T cell(T x, T y, T best) {
    const T d = __fsub_rn(x, y);
    return __fadd_rn(__fmul_rn(d, d), best);
  }
  static __device__ __forceinline__ T load(const FillArgs& A, int64_t idx) {
    return __ldg(A.samples32 + idx);
  }
};

struct PairInfo {
  int64_t slot;
  const int64_t* dummy;
  int64_t xoff, yoff;  // rows series (longer), columns series (shorter)
  int64_t n, m;        // n >= m
  int64_t hw;          // effective half width (pair_window, pairwise.hpp:29-33)
};

__device__ __forceinline__ PairInfo load_pair(const FillArgs& A, int64_t item) {
  PairInfo P;
  P.slot = A.list ? A.list[item] : A.begin + item;
  int64_t a, b;
  decode_slot(P.slot, A.p, a, b);
  const int64_t oa = A.offsets[a], la = A.offsets[a + 1] - oa;
  const int64_t ob = A.offsets[b], lb = A.offsets[b + 1] - ob;
  if (la >= lb) {
    P.xoff = oa; P.n = la; P.yoff = ob; P.m = lb;
  } else {
    P.xoff = ob; P.n = lb; P.yoff = oa; P.m = la;
  }
  if (A.half_width < 0) {
    P.hw = P.n;  // warp_window.hpp:33-35: unlimited -> max(n, m)
  } else {
    const int64_t gap = P.n - P.m;
    P.hw = (A.auto_widen && gap > A.half_width) ? gap : A.half_width;
  }
  return P;
}

// ===================================================================================
// Full family: column strips, multi-pass, optional band mask.
// ===================================================================================
template <int G, int R, bool MASK, class Ar>
__global__ void __launch_bounds__(kThreads) dtw_full_kernel(const FillArgs A) {
  using T = typename Ar::T;
  constexpr bool kF32 = sizeof(T) == 4;
  const int lane = threadIdx.x & 31;
  const int gl = lane % G;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane - gl));
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  double* bnd = A.scratch ? A.scratch + gid * A.scratch_stride : nullptr;
  const T INF = Ar::inf();

  for (int64_t item = gid; item < A.count; item += ngroups) {
    const PairInfo P = load_pair(A, item);
    const int64_t n = P.n, m = P.m, hw = P.hw;
    constexpr int64_t W = (int64_t)G * R;
    const int64_t npass = (m + W - 1) / W;
    int64_t written_hi = 0;  // boundary column rows valid from the previous pass
    double result = 0.0;
    const int64_t res_col = m - 1;  // 0-based column of cell (n, m)

    for (int64_t pass = 0; pass < npass; ++pass) {
      const int64_t c0 = pass * W;
      int64_t rs = 1, re = n;
      if (MASK) {
        rs = c0 + 1 - hw > 1 ? c0 + 1 - hw : 1;
        re = c0 + W + hw < n ? c0 + W + hw : n;
      }
      const int64_t jl = c0 + (int64_t)gl * R + 1;  // 1-based first column of this lane
      T yv[R], pv[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int64_t j = jl + r;
        yv[r] = (j <= m) ? Ar::load(A, P.yoff + j - 1) : T(0);
        pv[r] = INF;
      }
      // fp32 mode: values are stored relative to a per-lane fp64 offset.
      double off = 0.0;
      T diag0;  // cell (row-1, jl-1): the strip's top-left neighbour
      if (gl == 0) {
        if (pass == 0) {
          diag0 = (rs == 1) ? T(0) : INF;
        } else {
          diag0 = (rs - 1 >= 1 && rs - 1 <= written_hi) ? (T)bnd[rs - 1] : INF;
        }
      } else {
        diag0 = INF;
      }
      T send = INF;
      double send_off = 0.0;
      const int64_t nsteps = (re - rs + 1) + G - 1;
      const bool last_pass = pass == npass - 1;
      const bool hold_res = last_pass && (res_col - c0) / R == gl;
      const int r_res = (int)((res_col - c0) % R);
      const bool write_bnd = (gl == G - 1) && !last_pass;

      // Prefetch of this lane's row sample and lane 0's boundary value (one step ahead).
      int64_t i1 = rs - gl;
      T xq = (i1 >= rs && i1 <= re) ? Ar::load(A, P.xoff + i1 - 1) : T(0);
      double bq = (gl == 0 && pass > 0 && i1 <= written_hi) ? bnd[i1] : (double)INF;

      for (int64_t s = 0; s < nsteps; ++s, ++i1) {
        const bool active = (i1 >= rs) && (i1 <= re);
        const T x = xq;
        const double bcur = bq;
        if (i1 + 1 >= rs && i1 + 1 <= re) xq = Ar::load(A, P.xoff + i1);
        if (gl == 0 && pass > 0) bq = (i1 + 1 <= written_hi) ? bnd[i1 + 1] : (double)INF;

        T L = __shfl_up_sync(gmask, send, 1, G);
        double Loff = 0.0;
        if constexpr (kF32) Loff = __shfl_up_sync(gmask, send_off, 1, G);
        if (gl == 0) {
          if constexpr (kF32) {
            L = (T)(bcur - off);
            Loff = off;
          } else {
            L = (pass == 0) ? INF : (T)bcur;
          }
          if (pass == 0) L = INF;
        }
        if constexpr (kF32) {
          // Re-express the neighbour's value relative to this lane's offset.
          if (gl != 0) L = (L == INF) ? INF : (T)((double)L + (Loff - off));
        }
        bool all_in = true;
        if (MASK) all_in = !active || ((jl >= i1 - hw) && (jl + R - 1 <= i1 + hw));
        const bool fast = !MASK || __all_sync(gmask, all_in);
        if (active) {
          T d = diag0;
          T left = L;
          if (fast) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const T up = pv[r];
              const T v = Ar::cell(x, yv[r], Ar::mn(Ar::mn(d, up), left));
              d = up;
              pv[r] = v;
              left = v;
            }
          } else {
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const T up = pv[r];
              T v = Ar::cell(x, yv[r], Ar::mn(Ar::mn(d, up), left));
              const int64_t j = jl + r;
              v = (j >= i1 - hw && j <= i1 + hw) ? v : INF;
              d = up;
              pv[r] = v;
              left = v;
            }
          }
          diag0 = L;
          if constexpr (kF32) {
            // Periodic renormalisation: shift the strip so its minimum is ~0.
            if (((i1 - rs) % kRenorm) == kRenorm - 1) {
              T mn = pv[0];
#pragma unroll
              for (int r = 1; r < R; ++r) mn = Ar::mn(mn, pv[r]);
              if (mn != INF) {
#pragma unroll
                for (int r = 0; r < R; ++r) pv[r] = __fsub_rn(pv[r], mn);
                diag0 = (diag0 == INF) ? INF : __fsub_rn(diag0, mn);
                off += (double)mn;
              }
            }
          }
          send = pv[R - 1];
          if constexpr (kF32) send_off = off;
          if (write_bnd) {
            if constexpr (kF32) bnd[i1] = (send == INF) ? (double)INF : (double)send + off;
            else bnd[i1] = (double)send;
          }
          if (hold_res && i1 == n) {
            T rv = pv[0];
#pragma unroll
            for (int r = 1; r < R; ++r) rv = (r == r_res) ? pv[r] : rv;
            if constexpr (kF32) result = (double)rv + off;
            else result = (double)rv;
          }
        }
      }
      written_hi = re;
      __syncwarp(gmask);
    }
    if (((res_col - (npass - 1) * W) / R) == gl) A.out[P.slot - A.out_base] = result;
  }
}

// ===================================================================================
// Band family: sheared band coordinates, one group covers the whole band.
// ===================================================================================
// pv[rK] = inf for a uniform runtime rK: one jump-table branch instead of R selects.
template <int R, class T>
__device__ __forceinline__ void kill_cell(T (&pv)[R], int rK, T inf) {
  switch (rK) {
#define DTWG_KILL(c) \
  case c:            \
    if constexpr (c < R) pv[c] = inf; \
    break;
    DTWG_KILL(1) DTWG_KILL(2) DTWG_KILL(3) DTWG_KILL(4) DTWG_KILL(5) DTWG_KILL(6) DTWG_KILL(7)
    DTWG_KILL(8) DTWG_KILL(9) DTWG_KILL(10) DTWG_KILL(11) DTWG_KILL(12) DTWG_KILL(13)
    DTWG_KILL(14) DTWG_KILL(15)
#undef DTWG_KILL
    default:
      break;
  }
}

template <int G, int R, class Ar>
__device__ __forceinline__ typename Ar::T band_y(const FillArgs& A, const PairInfo& P, int64_t j) {
  return (j >= 1 && j <= P.m) ? Ar::load(A, P.yoff + j - 1) : Ar::inf();
}

template <int G, int R, class Ar>
__global__ void __launch_bounds__(kThreads) dtw_band_kernel(const FillArgs A) {
  static_assert(R >= 2, "band family needs R >= 2");
  using T = typename Ar::T;
  constexpr bool kF32 = sizeof(T) == 4;
  const int lane = threadIdx.x & 31;
  const int gl = lane % G;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane - gl));
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  const T INF = Ar::inf();

  for (int64_t item = gid; item < A.count; item += ngroups) {
    const PairInfo P = load_pair(A, item);
    const int64_t n = P.n, m = P.m, hw = P.hw;
    const int64_t K = 2 * hw + 1;          // band width; k = j - i + hw in [0, K)
    const int lK = (int)(K / R);           // lane holding k == K (first cell right of band)
    const int rK = (int)(K % R);
    const bool kill_lane = (lK == gl);
    const int64_t kres = m - n + hw;       // k of cell (n, m)
    const bool hold_res = (kres / R) == gl;
    const int r_res = (int)(kres % R);
    const int64_t kbase = (int64_t)gl * R;

    T pv[R], yb[R];
    double off = 0.0;  // fp32 renormalisation offset (per lane)
#pragma unroll
    for (int r = 0; r < R; ++r) pv[r] = (kbase + r == hw) ? T(0) : INF;  // row 0: cell (0,0) = 0
    // y window before step 0 is that of row -gl: yb[r] = y(-gl + kbase + r - hw).
#pragma unroll
    for (int r = 0; r < R; ++r) yb[r] = band_y<G, R, Ar>(A, P, -(int64_t)gl + kbase + r - hw);

    T send = INF;
    double send_off = 0.0;
    double result = 0.0;
    const int64_t nsteps = n + G - 1;
    int64_t i1 = 1 - gl;  // row of this lane at step 0
    T xq = (i1 >= 1 && i1 <= n) ? Ar::load(A, P.xoff + i1 - 1) : T(0);
    T yq = (gl == G - 1) ? band_y<G, R, Ar>(A, P, i1 + (int64_t)G * R - 1 - hw) : T(0);

    for (int64_t s0 = 0; s0 < nsteps; s0 += R) {
#pragma unroll
      for (int q = 0; q < R; ++q) {  // phase q: logical y[r] lives in yb[(r + q) % R]
        if (s0 + q < nsteps) {
          const bool active = (i1 >= 1) && (i1 <= n);
          const T x = xq;
          const T yfetch = yq;
          if (i1 + 1 >= 1 && i1 + 1 <= n) xq = Ar::load(A, P.xoff + i1);
          if (gl == G - 1) yq = band_y<G, R, Ar>(A, P, i1 + 1 + (int64_t)G * R - 1 - hw);

          // Slide the y window by one: the new last sample is lane l+1's logical y[1]
          // before its own slide (= y(i + lR + R - 1 - hw)); the last lane loads it.
          T ynew = __shfl_down_sync(gmask, yb[(1 + q) % R], 1, G);
          if (gl == G - 1) ynew = yfetch;
          yb[q % R] = ynew;  // physical slot of the dropped logical y[0]
          // From here on logical y[r] = yb[(r + q + 1) % R].

          T L = __shfl_up_sync(gmask, send, 1, G);
          double Loff = 0.0;
          if constexpr (kF32) Loff = __shfl_up_sync(gmask, send_off, 1, G);
          if (gl == 0) L = INF;  // k = -1 is outside the band
          if constexpr (kF32) {
            if (gl != 0) L = (L == INF) ? INF : (T)((double)L + (Loff - off));
          }

          // First cell of the strip (k = lR): needs only own previous row + L.
          T v0 = pv[0];
          if (active) v0 = Ar::cell(x, yb[(q + 1) % R], Ar::mn(Ar::mn(pv[0], pv[1]), L));
          if (kill_lane && rK == 0) v0 = INF;  // k == K is this lane's first cell
          // Up neighbour of the strip's last cell = lane l+1's first cell, previous row.
          T U = __shfl_down_sync(gmask, v0, 1, G);
          double Uoff = 0.0;
          if constexpr (kF32) Uoff = __shfl_down_sync(gmask, off, 1, G);
          if (gl == G - 1) U = INF;
          if constexpr (kF32) {
            if (gl != G - 1) U = (U == INF) ? INF : (T)((double)U + (Uoff - off));
          }
          if (active) {
            T left = v0;
#pragma unroll
            for (int r = 1; r < R; ++r) {
              const T up = (r < R - 1) ? pv[r + 1] : U;
              const T v = Ar::cell(x, yb[(r + q + 1) % R], Ar::mn(Ar::mn(pv[r], up), left));
              pv[r] = v;
              left = v;
            }
            pv[0] = v0;
            // Cell k == K lies right of the band: keep it at +inf (dtw.hpp:71). Cells
            // beyond it may hold garbage; only cell K feeds a valid cell (as "up").
            if (kill_lane && rK != 0) kill_cell<R>(pv, rK, INF);
            if constexpr (kF32) {
              if (((i1 - 1) % kRenorm) == kRenorm - 1) {
                T mn = pv[0];
#pragma unroll
                for (int r = 1; r < R; ++r) mn = Ar::mn(mn, pv[r]);
                if (mn != INF) {
#pragma unroll
                  for (int r = 0; r < R; ++r) pv[r] = __fsub_rn(pv[r], mn);
                  off += (double)mn;
                }
              }
            }
            send = pv[R - 1];
            if constexpr (kF32) send_off = off;
            if (hold_res && i1 == n) {
              T rv = pv[0];
#pragma unroll
              for (int r = 1; r < R; ++r) rv = (r == r_res) ? pv[r] : rv;
              if constexpr (kF32) result = (double)rv + off;
              else result = (double)rv;
            }
          }
          ++i1;
        }
      }
    }
    if (hold_res) A.out[P.slot - A.out_base] = result;
  }
}

}  // namespace

// ---- instantiation table ------------------------------------------------------------
#define DTWG_FULL_CFGS(X)                                                              \
  X(2, 23) X(4, 12) X(8, 8) X(16, 8) X(16, 16) X(32, 4) X(32, 8) X(32, 12) X(32, 15) \
  X(32, 16)
#define DTWG_BAND_CFGS(X) \
  X(16, 7) X(16, 9) X(16, 11) X(16, 13) X(32, 3) X(32, 5) X(32, 7) X(32, 9) X(32, 13)

template <class Fn>
static bool dispatch(const KernelCfg& c, Fn&& fn) {
#define DTWG_F(g, r)                                                                      \
  if (c.family == Family::Full && c.G == g && c.R == r) {                                 \
    if (c.fp32) {                                                                         \
      if (c.mask) fn((const void*)dtw_full_kernel<g, r, true, F32>);                     \
      else fn((const void*)dtw_full_kernel<g, r, false, F32>);                           \
    } else {                                                                              \
      if (c.mask) fn((const void*)dtw_full_kernel<g, r, true, F64>);                     \
      else fn((const void*)dtw_full_kernel<g, r, false, F64>);                           \
    }                                                                                     \
    return true;                                                                          \
  }
#define DTWG_B(g, r)                                                                      \
  if (c.family == Family::Band && c.G == g && c.R == r) {                                 \
    if (c.fp32) fn((const void*)dtw_band_kernel<g, r, F32>);                             \
    else fn((const void*)dtw_band_kernel<g, r, F64>);                                    \
    return true;                                                                          \
  }
  DTWG_FULL_CFGS(DTWG_F)
  DTWG_BAND_CFGS(DTWG_B)
#undef DTWG_F
#undef DTWG_B
  return false;
}

bool fill_cfg_supported(const KernelCfg& cfg) {
  return dispatch(cfg, [](const void*) {});
}

cudaError_t launch_fill(const KernelCfg& cfg, const FillArgs& args, int blocks,
                        cudaStream_t stream) {
  cudaError_t err = cudaErrorInvalidConfiguration;
  FillArgs a = args;
  void* params[] = {&a};
  dispatch(cfg, [&](const void* fn) {
    err = cudaLaunchKernel(fn, dim3(blocks), dim3(kThreads), params, 0, stream);
  });
  return err;
}

int fill_blocks_per_sm(const KernelCfg& cfg) {
  int nb = 0;
  dispatch(cfg, [&](const void* fn) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kThreads, 0) != cudaSuccess) nb = 1;
  });
  return nb > 0 ? nb : 1;
}

}  // namespace dtwgpu
