// dtw_kernels.cuh -- sm_100a kernels for the all-pairs banded DTW distance-matrix fill.
//
// Replaces the inside of dtwclust::build_matrix (pairwise.hpp:81-126), whose per-pair
// work is dtw_distance (dtw.hpp:40-75, hot loop :59-73):
//     cur[j] = (x_i - y_j)^2 + min(prev[j-1], prev[j], cur[j-1])
// Two kernel families, both "one group of G lanes per pair, R DP cells per lane per
// row, anti-diagonal wavefront across lanes, rolling rows in registers":
//
//  * Full  (column strips).  Lane l owns R consecutive columns of the shorter series
//    (y held in registers) and runs one step behind lane l-1; each step it advances TWO
//    rows, interleaving the two cell chains (ILP 2). The cells left of its strip arrive
//    from lane l-1 by __shfl_up_sync. Series longer than G*R columns are done in
//    passes; the strip's last column is handed to the next pass through a per-group
//    boundary column in global memory (L2-resident). Used for unlimited and wide
//    (auto-widened) bands; `MASK` adds warp-uniform band masking.
//  * Band  (sheared coordinates k = j - i + hw).  For narrow Sakoe-Chiba bands: lane l
//    owns band offsets [lR, lR+R), so the 2hw+1-wide band is covered by one group and
//    almost no out-of-band cell is computed. Dependencies become left (k-1, same row),
//    diag (k, prev row) and up (k+1, prev row): the left cell arrives from lane l-1
//    (shfl_up, previous step), the up cell of the strip's last column from lane l+1's
//    first cell of the previous row (shfl_down, same step). The y window slides one
//    sample per row; it rotates through registers (R steps unrolled) and is fed from
//    lane l+1 by shfl_down, so there are no per-cell loads.
//
// All loops are warp-uniform (groups of one warp run the warp's maximum trip count and
// idle through the surplus), so every shuffle uses the full mask and no divergence
// checks are emitted. Per-pair indices are 32-bit.
//
// Arithmetic (fp64): __dsub_rn / __dmul_rn / __dadd_rn (no FMA contraction) and a
// plain compare-select min -- bit-identical to the reference built without -march
// (SURVEY.md finding 4, hard part H1). Out-of-band and padding cells are +inf, as in
// dtw.hpp:61-71. Orientation (longer series on rows) follows dtw.hpp:45-47; the
// recurrence is bitwise transposable anyway.
//
// fp32 mode (precision == DTWG_FP32): samples rounded to fp32, squared differences
// and running sums in fp32, each lane keeping its values relative to a private fp64
// offset that is renormalised to the strip minimum every few rows, so fp32 magnitudes
// stay small. Cells crossing lanes are re-based with the
// neighbour's offset.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>
#include <cstdio>
#include <type_traits>

#include "dtw_fill.cuh"

namespace dtwgpu {
namespace kern {

constexpr unsigned kFull = 0xffffffffu;
// fp32 mode: steps between per-lane offset renormalisations. The Band kernels key them on
// the warp-uniform step index (not the lane's skewed row), so a whole warp renormalises
// together on 1 step in 8 instead of some lane on every step (which made the predicated
// renormalisation run every step: ~1.5 extra instructions per cell).
constexpr int kRenormSteps = 8;

#ifndef DTWG_UNIT_UNROLL  // steps unrolled per loop iteration in the unit-ring kernel
#define DTWG_UNIT_UNROLL 2
#endif
constexpr int kUnitUnroll = DTWG_UNIT_UNROLL;

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

// ---- bounds checks (DTWG_CHECK_BOUNDS builds only; tools/bounds_check.sh) -----------
// Every sample load of the Full/lane/strip kernels stays inside the guarded series buffer
// (lanes of a warp run to the warp's longest pair and prefetch past their own ends) and
// every boundary-column row inside the group's scratch column.
#ifdef DTWG_CHECK_BOUNDS
#define DTWG_CHK(cond, what, v)                                                              \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      printf("DTWG_CHECK_BOUNDS %s out of range: %lld (block %d thread %d)\n", what,      \
             (long long)(v), (int)blockIdx.x, (int)threadIdx.x);                           \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define DTWG_CHK(cond, what, v) \
  do {                          \
  } while (0)
#endif
template <class T>
__device__ __forceinline__ void chk_sample(const FillArgs& A, const T* S, const T* P, int64_t i) {
  const int64_t at = (int64_t)(P - S) + i;
  DTWG_CHK(at >= A.guard_lo && at < A.guard_hi, "sample", at);
}
__device__ __forceinline__ void chk_row(const FillArgs& A, int64_t row) {
  DTWG_CHK(row >= 0 && row < A.scratch_stride, "boundary row", row);
}

// ---- arithmetic policies ----------------------------------------------------------
// The fp64 cell has two instruction forms: selects only (F64::cell over two
// F64::mn, 5 fp64 + 4 ALU instructions) and the second minimum folded into a predicated
// DADD pair (F64::cell3pd, 6 fp64 + 2 ALU). Which cells take which form is a per-kernel
// choice, measured on the B200; the switches below exist for those measurements (the
// pattern macros are expanded where the unrolled row t / column r / unit h are in scope).
#ifndef DTWG_PD_CELL  // cell3pd allowed in: bit 0 the Full family, bit 1 the band family
#define DTWG_PD_CELL 3
#endif
#ifndef DTWG_PD_PATTERN  // register-y Full strips: checkerboard, odd (row + column) take it
#define DTWG_PD_PATTERN ((r + t) % 2 != 0)
#endif
#ifndef DTWG_PD_YSM_ALL  // shared-memory-y Full strips: every cell (0: the pattern above)
#define DTWG_PD_YSM_ALL 1
#endif
#ifndef DTWG_PD_LANE  // the one-lane single-strip kernel (c3): plain selects
#define DTWG_PD_LANE 0
#endif
#ifndef DTWG_PD_UNIT_PATTERN  // unit-ring band kernel: the even units' chains take it (c2:
#define DTWG_PD_UNIT_PATTERN (h % 2 == 0)  // 2167 GCUPS; every cell 2136, (c + h) odd 2144,
#endif                                     // odd columns 2136, h != 0 2152, h == 1 2134)
struct F64 {
  using T = double;
  static constexpr bool kFp32 = false;
  static __device__ __forceinline__ T inf() { return CUDART_INF; }
  static __device__ __forceinline__ T mn(T a, T b) { return b < a ? b : a; }
  // (x - y)^2 + best, each op rounded separately (dtw.hpp:16-19, :69).
  static __device__ __forceinline__ T cell(T x, T y, T best) {
    const T d = __dsub_rn(x, y);
    return __dadd_rn(__dmul_rn(d, d), best);
  }
  // (x - y)^2 + min(m, left) with the minimum folded into the add: the same predicate
  // that would select `left` or `m` picks one of two DADDs (`@q DADD v = dd + left;
  // @!q DADD v = dd + m`), bit-identical to cell(x, y, mn(m, left)). 6 fp64-pipe + 2 ALU
  // instructions per cell instead of 5 + 4. Written as PTX branches, which ptxas
  // if-converts into the predicated pair (predicated PTX adds come out as two DADDs and
  // four selects).
  static __device__ __forceinline__ T cell3pd(T x, T y, T m, T left) {
    T v;
    asm("{\n\t.reg .pred q;\n\t.reg .f64 d;\n\t"
        "sub.rn.f64 d, %1, %2;\n\t"
        "mul.rn.f64 d, d, d;\n\t"
        "setp.lt.f64 q, %4, %3;\n\t"
        "@q bra L1_%=;\n\t"
        "add.rn.f64 %0, d, %3;\n\t"
        "bra L2_%=;\n\t"
        "L1_%=:\n\t"
        "add.rn.f64 %0, d, %4;\n\t"
        "L2_%=:\n\t}"
        : "=d"(v)
        : "d"(x), "d"(y), "d"(m), "d"(left));
    return v;
  }
  // Band family: cell3pd on every cell unless the call site passes its own pattern.
  static __device__ __forceinline__ T cell3b(T x, T y, T m, T left, bool pd = true) {
#if DTWG_PD_CELL & 2
    if (pd) return cell3pd(x, y, m, left);
#endif
    return cell(x, y, mn(m, left));
  }
  static __device__ __forceinline__ const T* base(const FillArgs& A) { return A.samples; }
  static __device__ __forceinline__ const T* bbase(const FillArgs& A) { return A.bsamples; }
};

struct F32 {
  using T = float;
  static constexpr bool kFp32 = true;
  static __device__ __forceinline__ T inf() { return CUDART_INF_F; }
  static __device__ __forceinline__ T mn(T a, T b) { return fminf(a, b); }
  static __device__ __forceinline__ T cell(T x, T y, T best) {
    const T d = __fsub_rn(x, y);
    return __fadd_rn(__fmul_rn(d, d), best);
  }
  static __device__ __forceinline__ T cell3pd(T x, T y, T m, T left) {
    return cell(x, y, mn(m, left));
  }
  static __device__ __forceinline__ T cell3b(T x, T y, T m, T left, bool = true) {
    return cell(x, y, mn(m, left));
  }
  static __device__ __forceinline__ const T* base(const FillArgs& A) { return A.samples32; }
  static __device__ __forceinline__ const T* bbase(const FillArgs& A) { return A.bsamples32; }
};

// One pair's distance: into this launch's output and, for the fused fill + all-gather
// over peer memory (dtwg_exchange_*), into every other rank's copy of the matrix -- plain
// st.global to NVLink-mapped peer addresses, so the exchange overlaps the fill.
__device__ __forceinline__ void store_result(const FillArgs& A, int64_t slot, double v) {
  A.out[slot - A.out_base] = v;
  for (int r = 0; r < A.n_peer; ++r) A.peer_out[r][slot - A.peer_base] = v;
}

// Dynamic item scheduling: a warp takes its next `per` consecutive items of the launch from
// the class's counter (A.work, zeroed before the launch); without a counter, the static
// grid-stride item `static_base`. Classes run concurrently on side streams, so the CTAs of
// one class start as those of another exit; with a static split the late CTAs still held
// a full share (c5 shards of 8 GPUs: 254-318 ms for equal cells). Ragged classes list
// their pairs longest first, so taking items in order is longest-processing-time first.
__device__ __forceinline__ int64_t take_items(const FillArgs& A, int64_t static_base, int per) {
  if (A.work == nullptr) return static_base;
  unsigned long long b = 0;
  if ((threadIdx.x & 31) == 0) b = atomicAdd(A.work, (unsigned long long)per);
  return (int64_t)__shfl_sync(0xffffffffu, b, 0);
}
// The item after `base`: the next counter grab, or the static grid stride.
__device__ __forceinline__ int64_t next_items(const FillArgs& A, int64_t base, int64_t stride,
                                              int per) {
  return take_items(A, base + stride, per);
}

struct Pair {
  int64_t slot;
  int64_t xoff, yoff;  // rows series (longer), columns series (shorter)
  int n, m;            // n >= m
  int hw;              // effective half width (pair_window, pairwise.hpp:29-33)
};

__device__ __forceinline__ Pair load_pair(const FillArgs& A, int64_t item) {
  Pair P;
  P.slot = A.list ? A.list[item] : A.begin + item;
  int64_t a, b;
  decode_slot(P.slot, A.p, a, b);
  const int64_t oa = A.offsets[a], ob = A.offsets[b];
  const int la = (int)(A.offsets[a + 1] - oa), lb = (int)(A.offsets[b + 1] - ob);
  if (la >= lb) {
    P.xoff = oa; P.n = la; P.yoff = ob; P.m = lb;
  } else {
    P.xoff = ob; P.n = lb; P.yoff = oa; P.m = la;
  }
  if (A.half_width < 0 || A.half_width >= P.n) {
    P.hw = P.n;  // warp_window.hpp:33-35: unlimited -> max(n, m)
  } else {
    const int gap = P.n - P.m;
    P.hw = (A.auto_widen && gap > (int)A.half_width) ? gap : (int)A.half_width;
  }
  return P;
}


// ===================================================================================
// Full family: column strips, two rows per step, multi-pass, optional band mask.
// ===================================================================================
// Band edges in the Full family ("kill" semantics). With |i - j| <= hw, only ONE cell per
// row and edge has to be forced to +inf: the cell just past the lower edge, (i, i-hw-1),
// and the one just past the upper edge, (i, i+hw+1). Every other out-of-band cell then
// comes out +inf by itself, because all three of its inputs are out-of-band cells of the
// current or previous row (or the +inf column 0 / row rs-1 borders): left of the lower
// kill cell the diag/up/left inputs lie left of the previous rows' kill cells, right of
// the upper one they lie right of them. Moreover the kill cells' own inputs are known:
// the lower kill cell's diag and left inputs are +inf and only `up` (the edge cell above)
// is finite; the upper kill cell's diag and up inputs are +inf and only `left` is finite.
// So in fp64 the kill folds into the two compares of the min: "take up" is ANDed with
// "not the lower kill", "take left" with "not the upper kill" (DSETP with a predicate
// operand), i.e. one integer compare per cell and edge instead of two compares and two
// 64-bit selects per cell. KILL: bit 0 lower edge, bit 1 upper edge.
// (b < a && k != C) ? b : a -- fp64; the kill test is the compare's predicate operand
// (one ISETP + DSETP.LT.AND + 2 FSEL), which the compiler does not form from C++.
__device__ __forceinline__ double min_unless(double a, double b, int k, int c) {
  double r;
  asm("{\n\t.reg .pred q, p;\n\t"
      "setp.ne.s32 q, %3, %4;\n\t"
      "setp.lt.and.f64 p, %2, %1, q;\n\t"
      "selp.f64 %0, %2, %1, p;\n\t}"
      : "=d"(r)
      : "d"(a), "d"(b), "r"(k), "r"(c));
  return r;
}

constexpr bool kLanePd = DTWG_PD_LANE;
template <int R, int NR, int KILL, class Ar, bool PD = true>
struct FullRows {
  using T = typename Ar::T;
  // NR consecutive rows r0 .. r0+NR-1 of this lane's R-column strip. Row t's cell at
  // column r needs (row t-1, col r-1) [diag], (row t-1, col r) [up] and (row t, col r-1)
  // [left]; row -1 is the previous step's last row, held in pv. The unrolled NR x R
  // block is a 2-D wavefront, so the compiler interleaves NR independent chains (ILP NR).
  // In: diag0 = (r0-1, jl-1); L[t] = (r0+t, jl-1) from lane l-1; klo = column (0-based in
  // the strip) of row r0's lower kill cell, khi = of its upper kill cell (row t: +t).
  // Out: out[t] = (r0+t, last column); pv becomes row r0+NR-1.
  // yv: the strip's R y samples -- a register array, or a pointer into shared memory
  // (dtw_lane_kernel), indexed with compile-time offsets either way.
  // Which cells fold their second minimum into a predicated DADD pair (F64::cell3pd).
  // Strips with y in registers lay the two cell forms out as a checkerboard -- each
  // anti-diagonal of the block is one form, consecutive anti-diagonals alternate -- which
  // keeps the fp64 pipe and the ALU pipe both busy (c4: selects only 2478, predicated adds
  // only 2533, checkerboard 2575 GCUPS; alternate rows 2538, alternate columns 2529); the
  // shared-memory-y strips (12 warps per SM) do best with predicated adds on every cell
  // (c5: 2255 against 2241 checkerboard).
  static __device__ __forceinline__ constexpr bool pd_row(bool ysm, int t, int r) {
    return !Ar::kFp32 && PD && (DTWG_PD_CELL & 1) && ((ysm && DTWG_PD_YSM_ALL) || DTWG_PD_PATTERN);
  }
  template <class YV>
  static __device__ __forceinline__ void run(T (&pv)[R], const YV& yv, const T (&x)[NR],
                                             T diag0, const T (&L)[NR], int klo, int khi,
                                             T (&out)[NR]) {
    const T INF = Ar::inf();
    constexpr bool kYsm = std::is_pointer<YV>::value;
    T d[NR], l[NR];
#pragma unroll
    for (int t = 0; t < NR; ++t) {
      d[t] = t == 0 ? diag0 : L[t - 1];
      l[t] = L[t];
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      T up = pv[r];
      const T yr = yv[r];  // one read per column (one LDS when y lives in shared memory)
#pragma unroll
      for (int t = 0; t < NR; ++t) {
        T v;
        if constexpr (KILL == 0) {
          if (pd_row(kYsm, t, r)) v = Ar::cell3pd(x[t], yr, Ar::mn(d[t], up), l[t]);
          else v = Ar::cell(x[t], yr, Ar::mn(Ar::mn(d[t], up), l[t]));
        } else if constexpr (Ar::kFp32) {
          v = Ar::cell(x[t], yr, Ar::mn(Ar::mn(d[t], up), l[t]));
          const bool k = ((KILL & 1) && r - t == klo) || ((KILL & 2) && r - t == khi);
          v = k ? INF : v;
        } else {
          const T m1 = (KILL & 1) ? min_unless(d[t], up, klo, r - t) : Ar::mn(d[t], up);
          if constexpr (KILL & 2) v = Ar::cell(x[t], yr, min_unless(m1, l[t], khi, r - t));
          else if (pd_row(kYsm, t, r)) v = Ar::cell3pd(x[t], yr, m1, l[t]);
          else v = Ar::cell(x[t], yr, Ar::mn(m1, l[t]));
        }
        d[t] = up;  // (t-1, r) is the diagonal of (t, r+1)
        l[t] = v;
        up = v;     // (t, r) is the up neighbour of (t+1, r)
      }
      pv[r] = up;
    }
#pragma unroll
    for (int t = 0; t < NR; ++t) out[t] = l[t];
  }
};

// Which kill edges a step of NR rows needs in this lane: bit 0 when a lower kill cell of
// rows r0 .. r0+NR-1 falls in the lane's R columns, bit 1 for an upper one. klo/khi are
// row r0's kill columns relative to the lane's first column; the kill columns move right
// by one per row, so row t's are klo + t and khi + t.
template <int R, int NR>
__device__ __forceinline__ int kill_need(int klo, int khi) {
  return ((klo <= R - 1 && klo + NR - 1 >= 0) ? 1 : 0) |
         ((khi <= R - 1 && khi + NR - 1 >= 0) ? 2 : 0);
}

// Experiments only (-DDTWG_FULL_MINB_N=k caps the Full kernels' registers for k CTAs per
// SM). The default passes no minimum: an explicit 1 lets ptxas take more registers
// (186 instead of <= 170 for G=32 R=16 T=2), dropping residency from 3 to 2 CTAs per SM.
#ifdef DTWG_FULL_MINB_N
#define DTWG_FULL_BOUNDS __launch_bounds__(kThreads, DTWG_FULL_MINB_N)
#else
#define DTWG_FULL_BOUNDS __launch_bounds__(kThreads)
#endif
// Full family. TR rows per step (ILP TR), warp-uniform loops, multi-pass over column
// strips of width G*R with a per-group boundary column between passes. MP = false: every
// pair of the launch fits one strip (m <= G*R), so the boundary-column machinery and its
// registers are compiled out (c3: 198 -> fewer registers per thread).
template <bool YSM, class P, class Arr>
__device__ __forceinline__ auto& pick_y(P& p, Arr& a) {
  if constexpr (YSM) return p;
  else return a;
}

// YSM: the lane's R y samples live in shared memory (ys, odd stride) instead
// of R registers, read once per column per step -- fewer registers, so more warps per SM
// (dtw_full1s_kernel below).
template <int G, int R, int TR, bool MASK, class Ar, bool MP, bool YSM>
__device__ __forceinline__ void full_body(const FillArgs& A, volatile typename Ar::T* ys) {
  using T = typename Ar::T;
  constexpr bool kF32 = sizeof(T) == 4;
  constexpr int GPW = 32 / G;
  constexpr int W = G * R;
  const int lane = threadIdx.x & 31;
  const int gl = lane % G;
  const int gw = lane / G;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // The warp's GPW boundary columns interleaved by row (column of group gw at
  // bnd[row * GPW]), so the boundary loads and stores of a warp's groups for one row are
  // GPW consecutive doubles (one or a few sectors) instead of GPW scattered ones.
  double* bnd = A.scratch ? A.scratch + warp * GPW * A.scratch_stride + gw : nullptr;
  const T INF = Ar::inf();
  const T* S = Ar::base(A);

  for (int64_t base = take_items(A, warp * GPW, GPW); base < A.count;
       base = next_items(A, base, nwarps * GPW, GPW)) {
    const int64_t item = base + gw;
    const bool valid = item < A.count;
    const Pair P = load_pair(A, valid ? item : base);
    const T* X = S + P.xoff;
    const T* Y = S + P.yoff;
    const int n = P.n, m = P.m, hw = P.hw;
    const int npass_g = MP ? (m + W - 1) / W : 1;
    const int npass = MP ? __reduce_max_sync(kFull, npass_g) : 1;
    int written_hi = 0;
    double result = 0.0;

    for (int pass = 0; pass < npass; ++pass) {
      const bool pvalid = pass < npass_g;
      const int c0 = pass * W;
      int rs = 1, re = n;
      if (MASK) {
        rs = max(1, c0 + 1 - hw);
        re = min(n, c0 + W + hw);
      }
      if (!pvalid) re = rs - 1;
      const int my_steps = pvalid ? ((re - rs + TR) / TR) + G - 1 : 0;
      const int nsteps = __reduce_max_sync(kFull, my_steps);
      const int jl = c0 + gl * R + 1;  // 1-based first column of this lane
      T yreg[YSM ? 1 : R], pv[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (jl + r <= m) chk_sample(A, S, Y, jl + r - 1);
        const T yj = (jl + r <= m) ? __ldg(Y + jl + r - 1) : T(0);
        if constexpr (YSM) ys[r] = yj;
        else yreg[r] = yj;
        pv[r] = INF;
      }
      // the strip's y: registers, or this lane's own shared-memory row (no sync needed)
      auto& yv = pick_y<YSM>(ys, yreg);
      T diag0 = INF;  // cell (r0-1, jl-1)
      if (gl == 0) {
        if (pass == 0) diag0 = (rs == 1) ? T(0) : INF;
        else if (rs - 1 >= 1 && rs - 1 <= written_hi) {
          chk_row(A, rs - 1);
          diag0 = (T)bnd[(rs - 1) * GPW];
        }
      }
      double off = 0.0;  // fp32: this lane's offset
      T send[TR];
#pragma unroll
      for (int t = 0; t < TR; ++t) send[t] = INF;
      double send_off = 0.0;
      const bool last_pass = pass == npass_g - 1;
      const bool hold = pvalid && last_pass && ((m - 1 - c0) / R) == gl;
      const int r_res = hold ? (m - 1 - c0) % R : -1;
      const bool wb = MP && pvalid && !last_pass && gl == G - 1;
      const bool use_bnd = MP && gl == 0 && pass > 0;

      int r0 = rs - TR * gl;  // this lane's first row at step 0
      // Rows outside [1, n] read the zero guard around the packed series (never used).
      T xq[TR];
      double bq[TR];
#pragma unroll
      for (int t = 0; t < TR; ++t) {
        chk_sample(A, S, X, r0 + t - 1);
        xq[t] = __ldg(X + (r0 + t - 1));
        bq[t] = (double)Ar::inf();
        if constexpr (MP)
          if (use_bnd) {
            chk_row(A, r0 + t);
            bq[t] = bnd[(r0 + t) * GPW];
          }
      }

      for (int s = 0; s < nsteps; ++s, r0 += TR) {
        T x[TR], L[TR];
        double b[TR];
#pragma unroll
        for (int t = 0; t < TR; ++t) {
          x[t] = xq[t];
          b[t] = MP ? bq[t] : (double)Ar::inf();  // single strip: column 0 is +inf
          chk_sample(A, S, X, r0 + TR + t - 1);
          xq[t] = __ldg(X + (r0 + TR + t - 1));
          // Rows past the previous pass's last row hold +inf (written at its end), so
          // lane 0 loads its boundary rows unconditionally: a predicated load, no branch.
          if constexpr (MP)
            if (use_bnd) {
              chk_row(A, r0 + TR + t);
              bq[t] = bnd[(r0 + TR + t) * GPW];
            }
          // G = 1: no left neighbour (lane 0 of its own group takes the boundary below)
          if constexpr (G > 1) L[t] = __shfl_up_sync(kFull, send[t], 1, G);
          else L[t] = INF;
        }
        if constexpr (kF32) {
          // Neighbour values are relative to its offset: add the (fp32-rounded) offset
          // difference once per row (inf stays inf). Lane 0 reads absolute fp64 values.
          const double loff = G > 1 ? __shfl_up_sync(kFull, send_off, 1, G) : 0.0;
          const T delta = (T)(loff - off);
#pragma unroll
          for (int t = 0; t < TR; ++t) {
            if (gl == 0) L[t] = (T)(b[t] - off);
            else L[t] = L[t] + delta;
          }
        } else {
          if (gl == 0) {
#pragma unroll
            for (int t = 0; t < TR; ++t) L[t] = (T)b[t];
          }
        }
        const bool work = s >= gl && r0 <= re;
        // Band-edge kill cells of this step (see FullRows), warp-uniform variant choice.
        const int klo = r0 - hw - 1 - jl, khi = r0 + hw + 1 - jl;
        int need = 0;
        if (MASK) {
          const int mine = work ? kill_need<R, TR>(klo, khi) : 0;
          need = (__any_sync(kFull, mine & 1) ? 1 : 0) | (__any_sync(kFull, mine & 2) ? 2 : 0);
        }
        if (work) {
          T out[TR];
          const int nr = min(TR, re - r0 + 1);  // rows of this step inside [rs, re]
          if (nr == TR) {
            if (need == 0)
              FullRows<R, TR, 0, Ar>::run(pv, yv, x, diag0, L, klo, khi, out);
            else if (need == 1)
              FullRows<R, TR, 1, Ar>::run(pv, yv, x, diag0, L, klo, khi, out);
            else if (need == 2)
              FullRows<R, TR, 2, Ar>::run(pv, yv, x, diag0, L, klo, khi, out);
            else
              FullRows<R, TR, 3, Ar>::run(pv, yv, x, diag0, L, klo, khi, out);
            diag0 = L[TR - 1];
          } else {
            // Tail of the pass: the remaining rows one at a time.
#pragma unroll
            for (int t = 0; t < TR; ++t) {
              if (t < nr) {
                const T xt[1] = {x[t]};
                const T Lt[1] = {L[t]};
                T ot[1];
                FullRows<R, 1, MASK ? 3 : 0, Ar>::run(pv, yv, xt, diag0, Lt, klo + t, khi + t, ot);
                out[t] = ot[0];
                diag0 = L[t];
              } else {
                out[t] = INF;
              }
            }
          }
          if constexpr (kF32) {
            if ((s & (kRenormSteps - 1)) == kRenormSteps - 1) {
              T mnv = pv[0];
#pragma unroll
              for (int r = 1; r < R; ++r) mnv = Ar::mn(mnv, pv[r]);
              if (mnv != INF) {
#pragma unroll
                for (int r = 0; r < R; ++r) pv[r] = __fsub_rn(pv[r], mnv);
                diag0 = __fsub_rn(diag0, mnv);  // +inf stays +inf (mnv finite)
#pragma unroll
                for (int t = 0; t < TR; ++t) out[t] = __fsub_rn(out[t], mnv);
                off += (double)mnv;
              }
            }
            send_off = off;
          }
#pragma unroll
          for (int t = 0; t < TR; ++t) {
            send[t] = out[t];
            if (wb && t < nr) {
              chk_row(A, r0 + t);
              if constexpr (kF32) bnd[(r0 + t) * GPW] = (double)out[t] + off;  // +inf + off = +inf
              else bnd[(r0 + t) * GPW] = out[t];
            }
          }
          // pv now holds row r0 + nr - 1; row n is the last row of the last pass (re = n).
          if (hold && r0 + nr - 1 == n) {
            T rv = pv[0];
#pragma unroll
            for (int r = 1; r < R; ++r) rv = (r == r_res) ? pv[r] : rv;
            result = (double)rv + (kF32 ? off : 0.0);
          }
        }
      }
      if constexpr (MP && MASK) {
        // The next pass ends at most W rows lower; its rows past this pass's last one
        // lie outside the band at this pass's last column (+inf).
        if (wb)
          for (int r = re + 1; r <= min(n, re + W); ++r) {
            chk_row(A, r);
            bnd[r * GPW] = (double)INF;
          }
      }
      written_hi = re;
      __syncwarp();
    }
    const int last_c0 = (npass_g - 1) * W;
    if (valid && ((m - 1 - last_c0) / R) == gl) store_result(A, P.slot, result);
  }
}

template <int G, int R, int TR, bool MASK, class Ar, bool MP = true>
__global__ void DTWG_FULL_BOUNDS dtw_full_kernel(const FillArgs A) {
  full_body<G, R, TR, MASK, Ar, MP, false>(A, nullptr);
}

// Full strips with y in shared memory (every lane its own R samples, odd stride), one LDS
// per column per 4-row step: <= 168 registers, 3 CTAs (12 warps) per SM instead of 2.
// Planned with G = 1 (one lane per pair) for banded multi-pass shapes (c5). The register
// file is split per SM sub-partition, so 3 warps per scheduler cap a thread at 168
// registers whatever the CTA shape (R = 32 spills). (8 rows per step at 2 CTAs/SM
// measured slower: c4 2340, c5 1274 GCUPS.)
template <int G, int R, int TR, bool MASK, class Ar, bool MP = true>
__global__ void __launch_bounds__(kThreads, 3) dtw_full1s_kernel(const FillArgs A) {
  using T = typename Ar::T;
  constexpr int YS = (R % 2) ? R : R + 1;
  __shared__ T ysm[kThreads * YS];
  full_body<G, R, TR, MASK, Ar, MP, true>(A, ysm + threadIdx.x * YS);
}

// ===================================================================================
// One lane per pair (fp64, single strip: m <= R). The Full family with G = 1, except
// that the pair's R y samples live in shared memory (a lane's 2R row registers do not fit
// in fp64): each lane stages its own y once per pair and reads it with immediate-offset
// LDS, one per cell. No neighbour shuffles, no boundary column and no wavefront
// fill/drain: each pair's rows run back to back (c3: 1.0x the in-band cells computed
// instead of 1.09x for G = 2). Lanes of a warp run their own pairs in lockstep up to the
// warp's longest pair; band edges use the Full family's kill cells.
// ===================================================================================
template <int R, int TR, bool MASK, class Ar>
__global__ void __launch_bounds__(kThreads) dtw_lane_kernel(const FillArgs A) {
  using T = typename Ar::T;
  constexpr int YS = (R % 2) ? R : R + 1;  // odd stride (doubles): conflict-free LDS.64
  __shared__ T ysm[kThreads * YS];
  // volatile: one LDS per cell, not hoisted into (2R more) registers
  volatile T* ys = ysm + threadIdx.x * YS;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const T INF = Ar::inf();
  const T* S = Ar::base(A);
  const int64_t base0 = tid - (threadIdx.x & 31);  // the warp's first item

  for (int64_t base = take_items(A, base0, 32); base < A.count;
       base = next_items(A, base, nthreads, 32)) {
    const int64_t item = base + (threadIdx.x & 31);
    const bool valid = item < A.count;
    const Pair P = load_pair(A, valid ? item : base);
    const T* X = S + P.xoff;
    const T* Y = S + P.yoff;
    const int n = valid ? P.n : 0, m = P.m, hw = P.hw;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r < m) chk_sample(A, S, Y, r);
      ys[r] = (r < m) ? __ldg(Y + r) : T(0);  // this lane's own
    }
    T pv[R];
#pragma unroll
    for (int r = 0; r < R; ++r) pv[r] = INF;
    T diag0 = T(0);  // cell (0, 0); column 0 is +inf below it
    T L[TR];
#pragma unroll
    for (int t = 0; t < TR; ++t) L[t] = INF;
    const int rows = __reduce_max_sync(kFull, n);
    double result = 0.0;
    T xq[TR];
#pragma unroll
    for (int t = 0; t < TR; ++t) {
      chk_sample(A, S, X, t);
      xq[t] = __ldg(X + t);
    }
    for (int r0 = 1; r0 <= rows; r0 += TR) {
      T x[TR];
#pragma unroll
      for (int t = 0; t < TR; ++t) {
        x[t] = xq[t];
        chk_sample(A, S, X, r0 + TR + t - 1);
        xq[t] = __ldg(X + (r0 + TR + t - 1));  // rows past n read the zero guard (unused)
      }
      const int klo = r0 - hw - 2, khi = r0 + hw;  // kill columns of row r0, 0-based
      int need = 0;
      if (MASK) {
        const int mine = (r0 <= n) ? kill_need<R, TR>(klo, khi) : 0;
        need = (__any_sync(kFull, mine & 1) ? 1 : 0) | (__any_sync(kFull, mine & 2) ? 2 : 0);
      }
      T out[TR];
      if (r0 + TR - 1 <= n) {
        if (need == 0) FullRows<R, TR, 0, Ar, kLanePd>::run(pv, ys, x, diag0, L, klo, khi, out);
        else if (need == 1) FullRows<R, TR, 1, Ar, kLanePd>::run(pv, ys, x, diag0, L, klo, khi, out);
        else if (need == 2) FullRows<R, TR, 2, Ar, kLanePd>::run(pv, ys, x, diag0, L, klo, khi, out);
        else FullRows<R, TR, 3, Ar, kLanePd>::run(pv, ys, x, diag0, L, klo, khi, out);
        if (r0 + TR - 1 == n) {
          T rv = pv[0];
#pragma unroll
          for (int r = 1; r < R; ++r) rv = (r == m - 1) ? pv[r] : rv;
          result = (double)rv;
        }
      } else if (r0 <= n) {
        // The pair's last n - r0 + 1 < TR rows, one at a time.
        T dg = diag0;
#pragma unroll
        for (int t = 0; t < TR - 1; ++t) {
          if (r0 + t <= n) {
            const T xt[1] = {x[t]};
            const T Lt[1] = {INF};
            T ot[1];
            FullRows<R, 1, MASK ? 3 : 0, Ar, kLanePd>::run(pv, ys, xt, dg, Lt, klo + t, khi + t, ot);
            dg = INF;
          }
        }
        T rv = pv[0];
#pragma unroll
        for (int r = 1; r < R; ++r) rv = (r == m - 1) ? pv[r] : rv;
        result = (double)rv;
      }
      diag0 = INF;  // column 0 below row 0
    }
    if (valid) store_result(A, P.slot, result);
  }
}

// ===================================================================================
// Strip family: long pairs. The Full family's column strips of ONE pair are spread over
// many warps (all SMs) instead of being run as sequential passes by one group: strip s
// of a pair is a work item taken (in order, from a global counter) by any warp of a
// persistent grid; it trails strip s-1 through the boundary column strip s-1 writes
// (global memory, read through L2) and a per-strip progress counter published with
// release/acquire ordering every few steps. Items are handed out in dependency order
// and a warp finishes its item before taking the next, so every wait is on an item that
// a running warp holds: no deadlock, whatever the residency. Two boundary columns per
// pair suffice: strip s+2 overwrites row r of strip s's column only after strip s+1 has
// published row r, i.e. after it has read it.
// ===================================================================================
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int R, int TR, bool MASK, class Ar>
__global__ void __launch_bounds__(kThreads) dtw_strip_kernel(const FillArgs A) {
  using T = typename Ar::T;
  constexpr bool kF32 = sizeof(T) == 4;
  constexpr int G = 32;
  constexpr int W = G * R;
  constexpr int kPublish = 8;  // steps between progress publications
  const int gl = threadIdx.x & 31;
  const T INF = Ar::inf();
  const T* S = Ar::base(A);
  const int64_t total =
      A.strip_base ? A.strip_base[A.count] : A.count * (int64_t)A.strips_per_pair;

  for (;;) {
    unsigned long long it0 = 0;
    if (gl == 0) it0 = atomicAdd(A.work, 1ull);
    const int64_t it = (int64_t)__shfl_sync(kFull, it0, 0);
    if (it >= total) break;
    int64_t q;
    int s, nstrip;
    if (A.strip_base) {
      int64_t lo = 0, hi = A.count;  // strip_base[lo] <= it < strip_base[hi]
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (A.strip_base[mid] <= it) lo = mid;
        else hi = mid;
      }
      q = lo;
      s = (int)(it - A.strip_base[q]);
      nstrip = (int)(A.strip_base[q + 1] - A.strip_base[q]);
    } else {
      q = it / A.strips_per_pair;
      s = (int)(it - q * A.strips_per_pair);
      nstrip = A.strips_per_pair;
    }
    const Pair P = load_pair(A, q);
    const T* X = S + P.xoff;
    const T* Y = S + P.yoff;
    const int n = P.n, m = P.m, hw = P.hw;
    double* colq = A.cols + q * 2 * A.col_stride;
    const double* bin = s > 0 ? colq + ((s - 1) & 1) * A.col_stride : nullptr;
    double* bout = s < nstrip - 1 ? colq + (s & 1) * A.col_stride : nullptr;
    const int* pin = s > 0 ? A.prog + (it - 1) : nullptr;
    int* pout = A.prog + it;

    const int c0 = s * W;
    int rs = 1, re = n;
    if (MASK) {
      rs = max(1, c0 + 1 - hw);
      re = min(n, c0 + W + hw);
    }
    const int written_hi = s > 0 ? (MASK ? min(n, c0 + hw) : n) : 0;  // strip s-1's last row
    int avail = 0;  // rows of the boundary column published so far (warp-uniform)
    // Block until strip s-1 has published every row <= need that it writes.
    auto wait_rows = [&](int need) {
      need = min(need, written_hi);
      if (need <= avail) return;
      int v = 0;
      for (;;) {
        if (gl == 0) v = ld_acquire_gpu(pin);
        v = __shfl_sync(kFull, v, 0);
        if (v >= need) break;
        __nanosleep(100);
      }
      avail = v;
    };

    const int nsteps = ((re - rs + TR) / TR) + G - 1;
    const int jl = c0 + gl * R + 1;  // 1-based first column of this lane
    T yv[R], pv[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      yv[r] = (jl + r <= m) ? __ldg(Y + jl + r - 1) : T(0);
      pv[r] = INF;
    }
    const bool use_bnd = gl == 0 && s > 0;
    wait_rows(rs + 2 * TR - 1);
    T diag0 = INF;  // cell (r0-1, jl-1)
    if (gl == 0) {
      if (s == 0) diag0 = (rs == 1) ? T(0) : INF;
      else if (rs - 1 >= 1 && rs - 1 <= written_hi) diag0 = (T)__ldcg(bin + rs - 1);
    }
    double off = 0.0;
    T send[TR];
#pragma unroll
    for (int t = 0; t < TR; ++t) send[t] = INF;
    double send_off = 0.0;
    const bool hold = s == nstrip - 1 && ((m - 1 - c0) / R) == gl;
    const int r_res = hold ? (m - 1 - c0) % R : -1;
    const bool wb = bout != nullptr && gl == G - 1;
    double result = 0.0;

    int r0 = rs - TR * gl;
    T xq[TR];
    double bq[TR];
#pragma unroll
    for (int t = 0; t < TR; ++t) {
      xq[t] = __ldg(X + (r0 + t - 1));
      bq[t] = (use_bnd && r0 + t <= written_hi) ? __ldcg(bin + r0 + t) : (double)Ar::inf();
    }
    int last_written = 0;
    for (int st = 0; st < nsteps; ++st, r0 += TR) {
      wait_rows(rs + TR * (st + 2) - 1);  // lane 0's prefetch below
      T x[TR], L[TR];
      double b[TR];
#pragma unroll
      for (int t = 0; t < TR; ++t) {
        x[t] = xq[t];
        b[t] = bq[t];
        xq[t] = __ldg(X + (r0 + TR + t - 1));
        if (use_bnd)
          bq[t] = (r0 + TR + t <= written_hi) ? __ldcg(bin + r0 + TR + t) : (double)Ar::inf();
        L[t] = __shfl_up_sync(kFull, send[t], 1, G);
      }
      if constexpr (kF32) {
        const double loff = __shfl_up_sync(kFull, send_off, 1, G);
        const T delta = (T)(loff - off);
#pragma unroll
        for (int t = 0; t < TR; ++t) {
          if (gl == 0) L[t] = (T)(b[t] - off);
          else L[t] = L[t] + delta;
        }
      } else {
        if (gl == 0) {
#pragma unroll
          for (int t = 0; t < TR; ++t) L[t] = (T)b[t];
        }
      }
      const bool work = st >= gl && r0 <= re;
      const int klo = r0 - hw - 1 - jl, khi = r0 + hw + 1 - jl;  // band-edge kill cells
      int need = 0;
      if (MASK) {
        const int mine = work ? kill_need<R, TR>(klo, khi) : 0;
        need = (__any_sync(kFull, mine & 1) ? 1 : 0) | (__any_sync(kFull, mine & 2) ? 2 : 0);
      }
      if (work) {
        T out[TR];
        const int nr = min(TR, re - r0 + 1);
        if (nr == TR) {
          if (need == 0)
            FullRows<R, TR, 0, Ar>::run(pv, yv, x, diag0, L, klo, khi, out);
          else if (need == 1)
            FullRows<R, TR, 1, Ar>::run(pv, yv, x, diag0, L, klo, khi, out);
          else if (need == 2)
            FullRows<R, TR, 2, Ar>::run(pv, yv, x, diag0, L, klo, khi, out);
          else
            FullRows<R, TR, 3, Ar>::run(pv, yv, x, diag0, L, klo, khi, out);
          diag0 = L[TR - 1];
        } else {
#pragma unroll
          for (int t = 0; t < TR; ++t) {
            if (t < nr) {
              const T xt[1] = {x[t]};
              const T Lt[1] = {L[t]};
              T ot[1];
              FullRows<R, 1, MASK ? 3 : 0, Ar>::run(pv, yv, xt, diag0, Lt, klo + t, khi + t, ot);
              out[t] = ot[0];
              diag0 = L[t];
            } else {
              out[t] = INF;
            }
          }
        }
        if constexpr (kF32) {
          if ((st & (kRenormSteps - 1)) == kRenormSteps - 1) {
            T mnv = pv[0];
#pragma unroll
            for (int r = 1; r < R; ++r) mnv = Ar::mn(mnv, pv[r]);
            if (mnv != INF) {
#pragma unroll
              for (int r = 0; r < R; ++r) pv[r] = __fsub_rn(pv[r], mnv);
              diag0 = __fsub_rn(diag0, mnv);  // +inf stays +inf (mnv finite)
#pragma unroll
              for (int t = 0; t < TR; ++t) out[t] = __fsub_rn(out[t], mnv);
              off += (double)mnv;
            }
          }
          send_off = off;
        }
#pragma unroll
        for (int t = 0; t < TR; ++t) {
          send[t] = out[t];
          if (wb && t < nr) {
            if constexpr (kF32) bout[r0 + t] = (double)out[t] + off;  // +inf + off = +inf
            else bout[r0 + t] = out[t];
          }
        }
        if (wb) last_written = r0 + nr - 1;
        if (hold && r0 + nr - 1 == n) {
          T rv = pv[0];
#pragma unroll
          for (int r = 1; r < R; ++r) rv = (r == r_res) ? pv[r] : rv;
          result = (double)rv + (kF32 ? off : 0.0);
        }
      }
      if (wb && (st % kPublish) == kPublish - 1 && last_written > 0) st_release_gpu(pout, last_written);
    }
    if (wb) st_release_gpu(pout, 1 << 30);  // strip done
    if (hold) store_result(A, P.slot, result);
    __syncwarp();
  }
}

// ===================================================================================
// Band family: sheared band coordinates, one group covers the whole band.
// ===================================================================================
// pv[rK] = inf for a uniform runtime rK: one jump-table branch instead of R selects.
template <int R, class T>
__device__ __forceinline__ void kill_cell(T (&pv)[R], int rK, T inf) {
  static_assert(R <= 32, "kill_cell handles R <= 32");
  switch (rK) {
#define DTWG_KILL(c) \
  case c:            \
    if constexpr (c < R) pv[c] = inf; \
    break;
    DTWG_KILL(1) DTWG_KILL(2) DTWG_KILL(3) DTWG_KILL(4) DTWG_KILL(5) DTWG_KILL(6) DTWG_KILL(7)
    DTWG_KILL(8) DTWG_KILL(9) DTWG_KILL(10) DTWG_KILL(11) DTWG_KILL(12) DTWG_KILL(13)
    DTWG_KILL(14) DTWG_KILL(15) DTWG_KILL(16) DTWG_KILL(17) DTWG_KILL(18) DTWG_KILL(19)
    DTWG_KILL(20) DTWG_KILL(21) DTWG_KILL(22) DTWG_KILL(23) DTWG_KILL(24) DTWG_KILL(25)
    DTWG_KILL(26) DTWG_KILL(27) DTWG_KILL(28) DTWG_KILL(29) DTWG_KILL(30) DTWG_KILL(31)
#undef DTWG_KILL
    default:
      break;
  }
}

// Band family. KR >= 0: K % R known at compile time (static kill position); KR < 0:
// runtime switch. P pairs per lane group run interleaved (independent chains, ILP P);
// pairs of one group share the step counter, so each pair's result is captured when
// its own last row is reached (shared-memory stash, read after the loop). Series are
// read from the +inf-padded copy (A.bsamples), so no load needs a range check.
template <int G, int R, int KR, int P, class Ar, bool CHECK>
__device__ __forceinline__ void band_steps(
    int& i1, const typename Ar::T* (&xp)[P], const typename Ar::T* (&yp)[P],
    typename Ar::T (&xq)[P], typename Ar::T (&yq)[P], typename Ar::T (&pv)[P][R],
    typename Ar::T (&yb)[P][R], typename Ar::T (&send)[P], double (&send_off)[P],
    double (&off)[P], const int (&n)[P], const int (&lK)[P], const int (&rK)[P], int gl) {
  using T = typename Ar::T;
  constexpr bool kF32 = sizeof(T) == 4;
  const T INF = Ar::inf();
  const bool last = gl == G - 1;
#pragma unroll
  for (int q = 0; q < R; ++q) {  // phase q: logical y[r] lives in yb[(r + q) % R]
    T x[P], v0[P], U[P];
    // CHECK blocks (wavefront fill and drain) hold each lane to rows 1..n of each pair:
    // before row 1 a lane keeps the row-0 state, after row n it keeps row n, which is
    // read after the loop. Steady-state blocks compute unconditionally.
    bool act[P];
    bool any = false, all = true;
#pragma unroll
    for (int p = 0; p < P; ++p) {
      act[p] = CHECK ? (i1 >= 1 && i1 <= n[p]) : true;
      any |= act[p];
      all &= act[p];
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      x[p] = xq[p];
      const T yf = yq[p];
      xq[p] = __ldg(++xp[p]);
      yq[p] = __ldg(++yp[p]);
      // Slide the y window by one: the new last sample is lane l+1's logical y[1]
      // before its own slide (= y(i + lR + R - 1 - hw)); the last lane loads it.
      const T ynb = __shfl_down_sync(kFull, yb[p][(1 + q) % R], 1, G);
      yb[p][q % R] = last ? yf : ynb;  // physical slot of the dropped logical y[0]
      // From here on logical y[r] = yb[p][(r + q + 1) % R].
      T L = __shfl_up_sync(kFull, send[p], 1, G);
      if constexpr (kF32) {
        const double loff = __shfl_up_sync(kFull, send_off[p], 1, G);
        L = L + (T)(loff - off[p]);  // re-base to this lane's offset (inf stays inf)
      }
      if (gl == 0) L = INF;  // k = -1 is outside the band
      // First cell of the strip (k = lR): needs only own previous row + L.
      T v = Ar::cell3b(x[p], yb[p][(q + 1) % R], Ar::mn(pv[p][0], pv[p][1]), L);
      if (CHECK) v = act[p] ? v : pv[p][0];
      if (KR == 0 || KR < 0) {
        if (lK[p] == gl && rK[p] == 0) v = INF;  // k == K is this lane's first cell
      }
      v0[p] = v;
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      // Up neighbour of the strip's last cell = lane l+1's first cell, previous row.
      T u = __shfl_down_sync(kFull, v0[p], 1, G);
      if constexpr (kF32) {
        const double uoff = __shfl_down_sync(kFull, off[p], 1, G);
        u = u + (T)(uoff - off[p]);
      }
      U[p] = last ? INF : u;
    }
    if (any) {
      T left[P];
#pragma unroll
      for (int p = 0; p < P; ++p) left[p] = v0[p];
#pragma unroll
      for (int r = 1; r < R; ++r) {
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const T up = (r < R - 1) ? pv[p][r + 1] : U[p];
          T v = Ar::cell3b(x[p], yb[p][(r + q + 1) % R], Ar::mn(pv[p][r], up), left[p]);
          if (CHECK && P > 1 && !all) v = act[p] ? v : pv[p][r];
          pv[p][r] = v;
          left[p] = v;
        }
      }
#pragma unroll
      for (int p = 0; p < P; ++p) {
        if (CHECK && !act[p]) continue;
        pv[p][0] = v0[p];
        // Cell k == K lies right of the band: keep it at +inf (dtw.hpp:71). Cells
        // beyond it may hold garbage; only cell K feeds a valid cell (as "up").
        if constexpr (KR > 0) {
          if (lK[p] == gl) pv[p][KR] = INF;
        } else if constexpr (KR < 0) {
          if (lK[p] == gl && rK[p] != 0) kill_cell<R>(pv[p], rK[p], INF);
        }
        if constexpr (kF32) {
          if (((i1 - 1 + gl) & (kRenormSteps - 1)) == kRenormSteps - 1) {
            T mnv = pv[p][0];
#pragma unroll
            for (int r = 1; r < R; ++r) mnv = Ar::mn(mnv, pv[p][r]);
            if (mnv != INF) {
#pragma unroll
              for (int r = 0; r < R; ++r) pv[p][r] = __fsub_rn(pv[p][r], mnv);
              off[p] += (double)mnv;
            }
          }
          send_off[p] = off[p];
        }
        send[p] = pv[p][R - 1];
      }
    }
    ++i1;
  }
}

// Register cap: 5 CTAs of 128 threads per SM for the single-pair variants (<= 102 regs).
template <int G, int R, int KR, int P, class Ar>
__global__ void __launch_bounds__(kThreads, P == 1 ? 5 : 3) dtw_band_kernel(const FillArgs A) {
  static_assert(R >= 2, "band family needs R >= 2");
  using T = typename Ar::T;
  constexpr bool kF32 = sizeof(T) == 4;
  constexpr int GPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int gl = lane % G;
  const int gw = lane / G;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const T INF = Ar::inf();
  const T* S = Ar::bbase(A);

  for (int64_t base = take_items(A, warp * GPW * P, GPW * P); base < A.count;
       base = next_items(A, base, nwarps * GPW * P, GPW * P)) {
    const T* xp[P];
    const T* yp[P];
    const T* Y[P];
    int n[P], m[P], K[P], lK[P], rK[P], r_res[P];
    bool hold[P];
    int64_t slot[P];
    int nmax = 0, nmin = 1 << 30;
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const int64_t item = base + (int64_t)gw * P + p;
      const bool valid = item < A.count;
      const Pair Pp = load_pair(A, valid ? item : base);
      slot[p] = Pp.slot;
      // Same pair, addressed in the padded copy (lengths/orientation from load_pair).
      int64_t a, b;
      decode_slot(Pp.slot, A.p, a, b);
      const bool a_rows = (A.offsets[a + 1] - A.offsets[a]) >= (A.offsets[b + 1] - A.offsets[b]);
      const int64_t xo = A.boffsets[a_rows ? a : b], yo = A.boffsets[a_rows ? b : a];
      Y[p] = S + yo;
      xp[p] = S + xo;
      n[p] = Pp.n;
      m[p] = Pp.m;
      K[p] = 2 * Pp.hw + 1;             // band width; k = j - i + hw in [0, K)
      lK[p] = K[p] / R;                 // lane holding k == K (first cell right of band)
      rK[p] = KR >= 0 ? KR : K[p] % R;
      const int kres = m[p] - n[p] + Pp.hw;  // k of cell (n, m)
      hold[p] = valid && (kres / R) == gl;
      r_res[p] = kres % R;
      nmax = max(nmax, n[p]);
      nmin = min(nmin, n[p]);
    }
    const int kbase = gl * R;
    T pv[P][R], yb[P][R];
    double off[P], send_off[P];
    T send[P], xq[P], yq[P];
    int i1 = 1 - gl;  // this lane's row at step 0 (all pairs of the group)
#pragma unroll
    for (int p = 0; p < P; ++p) {
      off[p] = 0.0;
      send_off[p] = 0.0;
      send[p] = INF;
      const int hw = (K[p] - 1) / 2;
#pragma unroll
      for (int r = 0; r < R; ++r) pv[p][r] = (kbase + r == hw) ? T(0) : INF;  // row 0
      // y window before step 0 is that of row -gl: yb[r] = y(-gl + kbase + r - hw).
#pragma unroll
      for (int r = 0; r < R; ++r) yb[p][r] = __ldg(Y[p] + (-gl + kbase + r - hw - 1));
      // Streaming pointers: this lane's x (row i1 - 1, 0-based) and the last lane's
      // next y (index i1 + G*R - 1 - hw), both one step ahead.
      xp[p] += i1 - 1;
      xq[p] = __ldg(xp[p]);
      yp[p] = Y[p] + (i1 + G * R - 1 - hw - 1);
      yq[p] = __ldg(yp[p]);
    }
    // Steps in blocks of R (the y-rotation period). Blocks with a lane before its row 1
    // (fill) or past some pair's row n (drain) are checked; the rest run unconditionally.
    const int nsteps = __reduce_max_sync(kFull, nmax + G - 1);
    const int fill_end = ((G - 1 + R - 1) / R) * R;
    const int drain_start = (__reduce_min_sync(kFull, nmin) / R) * R;
    for (int s0 = 0; s0 < nsteps; s0 += R) {
      if (s0 < fill_end || s0 >= drain_start)
        band_steps<G, R, KR, P, Ar, true>(i1, xp, yp, xq, yq, pv, yb, send, send_off, off, n,
                                          lK, rK, gl);
      else
        band_steps<G, R, KR, P, Ar, false>(i1, xp, yp, xq, yq, pv, yb, send, send_off, off, n,
                                           lK, rK, gl);
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if (hold[p]) {  // pv holds row n
        T rv = pv[p][0];
#pragma unroll
        for (int r = 1; r < R; ++r) rv = (r == r_res[p]) ? pv[p][r] : rv;
        double result = (double)rv;
        if constexpr (kF32) result += off[p];
        store_result(A, slot[p], result);
      }
    }
  }
}

// ===================================================================================
// Band family, shared-memory y variant ("ring"): same sheared coordinates and cell
// dependencies as dtw_band_kernel, but the sliding y window lives in a per-group ring
// in shared memory (read with immediate offsets, one LDS per cell) instead of rotating
// through R registers. That frees 2R registers (more resident warps to cover the
// 29-cycle cell chain) and removes the R-fold unrolled loop body (I-cache).
// Ring: 256 slots (+R duplicated so a lane's R reads never wrap), refilled 32 samples at
// a time from the +inf-padded series, one chunk ahead.
// ===================================================================================
constexpr int kRing = 256;

template <int G, int R, int KR, class Ar, bool CHECK>
__device__ __forceinline__ void ring_steps(int nst, int& i1, const typename Ar::T*& xp,
                                           typename Ar::T& xq, int& b, const typename Ar::T* ring,
                                           typename Ar::T (&pv)[R], typename Ar::T& send,
                                           double& send_off, double& off, int n, int lK, int rK,
                                           int gl) {
  using T = typename Ar::T;
  constexpr bool kF32 = sizeof(T) == 4;
  const T INF = Ar::inf();
  const bool last = gl == G - 1;
#pragma unroll 2
  for (int q = 0; q < nst; ++q) {
    const bool act = CHECK ? (i1 >= 1 && i1 <= n) : true;
    const T x = xq;
    xq = __ldg(++xp);
    const T* yr = ring + b;
    T L = __shfl_up_sync(kFull, send, 1, G);
    if constexpr (kF32) {
      const double loff = __shfl_up_sync(kFull, send_off, 1, G);
      L = L + (T)(loff - off);
    }
    if (gl == 0) L = INF;
    T v0 = Ar::cell3b(x, yr[0], Ar::mn(pv[0], pv[1]), L);
    if (CHECK) v0 = act ? v0 : pv[0];
    if (KR == 0 || KR < 0) {
      if (lK == gl && rK == 0) v0 = INF;
    }
    T U = __shfl_down_sync(kFull, v0, 1, G);
    if constexpr (kF32) {
      const double uoff = __shfl_down_sync(kFull, off, 1, G);
      U = U + (T)(uoff - off);
    }
    U = last ? INF : U;
    if (act) {
      T left = v0;
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const T up = (r < R - 1) ? pv[r + 1] : U;
        const T v = Ar::cell3b(x, yr[r], Ar::mn(pv[r], up), left);
        pv[r] = v;
        left = v;
      }
      pv[0] = v0;
      if constexpr (KR > 0) {
        if (lK == gl) pv[KR] = INF;
      } else if constexpr (KR < 0) {
        if (lK == gl && rK != 0) kill_cell<R>(pv, rK, INF);
      }
      if constexpr (kF32) {
        if (((i1 - 1 + gl) & (kRenormSteps - 1)) == kRenormSteps - 1) {
          T mnv = pv[0];
#pragma unroll
          for (int r = 1; r < R; ++r) mnv = Ar::mn(mnv, pv[r]);
          if (mnv != INF) {
#pragma unroll
            for (int r = 0; r < R; ++r) pv[r] = __fsub_rn(pv[r], mnv);
            off += (double)mnv;
          }
        }
        send_off = off;
      }
      send = pv[R - 1];
    }
    b = (b + 1) & (kRing - 1);
    ++i1;
  }
}

#ifdef DTWG_RING_MINB  // experiments only; see DTWG_FULL_BOUNDS
#define DTWG_RING_BOUNDS __launch_bounds__(kThreads, DTWG_RING_MINB)
#else
#define DTWG_RING_BOUNDS __launch_bounds__(kThreads)
#endif
template <int G, int R, int KR, class Ar>
__global__ void DTWG_RING_BOUNDS dtw_bandring_kernel(const FillArgs A) {
  static_assert(R >= 2, "band family needs R >= 2");
  static_assert(G * R - G <= kRing - 33, "ring too small for this band width");
  // Lane l's window starts l*(R-1) slots after lane 0's: with R-1 odd the 8-byte reads
  // of a warp hit distinct bank pairs (conflict-free); even R-1 would serialise them.
  static_assert((R - 1) % 2 == 1, "ring variant needs even R (bank-conflict-free reads)");
  using T = typename Ar::T;
  constexpr int GPW = 32 / G;
  constexpr int C = 32;           // samples per refill chunk (= steps per chunk)
  constexpr int PER = C / G;      // chunk samples loaded by each lane
  const int lane = threadIdx.x & 31;
  const int gl = lane % G;
  const int gw = lane / G;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const T INF = Ar::inf();
  const T* S = Ar::bbase(A);
  // Ring stride = 8 (mod 16) slots: lane l of group g reads slot base + g*stride + l*(R-1)
  // (+r); with R-1 odd one group covers 8 of the 16 bank pairs and the next group (shifted
  // by 8) the other 8, so a half-warp of 8-byte reads is conflict-free.
  constexpr int kStride = ((kRing + R + 7) / 16) * 16 + 8;
  __shared__ T rings[kThreads / G][kStride];
  T* ring = rings[threadIdx.x / G];
  constexpr int JOFF = 4 * kRing;  // keeps ring indices of j >= 1 - hw - G non-negative

  for (int64_t base = take_items(A, warp * GPW, GPW); base < A.count;
       base = next_items(A, base, nwarps * GPW, GPW)) {
    const int64_t item = base + gw;
    const bool valid = item < A.count;
    const Pair Pp = load_pair(A, valid ? item : base);
    int64_t a, bb;
    decode_slot(Pp.slot, A.p, a, bb);
    const bool a_rows =
        (A.offsets[a + 1] - A.offsets[a]) >= (A.offsets[bb + 1] - A.offsets[bb]);
    const T* Y = S + A.boffsets[a_rows ? bb : a];
    const T* xp = S + A.boffsets[a_rows ? a : bb];
    const int n = Pp.n, m = Pp.m, hw = Pp.hw;
    const int K = 2 * hw + 1;
    const int lK = K / R;
    const int rK = KR >= 0 ? KR : K % R;
    const int kres = m - n + hw;
    const bool hold = valid && (kres / R) == gl;
    const int r_res = kres % R;
    const int kbase = gl * R;
    const int D = G * R - G + 2 - hw;  // first sample index of the chunk written at step 0

    // Ring prologue: samples j in [1 - hw, D) before step 0; chunk c (j in [32c + D,
    // 32c + D + 32)) is written at step 32c from registers loaded one chunk ahead.
    auto put = [&](int j, T v) {
      const int slot = (j + JOFF) & (kRing - 1);
      ring[slot] = v;
      if (slot < R) ring[slot + kRing] = v;
    };
    for (int j = 1 - hw + gl; j < D; j += G) put(j, __ldg(Y + (j - 1)));
    T chunk[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) chunk[u] = __ldg(Y + (D + gl + u * G - 1));

    T pv[R];
#pragma unroll
    for (int r = 0; r < R; ++r) pv[r] = (kbase + r == hw) ? T(0) : INF;  // row 0
    T send = INF;
    double off = 0.0, send_off = 0.0;
    int i1 = 1 - gl;
    xp += i1 - 1;
    T xq = __ldg(xp);
    int b = (i1 + kbase - hw + JOFF) & (kRing - 1);
    const int nsteps = __reduce_max_sync(kFull, n + G - 1);
    const int fill_end = ((G - 1 + C - 1) / C) * C;
    const int drain_start = (__reduce_min_sync(kFull, n) / C) * C;
    for (int s0 = 0; s0 < nsteps; s0 += C) {
      // write chunk s0/C, prefetch the next one
#pragma unroll
      for (int u = 0; u < PER; ++u) put(s0 + D + gl + u * G, chunk[u]);
#pragma unroll
      for (int u = 0; u < PER; ++u) chunk[u] = __ldg(Y + (s0 + C + D + gl + u * G - 1));
      __syncwarp();
      if (s0 < fill_end || s0 >= drain_start)
        ring_steps<G, R, KR, Ar, true>(C, i1, xp, xq, b, ring, pv, send, send_off, off, n, lK, rK,
                                       gl);
      else
        ring_steps<G, R, KR, Ar, false>(C, i1, xp, xq, b, ring, pv, send, send_off, off, n, lK,
                                        rK, gl);
      __syncwarp();
    }
    if (hold) {
      T rv = pv[0];
#pragma unroll
      for (int r = 1; r < R; ++r) rv = (r == r_res) ? pv[r] : rv;
      double result = (double)rv;
      if constexpr (sizeof(T) == 4) result += off;
      store_result(A, Pp.slot, result);
    }
    __syncwarp();
  }
}

// ===================================================================================
// Band family, ring variant with U units per lane ("unit" kernel). The lane's R band
// columns are split into U consecutive units; unit h of lane l is unit u = l*U + h of
// the group and runs one row behind unit u-1 (the wavefront skew moves inside the lane).
// Per step, unit h of a lane works on row i1 - h:
//   * its first cell's left neighbour is unit h-1's last column, same row, computed by
//     unit h-1 in the PREVIOUS step (register; for h = 0: lane l-1, shfl_up);
//   * its last cell's up neighbour is unit h+1's first cell of row i-1, computed in THIS
//     step (v0 of unit h+1; for h = U-1: lane l+1's v0 of unit 0, shfl_down).
// So after the U first cells (v0) of a step are done, the U cell chains are mutually
// independent: ILP U with chains of R/U cells, at the register cost of the U=1 kernel.
// Unit h's y window starts h*(width-1) samples into the lane's, so all reads are
// immediate offsets from one ring pointer; lanes are R-U samples apart, which must be
// odd for conflict-free 8-byte reads (cf. dtw_bandring_kernel).
// ===================================================================================
template <int R, int U>
struct Units {
  static constexpr int width(int h) { return R / U + (h < R % U ? 1 : 0); }
  static constexpr int start(int h) { return h * (R / U) + (h < R % U ? h : R % U); }
  static constexpr int maxw() { return R / U + (R % U ? 1 : 0); }
};

template <int G, int R, int U, int KR, class Ar, bool CHECK, int RING>
__device__ __forceinline__ void unit_steps(int nst, int& i1, const typename Ar::T*& xp,
                                           typename Ar::T& xq, typename Ar::T (&xs)[U], int& b,
                                           const typename Ar::T* ring, typename Ar::T (&pv)[R],
                                           typename Ar::T& send, double& send_off, double& off,
                                           int n, int lK, int rK, int gl) {
  using T = typename Ar::T;
  using Un = Units<R, U>;
  constexpr bool kF32 = sizeof(T) == 4;
  const T INF = Ar::inf();
  const bool last = gl == G - 1;
#pragma unroll kUnitUnroll
  for (int q = 0; q < nst; ++q) {
    bool act[U];
#pragma unroll
    for (int h = 0; h < U; ++h) act[h] = CHECK ? (i1 - h >= 1 && i1 - h <= n) : true;
#pragma unroll
    for (int h = U - 1; h > 0; --h) xs[h] = xs[h - 1];
    xs[0] = xq;
    xq = __ldg(++xp);
    const T* yr = ring + b;
    T L = __shfl_up_sync(kFull, send, 1, G);
    if constexpr (kF32) {
      const double loff = __shfl_up_sync(kFull, send_off, 1, G);
      L = L + (T)(loff - off);
    }
    if (gl == 0) L = INF;
    // First cells of the units (their left inputs are previous-step values).
    T v0[U];
#pragma unroll
    for (int h = 0; h < U; ++h) {
      const int s0 = Un::start(h);
      const T left = h == 0 ? L : pv[s0 - 1];
      T v = Ar::cell3b(xs[h], yr[s0 - h], Ar::mn(pv[s0], pv[s0 + 1]), left);
      if (CHECK) v = act[h] ? v : pv[s0];
      if (KR < 0 || KR == s0) {
        if (lK == gl && rK == s0) v = INF;  // k == K is this unit's first cell
      }
      v0[h] = v;
    }
    T Ud = __shfl_down_sync(kFull, v0[0], 1, G);
    if constexpr (kF32) {
      const double uoff = __shfl_down_sync(kFull, off, 1, G);
      Ud = Ud + (T)(uoff - off);
    }
    Ud = last ? INF : Ud;
    // Chains, interleaved across units (independent).
    T left[U];
#pragma unroll
    for (int h = 0; h < U; ++h) left[h] = v0[h];
#pragma unroll
    for (int c = 1; c < Un::maxw(); ++c) {
#pragma unroll
      for (int h = 0; h < U; ++h) {
        if (c < Un::width(h)) {
          const int r = Un::start(h) + c;
          const bool lastc = c == Un::width(h) - 1;
          const T up = !lastc ? pv[r + 1] : (h == U - 1 ? Ud : v0[h + 1]);
          T v = Ar::cell3b(xs[h], yr[r - h], Ar::mn(pv[r], up), left[h], DTWG_PD_UNIT_PATTERN);
          if (CHECK) v = act[h] ? v : pv[r];
          pv[r] = v;
          left[h] = v;
        }
      }
    }
#pragma unroll
    for (int h = 0; h < U; ++h) pv[Un::start(h)] = v0[h];
    // Cell k == K stays +inf (dtw.hpp:71); first-cell positions were handled above.
    if constexpr (KR > 0) {
      if (lK == gl) pv[KR] = INF;
    } else if constexpr (KR < 0) {
      if (lK == gl && rK != 0) kill_cell<R>(pv, rK, INF);
    }
    if constexpr (kF32) {
      if (((i1 - 1 + gl * U) & (kRenormSteps - 1)) == kRenormSteps - 1) {
        T mnv = pv[0];
#pragma unroll
        for (int r = 1; r < R; ++r) mnv = Ar::mn(mnv, pv[r]);
        if (mnv != INF) {
#pragma unroll
          for (int r = 0; r < R; ++r) pv[r] = __fsub_rn(pv[r], mnv);
          off += (double)mnv;
        }
      }
      send_off = off;
    }
    send = pv[R - 1];
    b = (b + 1) & (RING - 1);
    ++i1;
  }
}

// Resident CTAs the register allocation is capped for (ILP U needs fewer warps; wide R
// keeps 4 CTAs without spills, narrower ones fit 5).
#ifndef DTWG_UNIT_MINB
#define DTWG_UNIT_MINB(R) ((R) >= 40 ? 3 : ((R) >= 20 ? DTWG_UNIT_MINB20 : 5))
#endif
#ifndef DTWG_UNIT_MINB20
#define DTWG_UNIT_MINB20 4
#endif
#ifdef DTWG_UNIT_MINB32_N
#define DTWG_UNIT_MINB32(R) DTWG_UNIT_MINB32_N
#else
#define DTWG_UNIT_MINB32(R) DTWG_UNIT_MINB(R)
#endif
template <int G, int R, int U, int KR, class Ar>
__global__ void __launch_bounds__(kThreads, Ar::kFp32 ? DTWG_UNIT_MINB32(R) : DTWG_UNIT_MINB(R))
    dtw_bandunit_kernel(const FillArgs A) {
  static_assert(U >= 1 && R / U >= 2, "units need >= 2 columns");
  // ring slots: a power of two holding the group's window (G*(R-U)+1) plus one chunk ahead
  constexpr int RING = G * (R - U) <= 256 - 33 ? 256 : (G * (R - U) <= 512 - 33 ? 512 : 1024);
  static_assert(G * (R - U) <= RING - 33, "ring too small for this band width");
  static_assert((R - U) % 2 == 1, "unit variant needs odd R-U (bank-conflict-free reads)");
  using T = typename Ar::T;
  constexpr int GPW = 32 / G;
  constexpr int C = 32;
  constexpr int PER = C / G;
  const int lane = threadIdx.x & 31;
  const int gl = lane % G;
  const int gw = lane / G;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const T INF = Ar::inf();
  const T* S = Ar::bbase(A);
  // Per-group ring stride: 8 mod 16 words keeps the G = 8/16/32 groups of a warp on
  // distinct banks; G = 4 (8 groups of 4 lanes) needs 4 mod 32.
  constexpr int kStride = G == 4 ? ((RING + R + 1 - 4 + 31) / 32) * 32 + 4
                                 : ((RING + R + 7) / 16) * 16 + 8;
  __shared__ T rings[kThreads / G][kStride];
  T* ring = rings[threadIdx.x / G];
  constexpr int JOFF = 4 * RING;

  for (int64_t base = take_items(A, warp * GPW, GPW); base < A.count;
       base = next_items(A, base, nwarps * GPW, GPW)) {
    const int64_t item = base + gw;
    const bool valid = item < A.count;
    const Pair Pp = load_pair(A, valid ? item : base);
    int64_t a, bb;
    decode_slot(Pp.slot, A.p, a, bb);
    const bool a_rows =
        (A.offsets[a + 1] - A.offsets[a]) >= (A.offsets[bb + 1] - A.offsets[bb]);
    const T* Y = S + A.boffsets[a_rows ? bb : a];
    const T* xp = S + A.boffsets[a_rows ? a : bb];
    const int n = Pp.n, m = Pp.m, hw = Pp.hw;
    const int K = 2 * hw + 1;
    const int lK = K / R;
    const int rK = KR >= 0 ? KR : K % R;
    const int kres = m - n + hw;
    const bool hold = valid && (kres / R) == gl;
    const int r_res = kres % R;
    const int kbase = gl * R;
    const int D = G * (R - U) + 2 - hw;  // first sample index of the chunk written at step 0

    auto put = [&](int j, T v) {
      const int slot = (j + JOFF) & (RING - 1);
      ring[slot] = v;
      if (slot < R) ring[slot + RING] = v;
    };
    for (int j = 1 - hw + gl; j < D; j += G) put(j, __ldg(Y + (j - 1)));
    T chunk[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) chunk[u] = __ldg(Y + (D + gl + u * G - 1));

    T pv[R];
#pragma unroll
    for (int r = 0; r < R; ++r) pv[r] = (kbase + r == hw) ? T(0) : INF;  // row 0
    T send = INF;
    double off = 0.0, send_off = 0.0;
    int i1 = 1 - gl * U;  // row of unit 0 at step 0
    xp += i1 - 1;
    T xq = __ldg(xp);
    T xs[U];
#pragma unroll
    for (int h = 0; h < U - 1; ++h) xs[h] = __ldg(xp - 1 - h);  // shifted in at step 0
    xs[U - 1] = INF;
    int b = (i1 + kbase - hw + JOFF) & (RING - 1);
    const int nsteps = __reduce_max_sync(kFull, n + G * U - 1);
    const int fill_end = ((G * U - 1 + C - 1) / C) * C;
    const int drain_start = (__reduce_min_sync(kFull, n) / C) * C;
    for (int s0 = 0; s0 < nsteps; s0 += C) {
#pragma unroll
      for (int u = 0; u < PER; ++u) put(s0 + D + gl + u * G, chunk[u]);
#pragma unroll
      for (int u = 0; u < PER; ++u) chunk[u] = __ldg(Y + (s0 + C + D + gl + u * G - 1));
      __syncwarp();
      if (s0 < fill_end || s0 >= drain_start)
        unit_steps<G, R, U, KR, Ar, true, RING>(C, i1, xp, xq, xs, b, ring, pv, send, send_off,
                                                off, n, lK, rK, gl);
      else
        unit_steps<G, R, U, KR, Ar, false, RING>(C, i1, xp, xq, xs, b, ring, pv, send, send_off,
                                                 off, n, lK, rK, gl);
      __syncwarp();
    }
    if (hold) {
      T rv = pv[0];
#pragma unroll
      for (int r = 1; r < R; ++r) rv = (r == r_res) ? pv[r] : rv;
      double result = (double)rv;
      if constexpr (sizeof(T) == 4) result += off;
      store_result(A, Pp.slot, result);
    }
    __syncwarp();
  }
}

}  // namespace kern
}  // namespace dtwgpu
