// fill_table.h -- the compiled (G, R) instantiations of both fill families.
#pragma once

// Full family: (G, R, rows per step)
#define DTWG_FULL_CFGS(X)                                                                  \
  X(2, 23, 2) X(4, 12, 2) X(8, 8, 2) X(16, 8, 2) X(16, 16, 2) X(32, 4, 2) X(32, 8, 2)    \
  X(32, 12, 2) X(32, 15, 2) X(32, 16, 2) X(2, 23, 4) X(4, 12, 4) X(8, 8, 4) X(16, 16, 4) \
  X(32, 15, 4) X(32, 16, 4) X(2, 16, 4) X(1, 20, 4) X(1, 24, 4) X(1, 28, 4) X(1, 32, 4)
// Full family, fp32 only (wide strips: half the per-row overhead per cell; the fp64
// instantiation would need > 255 registers)
// Full strips with y in shared memory (dtw_full1s_kernel, 3 CTAs/SM): (G, R, rows per step)
#define DTWG_FULL1S_CFGS(X) X(1, 28, 4) X(1, 24, 4) X(1, 20, 4) X(1, 16, 4)
// Full family, fp64 only, multi-pass (long series: wider passes, fewer boundary columns)
#define DTWG_FULL_CFGS_F64(X) X(2, 30, 4) X(4, 30, 4) X(8, 30, 4)
#define DTWG_FULL_CFGS_F32(X) X(16, 30, 4) X(1, 46, 4) X(16, 32, 4) X(1, 56, 4) X(1, 64, 4)
// One lane per pair, fp64, single strip (dtw_lane_kernel): (R, rows per step)
#define DTWG_LANE_CFGS_F64(X) X(46, 2)
#define DTWG_BAND_CFGS_G16(X) X(16, 7) X(16, 9) X(16, 11) X(16, 13)
#define DTWG_BAND_CFGS_G32(X) X(32, 3) X(32, 5) X(32, 7) X(32, 9) X(32, 13)
// Band family, shared-memory y ring variant
#define DTWG_RING_CFGS(X) X(8, 16) X(8, 26) X(16, 8) X(16, 14) X(32, 6)
// Band family, ring variant with U units per lane: (G, R, U), R - U odd
// Strip family (G = 32): (R, rows per step)
#define DTWG_STRIP_CFGS(X) X(15, 4) X(8, 4)
// Band ring with U units, fp32 only (wide lanes: half the per-step shuffle and offset
// work per cell; fp64 would spill): (G, R, U)
#define DTWG_UNIT_CFGS_F32(X) X(4, 52, 3)
#define DTWG_UNIT_CFGS(X) X(8, 26, 3) X(8, 26, 5) X(16, 14, 3) X(16, 13, 2) X(16, 20, 3) \
  X(16, 26, 3) X(32, 20, 3) X(32, 26, 3)

namespace dtwgpu {
const void* full_kernel_ptr(int G, int R, int TR, bool mask, bool fp32, bool mp);
const void* full64_kernel_ptr(int G, int R, int TR, bool mask, bool mp);
const void* full1s_kernel_ptr(int G, int R, int TR, bool mask, bool fp32, bool mp);
const void* band16_kernel_ptr(int R, int kr, int P, bool fp32);
const void* band32_kernel_ptr(int R, int kr, int P, bool fp32);
const void* ring_kernel_ptr(int G, int R, int kr, bool fp32);
const void* unit_kernel_ptr(int G, int R, int U, int kr, bool fp32);
const void* strip_kernel_ptr(int R, int TR, bool mask, bool fp32);
}  // namespace dtwgpu
