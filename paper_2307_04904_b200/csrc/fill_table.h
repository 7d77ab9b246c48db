// fill_table.h -- the compiled (G, R) instantiations of both fill families.
#pragma once

#define DTWG_FULL_CFGS(X)                                                              \
  X(2, 23) X(4, 12) X(8, 8) X(16, 8) X(16, 16) X(32, 4) X(32, 8) X(32, 12) X(32, 15) \
  X(32, 16)
#define DTWG_BAND_CFGS_G16(X) X(16, 7) X(16, 9) X(16, 11) X(16, 13)
#define DTWG_BAND_CFGS_G32(X) X(32, 3) X(32, 5) X(32, 7) X(32, 9) X(32, 13)

namespace dtwgpu {
const void* full_kernel_ptr(int G, int R, bool mask, bool fp32);
const void* band16_kernel_ptr(int R, int kr, int P, bool fp32);
const void* band32_kernel_ptr(int R, int kr, int P, bool fp32);
}  // namespace dtwgpu
