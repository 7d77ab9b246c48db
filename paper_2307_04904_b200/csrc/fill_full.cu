// fill_full.cu -- instantiations of the Full (column-strip) family, see dtw_kernels.cuh.
#include "dtw_kernels.cuh"
#include "fill_table.h"

namespace dtwgpu {

const void* full_kernel_ptr(int G, int R, bool mask, bool fp32) {
  using namespace kern;
#define DTWG_F(g, r)                                                              \
  if (G == g && R == r) {                                                         \
    if (fp32) return mask ? (const void*)dtw_full_kernel<g, r, true, F32>         \
                          : (const void*)dtw_full_kernel<g, r, false, F32>;       \
    return mask ? (const void*)dtw_full_kernel<g, r, true, F64>                   \
                : (const void*)dtw_full_kernel<g, r, false, F64>;                 \
  }
  DTWG_FULL_CFGS(DTWG_F)
#undef DTWG_F
  return nullptr;
}

}  // namespace dtwgpu
