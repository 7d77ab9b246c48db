// fill_strip.cu -- instantiations of the Strip family (long pairs, dtw_kernels.cuh).
#include "dtw_kernels.cuh"
#include "fill_table.h"

namespace dtwgpu {
using namespace kern;

const void* strip_kernel_ptr(int R, int TR, bool mask, bool fp32) {
#define DTWG_ST(r, tr)                                                                     \
  if (R == r && TR == tr) {                                                                \
    if (fp32) return mask ? (const void*)dtw_strip_kernel<r, tr, true, F32>                \
                          : (const void*)dtw_strip_kernel<r, tr, false, F32>;              \
    return mask ? (const void*)dtw_strip_kernel<r, tr, true, F64>                          \
                : (const void*)dtw_strip_kernel<r, tr, false, F64>;                        \
  }
  DTWG_STRIP_CFGS(DTWG_ST)
#undef DTWG_ST
  return nullptr;
}

}  // namespace dtwgpu
