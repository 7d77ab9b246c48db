// fill_full64.cu -- fp64-only multi-pass instantiations of the Full family (see
// fill_table.h, DTWG_FULL_CFGS_F64), compiled in their own translation unit.
#include "dtw_kernels.cuh"
#include "fill_table.h"

namespace dtwgpu {

const void* full64_kernel_ptr(int G, int R, int TR, bool mask, bool mp) {
  using namespace kern;
  if (!mp) return nullptr;
#define DTWG_F64(g, r, tr)                                                                  \
  if (G == g && R == r && TR == tr)                                                         \
    return mask ? (const void*)dtw_full_kernel<g, r, tr, true, F64, true>                   \
                : (const void*)dtw_full_kernel<g, r, tr, false, F64, true>;
  DTWG_FULL_CFGS_F64(DTWG_F64)
#undef DTWG_F64
  return nullptr;
}

const void* full1s_kernel_ptr(int G, int R, int TR, bool mask, bool fp32, bool mp) {
  using namespace kern;
  if (fp32 || !mp) return nullptr;
#define DTWG_F1S(g, r, tr)                                                                  \
  if (G == g && R == r && TR == tr)                                                         \
    return mask ? (const void*)dtw_full1s_kernel<g, r, tr, true, F64, true>                 \
                : (const void*)dtw_full1s_kernel<g, r, tr, false, F64, true>;
  DTWG_FULL1S_CFGS(DTWG_F1S)
#undef DTWG_F1S
  return nullptr;
}

}  // namespace dtwgpu
