// fill_full.cu -- instantiations of the Full (column-strip) family, see dtw_kernels.cuh.
#include "dtw_kernels.cuh"
#include "fill_table.h"

namespace dtwgpu {

const void* full_kernel_ptr(int G, int R, int TR, bool mask, bool fp32, bool mp) {
  using namespace kern;
#define DTWG_F(g, r, tr)                                                                    \
  if (G == g && R == r && TR == tr) {                                                       \
    if (mp) {                                                                               \
      if (fp32) return mask ? (const void*)dtw_full_kernel<g, r, tr, true, F32, true>       \
                            : (const void*)dtw_full_kernel<g, r, tr, false, F32, true>;     \
      return mask ? (const void*)dtw_full_kernel<g, r, tr, true, F64, true>                 \
                  : (const void*)dtw_full_kernel<g, r, tr, false, F64, true>;               \
    }                                                                                       \
    if (fp32) return mask ? (const void*)dtw_full_kernel<g, r, tr, true, F32, false>        \
                          : (const void*)dtw_full_kernel<g, r, tr, false, F32, false>;      \
    return mask ? (const void*)dtw_full_kernel<g, r, tr, true, F64, false>                  \
                : (const void*)dtw_full_kernel<g, r, tr, false, F64, false>;                \
  }
  DTWG_FULL_CFGS(DTWG_F)
#undef DTWG_F
#define DTWG_F32(g, r, tr)                                                                  \
  if (fp32 && G == g && R == r && TR == tr) {                                               \
    if (mp) return mask ? (const void*)dtw_full_kernel<g, r, tr, true, F32, true>           \
                        : (const void*)dtw_full_kernel<g, r, tr, false, F32, true>;         \
    return mask ? (const void*)dtw_full_kernel<g, r, tr, true, F32, false>                  \
                : (const void*)dtw_full_kernel<g, r, tr, false, F32, false>;                \
  }
  DTWG_FULL_CFGS_F32(DTWG_F32)
#undef DTWG_F32
#define DTWG_L64(r, tr)                                                                     \
  if (!fp32 && G == 1 && R == r && TR == tr) {                                              \
    if (mp) return nullptr; /* multi-pass one-lane fp64: dtw_full_kernel<1, R, 4> */    \
    return mask ? (const void*)dtw_lane_kernel<r, tr, true, F64>                            \
                : (const void*)dtw_lane_kernel<r, tr, false, F64>;                          \
  }
  DTWG_LANE_CFGS_F64(DTWG_L64)
#undef DTWG_L64
  return nullptr;
}

}  // namespace dtwgpu
