// fill_unit32w.cu -- fp32-only instantiations of the units-per-lane ring Band variant
// with wide lanes (fill_table.h DTWG_UNIT_CFGS_F32): every static kill position (the fp32
// planner always uses one; no runtime-KR variant for R > 32), in their own translation
// unit (compile time).
#include "dtw_kernels.cuh"
#include "fill_table.h"

namespace dtwgpu {
namespace {
using namespace kern;
template <int G, int R, int U, int KR>
struct Unit32wTable {
  static const void* get(int kr) {
    if (kr == KR) return (const void*)dtw_bandunit_kernel<G, R, U, KR, F32>;
    if constexpr (KR > 0) return Unit32wTable<G, R, U, KR - 1>::get(kr);
    return nullptr;
  }
};
}  // namespace

const void* unit32w_kernel_ptr(int G, int R, int U, int kr) {
#define DTWG_UN32W(g, r, u)                                                       \
  if (G == g && R == r && U == u) {                                               \
    return kr < 0 ? nullptr : Unit32wTable<g, r, u, r - 1>::get(kr);              \
  }
  DTWG_UNIT_CFGS_F32(DTWG_UN32W)
#undef DTWG_UN32W
  return nullptr;
}

}  // namespace dtwgpu
