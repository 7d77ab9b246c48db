// fill_unit.cu -- instantiations of the units-per-lane ring Band variant (dtw_kernels.cuh).
// fp64 kernels for every static kill position KR = (2hw+1) % R; fp32 with a runtime KR.
#include "dtw_kernels.cuh"
#include "fill_table.h"

namespace dtwgpu {
namespace {
using namespace kern;
template <int G, int R, int U, int KR>
struct UnitTable {
  static const void* get(int kr) {
    if (kr == KR) return (const void*)dtw_bandunit_kernel<G, R, U, KR, F64>;
    if constexpr (KR > 0) return UnitTable<G, R, U, KR - 1>::get(kr);
    return nullptr;
  }
};
}  // namespace

const void* unit_kernel_ptr(int G, int R, int U, int kr, bool fp32) {
#define DTWG_UN(g, r, u)                                                          \
  if (G == g && R == r && U == u) {                                               \
    if (fp32) return (const void*)dtw_bandunit_kernel<g, r, u, -1, F32>;         \
    if (kr < 0) return (const void*)dtw_bandunit_kernel<g, r, u, -1, F64>;       \
    return UnitTable<g, r, u, r - 1>::get(kr);                                    \
  }
  DTWG_UNIT_CFGS(DTWG_UN)
#undef DTWG_UN
  return nullptr;
}

}  // namespace dtwgpu
