// fill_unit.cu -- fp64 instantiations of the units-per-lane ring Band variant
// (dtw_kernels.cuh) for every static kill position KR = (2hw+1) % R, plus the runtime-KR
// fallback; fp32 lives in fill_unit32.cu (compiled in parallel).
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

const void* unit32_kernel_ptr(int G, int R, int U, int kr);

const void* unit_kernel_ptr(int G, int R, int U, int kr, bool fp32) {
  if (fp32) return unit32_kernel_ptr(G, R, U, kr);
#define DTWG_UN(g, r, u)                                                          \
  if (G == g && R == r && U == u) {                                               \
    if (kr < 0) return (const void*)dtw_bandunit_kernel<g, r, u, -1, F64>;       \
    return UnitTable<g, r, u, r - 1>::get(kr);                                    \
  }
  DTWG_UNIT_CFGS(DTWG_UN)
#undef DTWG_UN
  return nullptr;
}

}  // namespace dtwgpu
