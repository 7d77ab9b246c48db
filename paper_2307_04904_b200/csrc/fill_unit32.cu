// fill_unit32.cu -- fp32 instantiations of the units-per-lane ring Band variant: every
// static kill position KR = (2hw+1) % R (a runtime KR costs a branch tree per step in the
// 4-instruction fp32 cell), plus the runtime-KR fallback.
#include "dtw_kernels.cuh"
#include "fill_table.h"

namespace dtwgpu {
namespace {
using namespace kern;
template <int G, int R, int U, int KR>
struct Unit32Table {
  static const void* get(int kr) {
    if (kr == KR) return (const void*)dtw_bandunit_kernel<G, R, U, KR, F32>;
    if constexpr (KR > 0) return Unit32Table<G, R, U, KR - 1>::get(kr);
    return nullptr;
  }
};
}  // namespace

const void* unit32w_kernel_ptr(int G, int R, int U, int kr);  // fill_unit32w.cu

const void* unit32_kernel_ptr(int G, int R, int U, int kr) {
#define DTWG_UN32(g, r, u)                                                        \
  if (G == g && R == r && U == u) {                                               \
    if (kr < 0) return (const void*)dtw_bandunit_kernel<g, r, u, -1, F32>;       \
    return Unit32Table<g, r, u, r - 1>::get(kr);                                  \
  }
  DTWG_UNIT_CFGS(DTWG_UN32)
#undef DTWG_UN32
  return unit32w_kernel_ptr(G, R, U, kr);
}

}  // namespace dtwgpu
