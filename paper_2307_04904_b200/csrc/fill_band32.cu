// fill_band32.cu -- instantiations of the Band family with G = 32 lanes per pair.
// fp64 kernels are instantiated for every static kill position KR = (2hw+1) % R so
// the out-of-band cell is cleared with one predicated move (dtw_kernels.cuh).
#include "dtw_kernels.cuh"
#include "fill_table.h"

namespace dtwgpu {
namespace {
using namespace kern;
template <int G, int R, int KR, int P>
struct BandTable {
  static const void* get(int kr) {
    if (kr == KR) return (const void*)dtw_band_kernel<G, R, KR, P, F64>;
    if constexpr (KR > 0) return BandTable<G, R, KR - 1, P>::get(kr);
    return nullptr;
  }
};
}  // namespace

const void* band32_kernel_ptr(int R, int kr, int P, bool fp32) {
#define DTWG_B(g, r)                                                              \
  if (g == 32 && R == r) {                                                        \
    if (P != 1) return nullptr; /* P = 2 measured slower everywhere; not built */  \
    if (fp32) return (const void*)dtw_band_kernel<g, r, -1, 1, F32>;             \
    if (kr < 0) return (const void*)dtw_band_kernel<g, r, -1, 1, F64>;           \
    return BandTable<g, r, r - 1, 1>::get(kr);                                    \
  }
  DTWG_BAND_CFGS_G32(DTWG_B)
#undef DTWG_B
  return nullptr;
}

}  // namespace dtwgpu
