// fill_ring.cu -- instantiations of the shared-memory-ring Band variant (dtw_kernels.cuh).
// fp64 kernels for every static kill position KR = (2hw+1) % R; fp32 with a runtime KR.
#include "dtw_kernels.cuh"
#include "fill_table.h"

namespace dtwgpu {
namespace {
using namespace kern;
template <int G, int R, int KR>
struct RingTable {
  static const void* get(int kr) {
    if (kr == KR) return (const void*)dtw_bandring_kernel<G, R, KR, F64>;
    if constexpr (KR > 0) return RingTable<G, R, KR - 1>::get(kr);
    return nullptr;
  }
};
}  // namespace

const void* ring_kernel_ptr(int G, int R, int kr, bool fp32) {
#define DTWG_RG(g, r)                                                             \
  if (G == g && R == r) {                                                         \
    if (fp32) return (const void*)dtw_bandring_kernel<g, r, -1, F32>;            \
    if (kr < 0) return (const void*)dtw_bandring_kernel<g, r, -1, F64>;          \
    return RingTable<g, r, r - 1>::get(kr);                                       \
  }
  DTWG_RING_CFGS(DTWG_RG)
#undef DTWG_RG
  return nullptr;
}

}  // namespace dtwgpu
