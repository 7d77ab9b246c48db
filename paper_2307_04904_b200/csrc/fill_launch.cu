// fill_launch.cu -- kernel lookup, occupancy and launch for the fill families.
#include <cuda_runtime.h>

#include "dtw_fill.cuh"
#include "fill_table.h"

namespace dtwgpu {

static const void* kernel_ptr(const KernelCfg& c) {
  if (c.family == Family::Full && c.ysm)
    return full1s_kernel_ptr(c.G, c.R, c.TR, c.mask, c.fp32, c.mp);
  if (c.family == Family::Full) {
    const void* f = full_kernel_ptr(c.G, c.R, c.TR, c.mask, c.fp32, c.mp);
    return (f || c.fp32) ? f : full64_kernel_ptr(c.G, c.R, c.TR, c.mask, c.mp);
  }
  if (c.family == Family::Strip) return c.G == 32 ? strip_kernel_ptr(c.R, c.TR, c.mask, c.fp32) : nullptr;
  if (c.ring && c.U > 1) return c.P == 1 ? unit_kernel_ptr(c.G, c.R, c.U, c.kr, c.fp32) : nullptr;
  if (c.ring) return c.P == 1 ? ring_kernel_ptr(c.G, c.R, c.kr, c.fp32) : nullptr;
  if (c.G == 16) return band16_kernel_ptr(c.R, c.kr, c.P, c.fp32);
  if (c.G == 32) return band32_kernel_ptr(c.R, c.kr, c.P, c.fp32);
  return nullptr;
}

bool fill_cfg_supported(const KernelCfg& cfg) { return kernel_ptr(cfg) != nullptr; }

cudaError_t launch_fill(const KernelCfg& cfg, const FillArgs& args, int blocks,
                        cudaStream_t stream) {
  const void* fn = kernel_ptr(cfg);
  if (!fn) return cudaErrorInvalidDeviceFunction;
  FillArgs a = args;
  void* params[] = {&a};
  return cudaLaunchKernel(fn, dim3(blocks), dim3(kThreads), params, 0, stream);
}

int fill_blocks_per_sm(const KernelCfg& cfg) {
  const void* fn = kernel_ptr(cfg);
  int nb = 0;
  if (!fn || cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kThreads, 0) != cudaSuccess)
    nb = 1;
  return nb > 0 ? nb : 1;
}

}  // namespace dtwgpu
