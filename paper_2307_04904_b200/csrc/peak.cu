// peak.cu -- live measurement of the cell-update ceiling (the roofline denominator).
//
// The DTW fill is min-plus, so neither the HBM copy nor the bf16 GEMM peak bounds it.
// Its ceiling is the issue/FP64-pipe rate of the cell body itself:
//   fp64:  DADD(sub) DMUL DSETP+2xFSEL DSETP+2xFSEL DADD   (5 fp64-pipe ops, 9 issues)
//   fp32:  FADD FMUL FMNMX3 FADD
// This kernel runs 8 independent chains of exactly that body per thread on every SM,
// so the result is the best cells/s the instruction mix can reach with no memory, no
// wavefront and no dependency stalls. bench.py reports roofline.frac against it.
#include <cuda_runtime.h>

#include <cstdint>

namespace dtwgpu {
namespace {

template <int CH, class T>
__global__ void cell_peak_kernel(const T* in, T* out, int iters) {
  T x = in[threadIdx.x & 7], y[CH], a[CH], b[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    y[c] = in[(c + 1) & 7];
    a[c] = in[(c + 2) & 7];
    b[c] = in[(c + 3) & 7];
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      T v;
      if constexpr (sizeof(T) == 8) {
        const T d = __dsub_rn(x, y[c]);
        const T m1 = b[c] < a[c] ? b[c] : a[c];
        const T m2 = y[c] < m1 ? y[c] : m1;
        v = __dadd_rn(__dmul_rn(d, d), m2);
      } else {
        const T d = __fsub_rn(x, y[c]);
        v = __fadd_rn(__fmul_rn(d, d), fminf(fminf(a[c], b[c]), y[c]));
      }
      a[c] = b[c];
      b[c] = v;
      y[c] = v;
    }
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += b[c];
  if (s == (T)-1) out[threadIdx.x] = s;
}

template <class T>
cudaError_t run(cudaStream_t st, int sms, double* cells_per_s) {
  T* buf = nullptr;
  cudaError_t e = cudaMalloc(&buf, 1024 * sizeof(T));
  if (e != cudaSuccess) return e;
  T h[8] = {1, 2, 3, 4, 5, 6, 7, 8};
  cudaMemcpyAsync(buf, h, sizeof(h), cudaMemcpyHostToDevice, st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2048, blocks = sms * 8;  // 32 warps per SM
  cell_peak_kernel<8, T><<<blocks, 128, 0, st>>>(buf, buf + 512, iters);
  cudaEventRecord(e0, st);
  cell_peak_kernel<8, T><<<blocks, 128, 0, st>>>(buf, buf + 512, iters);
  cudaEventRecord(e1, st);
  e = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  *cells_per_s = (double)blocks * 128 * 8 * iters / (ms * 1e-3);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  return e == cudaSuccess ? cudaGetLastError() : e;
}

}  // namespace

cudaError_t measure_cell_peak(cudaStream_t st, int sms, bool fp32, double* cells_per_s) {
  return fp32 ? run<float>(st, sms, cells_per_s) : run<double>(st, sms, cells_per_s);
}

}  // namespace dtwgpu
