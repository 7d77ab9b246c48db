// peak.cu -- live measurement of the cell-update ceiling (reported beside the roofline).
//
// The DTW fill is min-plus, so neither the HBM copy nor the bf16 GEMM peak bounds it.
// Its ceiling is the rate at which an SM issues the cell body itself:
//   fp64:  DADD(sub) DMUL DSETP+2xFSEL DSETP+2xFSEL DADD   (5 fp64-pipe ops, 9 issues), or
//          DADD DMUL DSETP+2xFSEL DSETP @q DADD @!q DADD    (6 fp64-pipe ops, 8 issues),
//          or the two forms on alternate cells
//   fp32:  FADD FMUL FMNMX3 FADD
// This kernel runs CH independent chains of exactly that body per thread on every SM
// with no memory and no wavefront. A chain's three registers rotate through the roles
// diag / up / left, so every cell's three inputs are distinct values. (Rounds 1-2 fed
// one value in as both `up` and `left`; the compiler then dropped a quarter of the
// compares and selects and the "ceiling" read 3045-3058 GCUPS, 12.3 SMSP-cycles per
// warp-cell. The real body measures 13.7-14.6: tools/dispatch_microbench.cu.)
#include <cuda_runtime.h>

#include <cstdint>

#include "dtw_kernels.cuh"

namespace dtwgpu {
namespace {

// FORM 0: selects; 1: predicated adds; 2: the two forms on alternate chains
template <int FORM, class T>
__device__ __forceinline__ T peak_cell(T x, T diag, T up, T left, int chain) {
  if constexpr (sizeof(T) == 8) {
    const T m = up < diag ? up : diag;
    if (FORM == 1 || (FORM == 2 && chain % 2 == 0)) return kern::F64::cell3pd(x, left, m, left);
    else return kern::F64::cell(x, left, left < m ? left : m);
  } else {
    const T d = __fsub_rn(x, left);
    return __fadd_rn(__fmul_rn(d, d), fminf(fminf(diag, up), left));
  }
}

template <int CH, int FORM, class T>
__global__ void cell_peak_kernel(const T* in, T* out, int iters) {
  T x = in[threadIdx.x & 7], a[CH], b[CH], c[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    a[i] = in[(i + 1) & 7];
    b[i] = in[(i + 2) & 7];
    c[i] = in[(i + 3) & 7];
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      c[i] = peak_cell<FORM>(x, c[i], b[i], a[i], i);  // newest value replaces the oldest
      b[i] = peak_cell<FORM>(x, b[i], a[i], c[i], i);
      a[i] = peak_cell<FORM>(x, a[i], c[i], b[i], i);
    }
  }
  T s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += a[i] + b[i] + c[i];
  if (s == (T)-1) out[threadIdx.x] = s;
}

template <int CH, int FORM, class T>
cudaError_t time_form(cudaStream_t st, int sms, T* buf, double* cells_per_s) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096, blocks = sms * 8;  // 32 warps per SM
  cell_peak_kernel<CH, FORM, T><<<blocks, 128, 0, st>>>(buf, buf + 512, iters);
  cudaEventRecord(e0, st);
  cell_peak_kernel<CH, FORM, T><<<blocks, 128, 0, st>>>(buf, buf + 512, iters);
  cudaEventRecord(e1, st);
  cudaError_t e = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  *cells_per_s = (double)blocks * 128 * CH * 3 * iters / (ms * 1e-3);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return e == cudaSuccess ? cudaGetLastError() : e;
}

template <class T>
cudaError_t run(cudaStream_t st, int sms, double* cells_per_s) {
  T* buf = nullptr;
  cudaError_t e = cudaMalloc(&buf, 1024 * sizeof(T));
  if (e != cudaSuccess) return e;
  T h[8] = {1, 2, 3, 4, 5, 6, 7, 8};
  cudaMemcpyAsync(buf, h, sizeof(h), cudaMemcpyHostToDevice, st);
  // best of the instruction forms the fill kernels use (fp64: selects / predicated adds)
  double best = 0, v = 0;
  e = time_form<2, 0, T>(st, sms, buf, &v);
  if (v > best) best = v;
  if (e == cudaSuccess && sizeof(T) == 8) {
    e = time_form<2, 1, T>(st, sms, buf, &v);
    if (v > best) best = v;
  }
  if (e == cudaSuccess && sizeof(T) == 8) {
    e = time_form<2, 2, T>(st, sms, buf, &v);
    if (v > best) best = v;
  }
  if (e == cudaSuccess && sizeof(T) == 8) {
    e = time_form<4, 2, T>(st, sms, buf, &v);
    if (v > best) best = v;
  }
  if (e == cudaSuccess) {
    e = time_form<4, 0, T>(st, sms, buf, &v);
    if (v > best) best = v;
  }
  *cells_per_s = best;
  cudaFree(buf);
  return e;
}

}  // namespace

cudaError_t measure_cell_peak(cudaStream_t st, int sms, bool fp32, double* cells_per_s) {
  return fp32 ? run<float>(st, sms, cells_per_s) : run<double>(st, sms, cells_per_s);
}

}  // namespace dtwgpu
