// block_microbench.cu -- the Full family's 4-row x R-column step (FullRows, the exact
// code of the fill kernels) in a register-only loop: no loads, no boundary column, no
// loop bookkeeping beyond the step counter. Compared with tools/mix_microbench.cu (the
// same cell body as independent 1-D chains) it isolates the cost of the block's 2-D
// dependency pattern as ptxas schedules it; compared with the c4 kernel it isolates the
// per-step memory and bookkeeping. One lane per pair layout: 1 thread = 1 strip.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2307_04904_b200/csrc \
//        -o block tools/block_microbench.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "dtw_kernels.cuh"

using namespace dtwgpu::kern;

template <int R, int TR>
__global__ void __launch_bounds__(128) block_kernel(const double* in, double* out, int steps) {
  double pv[R], yv[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    yv[r] = in[(r + threadIdx.x) & 63];
    pv[r] = in[(r + 7) & 63] * 1e-3;
  }
  double xs = in[threadIdx.x & 63];
  double diag0 = 0.0;
  for (int s = 0; s < steps; ++s) {
    double x[TR], L[TR], o[TR];
#pragma unroll
    for (int t = 0; t < TR; ++t) {
      x[t] = xs + (double)t;  // row samples (any values; DADD off the chain)
      L[t] = 1e300;            // left boundary (+large, like +inf for a first pass)
    }
    FullRows<R, TR, 0, F64>::run(pv, yv, x, diag0, L, 0, 0, o);
    diag0 = L[TR - 1];
    xs = o[TR - 1] * 1e-9;  // keep the loop dependent on the block
  }
  double acc = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) acc += pv[r];
  if (acc == -1.0) out[threadIdx.x] = acc;
}

// Two independent strips per thread (e.g. two pairs per lane), one FullRows block each per
// step: the scheduler can interleave two uncoupled wavefronts.
template <int R, int TR>
__global__ void __launch_bounds__(128) block2_kernel(const double* in, double* out, int steps) {
  double pv[R], yv[R], pw[R], yw[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    yv[r] = in[(r + threadIdx.x) & 63];
    pv[r] = in[(r + 7) & 63] * 1e-3;
    yw[r] = in[(r + threadIdx.x + 5) & 63];
    pw[r] = in[(r + 9) & 63] * 1e-3;
  }
  double xs = in[threadIdx.x & 63], xt = in[(threadIdx.x + 3) & 63];
  double d0 = 0.0, d1 = 0.0;
  for (int s = 0; s < steps; ++s) {
    double x[TR], L[TR], o[TR], x2[TR], L2[TR], o2[TR];
#pragma unroll
    for (int t = 0; t < TR; ++t) {
      x[t] = xs + (double)t;
      x2[t] = xt + (double)t;
      L[t] = 1e300;
      L2[t] = 1e300;
    }
    FullRows<R, TR, 0, F64>::run(pv, yv, x, d0, L, 0, 0, o);
    FullRows<R, TR, 0, F64>::run(pw, yw, x2, d1, L2, 0, 0, o2);
    d0 = L[TR - 1];
    d1 = L2[TR - 1];
    xs = o[TR - 1] * 1e-9;
    xt = o2[TR - 1] * 1e-9;
  }
  double acc = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) acc += pv[r] + pw[r];
  if (acc == -1.0) out[threadIdx.x] = acc;
}

template <int R, int TR>
void run2(int sms, int clk_khz, double* in, double* out, int blocks_per_sm) {
  const int steps = 2048;
  const int blocks = sms * blocks_per_sm;
  block2_kernel<R, TR><<<blocks, 128>>>(in, out, steps);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  block2_kernel<R, TR><<<blocks, 128>>>(in, out, steps);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double cells = 2.0 * blocks * 128 * steps * R * TR;
  const double gcups = cells / (ms * 1e-3) / 1e9;
  int regs = 0;
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, block2_kernel<R, TR>) == cudaSuccess) regs = fa.numRegs;
  printf("{\"two_strips\":1,\"R\":%d,\"T\":%d,\"ctas_per_sm\":%d,\"regs\":%d,\"gcups\":%.1f,"
         "\"smsp_cycles_per_warp_cell\":%.2f}\n",
         R, TR, blocks_per_sm, regs, gcups, (sms * 4.0 * clk_khz * 1e3) / (gcups * 1e9 / 32.0));
}

// The same 4 x R cells per step as a rolling parallelogram: slot t works on row
// rho + t at column d - t (d >= t) or finishes row rho - 4 + t at column R + d - t, so
// every anti-diagonal holds exactly 4 independent cells (no fill/drain per step).
template <int R>
__device__ __forceinline__ void pg_step(double (&pv)[R], const double (&yv)[R],
                                        const double (&xc)[4], const double (&xp)[4],
                                        double (&lv)[4], double (&dv)[4], double bl) {
#pragma unroll
  for (int d = 0; d < R; ++d) {
#pragma unroll
    for (int t = 3; t >= 0; --t) {
      const bool cur = d >= t;
      const int c = cur ? d - t : R + d - t;
      double up, dg;
      if (t == 0) {
        up = pv[c];
        dg = c == 0 ? bl : pv[c - 1];
      } else {
        up = lv[t - 1];
        dg = c == 0 ? bl : dv[t - 1];
      }
      const double left = c == 0 ? bl : lv[t];
      const double x = cur ? xc[t] : xp[t];
      const double v = F64::cell(x, yv[c], F64::mn(F64::mn(dg, up), left));
      dv[t] = lv[t];
      lv[t] = v;
      if (t == 3) pv[c] = v;
    }
  }
}

template <int R>
__global__ void __launch_bounds__(128) pg_kernel(const double* in, double* out, int steps) {
  double pv[R], yv[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    yv[r] = in[(r + threadIdx.x) & 63];
    pv[r] = in[(r + 7) & 63] * 1e-3;
  }
  double xs = in[threadIdx.x & 63];
  double xc[4], xp[4], lv[4], dv[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    xc[t] = xs + t;
    xp[t] = xs - t;
    lv[t] = dv[t] = 1e300;
  }
  for (int s = 0; s < steps; ++s) {
    pg_step<R>(pv, yv, xc, xp, lv, dv, 1e300);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      xp[t] = xc[t];
      xc[t] = xc[t] + lv[3] * 1e-12;
    }
  }
  double acc = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) acc += pv[r];
  if (acc == -1.0) out[threadIdx.x] = acc;
}

template <int R>
void run_pg(int sms, int clk_khz, double* in, double* out, int blocks_per_sm) {
  const int steps = 2048;
  const int blocks = sms * blocks_per_sm;
  pg_kernel<R><<<blocks, 128>>>(in, out, steps);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  pg_kernel<R><<<blocks, 128>>>(in, out, steps);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double cells = (double)blocks * 128 * steps * R * 4;
  const double gcups = cells / (ms * 1e-3) / 1e9;
  int regs = 0;
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, pg_kernel<R>) == cudaSuccess) regs = fa.numRegs;
  printf("{\"pg\":1,\"R\":%d,\"T\":4,\"ctas_per_sm\":%d,\"regs\":%d,\"gcups\":%.1f,"
         "\"smsp_cycles_per_warp_cell\":%.2f}\n",
         R, blocks_per_sm, regs, gcups, (sms * 4.0 * clk_khz * 1e3) / (gcups * 1e9 / 32.0));
}

template <int R, int TR>
void run(int sms, int clk_khz, double* in, double* out, int blocks_per_sm) {
  const int steps = 2048;
  const int blocks = sms * blocks_per_sm;
  block_kernel<R, TR><<<blocks, 128>>>(in, out, steps);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  block_kernel<R, TR><<<blocks, 128>>>(in, out, steps);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double cells = (double)blocks * 128 * steps * R * TR;
  const double gcups = cells / (ms * 1e-3) / 1e9;
  int regs = 0;
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, block_kernel<R, TR>) == cudaSuccess) regs = fa.numRegs;
  printf("{\"R\":%d,\"T\":%d,\"ctas_per_sm\":%d,\"regs\":%d,\"gcups\":%.1f,"
         "\"smsp_cycles_per_warp_cell\":%.2f}\n",
         R, TR, blocks_per_sm, regs, gcups, (sms * 4.0 * clk_khz * 1e3) / (gcups * 1e9 / 32.0));
}

int main() {
  double *in, *out;
  cudaMalloc(&in, 64 * sizeof(double));
  cudaMalloc(&out, 1024 * sizeof(double));
  double h[64];
  for (int i = 0; i < 64; ++i) h[i] = 0.01 * i;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  int sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  run<32, 4>(sms, clk_khz, in, out, 2);
  run<32, 2>(sms, clk_khz, in, out, 2);
  run<16, 4>(sms, clk_khz, in, out, 2);
  run<16, 4>(sms, clk_khz, in, out, 3);
  run<24, 4>(sms, clk_khz, in, out, 2);
  run<8, 8>(sms, clk_khz, in, out, 2);
  run<8, 4>(sms, clk_khz, in, out, 4);
  run2<16, 4>(sms, clk_khz, in, out, 2);
  run2<16, 2>(sms, clk_khz, in, out, 2);
  run2<12, 4>(sms, clk_khz, in, out, 2);
  run2<8, 4>(sms, clk_khz, in, out, 2);
  run2<16, 4>(sms, clk_khz, in, out, 3);
  run_pg<32>(sms, clk_khz, in, out, 2);
  run_pg<24>(sms, clk_khz, in, out, 2);
  run_pg<16>(sms, clk_khz, in, out, 2);
  run_pg<16>(sms, clk_khz, in, out, 3);
  return 0;
}
