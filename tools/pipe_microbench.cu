// pipe_microbench.cu -- sm_100a throughput of the instruction mixes in the DTW cell, in
// warp-instructions (or cells) per SM-clock, many independent chains per thread.
//   dadd     : DADD only                       (fp64 pipe)
//   dsetp    : DSETP + 2 FSEL (one fp64 min)    (fp64 pipe + ALU)
//   fsel     : FSEL only                        (ALU)
//   cell     : the fp64 cell body               (5 fp64 + 4 FSEL)
//   cell_lds : cell body + one LDS.64 per cell  (as the ring kernels)
//   cell_int : cell with both mins done on the integer pipe (non-negative doubles order
//              like their int64 bit patterns): 3 fp64 + 4 ISETP + 4 SEL
//   cell_mix : one min on the integer pipe, one DSETP: 4 fp64 + 2 ISETP + 4 SEL
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_microbench pipe_microbench.cu
#include <cuda_runtime.h>

#include <cstdio>

constexpr int CH = 8;

__device__ __forceinline__ double imin(double a, double b) {
  const long long x = __double_as_longlong(a), y = __double_as_longlong(b);
  return __longlong_as_double(y < x ? y : x);
}

template <int MODE>
__global__ void bench(const double* in, double* out, int iters) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = in[i & 7];
  __syncthreads();
  double x = in[threadIdx.x & 7], y[CH], a[CH], b[CH];
  unsigned fa[CH], fb[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    y[c] = in[(c + 1) & 7];
    a[c] = in[(c + 2) & 7];
    b[c] = in[(c + 3) & 7];
    fa[c] = (unsigned)c;
    fb[c] = (unsigned)(c * 7);
  }
  int p = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if constexpr (MODE == 0) {
        a[c] = __dadd_rn(a[c], x);
      } else if constexpr (MODE == 1) {
        a[c] = b[c] < a[c] ? b[c] : a[c];
        b[c] = __longlong_as_double(__double_as_longlong(b[c]) ^ 1);  // keep it alive (ALU)
      } else if constexpr (MODE == 2) {
        const bool pr = (fa[c] & 1u) != 0u;
        const unsigned t = pr ? fa[c] : fb[c];
        fb[c] = pr ? fb[c] : fa[c];
        fa[c] = t;
      } else {
        double yy = y[c];
        if constexpr (MODE == 4) yy = sm[(p + c * 33) & 1023];
        const double d = __dsub_rn(x, yy);
        double m;
        if constexpr (MODE == 5) m = imin(imin(a[c], b[c]), y[c]);
        else if constexpr (MODE == 6) {
          const double m1 = imin(a[c], b[c]);
          m = y[c] < m1 ? y[c] : m1;
        }
        else {
          const double m1 = b[c] < a[c] ? b[c] : a[c];
          m = y[c] < m1 ? y[c] : m1;
        }
        const double v = __dadd_rn(__dmul_rn(d, d), m);
        a[c] = b[c];
        b[c] = v;
        y[c] = v;
      }
    }
    if constexpr (MODE == 4) p += 1;
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += a[c] + b[c] + (double)(fa[c] + fb[c]);
  if (s == -1.0) out[threadIdx.x] = s;
}

template <int MODE>
void run(const char* name, double per_iter_units, const char* unit) {
  double* in;
  double* out;
  cudaMalloc(&in, 64 * sizeof(double));
  cudaMalloc(&out, 1024 * sizeof(double));
  double h[8] = {1, 2, 3, 4, 5, 6, 7, 8};
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {8, 16, 32}) {
    const int blocks = sms * warps / 4;
    bench<MODE><<<blocks, 128>>>(in, out, iters);
    cudaEventRecord(e0);
    bench<MODE><<<blocks, 128>>>(in, out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warp_units = (double)blocks * 4 * CH * iters * per_iter_units;
    const double per_sm_clk = warp_units / (ms * 1e-3) / (sms * (clk * 1e3));
    printf("{\"mode\":\"%s\",\"warps_per_sm\":%d,\"%s_per_sm_clk\":%.3f,\"ms\":%.3f}\n", name,
           warps, unit, per_sm_clk, ms);
  }
}

int main() {
  run<0>("dadd", 1, "warp_inst");
  run<1>("dsetp_min", 1, "warp_min");
  run<2>("fsel_x2", 2, "warp_sel");
  run<3>("cell", 1, "warp_cell");
  run<4>("cell_lds", 1, "warp_cell");
  run<5>("cell_int", 1, "warp_cell");
  run<6>("cell_mix", 1, "warp_cell");
  return 0;
}
