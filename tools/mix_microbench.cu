// mix_microbench.cu -- which pipe should do the two minima of the fp64 DTW cell?
// NOTE (round 2, session 4): this harness feeds one chain's previous value in as both
// `up` and `left`, so the compiler drops part of the compares/selects, and its V4/V5
// "predicated IMAD" come out as IMAD + SEL; its absolute cycles per cell are too low.
// tools/dispatch_microbench.cu is the corrected measurement.
//
//
// All DTW cell values are +0, positive or +inf doubles (squares and sums of them; no -0,
// no NaN), and such doubles order exactly like their bit patterns as unsigned 64-bit
// integers, with equal bits <=> equal values. So `b < a ? b : a` can be decided by DSETP
// (fp64 pipe) or by a 64-bit integer compare (ISETP lo + ISETP.EX hi, ALU pipe) with a
// bit-identical result. V selects where each of the cell's two compares runs:
//   V0: both DSETP (the fill kernels' body)     V1: min(diag, up) integer, min(., left) DSETP
//   V2: min(diag, up) DSETP, min(., left) int   V3: both integer
//   V4: min(diag, up) as DSETP + 2 predicated IMADs (FMA pipe), min(., left) DSETP + 2 FSEL
//   V5: both as DSETP + predicated IMADs
// Throughput: CH independent chains per thread, W warps per SM; latency: one dependent
// chain. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mix mix_microbench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ double imin(double a, double b) {  // b < a ? b : a, by bits
  const unsigned long long ab = __double_as_longlong(a), bb = __double_as_longlong(b);
  return bb < ab ? b : a;
}
__device__ __forceinline__ double fmin_(double a, double b) { return b < a ? b : a; }

// b < a ? b : a as DSETP + two predicated IMADs by a run-time 1 (FMA pipe instead of the
// ALU's two FSEL; ptxas cannot fold a multiply by an unknown value into a select)
__device__ __forceinline__ double pmin(double a, double b, unsigned one) {
  unsigned alo, ahi;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(alo), "=r"(ahi) : "d"(a));
  unsigned blo, bhi;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(blo), "=r"(bhi) : "d"(b));
  asm("{\n\t.reg .pred p;\n\t"
      "setp.lt.f64 p, %4, %5;\n\t"
      "@p mul.lo.u32 %0, %2, %6;\n\t"
      "@p mul.lo.u32 %1, %3, %6;\n\t}"
      : "+r"(alo), "+r"(ahi)
      : "r"(blo), "r"(bhi), "d"(b), "d"(a), "r"(one));
  double r;
  asm("mov.b64 %0, {%1, %2};" : "=d"(r) : "r"(alo), "r"(ahi));
  return r;
}

template <int V>
__device__ __forceinline__ double cell(double x, double y, double diag, double up, double left,
                                       unsigned one = 1) {
  const double d = __dsub_rn(x, y);
  double m1, m2;
  if constexpr (V >= 4) {
    m1 = pmin(diag, up, one);
    m2 = V == 5 ? pmin(m1, left, one) : fmin_(m1, left);
  } else {
    m1 = (V == 1 || V == 3) ? imin(diag, up) : fmin_(diag, up);
    m2 = (V == 2 || V == 3) ? imin(m1, left) : fmin_(m1, left);
  }
  return __dadd_rn(__dmul_rn(d, d), m2);
}

template <int V, int CH>
__global__ void tput(const double* in, double* out, int iters) {
  const unsigned one = iters > 0 ? 1u : 0u;  // a run-time 1
  double x = in[threadIdx.x & 7], y[CH], a[CH], b[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    y[c] = in[(c + 1) & 7];
    a[c] = in[(c + 2) & 7];
    b[c] = in[(c + 3) & 7];
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const double v = cell<V>(x, y[c], a[c], b[c], y[c], one);
      a[c] = b[c];
      b[c] = v;
      y[c] = v;
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += b[c];
  if (s == -1.0) out[threadIdx.x] = s;
}

template <int V>
__global__ void lat(const double* in, double* out, int iters, long long* clk) {
  double x = in[threadIdx.x & 7], y = in[1], a = in[2], b = in[3], left = in[4];
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    left = cell<V>(x, y, a, b, left);
    y = y + 1.0;
    a = a + 1.0;
    b = b + 2.0;
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) *clk = t1 - t0;
  if (left == -1.0) out[0] = left;
}

template <int V, int CH>
void run_tput(int sms, int clk_khz, double* in, double* out) {
  const int iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {8, 12, 16, 32}) {
    const int blocks = sms * warps / 4;
    tput<V, CH><<<blocks, 128>>>(in, out, iters);
    cudaEventRecord(e0);
    tput<V, CH><<<blocks, 128>>>(in, out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double cells = (double)blocks * 128 * CH * iters;
    const double gcups = cells / (ms * 1e-3) / 1e9;
    printf("{\"variant\":%d,\"chains\":%d,\"warps_per_sm\":%d,\"gcups\":%.1f,"
           "\"smsp_cycles_per_warp_cell\":%.2f}\n",
           V, CH, warps, gcups, (sms * 4.0 * clk_khz * 1e3) / (gcups * 1e9 / 32.0));
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

template <int V>
void run_lat(double* in, double* out, long long* clk) {
  const int iters = 1 << 16;
  lat<V><<<1, 32>>>(in, out, iters, clk);
  lat<V><<<1, 32>>>(in, out, iters, clk);
  long long c = 0;
  cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  printf("{\"variant\":%d,\"chain_cycles_per_cell\":%.2f}\n", V, (double)c / iters);
}

int main() {
  double *in, *out;
  long long* clk;
  cudaMalloc(&in, 64 * sizeof(double));
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMalloc(&clk, 8);
  double h[8] = {1, 2, 3, 4, 5, 6, 7, 8};
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  int sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  run_tput<0, 8>(sms, clk_khz, in, out);
  run_tput<0, 4>(sms, clk_khz, in, out);
  run_tput<4, 4>(sms, clk_khz, in, out);
  run_tput<5, 4>(sms, clk_khz, in, out);
  run_tput<4, 8>(sms, clk_khz, in, out);
  run_tput<5, 8>(sms, clk_khz, in, out);
  run_lat<0>(in, out, clk);
  run_lat<1>(in, out, clk);
  run_lat<2>(in, out, clk);
  run_lat<3>(in, out, clk);
  run_lat<4>(in, out, clk);
  run_lat<5>(in, out, clk);
  return 0;
}
