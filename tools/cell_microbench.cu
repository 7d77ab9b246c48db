// cell_microbench.cu -- measures the sm_100a ceiling of the DTW cell update itself.
// NOTE (round 2, session 4): the throughput kernels here feed one chain's previous value
// in as both `up` and `left`, which lets the compiler drop part of the compares/selects
// (their ~3045-3080 GCUPS overstates the fp64 cell; the chain latency figures stand).
// tools/dispatch_microbench.cu and csrc/peak.cu are the corrected measurements.
//
// Each thread runs CH independent chains of the exact fp64 cell body used by the fill
//   v = (x - y)^2 + min(min(diag, up), left)     (DADD, DMUL, 2x DSETP+2 FSEL, DADD)
// (and the fp32 body FADD, FMUL, FMNMX3, FADD), so the result is the issue/pipe-bound
// peak in cells per SM-clock, independent of memory and of the wavefront. Reported as
// GCUPS at the measured SM clock; compare with the 148*64*f/5 fp64 estimate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cell_microbench cell_microbench.cu
#include <cuda_runtime.h>

#include <cstdio>

template <int CH, class T>
__global__ void cells(const T* in, T* out, int iters) {
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
      T d, v;
      if constexpr (sizeof(T) == 8) {
        d = __dsub_rn(x, y[c]);
        const T m1 = b[c] < a[c] ? b[c] : a[c];
        const T m2 = y[c] < m1 ? y[c] : m1;
        v = __dadd_rn(__dmul_rn(d, d), m2);
      } else {
        d = __fsub_rn(x, y[c]);
        v = __fadd_rn(__fmul_rn(d, d), fminf(fminf(a[c], b[c]), y[c]));
      }
      a[c] = b[c];
      b[c] = v;
      y[c] = v;  // keep the chain dependent like cur[j-1]
    }
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += b[c];
  if (s == (T)-1) out[threadIdx.x] = s;
}

template <class T>
void run(const char* name) {
  T* in;
  T* out;
  cudaMalloc(&in, 64 * sizeof(T));
  cudaMalloc(&out, 1024 * sizeof(T));
  T h[8] = {1, 2, 3, 4, 5, 6, 7, 8};
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    const int blocks = sms * warps / 4;
    cells<8, T><<<blocks, 128>>>(in, out, iters);
    cudaEventRecord(e0);
    cells<8, T><<<blocks, 128>>>(in, out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double cellsn = (double)blocks * 128 * 8 * iters;
    const double gcups = cellsn / (ms * 1e-3) / 1e9;
    printf("{\"body\":\"%s\",\"warps_per_sm\":%d,\"gcups\":%.1f,\"cells_per_sm_clk_at_max\":%.2f}\n",
           name, warps, gcups, gcups * 1e9 / (sms * (clk * 1e3)));
  }
  cudaFree(in);
  cudaFree(out);
}

// Latency of one dependent cell chain (1 warp per SM, 1 chain per thread), in SM clocks.
template <class T>
__global__ void chain_lat(const T* in, T* out, int iters, long long* clk) {
  // The DTW left-chain: v_j = (x - y_j)^2 + min(min(d_j, u_j), v_{j-1}); only v_{j-1}
  // is loop-carried, as in the fill (d/u come from the previous row).
  T x = in[threadIdx.x & 7], y = in[1], a = in[2], b = in[3], left = in[4];
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    T d, v;
    if constexpr (sizeof(T) == 8) {
      d = __dsub_rn(x, y);
      const T m1 = b < a ? b : a;
      const T m2 = left < m1 ? left : m1;
      v = __dadd_rn(__dmul_rn(d, d), m2);
    } else {
      d = __fsub_rn(x, y);
      v = __fadd_rn(__fmul_rn(d, d), fminf(fminf(a, b), left));
    }
    left = v;
    y = y + (T)1;
    a = a + (T)1;
    b = b + (T)2;
  }
  const T b_out = left;
  const long long t1 = clock64();
  if (threadIdx.x == 0) *clk = t1 - t0;
  if (b_out == (T)-1) out[0] = b_out;
}

template <class T>
void lat(const char* name) {
  T* in;
  T* out;
  long long* clk;
  cudaMalloc(&in, 64 * sizeof(T));
  cudaMalloc(&out, 64 * sizeof(T));
  cudaMalloc(&clk, 8);
  T h[8] = {1, 2, 3, 4, 5, 6, 7, 8};
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  const int iters = 1 << 16;
  chain_lat<T><<<1, 32>>>(in, out, iters, clk);
  chain_lat<T><<<1, 32>>>(in, out, iters, clk);
  long long c = 0;
  cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  // the chain here runs through y = v: sub -> mul -> add plus the min chain
  printf("{\"body\":\"%s\",\"chain_cycles_per_cell\":%.2f}\n", name, (double)c / iters);
}

int main() {
  run<double>("fp64");
  run<float>("fp32");
  lat<double>("fp64");
  lat<float>("fp32");
  return 0;
}
