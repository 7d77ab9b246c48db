// dtw_fill.cuh -- shared declarations of the sm_100a DTW fill kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dtwgpu {

// Work description for one fill launch. Pairs are condensed slots (row-major upper
// triangle, pairwise.hpp:36-53); either the contiguous range [begin, begin+count) or
// the explicit slot list list[0..count).
struct FillArgs {
  const double* samples;   // packed series, fp64
  const float* samples32;  // same series rounded to fp32 (precision == fp32 only)
  const int64_t* offsets;  // p + 1
  int64_t p;
  int64_t half_width;      // < 0: unlimited
  int auto_widen;
  const int64_t* list;     // nullptr: range mode
  int64_t begin;
  int64_t count;
  int64_t out_base;        // out[slot - out_base]
  double* out;
  double* scratch;         // boundary columns for multi-pass fills (one per group)
  int64_t scratch_stride;  // doubles per group
  // Readable sample indices relative to samples/samples32 (the zero guards included);
  // checked by DTWG_CHECK_BOUNDS builds (tools/bounds_check.sh).
  int64_t guard_lo, guard_hi;
  // Band family: the same series, each surrounded by kBandPad +inf samples, so band
  // columns outside [1, m] (and rows outside [1, n]) load +inf without a range check.
  const double* bsamples;
  const float* bsamples32;
  const int64_t* boffsets;  // start of series i inside bsamples
  // Strip family (long pairs; column strips of one pair pipelined over many warps):
  const int64_t* strip_base;     // count + 1 prefix sums of strips per pair (nullptr: uniform)
  int strips_per_pair;           // uniform mode
  unsigned long long* work;      // item counter (zeroed before the launch)
  int* prog;                     // per strip item: last row published (zeroed before the launch)
  double* cols;                  // two boundary columns per pair, col_stride doubles each
  int64_t col_stride;
  // Fused exchange: every result is also stored to peer_out[r][slot - peer_base]
  static constexpr int kMaxPeers = 7;
  double* peer_out[kMaxPeers];
  int n_peer;
  int64_t peer_base;
};

constexpr int kBandPad = 1024;  // >= hw + G + G*R (+3 ring chunks) for every band instantiation

enum class Family : int { Full = 0, Band = 1, Strip = 2 };

// One kernel configuration: family, lanes per pair (G), DP cells per lane per row (R),
// and whether per-cell band masking may be needed (Full family only).
struct KernelCfg {
  Family family;
  int G;
  int R;
  bool mask;
  bool fp32;
  int kr = -1;  // Band family: (2hw+1) % R when every pair of the launch shares it, else -1
  int P = 1;    // Band family: pairs per lane group (independent chains per lane)
  int TR = 2;   // Full family: rows per step (independent chains per lane)
  bool ring = false;  // Band family: y window in a shared-memory ring instead of registers
  int U = 1;          // ring variant: units per lane (independent cell chains per lane)
  bool mp = true;     // Full family: some pair needs several strips (boundary column)
  bool ysm = false;   // Full family: y in shared memory (dtw_full1s_kernel)
};

// Launches cfg over args on stream with `blocks` CTAs of kThreads threads.
cudaError_t launch_fill(const KernelCfg& cfg, const FillArgs& args, int blocks,
                        cudaStream_t stream);
// CTAs per SM the configuration can keep resident.
int fill_blocks_per_sm(const KernelCfg& cfg);
// Whether (family, G, R, fp32) has a compiled instantiation.
bool fill_cfg_supported(const KernelCfg& cfg);

constexpr int kThreads = 128;

// ---- cell-body ceiling (peak.cu) -------------------------------------------------
cudaError_t measure_cell_peak(cudaStream_t st, int sms, bool fp32, double* cells_per_s);

// ---- k-medoids sweep kernels (kmedoids.cu) -------------------------------------
// The sweep kernels read the dense square (condensed = false) or the condensed matrix.
cudaError_t launch_silhouette(const double* matrix, bool condensed, int64_t p,
                              const int32_t* members, const int64_t* cluster_begin,
                              const int32_t* cls, int64_t k, double* sil, cudaStream_t s);
cudaError_t launch_to_f32(const double* in, int64_t n, float* out, cudaStream_t s);
cudaError_t launch_band_pad(const double* samples, const int64_t* off, const int64_t* boff,
                            int64_t p, int64_t pad, void* out, bool fp32, cudaStream_t s);
cudaError_t launch_expand_square(const double* condensed, int64_t p, double* square,
                                 cudaStream_t s);
cudaError_t launch_validate_condensed(const double* condensed, int64_t total, int* flags,
                                      cudaStream_t s);
cudaError_t launch_nearest_update(const double* matrix, bool condensed, int64_t p,
                                  int64_t current, const uint8_t* chosen, double* nearest,
                                  cudaStream_t s);
cudaError_t launch_assign(const double* matrix, bool condensed, int64_t p,
                          const int64_t* medoids, int64_t k, int64_t* assignment, double* dist,
                          cudaStream_t s);
cudaError_t launch_update(const double* matrix, bool condensed, int64_t p,
                          const int32_t* members, const int64_t* cluster_begin, int64_t k,
                          int64_t* best_member, double* best_sum, cudaStream_t s);
// round 2: device-side bucketing, slot-writing assignment, cluster-ordered square
cudaError_t launch_assign_slots(const double* matrix, bool condensed, int64_t p,
                                const int64_t* medoids, int64_t k, int64_t* assignment,
                                double* dist, int32_t* lab, cudaStream_t s,
                                int32_t* counts = nullptr);
cudaError_t launch_slots_of(const double* matrix, bool condensed, int64_t p,
                            const int64_t* medoids, int64_t k, const int64_t* assignment,
                            double* dist, int32_t* lab, cudaStream_t s);
cudaError_t launch_seed_step(const double* matrix, bool condensed, int64_t p, int64_t current,
                             uint8_t* chosen, double* nearest, cudaStream_t s);
size_t bucket_temp_bytes(int64_t p);
cudaError_t launch_iota(int32_t* out, int64_t n, cudaStream_t s);
cudaError_t launch_fill_inf(double* out, int64_t n, cudaStream_t s);
cudaError_t launch_bucket(const int32_t* lab, const int32_t* perm, const int32_t* iota, int64_t p,
                          int64_t k, int32_t* keys_a, int32_t* keys_b, int32_t* members,
                          int32_t* members_perm, int64_t* cb, void* tmp, size_t tmp_bytes,
                          cudaStream_t s, bool counted = false);
cudaError_t launch_update2(const double* matrix, bool condensed, const void* psq, bool psq32,
                           const int32_t* pinv, int64_t p, const int32_t* members,
                           const int32_t* members_perm, const int64_t* cluster_begin,
                           int64_t k, int64_t* best_member, double* best_sum, cudaStream_t s);
cudaError_t launch_cluster_layout(const double* sq, int64_t p, int n_anchor, const int64_t* anchors,
                                  int64_t* asg_tmp, double* dist_tmp, int32_t* lab,
                                  int32_t* keys_tmp, const int32_t* iota, int32_t* perm,
                                  int32_t* pinv, void* psq, bool psq32, void* tmp,
                                  size_t tmp_bytes, int num_sms, cudaStream_t s);

}  // namespace dtwgpu
