/*
 * dtwgpu.h -- C-ABI of the B200 DTW distance-matrix fill + k-medoids sweeps.
 *
 * This is the drop-in boundary for the reference's hot path (arXiv 2307.04904,
 * dtwclust). The reference exposes that path only as C++ inline/template
 * functions in namespace dtwclust; these entry points are what
 * an FFI/plugin seam for that path binds. Plain pointers and sizes, no exceptions
 * across the boundary, no torch types. The C++ drop-in with the reference's own
 * signatures sits on top of this in include/dtwgpu/dtwclust_gpu.hpp.
 *
 * Return codes: 0 = OK; 2..14 mirror dtwclust::ErrorCode (errors.hpp:11-25), so a
 * wrapper rethrows the same exception class; >= 100 = CUDA / internal failure
 * (message in dtwg_last_error). Threading: one context per host thread; calls on
 * one context are serialised on its stream.
 *
 * Series are passed packed CSR: series i is samples[offsets[i] .. offsets[i+1]),
 * offsets has p+1 entries. half_width < 0 means WarpWindow::unlimited().
 * The condensed matrix is the reference's layout (distance_matrix.hpp:20-78):
 * p(p-1)/2 doubles, row-major upper triangle, slot(i,j) = i*p - i*(i+1)/2 + j-i-1.
 */
#ifndef DTWGPU_H_
#define DTWGPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes (errors.hpp:11-25) plus device failures. */
enum {
  DTWG_OK = 0,
  DTWG_INVALID_ARGUMENTS = 2,
  DTWG_INVALID_SERIES = 5,
  DTWG_EMPTY_DATASET = 7,
  DTWG_BAND_INFEASIBLE = 8,
  DTWG_K_OUT_OF_RANGE = 10,
  DTWG_DISTANCE_MATRIX_INVALID = 11,
  DTWG_INDEX_OUT_OF_RANGE = 12,
  DTWG_SINGLE_CLUSTER_UNDEFINED = 13,
  DTWG_CUDA_ERROR = 100,
  DTWG_NO_DEVICE = 101,
  DTWG_INTERNAL = 102
};

/* Arithmetic of the fill. FP64 is bit-exact with the reference (dtw.hpp:59-73). */
enum { DTWG_FP64 = 0, DTWG_FP32 = 1 };

typedef struct dtwg_ctx dtwg_ctx;

/* Context: owns device buffers, a stream, the resident series and matrix. */
int dtwg_create(int device, dtwg_ctx** out);
void dtwg_destroy(dtwg_ctx* ctx);
/* One context driving several GPUs from one host thread (the C++ drop-in's default on a
 * multi-GPU node; devices may repeat, e.g. {0, 0} in tests): dtwg_build_matrix gives each
 * device a contiguous, cell-balanced slot range, fills the ranges concurrently and copies
 * each straight into the caller's buffer; dtwg_adopt_condensed places the matrix on every
 * device; dtwg_kmedoids runs contiguous blocks of restarts on the devices concurrently,
 * replays observer calls in restart order and reduces the best restart in restart order
 * with strict < (kmedoids.hpp:182). The other entry points act on the first device. */
int dtwg_create_multi(const int* devices, int n_devices, dtwg_ctx** out);
int dtwg_device_count(const dtwg_ctx* ctx);
/* CUDA devices visible to this process (0 when none). */
int dtwg_visible_devices(void);
const char* dtwg_last_error(const dtwg_ctx* ctx);
/* Pair reported by the last BandInfeasible error (pairwise.hpp:70-79), else -1,-1. */
void dtwg_last_error_pair(const dtwg_ctx* ctx, int64_t* i, int64_t* j);
/* Run on a caller-owned cudaStream_t (e.g. torch.cuda.current_stream()). NULL = own stream. */
int dtwg_set_stream(dtwg_ctx* ctx, void* cuda_stream);
int dtwg_synchronize(dtwg_ctx* ctx);

/*
 * Replaces dtwclust::build_matrix (pairwise.hpp:62-127) end to end, host buffers in
 * and out: validation in the reference's order (EmptyDataset, workers==0,
 * InvalidSeries, first infeasible pair when banded without auto_widen), the fill,
 * and from_condensed's finite/non-negative check (distance_matrix.hpp:27-41).
 * `workers` is validated (>= 1) and otherwise ignored. out_condensed: p(p-1)/2
 * doubles (may be NULL when p < 2). evaluations (may be NULL) = p(p-1)/2
 * (BuildStats, pairwise.hpp:21-23). The filled matrix stays resident on the device
 * for the k-medoids calls below.
 */
int dtwg_build_matrix(dtwg_ctx* ctx, const double* samples, const int64_t* offsets, int64_t p,
                      int64_t half_width, int auto_widen, unsigned workers, int precision,
                      double* out_condensed, uint64_t* evaluations);

/*
 * Lower-level pieces of the same call, for sharded / device-resident use:
 * upload + validate the series (time_series.hpp:24-45, per-series checks only; id
 * uniqueness is the caller's), then fill condensed slots [slot_begin, slot_end)
 * into a DEVICE buffer (slot s written at d_out[s - slot_begin]). d_out == NULL
 * fills the context's resident matrix (allocated for all p(p-1)/2 slots).
 * The band-feasibility error is reported for the first infeasible pair of the
 * whole dataset, as the reference does.
 */
int dtwg_upload_series(dtwg_ctx* ctx, const double* samples, const int64_t* offsets, int64_t p);
int dtwg_fill_slots(dtwg_ctx* ctx, int64_t half_width, int auto_widen, int precision,
                    int64_t slot_begin, int64_t slot_end, double* d_out);
/* In-band DP cells of slots [slot_begin, slot_end) (the GCUPS numerator). */
int dtwg_count_cells(dtwg_ctx* ctx, int64_t half_width, int auto_widen, int64_t slot_begin,
                     int64_t slot_end, uint64_t* cells);
/* Device-event time of the last dtwg_fill_slots / dtwg_build_matrix fill, in ms. */
int dtwg_last_fill_ms(dtwg_ctx* ctx, float* ms);
/* Number of kernels this context has launched so far (bench `gpu_launches`). */
uint64_t dtwg_launch_count(const dtwg_ctx* ctx);
/* Roofline denominator, measured live: cells/s of the bare cell body (5 fp64-pipe ops:
 * sub, mul, two compare-selects, add; or the fp32 body) on every SM with no memory or
 * dependency stalls. */
int dtwg_measure_cell_peak(dtwg_ctx* ctx, int precision, double* cells_per_s);
/* Diagnostics/tests: force kernel family (0 = full with 2 rows per step, 1 = band, 3 = full
 * with 4 rows per step, 4 = band with a shared-memory y ring, 10 + U = ring band with U units
 * per lane, 5 = strip pipeline for long pairs, G = 32, 6 = Full strips with y in shared
 * memory, 4 rows per step) and (G, R) for every pair shape it can legally run;
 * family < 0 restores the cost-model planner. */
int dtwg_force_kernel(dtwg_ctx* ctx, int family, int G, int R);
/* Human-readable plan of the last fill (kernel family, group lanes, cells per lane). */
const char* dtwg_last_plan(const dtwg_ctx* ctx);

/*
 * Adopt a condensed matrix as the resident k-medoids source (DistanceMatrix::
 * from_condensed, distance_matrix.hpp:27-41: entries must be finite and >= 0).
 * on_device != 0: `condensed` is a device pointer (e.g. the all-gathered result).
 */
int dtwg_adopt_condensed(dtwg_ctx* ctx, const double* condensed, int64_t p, int on_device);
/* Copy the resident condensed matrix to host memory (p(p-1)/2 doubles). */
int dtwg_download_condensed(dtwg_ctx* ctx, double* out_condensed);
/* Copy slots [slot_begin, slot_end) of the resident (or, during a fused exchange, the
 * rank's own exchange) matrix to host memory -- a rank's own slice after its fill. */
int dtwg_download_range(dtwg_ctx* ctx, int64_t slot_begin, int64_t slot_end, double* out);

typedef void (*dtwg_observer_fn)(void* user, int64_t restart, int64_t iteration, double cost);

/*
 * Replaces dtwclust::kmedoids (kmedoids.hpp:148-189) over the resident matrix.
 * Restarts [restart_begin, restart_end) of a run with `restarts` total are executed
 * (restart_stream(seed, r), rng.hpp:37-41), so restarts can be sharded over GPUs;
 * pass 0, restarts for the whole run. The best restart (strict <, earliest wins,
 * kmedoids.hpp:182) is returned: medoids_out[k] ascending, assignment_out[p],
 * *cost_out, *best_restart_out. Errors: KOutOfRange (k<1 || k>p), InvalidArguments
 * (restarts < 1 || max_iterations < 1) -- kmedoids.hpp:152-154.
 */
int dtwg_kmedoids(dtwg_ctx* ctx, int64_t k, int64_t restarts, int64_t max_iterations,
                  uint64_t seed, int64_t restart_begin, int64_t restart_end,
                  dtwg_observer_fn observer, void* user, int64_t* medoids_out,
                  int64_t* assignment_out, double* cost_out, int64_t* best_restart_out);

/* k-medoids sweep statistics since the last reset (out: 8 doubles): out[0] sweeps,
 * out[1] assignment kernel ms, out[2] its algorithmic bytes (8 per distance read), out[3]
 * update kernels ms (device bucketing + candidate sums + selection), out[4] their
 * algorithmic bytes (8 * sum |C|^2 + index traffic), out[5] ms spent preparing the sweep
 * views (square expansion), out[6] 1 if the cluster-ordered copy is in use (2: as fp32), out[7] its
 * build time in ms (device; it overlaps the seeding). With concurrent restart workers the
 * per-sweep times overlap each other. */
int dtwg_km_stats(dtwg_ctx* ctx, double* out, int reset);

/*
 * Replaces dtwclust::silhouette_scores (validation.hpp:30-79) over the resident matrix:
 * silhouette_out[p] per series and *mean_out, bit-identical to the reference (same
 * ascending-member summation order). Errors: InvalidArguments (p_assign != p, or a series
 * assigned to a non-medoid), 13 = SingleClusterUndefined (k < 2).
 */
int dtwg_silhouette(dtwg_ctx* ctx, const int64_t* medoids, int64_t k, const int64_t* assignment,
                    int64_t p_assign, double* silhouette_out, double* mean_out);

/* One sweep's pieces (cluster_result.hpp:40-72; kmedoids.hpp:48-52, 84-139). */
int dtwg_km_nearest_update(dtwg_ctx* ctx, int64_t current, const uint8_t* chosen,
                           double* nearest_inout);
int dtwg_km_assign(dtwg_ctx* ctx, const int64_t* medoids, int64_t k, int64_t* assignment_out,
                   double* dist_to_assigned_out);
int dtwg_km_update(dtwg_ctx* ctx, const int64_t* medoids, int64_t k, const int64_t* assignment,
                   int64_t* updated_out);

/* ---- fused fill + all-gather over peer memory (one process per GPU, NVLink/NVSwitch) ----
 * Replaces the fill-then-NCCL-all-gather of a sharded build: every rank exports its
 * resident matrix buffer (sized for p series), opens every other rank's through CUDA IPC,
 * and fills its own slot range; the fill kernels store each distance into ALL ranks'
 * buffers (st.global to peer-mapped addresses), so the exchange overlaps the fill tile by
 * tile and no collective follows. After every rank's dtwg_exchange_fill has returned
 * (host barrier), dtwg_exchange_complete validates the matrix and makes it resident for
 * k-medoids. Handles are 64 bytes per rank (cudaIpcMemHandle_t), handles[r] for rank r.
 */
int dtwg_exchange_export(dtwg_ctx* ctx, int64_t p, unsigned char* handle_out);
int dtwg_exchange_open(dtwg_ctx* ctx, const unsigned char* handles, int n_ranks, int my_rank);
int dtwg_exchange_fill(dtwg_ctx* ctx, int64_t half_width, int auto_widen, int precision,
                       int64_t slot_begin, int64_t slot_end);
int dtwg_exchange_complete(dtwg_ctx* ctx);
int dtwg_exchange_close(dtwg_ctx* ctx);

/* ---- host-side data path either side of the fill ------------
 * No device or context needed. Errors: the dtwclust::ErrorCode values (3 IoFailure,
 * 4 ParseFailure, 5 InvalidSeries, 6 EmptySeries, 7 EmptyDataset, 9 FormatViolation,
 * 11 DistanceMatrixInvalid); message, line and column of the last error on this thread
 * from dtwg_io_last_error (line/column -1 when not applicable), the file (ParseFailure,
 * EmptySeries) or series id (InvalidSeries) from dtwg_io_last_file. `threads` <= 0 uses
 * every core. Buffers returned through double** are released with dtwg_free.
 */
const char* dtwg_io_last_error(int64_t* line, int64_t* column);
const char* dtwg_io_last_file(void);
void dtwg_free(void* ptr);

/* Replaces dtwclust::save_matrix (distance_matrix.hpp:104-122): the same text format,
 * byte for byte, with rows formatted by several threads. */
int dtwg_save_matrix_text(const double* condensed, int64_t p, const char* path, int threads);
/* Replaces dtwclust::load_matrix (distance_matrix.hpp:127-192): same checks, same first
 * error (FormatViolation with its line); rows parsed by several threads. */
int dtwg_load_matrix_text(const char* path, int threads, int64_t* p_out, double** condensed_out);
/* Binary sidecar: "DTWGMAT1", uint64 p, the p(p-1)/2 condensed doubles (little-endian);
 * loading validates like DistanceMatrix::from_condensed (distance_matrix.hpp:27-41). */
int dtwg_save_matrix_binary(const double* condensed, int64_t p, const char* path);
int dtwg_load_matrix_binary(const char* path, int64_t* p_out, double** condensed_out);

/* Replaces dtwclust::ingest (csv.hpp:55-106): one series per row of each file, in file
 * order; label_column drops each row's first cell; delimiter 0 = ',' (tab for .tsv).
 * The packed result (samples + offsets[p+1] + ids "<file name>:<row>") is what
 * dtwg_build_matrix / dtwg_upload_series take. */
typedef struct dtwg_dataset dtwg_dataset;
int dtwg_ingest_csv(const char* const* paths, int64_t npaths, int label_column, int delimiter,
                    int threads, dtwg_dataset** out);
int64_t dtwg_dataset_size(const dtwg_dataset* ds);
double* dtwg_dataset_samples(dtwg_dataset* ds);
const int64_t* dtwg_dataset_offsets(const dtwg_dataset* ds);
const char* dtwg_dataset_id(const dtwg_dataset* ds, int64_t i);
void dtwg_dataset_free(dtwg_dataset* ds);
/* runner.hpp:82-95 in place, per series in parallel (bit-identical: sequential sums). */
int dtwg_z_normalize(double* samples, const int64_t* offsets, int64_t p, int threads);

#ifdef __cplusplus
}
#endif

#endif /* DTWGPU_H_ */
