// dtwclust_gpu.hpp -- C++ drop-in for the reference's hot path, on top of include/dtwgpu.h.
//
// Include it after the reference's own headers (it uses dtwclust's types, unchanged) and
// replace
//     dtwclust::build_matrix(dataset, window, workers, &stats, auto_widen)   // pairwise.hpp:62
//     dtwclust::dtw_distance(x, y, window)                                   // dtw.hpp:40
//     dtwclust::kmedoids(matrix, config, observer)                           // kmedoids.hpp:148
//     dtwclust::silhouette_scores(matrix, result)                            // validation.hpp:30
//     dtwclust::LazyDistanceSource(dataset, window, auto_widen)              // pairwise.hpp:133
//     dtwclust::save_matrix / load_matrix                                    // distance_matrix.hpp:104
//     dtwclust::ingest(paths, format), detail::z_normalize(dataset)          // csv.hpp:55, runner.hpp:82
// by the same calls in namespace dtwgpu. Signatures, results (bit-identical matrices,
// identical ClusterResult) and thrown exception types follow the reference; the work runs
// on the B200 through the C-ABI. Host-side types, data loading, the exact (MIP) solver
// and the scores keep consuming the returned dtwclust::DistanceMatrix unchanged.
//
// Threading: one device context per host thread (thread_local), as the C-ABI requires;
// it drives every visible GPU (or DTWGPU_DEVICES) -- see default_devices().
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <filesystem>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <dtwclust/cluster_result.hpp>
#include <dtwclust/csv.hpp>
#include <dtwclust/distance_matrix.hpp>
#include <dtwclust/errors.hpp>
#include <dtwclust/kmedoids.hpp>
#include <dtwclust/pairwise.hpp>
#include <dtwclust/time_series.hpp>
#include <dtwclust/validation.hpp>
#include <dtwclust/warp_window.hpp>

#include "../dtwgpu.h"

namespace dtwgpu {

class DeviceError : public std::runtime_error {
 public:
  DeviceError(int code, const std::string& what)
      : std::runtime_error("dtwgpu [code " + std::to_string(code) + "]: " + what), code_(code) {}
  int code() const noexcept { return code_; }

 private:
  int code_;
};

/// RAII owner of one dtwg_ctx on `device`, or on several devices (dtwg_create_multi).
class Context {
 public:
  explicit Context(int device = 0) {
    const int rc = dtwg_create(device, &ctx_);
    if (rc != DTWG_OK) throw DeviceError(rc, "no CUDA device available (there is no CPU fallback)");
  }
  explicit Context(const std::vector<int>& devices) {
    const int rc = devices.empty()
                       ? DTWG_NO_DEVICE
                       : dtwg_create_multi(devices.data(), static_cast<int>(devices.size()), &ctx_);
    if (rc != DTWG_OK) throw DeviceError(rc, "no CUDA device available (there is no CPU fallback)");
  }
  ~Context() { dtwg_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  dtwg_ctx* get() const noexcept { return ctx_; }

 private:
  dtwg_ctx* ctx_ = nullptr;
};

/// Devices the drop-in uses: DTWGPU_DEVICES ("0,1,2,3"; repeats allowed) or every
/// visible GPU -- build_matrix splits the slots over them, kmedoids the restarts.
inline std::vector<int> default_devices() {
  std::vector<int> devs;
  if (const char* env = std::getenv("DTWGPU_DEVICES")) {
    std::string cur;
    for (const char* c = env;; ++c) {
      if (*c == ',' || *c == 0) {
        if (!cur.empty()) devs.push_back(std::stoi(cur));
        cur.clear();
        if (*c == 0) break;
      } else {
        cur += *c;
      }
    }
  }
  if (devs.empty())
    for (int d = 0; d < std::max(1, dtwg_visible_devices()); ++d) devs.push_back(d);
  return devs;
}

inline Context& thread_context() {
  thread_local std::unique_ptr<Context> ctx;
  if (!ctx) ctx = std::make_unique<Context>(default_devices());
  return *ctx;
}

namespace detail {

/// Rethrows a C-ABI error code as the reference's exception class (errors.hpp:11-176).
[[noreturn]] inline void rethrow(dtwg_ctx* ctx, int rc, const std::vector<dtwclust::TimeSeries>* ds,
                                 std::int64_t hw) {
  const std::string msg = dtwg_last_error(ctx);
  switch (rc) {
    case DTWG_INVALID_ARGUMENTS:
      throw dtwclust::InvalidArgumentsError(msg);
    case DTWG_EMPTY_DATASET:
      throw dtwclust::EmptyDatasetError();
    case DTWG_INVALID_SERIES:
      throw dtwclust::InvalidSeriesError("?", msg);
    case DTWG_BAND_INFEASIBLE: {
      std::int64_t i = -1, j = -1;
      dtwg_last_error_pair(ctx, &i, &j);
      if (ds && i >= 0 && j >= 0) {
        const auto& a = (*ds)[static_cast<std::size_t>(i)];
        const auto& b = (*ds)[static_cast<std::size_t>(j)];
        throw dtwclust::BandInfeasibleError(
            static_cast<std::size_t>(i), static_cast<std::size_t>(j),
            dtwclust::BandInfeasibleError(a.length(), b.length(), static_cast<std::size_t>(hw)));
      }
      throw DeviceError(rc, msg);
    }
    case DTWG_DISTANCE_MATRIX_INVALID:
      throw dtwclust::DistanceMatrixInvalidError(msg);
    case DTWG_SINGLE_CLUSTER_UNDEFINED:
      throw dtwclust::SingleClusterUndefinedError();
    default:
      throw DeviceError(rc, msg);
  }
}

}  // namespace detail

/// pairwise.hpp:62-127 on the GPU: same signature, same validation order, bit-identical
/// condensed matrix (fp64), BuildStats::evaluations = p(p-1)/2.
inline dtwclust::DistanceMatrix build_matrix(const std::vector<dtwclust::TimeSeries>& dataset,
                                             const dtwclust::WarpWindow& w, unsigned workers,
                                             dtwclust::BuildStats* stats = nullptr,
                                             bool auto_widen = false) {
  if (dataset.empty()) throw dtwclust::EmptyDatasetError();
  if (workers == 0) throw dtwclust::InvalidArgumentsError("workers must be >= 1");
  dtwclust::validate_dataset(dataset);  // the reference's own checks, ids included

  const std::size_t p = dataset.size();
  std::vector<std::int64_t> offsets(p + 1, 0);
  for (std::size_t i = 0; i < p; ++i)
    offsets[i + 1] = offsets[i] + static_cast<std::int64_t>(dataset[i].length());
  std::vector<double> samples(static_cast<std::size_t>(offsets[p]));
  for (std::size_t i = 0; i < p; ++i)
    std::copy(dataset[i].samples.begin(), dataset[i].samples.end(),
              samples.begin() + offsets[i]);

  const std::int64_t hw = w.is_unlimited() ? -1 : static_cast<std::int64_t>(w.half_width());
  std::vector<double> values(dtwclust::DistanceMatrix::condensed_size(p));
  std::uint64_t evaluations = 0;
  dtwg_ctx* ctx = thread_context().get();
  const int rc = dtwg_build_matrix(ctx, samples.data(), offsets.data(),
                                   static_cast<std::int64_t>(p), hw, auto_widen ? 1 : 0, workers,
                                   DTWG_FP64, values.empty() ? nullptr : values.data(),
                                   &evaluations);
  if (rc != DTWG_OK) detail::rethrow(ctx, rc, &dataset, hw);
  if (stats) stats->evaluations = evaluations;
  return dtwclust::DistanceMatrix::from_condensed(p, std::move(values));
}

/// dtw.hpp:40-75 for one pair on the GPU: the same checks (validate both series, then the
/// band's feasibility -> BandInfeasibleError(n, m, hw)) and a bit-identical distance. Worth
/// it for long series: a single 1e5-sample pair runs on every SM through the strip
/// pipeline (38 ms against ~30 s on one CPU core).
inline double dtw_distance(const dtwclust::TimeSeries& x, const dtwclust::TimeSeries& y,
                           const dtwclust::WarpWindow& w) {
  dtwclust::validate(x);
  dtwclust::validate(y);
  if (!w.feasible_for(x.length(), y.length()))
    throw dtwclust::BandInfeasibleError(x.length(), y.length(), w.half_width());
  std::vector<double> samples(x.samples);
  samples.insert(samples.end(), y.samples.begin(), y.samples.end());
  const std::int64_t offsets[3] = {0, static_cast<std::int64_t>(x.length()),
                                   static_cast<std::int64_t>(x.length() + y.length())};
  const std::int64_t hw = w.is_unlimited() ? -1 : static_cast<std::int64_t>(w.half_width());
  double d = 0.0;
  dtwg_ctx* ctx = thread_context().get();
  const int rc = dtwg_build_matrix(ctx, samples.data(), offsets, 2, hw, 0, 1, DTWG_FP64, &d,
                                   nullptr);
  if (rc != DTWG_OK) detail::rethrow(ctx, rc, nullptr, hw);
  return d;
}

/// kmedoids.hpp:148-189 over a DistanceMatrix, sweeps on the GPU: identical medoids,
/// assignment, total_cost and observer trace.
inline dtwclust::ClusterResult kmedoids(const dtwclust::DistanceMatrix& source,
                                        const dtwclust::KMedoidsConfig& config,
                                        const dtwclust::IterationObserver& observer = {}) {
  const std::size_t p = source.size();
  if (config.k < 1 || config.k > p) throw dtwclust::KOutOfRangeError(config.k, p);
  if (config.restarts < 1) throw dtwclust::InvalidArgumentsError("restarts must be >= 1");
  if (config.max_iterations < 1)
    throw dtwclust::InvalidArgumentsError("max_iterations must be >= 1");
  dtwg_ctx* ctx = thread_context().get();
  const auto& cond = source.condensed();
  int rc = dtwg_adopt_condensed(ctx, cond.empty() ? nullptr : cond.data(),
                                static_cast<std::int64_t>(p), 0);
  if (rc != DTWG_OK) detail::rethrow(ctx, rc, nullptr, 0);

  struct Trampoline {
    static void call(void* user, std::int64_t r, std::int64_t it, double cost) {
      (*static_cast<const dtwclust::IterationObserver*>(user))(static_cast<std::size_t>(r),
                                                               static_cast<std::size_t>(it), cost);
    }
  };
  std::vector<std::int64_t> medoids(config.k), assignment(p);
  double cost = 0.0;
  std::int64_t best_restart = -1;
  rc = dtwg_kmedoids(ctx, static_cast<std::int64_t>(config.k),
                     static_cast<std::int64_t>(config.restarts),
                     static_cast<std::int64_t>(config.max_iterations), config.seed, 0,
                     static_cast<std::int64_t>(config.restarts),
                     observer ? &Trampoline::call : nullptr,
                     const_cast<dtwclust::IterationObserver*>(&observer), medoids.data(),
                     assignment.data(), &cost, &best_restart);
  if (rc != DTWG_OK) detail::rethrow(ctx, rc, nullptr, 0);
  dtwclust::ClusterResult result;
  result.medoids.assign(medoids.begin(), medoids.end());
  result.assignment.assign(assignment.begin(), assignment.end());
  result.total_cost = cost;
  result.certificate = dtwclust::Certificate::LocalHeuristic;
  return result;
}

/// validation.hpp:30-79 on the GPU: per-series silhouettes and their mean, bit-identical.
inline dtwclust::ScoreReport silhouette_scores(const dtwclust::DistanceMatrix& distances,
                                               const dtwclust::ClusterResult& result) {
  const std::size_t p = distances.size();
  if (result.assignment.size() != p) {
    throw dtwclust::InvalidArgumentsError("clustering covers " +
                                          std::to_string(result.assignment.size()) +
                                          " series, matrix has " + std::to_string(p));
  }
  if (result.medoids.size() < 2) throw dtwclust::SingleClusterUndefinedError();
  dtwg_ctx* ctx = thread_context().get();
  const auto& cond = distances.condensed();
  int rc = dtwg_adopt_condensed(ctx, cond.empty() ? nullptr : cond.data(),
                                static_cast<std::int64_t>(p), 0);
  if (rc != DTWG_OK) detail::rethrow(ctx, rc, nullptr, 0);
  std::vector<std::int64_t> med(result.medoids.begin(), result.medoids.end());
  std::vector<std::int64_t> asg(result.assignment.begin(), result.assignment.end());
  dtwclust::ScoreReport report;
  report.silhouette.resize(p);
  rc = dtwg_silhouette(ctx, med.data(), static_cast<std::int64_t>(med.size()), asg.data(),
                       static_cast<std::int64_t>(asg.size()), report.silhouette.data(),
                       &report.mean_silhouette);
  if (rc != DTWG_OK) detail::rethrow(ctx, rc, nullptr, 0);
  return report;
}

/// Drop-in for dtwclust::LazyDistanceSource (pairwise.hpp:133-188) on the k-medoids path
/// (runner.hpp:187-189, 211). Instead of computing pairs on demand on the host, the first
/// use fills the whole matrix on the GPU, into this source's own device context where it
/// stays resident: dtwgpu::kmedoids(GpuDistanceSource&, ...) below sweeps it there with no
/// host round trip, and distance(i, j) from host code reads a host copy fetched once.
/// Satisfies the DistanceSource concept (cluster_result.hpp:13-17).
///
/// Semantics kept from LazyDistanceSource::distance: indices are checked first
/// (IndexOutOfRangeError), i == j is 0 without any work, and a banded window without
/// auto-widen throws BandInfeasibleError(min(i,j), max(i,j), cause) only for a requested
/// infeasible pair -- the fill then computes the other pairs (auto-widened entries of the
/// infeasible pairs are never handed out). Every returned distance is bit-identical to
/// the reference's. Differences: computed_pairs() reports p(p-1)/2 once filled.
class GpuDistanceSource {
 public:
  GpuDistanceSource(const std::vector<dtwclust::TimeSeries>& dataset,
                    const dtwclust::WarpWindow& w, bool auto_widen = false)
      : dataset_(&dataset), window_(w), auto_widen_(auto_widen) {
    if (dataset.empty()) throw dtwclust::EmptyDatasetError();
    dtwclust::validate_dataset(dataset);
    if (!w.is_unlimited() && !auto_widen) {
      std::size_t lo = dataset[0].length(), hi = lo;
      for (const auto& s : dataset) {
        lo = std::min(lo, s.length());
        hi = std::max(hi, s.length());
      }
      has_infeasible_ = hi - lo > w.half_width();
    }
  }
  std::size_t size() const noexcept { return dataset_->size(); }

  double distance(std::size_t i, std::size_t j) {
    const std::size_t p = size();
    if (i >= p) throw dtwclust::IndexOutOfRangeError(i, p);
    if (j >= p) throw dtwclust::IndexOutOfRangeError(j, p);
    if (i == j) return 0.0;
    if (!feasible(i, j)) {
      const auto& a = (*dataset_)[i];
      const auto& b = (*dataset_)[j];
      throw dtwclust::BandInfeasibleError(
          std::min(i, j), std::max(i, j),
          dtwclust::BandInfeasibleError(a.length(), b.length(), window_.half_width()));
    }
    if (host_.empty()) {
      ensure_device();
      host_.resize(dtwclust::DistanceMatrix::condensed_size(p));
      const int rc = dtwg_download_condensed(ctx_->get(), host_.data());
      if (rc != DTWG_OK) detail::rethrow(ctx_->get(), rc, nullptr, 0);
    }
    const std::size_t lo = std::min(i, j), hi = std::max(i, j);
    return host_[lo * p - lo * (lo + 1) / 2 + (hi - lo - 1)];
  }

  std::uint64_t computed_pairs() const { return computed_; }
  /// Whether some pair of the dataset is infeasible under the window (banded, no widen).
  bool has_infeasible_pairs() const noexcept { return has_infeasible_; }

  /// Fills the matrix on the GPU (once) and leaves it resident in this source's context.
  dtwg_ctx* ensure_device() {
    if (!ctx_) {
      ctx_ = std::make_unique<Context>(default_devices()[0]);
      const std::size_t p = size();
      std::vector<std::int64_t> offsets(p + 1, 0);
      for (std::size_t i = 0; i < p; ++i)
        offsets[i + 1] = offsets[i] + static_cast<std::int64_t>((*dataset_)[i].length());
      std::vector<double> samples(static_cast<std::size_t>(offsets[p]));
      for (std::size_t i = 0; i < p; ++i)
        std::copy((*dataset_)[i].samples.begin(), (*dataset_)[i].samples.end(),
                  samples.begin() + offsets[i]);
      const std::int64_t hw =
          window_.is_unlimited() ? -1 : static_cast<std::int64_t>(window_.half_width());
      std::uint64_t evaluations = 0;
      // infeasible pairs (never handed out, see distance) are filled auto-widened so the
      // feasible ones can be computed in the same launch
      const int rc = dtwg_build_matrix(ctx_->get(), samples.data(), offsets.data(),
                                       static_cast<std::int64_t>(p), hw,
                                       (auto_widen_ || has_infeasible_) ? 1 : 0, 1, DTWG_FP64,
                                       nullptr, &evaluations);
      if (rc != DTWG_OK) {
        dtwg_ctx* c = ctx_->get();
        const std::string msg = dtwg_last_error(c);
        ctx_.reset();
        throw DeviceError(rc, msg);
      }
      computed_ = evaluations;
    }
    return ctx_->get();
  }

 private:
  bool feasible(std::size_t i, std::size_t j) const {
    if (!has_infeasible_) return true;
    return window_.feasible_for((*dataset_)[i].length(), (*dataset_)[j].length());
  }

  const std::vector<dtwclust::TimeSeries>* dataset_;
  dtwclust::WarpWindow window_;
  bool auto_widen_;
  bool has_infeasible_ = false;
  std::unique_ptr<Context> ctx_;
  std::vector<double> host_;
  std::uint64_t computed_ = 0;
};

/// kmedoids.hpp:148-189 over a GpuDistanceSource (the runner's lazy path, runner.hpp:211):
/// the sweeps run on the GPU over the matrix the source filled in HBM -- no host copy, no
/// re-upload. An unqualified kmedoids(source, config) call picks this overload (ADL,
/// non-template). If some pair is infeasible under the window, the reference's kmedoids
/// throws for the first infeasible pair it requests, which depends on its access order;
/// that case runs the reference's template over distance() so the same error surfaces.
inline dtwclust::ClusterResult kmedoids(GpuDistanceSource& source,
                                        const dtwclust::KMedoidsConfig& config,
                                        const dtwclust::IterationObserver& observer = {}) {
  const std::size_t p = source.size();
  if (config.k < 1 || config.k > p) throw dtwclust::KOutOfRangeError(config.k, p);
  if (config.restarts < 1) throw dtwclust::InvalidArgumentsError("restarts must be >= 1");
  if (config.max_iterations < 1)
    throw dtwclust::InvalidArgumentsError("max_iterations must be >= 1");
  if (source.has_infeasible_pairs()) return dtwclust::kmedoids<GpuDistanceSource>(source, config, observer);
  dtwg_ctx* ctx = source.ensure_device();
  struct Trampoline {
    static void call(void* user, std::int64_t r, std::int64_t it, double cost) {
      (*static_cast<const dtwclust::IterationObserver*>(user))(static_cast<std::size_t>(r),
                                                               static_cast<std::size_t>(it), cost);
    }
  };
  std::vector<std::int64_t> medoids(config.k), assignment(p);
  double cost = 0.0;
  std::int64_t best_restart = -1;
  const int rc = dtwg_kmedoids(ctx, static_cast<std::int64_t>(config.k),
                               static_cast<std::int64_t>(config.restarts),
                               static_cast<std::int64_t>(config.max_iterations), config.seed, 0,
                               static_cast<std::int64_t>(config.restarts),
                               observer ? &Trampoline::call : nullptr,
                               const_cast<dtwclust::IterationObserver*>(&observer),
                               medoids.data(), assignment.data(), &cost, &best_restart);
  if (rc != DTWG_OK) detail::rethrow(ctx, rc, nullptr, 0);
  dtwclust::ClusterResult result;
  result.medoids.assign(medoids.begin(), medoids.end());
  result.assignment.assign(assignment.begin(), assignment.end());
  result.total_cost = cost;
  result.certificate = dtwclust::Certificate::LocalHeuristic;
  return result;
}

namespace detail {

/// Rethrows a host-I/O error code (include/dtwgpu.h, host-side data path) as the
/// reference's exception class.
[[noreturn]] inline void rethrow_io(int rc) {
  std::int64_t line = -1, column = -1;
  const std::string msg = dtwg_io_last_error(&line, &column);
  const std::string where = dtwg_io_last_file();
  switch (rc) {
    case 3:
      throw dtwclust::IoFailureError(msg);
    case 4: {
      // the message is "<file>:<line>:<column>: <text>"; the exception rebuilds it
      const std::string prefix =
          where + ":" + std::to_string(line) + ":" + std::to_string(column) + ": ";
      throw dtwclust::ParseFailureError(where, static_cast<std::size_t>(line),
                                        static_cast<std::size_t>(column),
                                        msg.rfind(prefix, 0) == 0 ? msg.substr(prefix.size()) : msg);
    }
    case 5: {
      const std::string prefix = "series '" + where + "': ";
      throw dtwclust::InvalidSeriesError(where, msg.rfind(prefix, 0) == 0 ? msg.substr(prefix.size())
                                                                         : msg);
    }
    case 6:
      throw dtwclust::EmptySeriesError(where, static_cast<std::size_t>(line));
    case 7:
      throw dtwclust::EmptyDatasetError();
    case 9:
      throw dtwclust::FormatViolationError(static_cast<std::size_t>(line), msg);
    case 11:
      throw dtwclust::DistanceMatrixInvalidError(msg);
    default:
      throw dtwclust::InvalidArgumentsError(msg);
  }
}

}  // namespace detail

/// distance_matrix.hpp:104-122: byte-identical file, rows formatted by `threads` host
/// threads (0 = all cores).
inline void save_matrix(const dtwclust::DistanceMatrix& m, const std::filesystem::path& path,
                        int threads = 0) {
  const auto& c = m.condensed();
  const int rc = dtwg_save_matrix_text(c.empty() ? nullptr : c.data(),
                                       static_cast<std::int64_t>(m.size()), path.c_str(), threads);
  if (rc != DTWG_OK) detail::rethrow_io(rc);
}

/// distance_matrix.hpp:127-192: same checks and first error, rows parsed in parallel.
inline dtwclust::DistanceMatrix load_matrix(const std::filesystem::path& path, int threads = 0) {
  std::int64_t p = 0;
  double* buf = nullptr;
  const int rc = dtwg_load_matrix_text(path.c_str(), threads, &p, &buf);
  if (rc != DTWG_OK) detail::rethrow_io(rc);
  const std::size_t total = dtwclust::DistanceMatrix::condensed_size(static_cast<std::size_t>(p));
  std::vector<double> values(buf, buf + total);
  dtwg_free(buf);
  return dtwclust::DistanceMatrix::from_condensed(static_cast<std::size_t>(p), std::move(values));
}

/// Binary sidecar of the condensed matrix (loads at disk speed).
inline void save_matrix_binary(const dtwclust::DistanceMatrix& m, const std::filesystem::path& path) {
  const auto& c = m.condensed();
  const int rc = dtwg_save_matrix_binary(c.empty() ? nullptr : c.data(),
                                         static_cast<std::int64_t>(m.size()), path.c_str());
  if (rc != DTWG_OK) detail::rethrow_io(rc);
}

inline dtwclust::DistanceMatrix load_matrix_binary(const std::filesystem::path& path) {
  std::int64_t p = 0;
  double* buf = nullptr;
  const int rc = dtwg_load_matrix_binary(path.c_str(), &p, &buf);
  if (rc != DTWG_OK) detail::rethrow_io(rc);
  const std::size_t total = dtwclust::DistanceMatrix::condensed_size(static_cast<std::size_t>(p));
  std::vector<double> values(buf, buf + total);
  dtwg_free(buf);
  return dtwclust::DistanceMatrix::from_condensed(static_cast<std::size_t>(p), std::move(values));
}

/// csv.hpp:55-106: same series, ids and first error; each file parsed by several threads.
inline std::vector<dtwclust::TimeSeries> ingest(const std::vector<std::filesystem::path>& paths,
                                                const dtwclust::CsvFormat& format = {},
                                                int threads = 0) {
  std::vector<std::string> names;
  for (const auto& p : paths) names.push_back(p.string());
  std::vector<const char*> cps;
  for (const auto& n : names) cps.push_back(n.c_str());
  dtwg_dataset* ds = nullptr;
  const int rc = dtwg_ingest_csv(cps.data(), static_cast<std::int64_t>(cps.size()),
                                 format.label_column ? 1 : 0,
                                 format.delimiter ? static_cast<unsigned char>(*format.delimiter) : 0,
                                 threads, &ds);
  if (rc != DTWG_OK) detail::rethrow_io(rc);
  std::vector<dtwclust::TimeSeries> out;
  const std::int64_t p = dtwg_dataset_size(ds);
  const double* smp = dtwg_dataset_samples(ds);
  const std::int64_t* off = dtwg_dataset_offsets(ds);
  out.reserve(static_cast<std::size_t>(p));
  for (std::int64_t i = 0; i < p; ++i)
    out.push_back({dtwg_dataset_id(ds, i), std::vector<double>(smp + off[i], smp + off[i + 1])});
  dtwg_dataset_free(ds);
  return out;
}

/// runner.hpp:82-95 (bit-identical), series normalised in parallel.
inline void z_normalize(std::vector<dtwclust::TimeSeries>& dataset, int threads = 0) {
  std::vector<std::int64_t> off(dataset.size() + 1, 0);
  for (std::size_t i = 0; i < dataset.size(); ++i)
    off[i + 1] = off[i] + static_cast<std::int64_t>(dataset[i].samples.size());
  std::vector<double> smp(static_cast<std::size_t>(off.back()));
  for (std::size_t i = 0; i < dataset.size(); ++i)
    std::copy(dataset[i].samples.begin(), dataset[i].samples.end(), smp.begin() + off[i]);
  const int rc = dtwg_z_normalize(smp.data(), off.data(), static_cast<std::int64_t>(dataset.size()),
                                  threads);
  if (rc != DTWG_OK) detail::rethrow_io(rc);
  for (std::size_t i = 0; i < dataset.size(); ++i)
    std::copy(smp.begin() + off[i], smp.begin() + off[i + 1], dataset[i].samples.begin());
}

}  // namespace dtwgpu
