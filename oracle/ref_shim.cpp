// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// An extern "C" face over the UNMODIFIED reference headers, compiled in place from
// /root/reference/proj/include (see oracle/Makefile) into oracle/_ref/libdtwclust_ref.so.
// No reference source is copied into this repository: this file only calls the
// reference's public entry points:
//   dtwclust::build_matrix   pairwise.hpp:62-127
//   dtwclust::dtw_distance   dtw.hpp:40-75
//   dtwclust::kmedoids       kmedoids.hpp:148-189
//   dtwclust::assign_to_medoids / assignment_cost  cluster_result.hpp:40-72
//   dtwclust::testing::dtw_brute_force_oracle      tests/support/oracles.hpp:44-59
//   dtwclust::silhouette_scores                    validation.hpp:30-79
//   dtwclust::save_matrix / load_matrix            distance_matrix.hpp:104-192
//   dtwclust::ingest                               csv.hpp:55-106
//   dtwclust::detail::z_normalize                  runner.hpp:82-95
// It is used (a) to pin oracle/dtw_oracle.c and the golden fixtures, and (b) as the
// "reference" arm of bench.py (the reference's own multithreaded CPU fill).
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <dtwclust/cluster_result.hpp>
#include <dtwclust/distance_matrix.hpp>
#include <dtwclust/dtw.hpp>
#include <dtwclust/errors.hpp>
#include <dtwclust/kmedoids.hpp>
#include <dtwclust/csv.hpp>
#include <dtwclust/pairwise.hpp>
#include <dtwclust/runner.hpp>
#include <dtwclust/validation.hpp>

#include "support/oracles.hpp"

namespace {

thread_local std::string g_last_error;
thread_local std::int64_t g_pair_i = -1;
thread_local std::int64_t g_pair_j = -1;

dtwclust::WarpWindow window_of(std::int64_t hw) {
  return hw < 0 ? dtwclust::WarpWindow::unlimited()
                : dtwclust::WarpWindow::banded(static_cast<std::size_t>(hw));
}

std::vector<dtwclust::TimeSeries> dataset_of(const double* samples, const std::int64_t* offsets,
                                             std::int64_t p) {
  std::vector<dtwclust::TimeSeries> ds;
  ds.reserve(static_cast<std::size_t>(p));
  for (std::int64_t i = 0; i < p; ++i) {
    ds.push_back({"s" + std::to_string(i),
                  std::vector<double>(samples + offsets[i], samples + offsets[i + 1])});
  }
  return ds;
}

template <class F>
int guarded(F&& f) {
  g_pair_i = g_pair_j = -1;
  try {
    f();
    return 0;
  } catch (const dtwclust::BandInfeasibleError& e) {
    g_last_error = e.what();
    if (e.has_pair()) {
      g_pair_i = static_cast<std::int64_t>(e.pair_i());
      g_pair_j = static_cast<std::int64_t>(e.pair_j());
    }
    return static_cast<int>(e.code());
  } catch (const dtwclust::Error& e) {
    g_last_error = e.what();
    return static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return 1;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }
void ref_last_pair(std::int64_t* i, std::int64_t* j) {
  *i = g_pair_i;
  *j = g_pair_j;
}

// dtwclust::build_matrix over a packed CSR dataset; writes p(p-1)/2 condensed values.
int ref_build_condensed(const double* samples, const std::int64_t* offsets, std::int64_t p,
                        std::int64_t half_width, int auto_widen, unsigned workers, double* out,
                        std::uint64_t* evaluations) {
  return guarded([&] {
    const auto ds = dataset_of(samples, offsets, p);
    dtwclust::BuildStats stats;
    const dtwclust::DistanceMatrix m =
        dtwclust::build_matrix(ds, window_of(half_width), workers, &stats, auto_widen != 0);
    const auto& c = m.condensed();
    if (!c.empty()) std::memcpy(out, c.data(), c.size() * sizeof(double));
    if (evaluations) *evaluations = stats.evaluations;
  });
}

// Same, for an arbitrary list of series ids (lets tests pass empty/NaN/duplicate rows).
int ref_build_condensed_ids(const double* samples, const std::int64_t* offsets, std::int64_t p,
                            const char* const* ids, std::int64_t half_width, int auto_widen,
                            unsigned workers, double* out, std::uint64_t* evaluations) {
  return guarded([&] {
    auto ds = dataset_of(samples, offsets, p);
    for (std::int64_t i = 0; i < p; ++i) ds[static_cast<std::size_t>(i)].id = ids[i];
    dtwclust::BuildStats stats;
    const dtwclust::DistanceMatrix m =
        dtwclust::build_matrix(ds, window_of(half_width), workers, &stats, auto_widen != 0);
    const auto& c = m.condensed();
    if (!c.empty()) std::memcpy(out, c.data(), c.size() * sizeof(double));
    if (evaluations) *evaluations = stats.evaluations;
  });
}

int ref_dtw(const double* x, std::int64_t n, const double* y, std::int64_t m,
            std::int64_t half_width, double* out) {
  return guarded([&] {
    const dtwclust::TimeSeries a{"x", std::vector<double>(x, x + n)};
    const dtwclust::TimeSeries b{"y", std::vector<double>(y, y + m)};
    *out = dtwclust::dtw_distance(a, b, window_of(half_width));
  });
}

int ref_dtw_brute_force(const double* x, std::int64_t n, const double* y, std::int64_t m,
                        std::int64_t half_width, double* out) {
  return guarded([&] {
    const dtwclust::TimeSeries a{"x", std::vector<double>(x, x + n)};
    const dtwclust::TimeSeries b{"y", std::vector<double>(y, y + m)};
    *out = dtwclust::testing::dtw_brute_force_oracle(a, b, window_of(half_width));
  });
}

typedef void (*ref_observer_fn)(void* user, std::int64_t restart, std::int64_t iteration,
                                double cost);

// dtwclust::kmedoids over DistanceMatrix::from_condensed.
int ref_kmedoids(const double* condensed, std::int64_t p, std::int64_t k, std::int64_t restarts,
                 std::int64_t max_iterations, std::uint64_t seed, ref_observer_fn observer,
                 void* user, std::int64_t* medoids_out, std::int64_t* assignment_out,
                 double* cost_out) {
  return guarded([&] {
    const std::size_t total = dtwclust::DistanceMatrix::condensed_size(static_cast<std::size_t>(p));
    auto m = dtwclust::DistanceMatrix::from_condensed(
        static_cast<std::size_t>(p), std::vector<double>(condensed, condensed + total));
    dtwclust::KMedoidsConfig cfg;
    cfg.k = static_cast<std::size_t>(k);
    cfg.restarts = static_cast<std::size_t>(restarts);
    cfg.max_iterations = static_cast<std::size_t>(max_iterations);
    cfg.seed = seed;
    dtwclust::IterationObserver obs;
    if (observer) {
      obs = [&](std::size_t r, std::size_t it, double cost) {
        observer(user, static_cast<std::int64_t>(r), static_cast<std::int64_t>(it), cost);
      };
    }
    const dtwclust::ClusterResult res = dtwclust::kmedoids(m, cfg, obs);
    for (std::size_t t = 0; t < res.medoids.size(); ++t)
      medoids_out[t] = static_cast<std::int64_t>(res.medoids[t]);
    for (std::size_t t = 0; t < res.assignment.size(); ++t)
      assignment_out[t] = static_cast<std::int64_t>(res.assignment[t]);
    *cost_out = res.total_cost;
  });
}

// One assign + update sweep (cluster_result.hpp:40-72, kmedoids.hpp:84-139).
int ref_sweep(const double* condensed, std::int64_t p, const std::int64_t* medoids, std::int64_t k,
              std::int64_t* assignment_out, double* cost_out, std::int64_t* updated_out) {
  return guarded([&] {
    const std::size_t total = dtwclust::DistanceMatrix::condensed_size(static_cast<std::size_t>(p));
    auto m = dtwclust::DistanceMatrix::from_condensed(
        static_cast<std::size_t>(p), std::vector<double>(condensed, condensed + total));
    std::vector<std::size_t> med(medoids, medoids + k);
    const auto asg = dtwclust::assign_to_medoids(m, med);
    *cost_out = dtwclust::assignment_cost(m, asg);
    const auto upd = dtwclust::detail::update_medoids(m, med, asg);
    for (std::size_t t = 0; t < asg.size(); ++t) assignment_out[t] = static_cast<std::int64_t>(asg[t]);
    for (std::size_t t = 0; t < upd.size(); ++t) updated_out[t] = static_cast<std::int64_t>(upd[t]);
  });
}

// dtwclust::silhouette_scores (validation.hpp:30-79).
int ref_silhouette(const double* condensed, std::int64_t p, const std::int64_t* medoids,
                   std::int64_t k, const std::int64_t* assignment, std::int64_t p_assign,
                   double* sil_out, double* mean_out) {
  return guarded([&] {
    const std::size_t total = dtwclust::DistanceMatrix::condensed_size(static_cast<std::size_t>(p));
    auto m = dtwclust::DistanceMatrix::from_condensed(
        static_cast<std::size_t>(p), std::vector<double>(condensed, condensed + total));
    dtwclust::ClusterResult r;
    r.medoids.assign(medoids, medoids + k);
    r.assignment.assign(assignment, assignment + p_assign);
    const dtwclust::ScoreReport rep = dtwclust::silhouette_scores(m, r);
    for (std::size_t t = 0; t < rep.silhouette.size(); ++t) sil_out[t] = rep.silhouette[t];
    *mean_out = rep.mean_silhouette;
  });
}

void ref_free(void* ptr) { std::free(ptr); }

// dtwclust::save_matrix (distance_matrix.hpp:104-122).
int ref_save_matrix(const double* condensed, std::int64_t p, const char* path) {
  return guarded([&] {
    const std::size_t total = dtwclust::DistanceMatrix::condensed_size(static_cast<std::size_t>(p));
    auto m = dtwclust::DistanceMatrix::from_condensed(
        static_cast<std::size_t>(p), std::vector<double>(condensed, condensed + total));
    dtwclust::save_matrix(m, path);
  });
}

// dtwclust::load_matrix (distance_matrix.hpp:127-192); *cond_out is malloc'ed.
int ref_load_matrix(const char* path, std::int64_t* p_out, double** cond_out) {
  return guarded([&] {
    const dtwclust::DistanceMatrix m = dtwclust::load_matrix(path);
    const auto& c = m.condensed();
    double* buf = static_cast<double*>(std::malloc(std::max<std::size_t>(c.size(), 1) * 8));
    std::memcpy(buf, c.data(), c.size() * 8);
    *p_out = static_cast<std::int64_t>(m.size());
    *cond_out = buf;
  });
}

// dtwclust::ingest (csv.hpp:55-106) -> packed buffers (malloc'ed) and '\n'-joined ids.
int ref_ingest(const char* const* paths, std::int64_t n, int label_column, int delimiter,
               std::int64_t* p_out, double** samples_out, std::int64_t** offsets_out,
               char** ids_out) {
  return guarded([&] {
    std::vector<std::filesystem::path> ps(paths, paths + n);
    dtwclust::CsvFormat fmt;
    fmt.label_column = label_column != 0;
    if (delimiter > 0) fmt.delimiter = static_cast<char>(delimiter);
    const auto ds = dtwclust::ingest(ps, fmt);
    std::size_t total = 0;
    std::string ids;
    for (const auto& s : ds) {
      total += s.samples.size();
      ids += s.id;
      ids += '\n';
    }
    double* smp = static_cast<double*>(std::malloc(std::max<std::size_t>(total, 1) * 8));
    auto* off = static_cast<std::int64_t*>(std::malloc((ds.size() + 1) * 8));
    char* idb = static_cast<char*>(std::malloc(ids.size() + 1));
    std::size_t pos = 0;
    off[0] = 0;
    for (std::size_t i = 0; i < ds.size(); ++i) {
      std::memcpy(smp + pos, ds[i].samples.data(), ds[i].samples.size() * 8);
      pos += ds[i].samples.size();
      off[i + 1] = static_cast<std::int64_t>(pos);
    }
    std::memcpy(idb, ids.c_str(), ids.size() + 1);
    *p_out = static_cast<std::int64_t>(ds.size());
    *samples_out = smp;
    *offsets_out = off;
    *ids_out = idb;
  });
}

// dtwclust::z_normalize (runner.hpp:82-95), in place on packed series.
int ref_z_normalize(double* samples, const std::int64_t* offsets, std::int64_t p) {
  return guarded([&] {
    std::vector<dtwclust::TimeSeries> ds = dataset_of(samples, offsets, p);
    dtwclust::detail::z_normalize(ds);
    for (std::int64_t i = 0; i < p; ++i)
      std::memcpy(samples + offsets[i], ds[i].samples.data(), ds[i].samples.size() * 8);
  });
}

}  // extern "C"
