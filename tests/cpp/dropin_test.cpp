// dropin_test.cpp -- framework-free parity test of the C++ drop-in (include/dtwgpu/
// dtwclust_gpu.hpp) against the unmodified reference, in the style of the reference's
// acceptance suite (acceptance_main.cpp: Check{name, body}, PASS/FAIL lines, exit code).
// Built by tests/cpp/Makefile against /root/reference/proj headers + libdtwgpu.so; run
// on the GPU box by tests/test_gpu_dropin.py.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <functional>
#include <string>
#include <vector>

#include <dtwclust/dtw.hpp>
#include <dtwclust/kmedoids.hpp>
#include <dtwclust/pairwise.hpp>
#include <dtwclust/runner.hpp>

#include "support/synthetic.hpp"

#include <dtwgpu/dtwclust_gpu.hpp>

using namespace dtwclust;

namespace {

struct Check {
  std::string name;
  std::function<std::string()> body;
};

void require(bool ok, const std::string& what) {
  if (!ok) throw std::runtime_error(what);
}

std::vector<TimeSeries> walks(std::uint64_t seed, std::size_t p, std::size_t lo, std::size_t hi) {
  SplitMix64 rng(seed);
  std::vector<TimeSeries> ds;
  for (std::size_t i = 0; i < p; ++i) {
    const std::size_t len = lo + rng.next_below(hi - lo + 1);
    ds.push_back(testing::random_walk_series(rng, len, "s" + std::to_string(i)));
  }
  return ds;
}

std::string same_matrix(const std::vector<TimeSeries>& ds, const WarpWindow& w, bool widen) {
  BuildStats a, b;
  const DistanceMatrix ref = dtwclust::build_matrix(ds, w, 4, &a, widen);
  const DistanceMatrix gpu = dtwgpu::build_matrix(ds, w, 4, &b, widen);
  require(ref.condensed() == gpu.condensed(), "condensed matrices differ");
  require(a.evaluations == b.evaluations, "evaluation counts differ");
  return std::to_string(ds.size()) + " series, " + std::to_string(ref.condensed().size()) +
         " pairs bit-identical";
}

}  // namespace

int main() {
  std::vector<Check> checks = {
      {"matrix: unlimited window, ragged lengths",
       [] { return same_matrix(walks(1, 60, 20, 300), WarpWindow::unlimited(), false); }},
      {"matrix: banded window, equal lengths",
       [] { return same_matrix(walks(2, 40, 500, 500), WarpWindow::banded(50), false); }},
      {"matrix: auto-widen, ragged lengths",
       [] { return same_matrix(walks(3, 50, 50, 700), WarpWindow::banded(30), true); }},
      {"matrix: short series (many pairs)",
       [] { return same_matrix(walks(4, 300, 30, 46), WarpWindow::unlimited(), false); }},
      {"dtw_distance: one pair, same value and errors",
       [] {
         const auto ds = walks(9, 2, 3000, 3500);
         for (const WarpWindow& w : {WarpWindow::unlimited(), WarpWindow::banded(600)}) {
           const double a = dtwclust::dtw_distance(ds[0], ds[1], w);
           const double b = dtwgpu::dtw_distance(ds[0], ds[1], w);
           require(a == b, "distance differs");
         }
         std::string e1, e2;
         try { dtwclust::dtw_distance(ds[0], ds[1], WarpWindow::banded(1)); } catch (const BandInfeasibleError& e) { e1 = e.what(); }
         try { dtwgpu::dtw_distance(ds[0], ds[1], WarpWindow::banded(1)); } catch (const BandInfeasibleError& e) { e2 = e.what(); }
         require(!e1.empty() && e1 == e2, "errors differ: " + e1 + " / " + e2);
         return "3000-3500 samples, unlimited and banded(600) equal; '" + e2 + "'";
       }},
      {"errors: first band-infeasible pair",
       [] {
         const std::vector<TimeSeries> ds = {testing::make_series("a", {1, 2}),
                                             testing::make_series("b", {1, 2, 3}),
                                             testing::make_series("c", {1, 2, 3, 4, 5, 6})};
         try {
           dtwgpu::build_matrix(ds, WarpWindow::banded(1), 1);
         } catch (const BandInfeasibleError& e) {
           require(e.has_pair() && e.pair_i() == 0 && e.pair_j() == 2, "wrong pair");
           return std::string("BandInfeasibleError at (0, 2)");
         }
         throw std::runtime_error("no exception");
       }},
      {"errors: validation order",
       [] {
         int hits = 0;
         try { dtwgpu::build_matrix({}, WarpWindow::unlimited(), 1); } catch (const EmptyDatasetError&) { ++hits; }
         try { dtwgpu::build_matrix({testing::make_series("a", {1})}, WarpWindow::unlimited(), 0); } catch (const InvalidArgumentsError&) { ++hits; }
         try { dtwgpu::build_matrix({testing::make_series("a", {1}), testing::make_series("a", {2})}, WarpWindow::unlimited(), 1); } catch (const InvalidSeriesError&) { ++hits; }
         try { dtwgpu::build_matrix({testing::make_series("a", {1}), testing::make_series("b", {})}, WarpWindow::unlimited(), 1); } catch (const InvalidSeriesError&) { ++hits; }
         require(hits == 4, "expected 4 typed exceptions, got " + std::to_string(hits));
         return std::string("Empty/InvalidArguments/InvalidSeries x2 as the reference");
       }},
      {"kmedoids: identical ClusterResult and observer trace",
       [] {
         const auto ds = walks(5, 120, 100, 160);
         const DistanceMatrix m = dtwclust::build_matrix(ds, WarpWindow::banded(20), 4, nullptr, true);
         KMedoidsConfig cfg;
         cfg.k = 6;
         cfg.restarts = 5;
         cfg.seed = 0xDEED;
         std::vector<double> ta, tb;
         const ClusterResult a = dtwclust::kmedoids(m, cfg, [&](std::size_t, std::size_t, double c) { ta.push_back(c); });
         const ClusterResult b = dtwgpu::kmedoids(m, cfg, [&](std::size_t, std::size_t, double c) { tb.push_back(c); });
         require(a == b, "ClusterResult differs");
         require(ta == tb, "observer traces differ");
         return "k=6, 5 restarts: medoids, labels, cost bit-identical; " + std::to_string(ta.size()) + " sweeps";
       }},
      {"kmedoids: k == p and invalid configs",
       [] {
         SplitMix64 rng(1);
         const DistanceMatrix d = testing::random_distance_matrix(rng, 6);
         KMedoidsConfig cfg;
         cfg.k = 6;
         cfg.restarts = 2;
         require(dtwgpu::kmedoids(d, cfg) == dtwclust::kmedoids(d, cfg), "k == p differs");
         int hits = 0;
         cfg.k = 7;
         try { dtwgpu::kmedoids(d, cfg); } catch (const KOutOfRangeError&) { ++hits; }
         cfg.k = 2;
         cfg.restarts = 0;
         try { dtwgpu::kmedoids(d, cfg); } catch (const InvalidArgumentsError&) { ++hits; }
         require(hits == 2, "typed exceptions missing");
         return std::string("k == p equal; KOutOfRange, InvalidArguments thrown");
       }},
      {"silhouette: identical ScoreReport",
       [] {
         const auto ds = walks(6, 150, 80, 120);
         const DistanceMatrix m = dtwclust::build_matrix(ds, WarpWindow::unlimited(), 4);
         KMedoidsConfig cfg;
         cfg.k = 5;
         const ClusterResult r = dtwclust::kmedoids(m, cfg);
         const ScoreReport a = dtwclust::silhouette_scores(m, r);
         const ScoreReport b = dtwgpu::silhouette_scores(m, r);
         require(a.silhouette == b.silhouette, "silhouettes differ");
         require(a.mean_silhouette == b.mean_silhouette, "mean differs");
         ClusterResult one = r;
         one.medoids = {r.medoids[0]};
         try { dtwgpu::silhouette_scores(m, one); } catch (const SingleClusterUndefinedError&) {
           return "150 series, k=5: bit-identical; k=1 -> SingleClusterUndefinedError";
         }
         throw std::runtime_error("k=1 accepted");
       }},
      {"lazy source: GPU-backed DistanceSource gives the same clustering",
       [] {
         const auto ds = walks(7, 60, 40, 90);
         dtwclust::LazyDistanceSource lazy(ds, WarpWindow::banded(10), true);
         dtwgpu::GpuDistanceSource gpu(ds, WarpWindow::banded(10), true);
         KMedoidsConfig cfg;
         cfg.k = 3;
         cfg.seed = 2024;
         std::vector<double> ta, tb;
         const ClusterResult a =
             dtwclust::kmedoids(lazy, cfg, [&](std::size_t, std::size_t, double c) { ta.push_back(c); });
         // unqualified call, as runner.hpp:211 makes it: resolves to the GPU sweeps (ADL)
         const ClusterResult b = kmedoids(gpu, cfg, [&](std::size_t, std::size_t, double c) { tb.push_back(c); });
         require(a == b, "results differ");
         require(ta == tb, "observer traces differ");
         require(gpu.computed_pairs() == 60 * 59 / 2, "computed_pairs");
         // host-side reads equal the reference's lazily computed ones
         for (std::size_t i = 0; i < 60; i += 7)
           for (std::size_t j = 0; j < 60; j += 5)
             require(lazy.distance(i, j) == gpu.distance(i, j), "distance differs");
         return "kmedoids(lazy) == kmedoids(GpuDistanceSource) on the device, same trace";
       }},
      {"lazy source: lazy errors (index, diagonal, infeasible pair)",
       [] {
         // lengths 40..90 with a narrow band, no auto-widen: some pairs are infeasible
         const auto ds = walks(9, 30, 40, 90);
         dtwclust::LazyDistanceSource lazy(ds, WarpWindow::banded(5), false);
         dtwgpu::GpuDistanceSource gpu(ds, WarpWindow::banded(5), false);
         std::string e1, e2;
         try { lazy.distance(3, 30); } catch (const IndexOutOfRangeError& e) { e1 = e.what(); }
         try { gpu.distance(3, 30); } catch (const IndexOutOfRangeError& e) { e2 = e.what(); }
         require(!e1.empty() && e1 == e2, "index error differs");
         require(gpu.distance(4, 4) == 0.0 && gpu.computed_pairs() == 0, "diagonal did work");
         std::size_t checked = 0, infeasible = 0;
         for (std::size_t i = 0; i < 30; ++i)
           for (std::size_t j = 0; j < 30; ++j) {
             std::string a, b;
             double va = -1, vb = -2;
             try { va = lazy.distance(i, j); } catch (const BandInfeasibleError& e) { a = e.what(); }
             try { vb = gpu.distance(i, j); } catch (const BandInfeasibleError& e) { b = e.what(); }
             require(a == b, "errors differ at (" + std::to_string(i) + "," + std::to_string(j) + ")");
             if (a.empty()) require(va == vb, "distance differs");
             infeasible += !a.empty();
             ++checked;
           }
         require(infeasible > 0, "no infeasible pair in the test data");
         KMedoidsConfig cfg;
         cfg.k = 3;
         std::string k1, k2;
         try { dtwclust::kmedoids(lazy, cfg); } catch (const BandInfeasibleError& e) { k1 = e.what(); }
         try { kmedoids(gpu, cfg); } catch (const BandInfeasibleError& e) { k2 = e.what(); }
         require(k1 == k2, "kmedoids errors differ: '" + k1 + "' vs '" + k2 + "'");
         return std::to_string(checked) + " requests, " + std::to_string(infeasible) +
                " infeasible with the reference's message; kmedoids error '" + k2 + "'";
       }},
      {"matrix files: byte-identical text, round trips, same first error",
       [] {
         const auto ds = walks(8, 40, 30, 60);
         const DistanceMatrix m = dtwclust::build_matrix(ds, WarpWindow::unlimited(), 2);
         const std::filesystem::path dir = std::filesystem::temp_directory_path() / "dtwgpu_io";
         std::filesystem::create_directories(dir);
         dtwclust::save_matrix(m, dir / "ref.txt");
         dtwgpu::save_matrix(m, dir / "gpu.txt", 4);
         auto slurp = [](const std::filesystem::path& p) {
           std::ifstream f(p, std::ios::binary);
           std::stringstream ss;
           ss << f.rdbuf();
           return ss.str();
         };
         require(slurp(dir / "ref.txt") == slurp(dir / "gpu.txt"), "files differ");
         require(dtwgpu::load_matrix(dir / "ref.txt", 3) == m, "load differs");
         dtwgpu::save_matrix_binary(m, dir / "m.bin");
         require(dtwgpu::load_matrix_binary(dir / "m.bin") == m, "binary round trip");
         {
           std::ofstream f(dir / "bad.txt", std::ios::binary);
           f << "p=3\n0,1,2\n1,0,3\n2,4,0\n";
         }
         std::string a, b;
         try { dtwclust::load_matrix(dir / "bad.txt"); } catch (const FormatViolationError& e) { a = e.what(); }
         try { dtwgpu::load_matrix(dir / "bad.txt"); } catch (const FormatViolationError& e) { b = e.what(); }
         require(!a.empty() && a == b, "errors differ: '" + a + "' vs '" + b + "'");
         return "40x40 text identical; text/binary round trips; '" + b + "'";
       }},
      {"ingest + z-normalise: same series, ids, errors",
       [] {
         const std::filesystem::path dir = std::filesystem::temp_directory_path() / "dtwgpu_io";
         std::filesystem::create_directories(dir);
         {
           std::ofstream f(dir / "u.csv", std::ios::binary);
           f << "1,0.5,2.25,\n2,3e-2,-4,5\r\n3, +6 ,7\n";
         }
         CsvFormat fmt;
         fmt.label_column = true;
         auto a = dtwclust::ingest({dir / "u.csv"}, fmt);
         auto b = dtwgpu::ingest({dir / "u.csv"}, fmt, 2);
         require(a == b, "ingested series differ");
         dtwclust::detail::z_normalize(a);
         dtwgpu::z_normalize(b, 2);
         require(a == b, "z-normalised series differ");
         {
           std::ofstream f(dir / "v.csv", std::ios::binary);
           f << "1,2\n3,,4\n";
         }
         std::string e1, e2;
         try { dtwclust::ingest({dir / "v.csv"}); } catch (const ParseFailureError& e) { e1 = e.what(); }
         try { dtwgpu::ingest({dir / "v.csv"}); } catch (const ParseFailureError& e) { e2 = e.what(); }
         require(!e1.empty() && e1 == e2, "errors differ: '" + e1 + "' vs '" + e2 + "'");
         return "3 rows equal (label column, CRLF, '+'); ParseFailure '" + e2 + "'";
       }},
  };
  int failed = 0;
  for (const auto& c : checks) {
    try {
      const std::string detail = c.body();
      std::printf("PASS  %s -- %s\n", c.name.c_str(), detail.c_str());
    } catch (const std::exception& e) {
      ++failed;
      std::printf("FAIL  %s -- %s\n", c.name.c_str(), e.what());
    }
  }
  std::printf("%zu/%zu passed\n", checks.size() - failed, checks.size());
  return failed ? 1 : 0;
}
