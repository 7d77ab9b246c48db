"""GPU k-medoids sweeps vs the reference's kmedoids (oracle/_ref) and the C restatement.

Bar: medoids and labels identical, total cost bit-identical (test_kmedoids.cpp,
acceptance criterion 7, test_csv_runner.cpp:192-200 reconstructed cost).
"""
import numpy as np
import pytest

import oracle
from paper_2307_04904_b200 import api, generators as gen
from paper_2307_04904_b200.api import (DistanceMatrix, InvalidArgumentsError, KMedoidsConfig,
                                       KOutOfRangeError, TimeSeries, WarpWindow, build_matrix,
                                       kmedoids)
from tests.helpers import ScalarRng, blob_series, random_condensed

pytestmark = pytest.mark.gpu


def kref(D, p, cfg, observer=None):
    if oracle.have_ref():
        return oracle.ref_kmedoids(D, p, cfg.k, cfg.restarts, cfg.max_iterations, cfg.seed,
                                   observer)
    return oracle.kmedoids(D, p, cfg.k, cfg.restarts, cfg.max_iterations, cfg.seed, observer)


def check_same(D, p, cfg):
    m = DistanceMatrix.from_condensed(p, D)
    got = kmedoids(m, cfg)
    med, asg, cost = kref(D, p, cfg)
    assert got.medoids == [int(v) for v in med]
    assert got.assignment == [int(v) for v in asg]
    assert got.total_cost == cost
    return got


def test_k_equals_p():
    D = random_condensed(ScalarRng(1), 6)
    got = check_same(D, 6, KMedoidsConfig(k=6, restarts=2))
    assert got.total_cost == 0.0 and got.assignment == list(range(6))


def test_k_one_global_medoid():
    D = random_condensed(ScalarRng(2), 9)
    check_same(D, 9, KMedoidsConfig(k=1, restarts=1))


def test_two_blobs():
    data = []
    for i in range(5):
        data.append(TimeSeries(f"low{i}", [0.1 * i] * 4))
    for i in range(5):
        data.append(TimeSeries(f"high{i}", [100 + 0.1 * i] * 4))
    m = build_matrix(data, WarpWindow.unlimited(), 1)
    got = kmedoids(m, KMedoidsConfig(k=2, seed=11))
    med, asg, cost = kref(m.condensed(), 10, KMedoidsConfig(k=2, seed=11))
    assert got.total_cost == cost and got.medoids == list(med)
    assert len(set(got.assignment[:5])) == 1 and len(set(got.assignment[5:])) == 1


@pytest.mark.parametrize("p,k,seed", [(20, 4, 20240101), (15, 3, 5), (25, 4, 99), (30, 5, 1234),
                                      (200, 7, 0xDEED), (1000, 8, 0)])
def test_random_matrices_match_reference(p, k, seed):
    D = random_condensed(ScalarRng(p + k), p)
    check_same(D, p, KMedoidsConfig(k=k, restarts=6, seed=seed))


def test_observer_trace_matches_and_descends():
    D = random_condensed(ScalarRng(6), 25)
    cfg = KMedoidsConfig(k=4, restarts=6, seed=99)
    trace_gpu, trace_ref = [], []
    kmedoids(DistanceMatrix.from_condensed(25, D), cfg,
             lambda r, it, c: trace_gpu.append((r, it, c)))
    kref(D, 25, cfg, lambda r, it, c: trace_ref.append((r, it, c)))
    assert trace_gpu == trace_ref
    by_r = {}
    for r, it, c in trace_gpu:
        by_r.setdefault(r, []).append(c)
    for costs in by_r.values():
        assert all(b <= a for a, b in zip(costs, costs[1:]))


def test_best_of_restarts_monotone():
    """More restarts never raise the best cost (test_kmedoids.cpp:141-154): restart r's
    stream does not depend on the restart count, and the best is kept by strict <."""
    D = random_condensed(ScalarRng(31), 60)
    m = DistanceMatrix.from_condensed(60, D)
    costs = [kmedoids(m, KMedoidsConfig(k=5, restarts=r, seed=7)).total_cost
             for r in range(1, 9)]
    assert all(b <= a for a, b in zip(costs, costs[1:]))
    assert costs[-1] == kref(D, 60, KMedoidsConfig(k=5, restarts=8, seed=7))[2]


def test_duplicates_and_fixed_point():
    data = [TimeSeries(f"dup{i}", [1.0, 2.0, 3.0]) for i in range(6)]
    m = build_matrix(data, WarpWindow.unlimited(), 1)
    got = kmedoids(m, KMedoidsConfig(k=3, seed=9))
    med, asg, cost = kref(m.condensed(), 6, KMedoidsConfig(k=3, seed=9))
    assert got.total_cost == 0.0 == cost and got.medoids == list(med)
    D = random_condensed(ScalarRng(4), 15)
    mm = DistanceMatrix.from_condensed(15, D)
    res = kmedoids(mm, KMedoidsConfig(k=3, seed=5))
    assert api.assign_to_medoids(mm, res.medoids) == res.assignment
    assert api.update_medoids(mm, res.medoids, res.assignment) == res.medoids
    assert api.assignment_cost(mm, res.assignment) == res.total_cost


def test_invalid_configs():
    m = DistanceMatrix.from_condensed(4, random_condensed(ScalarRng(10), 4))
    with pytest.raises(KOutOfRangeError):
        kmedoids(m, KMedoidsConfig(k=5))
    with pytest.raises(KOutOfRangeError):
        kmedoids(m, KMedoidsConfig(k=0))
    with pytest.raises(InvalidArgumentsError):
        kmedoids(m, KMedoidsConfig(k=2, restarts=0))


def test_sweep_pieces_match_reference():
    p, k = 300, 9
    D = random_condensed(ScalarRng(77), p)
    m = DistanceMatrix.from_condensed(p, D)
    medoids = sorted(np.random.default_rng(0).choice(p, k, replace=False).tolist())
    asg_ref, cost_ref, upd_ref = oracle.ref_sweep(D, p, medoids) if oracle.have_ref() else (
        oracle.assign(D, p, medoids), None, None)
    assert api.assign_to_medoids(m, medoids) == list(asg_ref)
    if upd_ref is not None:
        assert api.update_medoids(m, medoids, list(asg_ref)) == list(upd_ref)


@pytest.mark.parametrize("cfgno,q", [(1, 100), (3, 600), (5, 150)])
def test_config_pipeline_matches_reference(eng, cfgno, q):
    ds = gen.make_config(cfgno).subset(q)
    m = api.build_matrix_packed(ds.samples, ds.offsets,
                                WarpWindow(None if ds.half_width < 0 else ds.half_width),
                                ds.auto_widen)
    cfg = KMedoidsConfig(k=ds.k, restarts=3, seed=0)
    got = kmedoids(m, cfg)
    med, asg, cost = kref(m.condensed(), ds.p, cfg)
    assert got.medoids == list(med) and got.assignment == list(asg) and got.total_cost == cost


# ---------------------------------------------------------------- silhouette (validation.hpp)
def sref(D, p, med, asg):
    return (oracle.ref_silhouette if oracle.have_ref() else oracle.silhouette)(D, p, med, asg)


@pytest.mark.parametrize("cfgno,q", [(1, 100), (3, 800), (5, 200)])
def test_silhouette_matches_reference(cfgno, q):
    ds = gen.make_config(cfgno).subset(q)
    m = api.build_matrix_packed(ds.samples, ds.offsets,
                                WarpWindow(None if ds.half_width < 0 else ds.half_width),
                                ds.auto_widen)
    res = kmedoids(m, KMedoidsConfig(k=ds.k, restarts=2))
    rep = api.silhouette_scores(m, res)
    sil, mean = sref(m.condensed(), ds.p, res.medoids, res.assignment)
    assert np.array_equal(np.array(rep.silhouette).view(np.uint64), sil.view(np.uint64))
    assert rep.mean_silhouette == mean


def test_silhouette_singletons_and_errors():
    D = random_condensed(ScalarRng(12), 12)
    m = DistanceMatrix.from_condensed(12, D)
    res = kmedoids(m, KMedoidsConfig(k=6, restarts=2))   # k large: singleton clusters likely
    rep = api.silhouette_scores(m, res)
    sil, mean = sref(D, 12, res.medoids, res.assignment)
    assert np.array_equal(np.array(rep.silhouette), sil) and rep.mean_silhouette == mean
    with pytest.raises(api.SingleClusterUndefinedError):
        api.silhouette_scores(m, api.ClusterResult([res.medoids[0]], [res.medoids[0]] * 12, 0.0))
    with pytest.raises(InvalidArgumentsError):
        api.silhouette_scores(m, api.ClusterResult(res.medoids, res.assignment[:-1], 0.0))
    bad = list(res.assignment)
    bad[0] = next(j for j in range(12) if j not in res.medoids)
    with pytest.raises(InvalidArgumentsError):
        api.silhouette_scores(m, api.ClusterResult(res.medoids, bad, 0.0))


@pytest.mark.parametrize("spread", [0.0, 1e-16, 1e-15, 1e-13])
def test_update_near_ties_match_reference(spread):
    """Candidate sums equal up to rounding: the warp-tree sums only pre-filter, the
    reference's sequential sums decide (ties and last-ulp differences included)."""
    p = 300
    rng = np.random.default_rng(int(spread * 1e17) + 1)
    D = 1.0 + spread * rng.integers(0, 8, size=p * (p - 1) // 2).astype(np.float64)
    D[::7] *= 3.0  # a few larger terms so summation order matters
    m = DistanceMatrix.from_condensed(p, D)
    for medoids in ([0], [3, 150, 299], list(range(0, 300, 30))):
        asg = api.assign_to_medoids(m, medoids)
        got = api.update_medoids(m, medoids, asg)
        if oracle.have_ref():
            asg_ref, _, upd_ref = oracle.ref_sweep(D, p, medoids)
            assert asg == list(asg_ref)
            assert got == list(upd_ref), (spread, medoids)
        cfg = KMedoidsConfig(k=len(medoids), restarts=2, seed=7)
        check_same(D, p, cfg)


@pytest.mark.parametrize("cfgno,q", [(3, 900), (5, 300)])
def test_condensed_view_matches_square(monkeypatch, cfgno, q):
    """Matrices whose p x p square does not fit in HBM are swept straight from the
    condensed storage; forced here, every result must equal the square path's and the
    reference's."""
    ds = gen.make_config(cfgno).subset(q)
    m = api.build_matrix_packed(ds.samples, ds.offsets,
                                WarpWindow(None if ds.half_width < 0 else ds.half_width),
                                ds.auto_widen)
    cfg = KMedoidsConfig(k=ds.k, restarts=3, seed=1)
    a = kmedoids(m, cfg)
    sa = api.silhouette_scores(m, a)
    monkeypatch.setenv("DTWGPU_KM_CONDENSED", "1")
    m2 = DistanceMatrix.from_condensed(ds.p, m.condensed())
    b = kmedoids(m2, cfg)
    sb = api.silhouette_scores(m2, b)
    assert (a.medoids, a.assignment, a.total_cost) == (b.medoids, b.assignment, b.total_cost)
    assert sa.silhouette == sb.silhouette and sa.mean_silhouette == sb.mean_silhouette
    med, asg, cost = kref(m.condensed(), ds.p, cfg)
    assert b.medoids == list(med) and b.assignment == list(asg) and b.total_cost == cost


@pytest.mark.parametrize("cfgno,q", [(2, 120), (5, 200)])
def test_multi_device_context_matches_single(cfgno, q):
    """One context over two device contexts (dtwg_create_multi, both on the one B200 here):
    the slot ranges and restart blocks are split between them; matrix, clustering,
    observer trace and silhouettes must equal the single-device results."""
    ds = gen.make_config(cfgno).subset(q)
    single = api.Engine(0)
    multi = api.Engine(devices=[0, 0])
    a = single.build_condensed(ds.samples, ds.offsets, ds.half_width, ds.auto_widen)
    b = multi.build_condensed(ds.samples, ds.offsets, ds.half_width, ds.auto_widen)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    for eng in (single, multi):
        eng.adopt(a, ds.p)
    res = []
    for eng in (single, multi):
        trace = []
        med, asg, cost, br = eng.kmedoids(ds.p, ds.k, 6, 100, 3, 0, 6,
                                          lambda r, it, c: trace.append((r, it, c)))
        res.append((list(med), list(asg), cost, br, trace))
    assert res[0] == res[1]
    med, asg, cost = kref(a, ds.p, KMedoidsConfig(k=ds.k, restarts=6, seed=3))
    assert res[1][0] == list(med) and res[1][1] == list(asg) and res[1][2] == cost
    multi.close()
    single.close()


def test_python_api_devices_option():
    """api.build_matrix / kmedoids with devices=[0, 0]: the same matrix and clustering."""
    ds = gen.make_config(1).subset(60)
    data = [TimeSeries(f"s{i}", ds.series(i)) for i in range(ds.p)]
    a = build_matrix(data, WarpWindow.unlimited(), 1)
    b = build_matrix(data, WarpWindow.unlimited(), 1, devices=[0, 0])
    assert np.array_equal(a.condensed().view(np.uint64), b.condensed().view(np.uint64))
    cfg = KMedoidsConfig(k=4, restarts=5, seed=2)
    ta, tb = [], []
    ra = kmedoids(a, cfg, lambda r, i, c: ta.append((r, i, c)))
    rb = kmedoids(b, cfg, lambda r, i, c: tb.append((r, i, c)), devices=[0, 0])
    assert (ra.medoids, ra.assignment, ra.total_cost) == (rb.medoids, rb.assignment, rb.total_cost)
    assert ta == tb


@pytest.mark.parametrize("workers", ["1", "3", "8"])
def test_restart_workers_identical(monkeypatch, workers):
    """Restarts run concurrently on restart-worker streams (DTWGPU_KM_WORKERS); the result
    and the observer trace equal the sequential loop's and the reference's."""
    monkeypatch.setenv("DTWGPU_KM_WORKERS", workers)
    D = random_condensed(ScalarRng(31), 400)
    cfg = KMedoidsConfig(k=7, restarts=9, seed=5)
    trace = []
    got = kmedoids(DistanceMatrix.from_condensed(400, D), cfg,
                   lambda r, it, c: trace.append((r, it, c)))
    ref_trace = []
    med, asg, cost = kref(D, 400, cfg, lambda r, it, c: ref_trace.append((r, it, c)))
    assert got.medoids == list(med) and got.assignment == list(asg) and got.total_cost == cost
    assert trace == ref_trace


def test_acceptance_silhouette_fuzz():
    """acceptance_main.cpp:420-436 (criterion 9): 200 fuzzed instances (seed 0x9C, p in
    [3, 12], k in [2, p]) -- silhouettes in [-1, 1] and bit-identical to the reference."""
    rng = ScalarRng(0x9C)
    for trial in range(200):
        p = 3 + rng.next_below(10)
        D = random_condensed(rng, p)
        k = 2 + rng.next_below(p - 1)
        m = DistanceMatrix.from_condensed(p, D)
        res = kmedoids(m, KMedoidsConfig(k=k, seed=trial))
        rep = api.silhouette_scores(m, res)
        assert all(-1.0 <= v <= 1.0 for v in rep.silhouette)
        sil, mean = sref(D, p, res.medoids, res.assignment)
        assert np.array_equal(np.array(rep.silhouette), sil) and rep.mean_silhouette == mean


# ---------------------------------------------------- cluster-ordered layout (round 2)
@pytest.mark.parametrize("cfgno,q,k", [(3, 900, 24), (5, 300, 10), (1, 100, 4), (3, 700, 60)])
def test_cluster_layout_identical(monkeypatch, cfgno, q, k):
    """The candidate sums read a cluster-ordered copy of the square (km_host.cu
    ensure_layout; normally only for p >= 4096, forced here): medoids, labels, cost and the
    observer trace equal the plain-square path's and the reference's."""
    ds = gen.make_config(cfgno).subset(q)
    m = api.build_matrix_packed(ds.samples, ds.offsets,
                                WarpWindow(None if ds.half_width < 0 else ds.half_width),
                                ds.auto_widen)
    cfg = KMedoidsConfig(k=k, restarts=4, seed=2)
    runs = []
    for layout in ("0", "1"):
        monkeypatch.setenv("DTWGPU_KM_LAYOUT", layout)
        monkeypatch.setenv("DTWGPU_KM_LAYOUT_MIN_P", "2")
        mm = DistanceMatrix.from_condensed(ds.p, m.condensed())
        trace = []
        r = kmedoids(mm, cfg, lambda rr, it, c: trace.append((rr, it, c)))
        runs.append((r.medoids, r.assignment, r.total_cost, trace))
    assert runs[0] == runs[1]
    ref_trace = []
    med, asg, cost = kref(m.condensed(), ds.p, cfg, lambda rr, it, c: ref_trace.append((rr, it, c)))
    assert runs[1][:3] == (list(med), list(asg), cost) and runs[1][3] == ref_trace


@pytest.mark.parametrize("p,k", [(64, 9), (300, 40)])
def test_cluster_layout_duplicates_and_empty_clusters(monkeypatch, p, k):
    """Duplicated series (zero distances, collapsed medoids, refill) and many small clusters
    with the layout forced: identical to the reference."""
    monkeypatch.setenv("DTWGPU_KM_LAYOUT_MIN_P", "2")
    rng = np.random.default_rng(p)
    base = random_condensed(ScalarRng(p), p)
    sq = np.zeros((p, p))
    iu = np.triu_indices(p, 1)
    sq[iu] = base
    sq = sq + sq.T
    dup = rng.integers(0, p // 4, size=p)  # series j is a copy of series dup[j]
    sq = sq[np.ix_(dup, dup)]
    D = np.ascontiguousarray(sq[iu])
    check_same(D, p, KMedoidsConfig(k=k, restarts=5, seed=3))


@pytest.mark.parametrize("layout", ["0", "1"])
def test_many_clusters_radix_bucketing(monkeypatch, layout):
    """k > 256 takes the radix-sort bucketing (cub) instead of the per-cluster compaction;
    with and without the cluster-ordered copy the result equals the reference's."""
    monkeypatch.setenv("DTWGPU_KM_LAYOUT", layout)
    monkeypatch.setenv("DTWGPU_KM_LAYOUT_MIN_P", "2")
    p = 700
    D = random_condensed(ScalarRng(77), p)
    check_same(D, p, KMedoidsConfig(k=300, restarts=2, seed=4))
    m = DistanceMatrix.from_condensed(p, D)
    medoids = sorted(np.random.default_rng(3).choice(p, 290, replace=False).tolist())
    if oracle.have_ref():
        asg_ref, _, upd_ref = oracle.ref_sweep(D, p, medoids)
        assert api.assign_to_medoids(m, medoids) == list(asg_ref)
        assert api.update_medoids(m, medoids, list(asg_ref)) == list(upd_ref)
