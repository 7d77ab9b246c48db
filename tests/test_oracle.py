"""CPU tests: pin the oracle (oracle/dtw_oracle.c) before trusting it.

Pins: the reference's own known answers (test_dtw.cpp, test_kmedoids.cpp), the golden
vectors produced by the reference itself (tests/golden, made by make_golden.py from
oracle/_ref), and -- when oracle/_ref is present -- a live comparison with the reference.
"""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2307_04904_b200 import generators as gen
from tests.helpers import ScalarRng, assert_bitwise, pack, random_condensed, random_int_series

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "golden.npz"))
META = json.load(open(os.path.join(HERE, "golden", "golden.json")))


# ---------------------------------------------------------------- known answers
def test_known_answers():
    assert oracle.dtw([1, 2, 3], [1, 2, 3]) == 0.0
    assert oracle.dtw([1, 2, 3], [1, 2, 3], 0) == 0.0
    assert oracle.dtw([0], [5]) == 25.0
    assert oracle.dtw([1, 2, 3], [1, 2, 2, 3]) == 0.0
    assert oracle.dtw([0, 0, 0, 10], [10, 0, 0, 0], 0) == 200.0
    assert oracle.dtw([0, 0, 0, 10], [10, 0, 0, 0]) == oracle.dtw_brute_force(
        [0, 0, 0, 10], [10, 0, 0, 0])
    assert oracle.dtw_brute_force([0, 0], [1, 1]) == 2.0
    assert oracle.dtw([1, 2, 3, 4, 5], [1, 2], 3) == oracle.dtw_brute_force([1, 2, 3, 4, 5],
                                                                              [1, 2], 3)


def test_golden_random_pairs_match_bruteforce_and_reference():
    s, o, w = GOLD["pairs_samples"], GOLD["pairs_offsets"], GOLD["pairs_windows"]
    n = len(w)
    for t in range(n):
        x = s[o[t]:o[t + 1]]
        y = s[o[n + t]:o[n + t + 1]]
        assert oracle.dtw(x, y, int(w[t])) == GOLD["pairs_dtw"][t]
        assert oracle.dtw_brute_force(x, y, int(w[t])) == GOLD["pairs_bruteforce"][t]


def test_symmetry_and_band_monotonicity():
    rng = ScalarRng(0xBA2D)
    for _ in range(200):
        x = random_int_series(rng, 24, -5, 5)
        y = random_int_series(rng, 24, -5, 5)
        gap = abs(len(x) - len(y))
        prev = np.inf
        for hw in range(gap, max(len(x), len(y)) + 1):
            c = oracle.dtw(x, y, hw)
            assert c <= prev and c == oracle.dtw(y, x, hw)
            prev = c
        assert prev == oracle.dtw(x, y, -1)


# ---------------------------------------------------------------- golden matrices
@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_golden_config_matrices(c):
    m = META["configs"][f"c{c}"]
    got = oracle.build_condensed(GOLD[f"c{c}_samples"], GOLD[f"c{c}_offsets"], m["half_width"],
                                 m["auto_widen"])
    assert_bitwise(got, GOLD[f"c{c}_condensed"], f"c{c}")
    assert m["evaluations"] == m["series"] * (m["series"] - 1) // 2


@pytest.mark.parametrize("key", ["c1", "c3", "c5", "rand20", "rand25", "rand30"])
def test_golden_kmedoids(key):
    km = META["kmedoids"][key]
    if key.startswith("rand"):
        D = GOLD[f"{key}_D"]
        p = int((1 + np.sqrt(1 + 8 * len(D))) / 2)
        trace = []
        med, asg, cost = oracle.kmedoids(D, p, km["k"], km["restarts"], km["max_iterations"],
                                         km["seed"], lambda r, i, c: trace.append((r, i, c)))
        np.testing.assert_array_equal(np.array(trace), GOLD[f"{key}_trace"])
    else:
        D = GOLD[f"{key}_condensed"]
        p = META["configs"][key]["series"]
        med, asg, cost = oracle.kmedoids(D, p, km["k"], km["restarts"], km["max_iterations"],
                                         km["seed"])
    np.testing.assert_array_equal(med, GOLD[f"{key}_km_medoids" if key[0] == "c" else f"{key}_medoids"])
    np.testing.assert_array_equal(asg, GOLD[f"{key}_km_assignment" if key[0] == "c" else f"{key}_assignment"])
    assert cost == GOLD[f"{key}_km_cost" if key[0] == "c" else f"{key}_cost"][0]


def test_kmedoids_k_equals_p_and_duplicates():
    D = random_condensed(ScalarRng(1), 6)
    med, asg, cost = oracle.kmedoids(D, 6, 6, 2)
    assert cost == 0.0 and list(asg) == list(range(6))
    samples, offsets = pack([[1.0, 2.0, 3.0]] * 6)
    D = oracle.build_condensed(samples, offsets)
    med, asg, cost = oracle.kmedoids(D, 6, 3, 10, 100, 9)
    assert cost == 0.0 and all(asg[m] == m for m in med)


# ---------------------------------------------------------------- live reference
needs_ref = pytest.mark.skipif(not oracle.have_ref(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("c,q", [(1, 25), (2, 12), (3, 80), (5, 25)])
def test_oracle_equals_reference_live(c, q):
    ds = gen.make_config(c).subset(q)
    a = oracle.build_condensed(ds.samples, ds.offsets, ds.half_width, ds.auto_widen)
    b, ev = oracle.ref_build_condensed(ds.samples, ds.offsets, ds.half_width, ds.auto_widen,
                                       workers=3)
    assert_bitwise(a, b)
    assert ev == q * (q - 1) // 2


@needs_ref
def test_reference_errors_and_first_infeasible_pair():
    samples, offsets = pack([[1, 2], [1, 2, 3], [1, 2, 3, 4, 5, 6]])
    with pytest.raises(oracle.RefError) as ei:
        oracle.ref_build_condensed(samples, offsets, 1)
    assert ei.value.code == 8 and ei.value.pair == (0, 2)
    assert oracle.first_infeasible(offsets, 1) == (0, 2)
    with pytest.raises(oracle.RefError) as ei:
        oracle.ref_build_condensed(samples, offsets, -1, workers=0)
    assert ei.value.code == 2


@needs_ref
def test_kmedoids_oracle_equals_reference_live():
    for p, k, seed in [(40, 3, 7), (60, 6, 11)]:
        D = random_condensed(ScalarRng(p), p)
        a = oracle.kmedoids(D, p, k, 4, 100, seed)
        b = oracle.ref_kmedoids(D, p, k, 4, 100, seed)
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])
        assert a[2] == b[2]


# ---------------------------------------------------------------- host helpers
def test_pair_cells_formula_matches_oracle():
    rng = np.random.default_rng(3)
    for _ in range(300):
        n, m = (int(v) for v in rng.integers(1, 300, size=2))
        for hw in (-1, 0, 1, 5, 50, abs(n - m), abs(n - m) + 3):
            if hw >= 0 and hw < abs(n - m):
                continue
            want = oracle.pair_cells(n, m, hw)
            got = int(gen.pair_cells(np.array([n]), np.array([m]), hw)[0])
            assert got == want, (n, m, hw)


def test_splitmix_matches_reference_rng():
    import ctypes
    st = ctypes.c_uint64(2307049042)
    want = [oracle.lib().oracle_splitmix_next(ctypes.byref(st)) for _ in range(100)]
    got = gen.SplitMix64(2307049042).next_u64(100)
    assert [int(v) for v in got] == want


def test_generators_shapes():
    assert gen.config1().p == 100 and set(gen.config1().lengths) == {500}
    ds = gen.config5(n=200)
    assert ds.lengths.min() >= 50 and ds.lengths.max() <= 1500 and ds.auto_widen
    # z-normalised: mean 0, population std 1
    s = gen.config2(n=3).series(1)
    assert abs(s.mean()) < 1e-12 and abs(s.std() - 1) < 1e-12


@pytest.mark.parametrize("c", [1, 3, 5])
def test_golden_silhouette(c):
    """validation.hpp:30-79 restated, against the reference's own ScoreReport."""
    p = META["configs"][f"c{c}"]["series"]
    sil, mean = oracle.silhouette(GOLD[f"c{c}_condensed"], p, GOLD[f"c{c}_km_medoids"],
                                  GOLD[f"c{c}_km_assignment"])
    assert_bitwise(sil, GOLD[f"c{c}_silhouette"], f"c{c} silhouette")
    assert mean == GOLD[f"c{c}_silhouette_mean"][0]
