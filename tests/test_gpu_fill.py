"""GPU parity of the DTW fill (through the C-ABI) against the oracle and the reference.

Bar (BASELINE.json north_star): fp64 distances bitwise-equal to the reference built
without FMA (the contract's 1e-12 relative is met with 0 ulp); fp32 mode within 1e-5
relative. Mirrors test_dtw.cpp, test_distance_matrix.cpp and acceptance criteria 1, 2, 7.
"""
import numpy as np
import pytest

import oracle
from paper_2307_04904_b200 import api, generators as gen
from paper_2307_04904_b200.api import (BandInfeasibleError, BuildStats, EmptyDatasetError,
                                       InvalidArgumentsError, InvalidSeriesError, TimeSeries,
                                       WarpWindow, build_matrix)
from tests.helpers import ScalarRng, assert_bitwise, pack, random_int_series

pytestmark = pytest.mark.gpu

U = WarpWindow.unlimited()


def ts(name, vals):
    return TimeSeries(name, np.array(vals, dtype=np.float64))


def gpu_pair(x, y, w):
    m = build_matrix([ts("x", x), ts("y", y)], w, 1)
    return m.distance(0, 1)


# ---------------------------------------------------------------- test_dtw.cpp:30-78
def test_identical_series_is_zero():
    assert gpu_pair([1, 2, 3], [1, 2, 3], U) == 0.0
    assert gpu_pair([1, 2, 3], [1, 2, 3], WarpWindow.banded(0)) == 0.0


def test_two_singletons():
    assert gpu_pair([0], [5], U) == 25.0


def test_one_to_many():
    assert gpu_pair([1, 2, 3], [1, 2, 2, 3], U) == 0.0


def test_zero_width_band_forces_diagonal():
    assert gpu_pair([0, 0, 0, 10], [10, 0, 0, 0], WarpWindow.banded(0)) == 200.0
    assert gpu_pair([0, 0, 0, 10], [10, 0, 0, 0], U) == oracle.dtw_brute_force(
        [0, 0, 0, 10], [10, 0, 0, 0])


def test_invalid_series_rejected():
    good = ts("good", [1, 2])
    with pytest.raises(InvalidSeriesError):
        build_matrix([ts("empty", []), good], U, 1)
    with pytest.raises(InvalidSeriesError):
        build_matrix([ts("nan", [1, np.nan]), good], U, 1)
    with pytest.raises(InvalidSeriesError):
        build_matrix([ts("inf", [np.inf]), good], U, 1)


def test_band_narrower_than_gap_rejected():
    x, y = [1, 2, 3, 4, 5], [1, 2]
    with pytest.raises(BandInfeasibleError):
        build_matrix([ts("x", x), ts("y", y)], WarpWindow.banded(2), 1)
    assert gpu_pair(x, y, WarpWindow.banded(3)) == oracle.dtw_brute_force(x, y, 3)


# ---------------------------------------------------------------- test_dtw.cpp:80-124
def _random_pairs(seed, count, max_len):
    rng = ScalarRng(seed)
    out = []
    for _ in range(count):
        x = random_int_series(rng, max_len, -5, 5)
        y = random_int_series(rng, max_len, -5, 5)
        gap = abs(len(x) - len(y))
        windows = [-1] + [hw for hw in (0, 1, 2) if hw >= gap]
        w = windows[rng.next_below(len(windows))]
        out.append((x, y, w))
    return out


@pytest.mark.parametrize("seed,count", [(20240601, 500), (0xAC5E01, 10000)])  # acceptance_main.cpp:101-125
def test_matches_exhaustive_oracle_on_random_small_pairs(eng, seed, count):
    pairs = _random_pairs(seed, count, 8)
    for w in (-1, 0, 1, 2):
        sel = [(x, y) for (x, y, ww) in pairs if ww == w]
        rows = []
        for x, y in sel:
            rows += [x, y]
        samples, offsets = pack(rows)
        # auto_widen so that cross pairs (not in the reference test) stay feasible
        got = eng.build_condensed(samples, offsets, w, auto_widen=True)
        want = oracle.build_condensed(samples, offsets, w, True)
        assert_bitwise(got, want, f"w={w}")
        p = len(rows)
        for t, (x, y) in enumerate(sel):
            i, j = 2 * t, 2 * t + 1
            slot = i * p - i * (i + 1) // 2 + (j - i - 1)
            assert got[slot] == oracle.dtw_brute_force(x, y, w)


def test_symmetric_and_band_monotone():
    rng = ScalarRng(99)
    for _ in range(30):
        x = random_int_series(rng, 8, -5, 5)
        y = random_int_series(rng, 8, -5, 5)
        gap = abs(len(x) - len(y))
        sat = max(len(x), len(y))
        prev = np.inf
        for hw in range(gap, sat + 1):
            c = gpu_pair(x, y, WarpWindow.banded(hw))
            assert c <= prev
            assert c == gpu_pair(y, x, WarpWindow.banded(hw))
            prev = c
        assert prev == gpu_pair(x, y, U)


# ---------------------------------------------------------------- every instantiation
FULL = [(2, 23), (4, 12), (8, 8), (16, 8), (16, 16), (32, 4), (32, 8), (32, 12), (32, 15),
        (32, 16)]
BAND = [(16, 7), (16, 9), (16, 11), (16, 13), (32, 3), (32, 5), (32, 7), (32, 9), (32, 13)]


def _walks(seed, lengths):
    rng = gen.SplitMix64(seed)
    rows = []
    for L in lengths:
        rows.append(np.cumsum(rng.gaussian(int(L))))
    return pack(rows)


FULL4 = [(2, 23), (4, 12), (8, 8), (16, 16), (32, 15), (32, 16), (2, 16), (1, 20), (1, 24),
         (1, 28), (1, 32)]


@pytest.mark.parametrize("G,R,fam", [(g, r, 0) for g, r in FULL] + [(g, r, 3) for g, r in FULL4])
@pytest.mark.parametrize("fp32", [False, True])
def test_full_family_every_instantiation(eng, G, R, fam, fp32):
    rng = np.random.default_rng(G * 100 + R)
    lengths = rng.integers(1, 700, size=14)
    lengths[:3] = [1, G * R, G * R + 1]
    samples, offsets = _walks(7 + G + R, lengths)
    for hw, aw in ((-1, False), (40, True), (3, True)):
        eng.force_kernel(fam, G, R)
        got = eng.build_condensed(samples, offsets, hw, aw, precision=1 if fp32 else 0)
        plan = eng.last_plan()
        assert f"full[G={G},R={R}" in plan and f"T={4 if fam == 3 else 2}" in plan, plan
        want = oracle.build_condensed(samples, offsets, hw, aw)
        if fp32:
            np.testing.assert_allclose(got, want, rtol=1e-5, atol=0)
        else:
            assert_bitwise(got, want, f"full G={G} R={R} hw={hw}")


@pytest.mark.parametrize("G,R,maxlen", [(16, 30, 1100), (1, 46, 200), (16, 32, 1100),
                                        (1, 56, 300), (1, 64, 300)])
def test_full_family_fp32_only_instantiations(eng, G, R, maxlen):
    """fp32-only Full instantiations (fill_table.h DTWG_FULL_CFGS_F32): every mask/pass
    variant within the fp32 tolerance (G = 1: one lane per pair, multi-pass when forced);
    fp64 requests fall back to the planner."""
    rng = np.random.default_rng(1630 + G)
    lengths = rng.integers(1, maxlen, size=12)
    lengths[:3] = [1, G * R, G * R + 1]
    samples, offsets = _walks(1630 + G, lengths)
    for hw, aw in ((-1, False), (40, True), (3, True)):
        eng.force_kernel(3, G, R)
        got = eng.build_condensed(samples, offsets, hw, aw, precision=1)
        assert f"full[G={G},R={R}" in eng.last_plan(), eng.last_plan()
        want = oracle.build_condensed(samples, offsets, hw, aw)
        np.testing.assert_allclose(got, want, rtol=1e-5, atol=0)
        eng.force_kernel(3, G, R)
        got64 = eng.build_condensed(samples, offsets, hw, aw, precision=0)
        assert f"full[G={G},R={R},T=4" not in eng.last_plan(), eng.last_plan()
        assert_bitwise(got64, want, f"fp64 fallback hw={hw}")


@pytest.mark.parametrize("G,R", [(2, 30), (4, 30), (8, 30)])
def test_full_family_fp64_multipass_instantiations(eng, G, R):
    """fp64-only multi-pass Full instantiations (fill_table.h DTWG_FULL_CFGS_F64): bitwise
    with unlimited, auto-widened and narrow bands over several passes; fp32 requests (and
    single-strip classes) fall back to the planner."""
    rng = np.random.default_rng(1730 + G)
    lengths = rng.integers(1, 4 * G * R, size=12)
    lengths[:4] = [1, G * R, G * R + 1, 3 * G * R + 7]
    samples, offsets = _walks(1730 + G, lengths)
    for hw, aw in ((-1, False), (40, True), (3, True), (G * R + 5, True)):
        eng.force_kernel(3, G, R)
        got = eng.build_condensed(samples, offsets, hw, aw, precision=0)
        assert f"full[G={G},R={R},T=4" in eng.last_plan(), eng.last_plan()
        want = oracle.build_condensed(samples, offsets, hw, aw)
        assert_bitwise(got, want, f"full64 G={G} R={R} hw={hw}")
        eng.force_kernel(3, G, R)
        got32 = eng.build_condensed(samples, offsets, hw, aw, precision=1)
        assert f"full[G={G},R={R},fp32" not in eng.last_plan(), eng.last_plan()
        np.testing.assert_allclose(got32, want, rtol=1e-5, atol=0)


@pytest.mark.parametrize("R,fam", [(28, 6), (24, 6), (20, 6), (16, 6)])
def test_full_one_lane_shared_y_instantiations(eng, R, fam):
    """One lane per pair with y in shared memory (dtw_full1s_kernel, fill_table.h
    DTWG_FULL1S_CFGS; forced as family 6): bitwise over several passes with unlimited,
    auto-widened and narrow bands, ragged lengths in one warp; fp32 falls back."""
    rng = np.random.default_rng(1830 + R)
    lengths = rng.integers(1, 12 * R, size=40)
    lengths[:4] = [1, R, R + 1, 9 * R + 7]
    samples, offsets = _walks(1830 + R, lengths)
    for hw, aw in ((-1, False), (40, True), (3, True), (2 * R + 5, True)):
        eng.force_kernel(fam, 1, R)
        got = eng.build_condensed(samples, offsets, hw, aw, precision=0)
        plan = eng.last_plan()
        assert f"full[G=1,R={R}" in plan and "ysm" in plan and f"T={4 if fam == 6 else 8}" in plan, plan
        want = oracle.build_condensed(samples, offsets, hw, aw)
        assert_bitwise(got, want, f"full1s R={R} hw={hw}")
        eng.force_kernel(fam, 1, R)
        got32 = eng.build_condensed(samples, offsets, hw, aw, precision=1)
        assert "ysm" not in eng.last_plan(), eng.last_plan()
        np.testing.assert_allclose(got32, want, rtol=1e-5, atol=0)


@pytest.mark.parametrize("G,R,fam", [(4, 12, 0), (4, 12, 3), (2, 23, 3), (8, 8, 0), (32, 4, 0),
                                     (32, 15, 3), (1, 20, 3), (2, 16, 3), (1, 28, 3)])
def test_full_family_band_edge_kill_cells(eng, G, R, fam):
    """Banded Full fills force only the cell just past each band edge per row to +inf (the
    rest of the out-of-band region comes out +inf by itself, dtw_kernels.cuh FullRows):
    narrow bands where both kill cells sit in one lane's strip (2hw+2 < R), bands around
    the strip width, equal and near-equal lengths (no auto-widening), multi-pass pairs."""
    W = G * R
    lengths = [1, 2, 5, W - 1, W, W + 1, 2 * W + 3, 150, 150, 151, 300, 301, 303]
    samples, offsets = _walks(4242 + G * R, lengths)
    for hw in (0, 1, 2, 5, R - 1, R, W // 2, W - 1, W, W + 1, 149):
        eng.force_kernel(fam, G, R)
        got = eng.build_condensed(samples, offsets, hw, True)
        assert f"full[G={G},R={R}" in eng.last_plan(), eng.last_plan()
        want = oracle.build_condensed(samples, offsets, hw, True)
        assert_bitwise(got, want, f"full G={G} R={R} fam={fam} hw={hw}")


RING = [(8, 16), (8, 26), (16, 8), (16, 14), (32, 6)]
UNIT = [(8, 26, 3), (8, 26, 5), (16, 14, 3), (16, 13, 2), (16, 20, 3), (16, 26, 3), (32, 20, 3),
        (32, 26, 3)]  # ring with U units per lane


@pytest.mark.parametrize("G,R,family", [(g, r, 1) for g, r in BAND] +
                         [(g, r, 4) for g, r in RING] +  # 4: smem ring
                         [(g, r, 10 + u) for g, r, u in UNIT])
@pytest.mark.parametrize("fp32", [False, True])
def test_band_family_every_instantiation(eng, G, R, fp32, family):
    rng = np.random.default_rng(G * 1000 + R)
    kmax = G * R
    for hw in sorted({0, 1, (kmax - 1) // 2, max((kmax - 1) // 2 - 3, 0), 7}):
        if 2 * hw + 1 > kmax:
            continue
        base = int(rng.integers(hw + 2, max(400, hw + 3)))
        lengths = [base + int(d) for d in rng.integers(-hw, hw + 1, size=10)]
        lengths = [max(L, 1) for L in lengths]
        samples, offsets = _walks(11 + hw, lengths)
        eng.force_kernel(family, G, R)
        got = eng.build_condensed(samples, offsets, hw, True, precision=1 if fp32 else 0)
        plan = eng.last_plan()
        want = oracle.build_condensed(samples, offsets, hw, True)
        if fp32:
            np.testing.assert_allclose(got, want, rtol=1e-5, atol=0)
        else:
            assert_bitwise(got, want, f"band G={G} R={R} hw={hw} plan={plan}")


def test_band_unit_fp32_only_wide_lanes(eng):
    """fp32-only unit-ring band kernel with wide lanes (fill_table.h DTWG_UNIT_CFGS_F32:
    G=4 R=52 U=3), over kill positions from hw = 0 to the widest band it covers."""
    G, R, U = 4, 52, 3
    rng = np.random.default_rng(452)
    for hw in (0, 1, 7, 40, 100, 101, 103):
        base = int(rng.integers(hw + 2, max(400, hw + 3)))
        lengths = [max(base + int(d), 1) for d in rng.integers(-hw, hw + 1, size=10)]
        samples, offsets = _walks(23 + hw, lengths)
        eng.force_kernel(10 + U, G, R)
        got = eng.build_condensed(samples, offsets, hw, True, precision=1)
        assert f"band[G={G},R={R},fp32" in eng.last_plan(), eng.last_plan()
        want = oracle.build_condensed(samples, offsets, hw, True)
        np.testing.assert_allclose(got, want, rtol=1e-5, atol=0)


STRIP = [15, 8]


@pytest.mark.parametrize("R", STRIP)
@pytest.mark.parametrize("fp32", [False, True])
def test_strip_family_every_instantiation(eng, R, fp32):
    """Long-pair family: column strips of one pair pipelined over warps (forced here on
    ragged pairs of 1..6 strips, unlimited, widened and narrow bands)."""
    rng = np.random.default_rng(R)
    lengths = rng.integers(1, 1500, size=12)
    lengths[:3] = [1, 32 * R, 32 * R + 1]
    samples, offsets = _walks(5 + R, lengths)
    for hw, aw in ((-1, False), (40, True), (3, True), (700, True)):
        eng.force_kernel(5, 32, R)
        got = eng.build_condensed(samples, offsets, hw, aw, precision=1 if fp32 else 0)
        plan = eng.last_plan()
        assert f"strip[G=32,R={R}" in plan, plan
        want = oracle.build_condensed(samples, offsets, hw, aw)
        if fp32:
            np.testing.assert_allclose(got, want, rtol=1e-5, atol=0)
        else:
            assert_bitwise(got, want, f"strip R={R} hw={hw}")


@pytest.mark.parametrize("lengths,hw", [([6000, 5000, 7000], -1), ([100000, 99000], 300),
                                        ([3000] * 5, -1)])
def test_few_long_pairs_use_the_strip_pipeline(eng, lengths, hw):
    """Few long pairs (the reference's 1e5-sample case, acceptance_main.cpp:153-187):
    the planner spreads each pair's strips over the GPU; bit-identical to the oracle."""
    samples, offsets = _walks(0x5771 + len(lengths), lengths)
    got = eng.build_condensed(samples, offsets, hw, True)
    assert "strip[" in eng.last_plan(), eng.last_plan()
    want = oracle.build_condensed(samples, offsets, hw, True)
    assert_bitwise(got, want, f"plan={eng.last_plan()}")


# ---------------------------------------------------------------- configs (oracle-sized)
@pytest.mark.parametrize("cfg,q", [(1, 100), (2, 60), (3, 400), (4, 6), (5, 70)])
def test_config_parity_bitwise(eng, cfg, q):
    ds = gen.make_config(cfg).subset(q)
    got = eng.build_condensed(ds.samples, ds.offsets, ds.half_width, ds.auto_widen)
    want = oracle.build_condensed(ds.samples, ds.offsets, ds.half_width, ds.auto_widen)
    assert_bitwise(got, want, f"c{cfg}[:{q}] plan={eng.last_plan()}")


def test_config4_fp32_within_tolerance(eng):
    ds = gen.config4().subset(8)
    got = eng.build_condensed(ds.samples, ds.offsets, -1, precision=1)
    want = oracle.build_condensed(ds.samples, ds.offsets, -1)
    rel = np.abs(got - want) / np.abs(want)
    assert rel.max() <= 1e-5, rel.max()


def test_slot_ranges_assemble_the_matrix(eng):
    import torch
    ds = gen.config5().subset(50)
    p = ds.p
    total = p * (p - 1) // 2
    full = eng.build_condensed(ds.samples, ds.offsets, ds.half_width, True)
    eng.upload(ds.samples, ds.offsets)
    parts = []
    cuts = [0, 1, 333, 334, 900, total]
    for b, e in zip(cuts[:-1], cuts[1:]):
        buf = torch.empty(max(e - b, 1), dtype=torch.float64, device="cuda")
        eng.fill_slots(ds.half_width, True, 0, b, e, buf.data_ptr())
        torch.cuda.synchronize()
        parts.append(buf[: e - b].cpu().numpy())
    assert_bitwise(np.concatenate(parts), full, "slot ranges")


# ---------------------------------------------------------------- matrix semantics
def test_single_series_gives_1x1():
    stats = BuildStats()
    m = build_matrix([ts("only", [1, 2, 3])], U, 1, stats)
    assert m.size() == 1 and m.distance(0, 0) == 0.0 and stats.evaluations == 0


def test_evaluations_and_worker_invariance():
    rng = ScalarRng(11)
    data = [ts(f"s{i}", random_int_series(rng, 12, -5, 5)) for i in range(17)]
    s1 = BuildStats()
    a = build_matrix(data, U, 1, s1)
    assert s1.evaluations == 17 * 16 // 2
    for w in (2, 3, 8, 64):
        st = BuildStats()
        b = build_matrix(data, U, w, st)
        assert st.evaluations == 17 * 16 // 2
        assert_bitwise(a.condensed(), b.condensed())
    samples, offsets = pack([d.samples for d in data])
    ref, ev = oracle.ref_build_condensed(samples, offsets, -1, workers=3) if oracle.have_ref() \
        else (oracle.build_condensed(samples, offsets), 136)
    assert_bitwise(a.condensed(), ref)


def test_build_rejects_bad_inputs():
    with pytest.raises(EmptyDatasetError):
        build_matrix([], U, 1)
    with pytest.raises(InvalidArgumentsError):
        build_matrix([ts("a", [1])], U, 0)
    with pytest.raises(InvalidSeriesError):
        build_matrix([ts("a", [1]), ts("a", [2])], U, 1)
    with pytest.raises(InvalidSeriesError):
        build_matrix([ts("a", [1]), ts("b", [])], U, 1)


def test_first_band_infeasible_pair():
    data = [ts("a", [1, 2]), ts("b", [1, 2, 3]), ts("c", [1, 2, 3, 4, 5, 6])]
    with pytest.raises(BandInfeasibleError) as ei:
        build_matrix(data, WarpWindow.banded(1), 1)
    assert ei.value.has_pair() and (ei.value.pair_i, ei.value.pair_j) == (0, 2)


def test_auto_widen_equals_gap_band():
    data = [ts("a", [1, 2]), ts("b", [1, 2, 3, 4, 5, 6])]
    widened = build_matrix(data, WarpWindow.banded(1), 1, None, True)
    assert widened.distance(0, 1) == gpu_pair([1, 2], [1, 2, 3, 4, 5, 6], WarpWindow.banded(4))


def test_memory_scale_long_pair(eng):
    """acceptance criterion 3 analogue: n = m = 20000 random walks, one pair."""
    rng = ScalarRng(0x3E)
    from tests.helpers import random_walk_series
    x = random_walk_series(rng, 20000)
    y = random_walk_series(rng, 20000)
    samples, offsets = pack([x, y])
    got = eng.build_condensed(samples, offsets, -1)
    assert got[0] == oracle.dtw(x, y, -1)


@pytest.mark.slow
def test_config4_fp32_full_matrix_error_histogram(eng):
    """fp32 mode on ALL 499,500 pairs of c4 (L=2844) against the bit-exact
    fp64 fill (itself equal to the reference): max relative error <= 1e-5."""
    import torch
    ds = gen.config4()
    eng.upload(ds.samples, ds.offsets)
    total = ds.p * (ds.p - 1) // 2
    a = torch.empty(total, dtype=torch.float64, device="cuda")
    b = torch.empty(total, dtype=torch.float64, device="cuda")
    eng.fill_slots(-1, False, 0, 0, total, a.data_ptr())
    eng.fill_slots(-1, False, 1, 0, total, b.data_ptr())
    rel = ((b - a).abs() / a.abs()).cpu().numpy()
    hist = np.histogram(np.log10(np.maximum(rel, 1e-16)), bins=[-16, -9, -8, -7, -6, -5.5, -5, 0])
    print("fp32 rel-error histogram (log10 bins):", hist[0].tolist(), "max", rel.max())
    assert rel.max() <= 1e-5, rel.max()


def test_streamed_build_matches_oracle():
    """Large outputs are filled in slot chunks and copied out through pinned staging while
    the fill continues; shrink the thresholds so a small input takes many chunks."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, oracle\n"
        "from paper_2307_04904_b200 import api, generators as gen\n"
        "from tests.helpers import assert_bitwise\n"
        "ds = gen.config3().subset(1500)\n"
        "m = api.build_matrix_packed(ds.samples, ds.offsets, api.WarpWindow(None), False)\n"
        "want = oracle.build_condensed(ds.samples, ds.offsets, -1, False)\n"
        "assert_bitwise(m.condensed(), want, 'streamed')\n"
        "ds = gen.config2().subset(300)\n"
        "m = api.build_matrix_packed(ds.samples, ds.offsets, api.WarpWindow(100), False)\n"
        "assert_bitwise(m.condensed(), oracle.build_condensed(ds.samples, ds.offsets, 100, False))\n"
        "print('ok')\n")
    env = dict(os.environ, DTWGPU_STREAM_MIN_BYTES="0", DTWGPU_CHUNK_FILL_MIN_BYTES="0",
               DTWGPU_STREAM_CHUNK="77777")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


# ---------------------------------------------------------------- full-size parity
@pytest.mark.slow
@pytest.mark.parametrize("cfg,q", [(1, 0), (2, 0), (3, 6000), (5, 1200)])
def test_full_size_matrix_bitwise_vs_reference(eng, cfg, q):
    """Whole matrices (c1, the headline c2; c3 and c5 at 6000 / 1200 series) against the
    UNMODIFIED reference's own multithreaded build_matrix (oracle/_ref) -- every pair,
    bit for bit, through the same kernels and plan the bench times."""
    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    import os
    ds = gen.make_config(cfg)
    if q:
        ds = ds.subset(q)
    got = eng.build_condensed(ds.samples, ds.offsets, ds.half_width, ds.auto_widen)
    plan = eng.last_plan()
    want, ev = oracle.ref_build_condensed(ds.samples, ds.offsets, ds.half_width, ds.auto_widen,
                                          workers=os.cpu_count() or 1)
    assert ev == ds.p * (ds.p - 1) // 2
    assert_bitwise(got, want, f"c{cfg} (p={ds.p}) plan={plan[:200]}")


@pytest.mark.parametrize("fp32", [False, True])
def test_one_lane_per_pair_kernels(eng, fp32):
    """One lane per pair, single strip (fp64: dtw_lane_kernel, y in shared memory; fp32:
    the Full family with G = 1): ragged lengths, unlimited, banded (kill cells) and
    auto-widened windows, pairs shorter than a row step; bit-exact in fp64. (Multi-pass
    one-lane fp64 strips are the G = 1 Full instantiations, tested above.)"""
    rng = np.random.default_rng(46)
    lengths = rng.integers(1, 47, size=40)
    lengths[:6] = [1, 2, 3, 45, 46, 46]
    samples, offsets = _walks(4646, lengths)
    for hw, aw in ((-1, False), (0, True), (1, True), (5, True), (20, True), (45, True)):
        eng.force_kernel(3 if fp32 else 0, 1, 46)
        got = eng.build_condensed(samples, offsets, hw, aw, precision=1 if fp32 else 0)
        assert "full[G=1,R=46" in eng.last_plan(), eng.last_plan()
        want = oracle.build_condensed(samples, offsets, hw, aw)
        if fp32:
            np.testing.assert_allclose(got, want, rtol=1e-5, atol=0)
        else:
            assert_bitwise(got, want, f"lane kernel hw={hw}")


@pytest.mark.parametrize("replan", ["0", "1"])
@pytest.mark.parametrize("prec", [0, 1])
def test_planner_mixed_classes_short_and_long(eng, prec, replan, monkeypatch):
    """Default planner over a ragged set whose short pairs (m <= 46) take the one-lane
    kernels and the rest the wavefront/band families, several classes in one fill. With
    the underfill re-plan (default) such tiny classes (435 one-lane pairs: 14 warps) are
    re-costed with their pair count and move to wider lane groups."""
    monkeypatch.setenv("DTWGPU_UNDERFILL_REPLAN", replan)
    rng = np.random.default_rng(4647)
    lengths = np.concatenate([rng.integers(2, 47, size=30), rng.integers(47, 400, size=20)])
    samples, offsets = _walks(4647, lengths)
    for hw, aw in ((-1, False), (12, True), (100, True)):
        got = eng.build_condensed(samples, offsets, hw, aw, precision=prec)
        want = oracle.build_condensed(samples, offsets, hw, aw)
        if prec:
            np.testing.assert_allclose(got, want, rtol=1e-5, atol=0)
        else:
            assert_bitwise(got, want, f"mixed hw={hw} plan={eng.last_plan()[:300]}")
        if hw < 0 and replan == "0":
            assert "G=1,R=46" in eng.last_plan(), eng.last_plan()
        if hw < 0 and replan == "1":
            assert "G=1,R=46" not in eng.last_plan(), eng.last_plan()


@pytest.mark.parametrize("prec", [0, 1])
def test_table_planner_equals_general_planner(eng, prec, monkeypatch):
    """The table-driven ragged planner (shape counts, parallel costing, one placement scan)
    makes exactly the plan of the general per-slot path: same classes, pair counts, cells
    and slot order (bitwise-equal matrices), on c5-like ragged data with underfilled
    classes (re-plan) and a slot sub-range."""
    ds = gen.config5(n=260, hi=700)
    total = ds.p * (ds.p - 1) // 2
    for sb, se in ((0, total), (1234, total - 777)):
        plans, outs = [], []
        for table in ("1", "0"):
            monkeypatch.setenv("DTWGPU_PLAN_TABLE", table)
            eng.upload(ds.samples, ds.offsets)
            import torch
            out = torch.empty(se - sb, dtype=torch.float64, device="cuda")
            eng.fill_slots(ds.half_width, ds.auto_widen, prec, sb, se, out.data_ptr())
            eng.synchronize()
            plans.append(eng.last_plan())
            outs.append(out.cpu().numpy())
        assert plans[0] == plans[1], plans
        assert np.array_equal(outs[0].view(np.uint64), outs[1].view(np.uint64))


@pytest.mark.parametrize("fam,G,R,prec", [(0, 1, 46, 0), (3, 1, 46, 1), (3, 16, 30, 1),
                                         (3, 2, 16, 0)])
def test_new_instantiations_on_tiny_inputs(eng, fam, G, R, prec):
    """Partial warps and single pairs through the one-lane, wide-lane and W = 32 kernels
    (p = 2, 3, 5; equal and unequal lengths; unlimited and auto-widened windows)."""
    for lens in ([7, 7], [1, 30], [46, 3, 17], [45, 46, 40, 12, 2]):
        samples, offsets = _walks(sum(lens), lens)
        for hw, aw in ((-1, False), (2, True)):
            eng.force_kernel(fam, G, R)
            got = eng.build_condensed(samples, offsets, hw, aw, precision=prec)
            want = oracle.build_condensed(samples, offsets, hw, aw)
            if prec:
                np.testing.assert_allclose(got, want, rtol=1e-5, atol=0)
            else:
                assert_bitwise(got, want, f"{G},{R} lens={lens} hw={hw}")


@pytest.mark.parametrize("cfg,prec,expect", [(1, 0, "full[G=32,R=16"),
                                             (2, 0, "band[G=8,R=26,kr=19,P=1,ring,U=3]"),
                                             (4, 0, "full[G=1,R=32,T=4]"),
                                             (4, 1, "full[G=1,R=64,fp32,T=4]"),
                                             (3, 1, "full[G=1,R=46,fp32,T=4,1strip]"),
                                             (3, 0, "full[G=1,R=46,T=2,1strip]"),
                                             (1, 1, "full[G=16,R=32,fp32,T=4,1strip]"),
                                             (2, 1, "band[G=4,R=52,fp32,kr=45,P=1,ring,U=3]")])
def test_planner_picks_the_measured_best(eng, cfg, prec, expect):
    """The cost model's choices on the benchmark configs (profiles/round1_*: the sweeps
    that calibrated it); guards against a model change silently regressing a config."""
    ds = gen.make_config(cfg)
    eng.upload(ds.samples, ds.offsets)
    p = ds.p
    import torch
    out = torch.empty(p * (p - 1) // 2, dtype=torch.float64, device="cuda")
    eng.fill_slots(ds.half_width, ds.auto_widen, prec, 0, p * (p - 1) // 2, out.data_ptr())
    assert expect in eng.last_plan(), eng.last_plan()


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [4, 5])
def test_full_size_properties(eng, cfg):
    """Full-size c4 / c5 (4e12 cells: beyond a CPU oracle in test time) through
    size-independent properties: the matrix of the REVERSED dataset is the same matrix
    with rows/columns permuted, bit for bit (DTW is symmetric bitwise: (a-b)^2 == (b-a)^2
    and min is commutative), and 64 random pairs equal the oracle."""
    import torch
    ds = gen.make_config(cfg)
    p = ds.p
    total = p * (p - 1) // 2
    a = torch.empty(total, dtype=torch.float64, device="cuda")
    eng.upload(ds.samples, ds.offsets)
    eng.fill_slots(ds.half_width, ds.auto_widen, 0, 0, total, a.data_ptr())
    A = a.cpu().numpy()
    lens = np.diff(ds.offsets)
    rows = [ds.samples[ds.offsets[i]:ds.offsets[i + 1]] for i in range(p)][::-1]
    rs, ro = pack(rows)
    b = torch.empty(total, dtype=torch.float64, device="cuda")
    eng.upload(rs, ro)
    eng.fill_slots(ds.half_width, ds.auto_widen, 0, 0, total, b.data_ptr())
    B = b.cpu().numpy()
    # slot of (i, j), i < j, in a p-series condensed matrix
    rng = np.random.default_rng(cfg)
    i = rng.integers(0, p, size=200000)
    j = rng.integers(0, p, size=200000)
    keep = i != j
    i, j = np.minimum(i[keep], j[keep]), np.maximum(i[keep], j[keep])
    off = lambda r: r * p - r * (r + 1) // 2
    sa = off(i) + (j - i - 1)
    ri, rj = p - 1 - j, p - 1 - i  # reversed indices, ri < rj
    sb = off(ri) + (rj - ri - 1)
    assert_bitwise(A[sa], B[sb], f"c{cfg} reversed-order symmetry")
    # and the whole matrices hold the same multiset of values
    assert np.array_equal(np.sort(A), np.sort(B))
    for t in range(64):
        x = ds.series(int(i[t]))
        y = ds.series(int(j[t]))
        hw = int(gen.effective_half_width(lens[i[t]], lens[j[t]], ds.half_width, ds.auto_widen))
        assert A[sa[t]] == oracle.dtw(x, y, hw), (cfg, int(i[t]), int(j[t]))


def test_multi_device_context_edge_cases():
    """One context over three device contexts (all on the one B200 here): tiny matrices
    (empty device ranges), ragged auto-widened pairs, and the first band-infeasible pair
    reported exactly as by a single device."""
    multi = api.Engine(devices=[0, 0, 0])
    single = api.Engine(0)
    try:
        for rows in ([[1.0, 2.0], [2.0, 3.0]], [[1.0], [2.0, 3.0], [4.0, 5.0, 6.0]]):
            s, o = pack(rows)
            assert_bitwise(multi.build_condensed(s, o), single.build_condensed(s, o))
        ds = gen.config5().subset(90)
        assert_bitwise(multi.build_condensed(ds.samples, ds.offsets, 40, True),
                       single.build_condensed(ds.samples, ds.offsets, 40, True))
        s, o = pack([[1, 2], [1, 2, 3], [1, 2, 3, 4, 5, 6]])
        with pytest.raises(BandInfeasibleError) as ei:
            multi.build_condensed(s, o, 1, False)
        assert (ei.value.pair_i, ei.value.pair_j) == (0, 2)
    finally:
        multi.close()
        single.close()


def test_single_pair_dtw_distance_api():
    """api.dtw_distance (dtw.hpp:40-75 on the GPU): KATs, a long pair, and the error."""
    assert api.dtw_distance(ts("a", [0]), ts("b", [5]), U) == 25.0
    assert api.dtw_distance(ts("a", [0, 0, 0, 10]), ts("b", [10, 0, 0, 0]),
                            WarpWindow.banded(0)) == 200.0
    rng = ScalarRng(0xD7)
    from tests.helpers import random_walk_series
    x, y = random_walk_series(rng, 6000), random_walk_series(rng, 5200)
    assert api.dtw_distance(ts("x", x), ts("y", y), WarpWindow.banded(900)) == \
        oracle.dtw(x, y, 900)
    with pytest.raises(BandInfeasibleError) as ei:
        api.dtw_distance(ts("x", x), ts("y", y), WarpWindow.banded(10))
    assert not ei.value.has_pair() and "length gap of 800" in str(ei.value)


def test_staged_build_validation_order(eng):
    """Outputs >= 1 MB overlap the per-series checks with the fill; the errors and their
    order stay the reference's (pairwise.hpp:65-79): InvalidSeries before BandInfeasible."""
    rng = np.random.default_rng(4)
    rows = [rng.normal(size=int(rng.integers(20, 60))) for _ in range(700)]  # 244 650 pairs
    s, o = pack(rows)
    got = eng.build_condensed(s, o, -1)
    assert_bitwise(got[:5000], oracle.build_condensed(s, o, -1)[:5000])
    bad = s.copy()
    bad[o[400] + 3] = np.nan
    with pytest.raises(InvalidSeriesError):
        eng.build_condensed(bad, o, 2)          # infeasible band too: the series error wins
    with pytest.raises(BandInfeasibleError) as ei:
        eng.build_condensed(s, o, 2)
    assert ei.value.has_pair()
    assert_bitwise(eng.build_condensed(s, o, -1), got)  # the context is usable afterwards


def test_acceptance_band_properties():
    """acceptance_main.cpp:129-149 (criterion 2) at its size: 1000 pairs (seed 0xBA2D, up to
    24 samples) -- cost non-increasing as the band widens from the gap to max(n, m), and
    equal to the unlimited window at saturation. All pairs go through the GPU together,
    one build per half-width (auto-widen keeps the cross pairs feasible)."""
    rng = ScalarRng(0xBA2D)
    pairs = [(random_int_series(rng, 24, -5, 5), random_int_series(rng, 24, -5, 5))
             for _ in range(1000)]
    rows = [r for xy in pairs for r in xy]
    s, o = pack(rows)
    p = len(rows)
    slot = [2 * t * p - 2 * t * (2 * t + 1) // 2 for t in range(len(pairs))]  # (2t, 2t+1)
    unl = api.engine(0).build_condensed(s, o, -1)
    prev = np.full(len(pairs), np.inf)
    for hw in range(0, 25):
        d = api.engine(0).build_condensed(s, o, hw, True)
        for t, (x, y) in enumerate(pairs):
            gap, sat = abs(len(x) - len(y)), max(len(x), len(y))
            if hw < gap or hw > sat:
                continue
            c = d[slot[t]]
            assert c <= prev[t], (t, hw)
            prev[t] = c
            if hw == sat:
                assert c == unl[slot[t]], (t, hw)


@pytest.mark.slow
def test_acceptance_memory_at_scale():
    """acceptance_main.cpp:153-187 (criterion 3): the 1e5-sample random-walk pair (seed 0x3E),
    through the strip pipeline, finite, the p = 2 build equal to dtw_distance, and bit-
    identical to the reference (one CPU core, ~30 s)."""
    from tests.helpers import random_walk_series
    rng = ScalarRng(0x3E)
    x = random_walk_series(rng, 100000)
    y = random_walk_series(rng, 100000)
    d = api.dtw_distance(ts("x", x), ts("y", y), U)
    s, o = pack([x, y])
    e = api.engine(0)
    assert e.build_condensed(s, o, -1)[0] == d and "strip[" in e.last_plan()
    assert np.isfinite(d) and d >= 0.0
    want = oracle.ref_dtw(x, y, -1) if oracle.have_ref() else oracle.dtw(x, y, -1)
    assert d == want
