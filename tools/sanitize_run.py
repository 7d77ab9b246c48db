"""Small fills of every kernel family checked bit for bit against the oracle (no timing):
masked multi-pass Full strips (lane 0's unconditional boundary-column prefetch runs up to
TR*(G+1)+4 rows past the pair's last row, inside the kScratchPad rows of its group's
column), single-strip Full, the band/ring/unit kernels, the strip pipeline and the
k-medoids sweeps. Meant for `compute-sanitizer --tool memcheck python tools/sanitize_run.py`
-- plus the ADVICE r1 case: one lane per pair with one long series among many short ones
(every lane of a warp runs to the warp's longest pair; its prefetches past its own pair's
last row must stay inside the tail guard and its own scratch column)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2307_04904_b200 import api, generators as gen  # noqa: E402


def check(eng, samples, offsets, hw, aw, what):
    got = eng.build_condensed(samples, offsets, hw, aw)
    want = oracle.build_condensed(samples, offsets, hw, aw)
    if not np.array_equal(got.view(np.uint64), want.view(np.uint64)):
        raise AssertionError(f"{what}: mismatch (plan {eng.last_plan()})")
    print(f"{what}: ok  {eng.last_plan()[:90]}", flush=True)


def main():
    eng = api.engine(0)
    # planner's own choices on c2/c5-shaped data (band unit kernels, masked Full)
    for ds in (gen.config2(n=12, length=300), gen.config5(n=14, hi=500), gen.config1(n=8)):
        check(eng, ds.samples, ds.offsets, ds.half_width, ds.auto_widen, ds.name)
    # forced families on ragged lengths, incl. multi-pass masked Full (lane 0's boundary
    # prefetch runs past the pair's last row into the padded scratch)
    rng = np.random.default_rng(5)
    lens = rng.integers(1, 260, size=10)
    lens[:3] = [1, 48, 49]
    rows = [np.cumsum(rng.standard_normal(int(L))) for L in lens]
    samples = np.concatenate(rows)
    offsets = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(lens, out=offsets[1:])
    for fam, G, R in ((3, 4, 12), (0, 2, 23), (3, 32, 15), (0, 32, 16), (5, 32, 8)):
        for hw, aw in ((-1, False), (20, True), (2, True)):
            eng.force_kernel(fam, G, R)
            check(eng, samples, offsets, hw, aw, f"forced fam={fam} G={G} R={R} hw={hw}")
    # one lane per pair (G = 1, register and shared-memory y), one long series among short
    # ones: lanes run to the warp's longest pair, prefetching far past their own ends
    lens = np.concatenate([[6000], rng.integers(2, 120, size=90)])
    rows = [np.cumsum(rng.standard_normal(int(L))) for L in lens]
    samples = np.concatenate(rows)
    offsets = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(lens, out=offsets[1:])
    for fam, G, R in ((3, 1, 32), (3, 1, 28), (6, 1, 24), (6, 1, 20), (0, 1, 46)):
        for hw, aw in ((-1, False), (50, True)):
            eng.force_kernel(fam, G, R)
            check(eng, samples, offsets, hw, aw, f"long+short fam={fam} G={G} R={R} hw={hw}")
    eng.force_kernel(-1, 0, 0)
    # k-medoids sweeps over the resident matrix
    ds = gen.config1(n=24)
    m = api.build_matrix_packed(ds.samples, ds.offsets, api.WarpWindow.unlimited())
    res = api.kmedoids(m, api.KMedoidsConfig(k=3, restarts=2))
    med, asg, cost = oracle.kmedoids(m.condensed(), ds.p, 3, 2, 100, 0)
    if res.medoids != list(med) or res.assignment != list(asg) or res.total_cost != cost:
        raise AssertionError("k-medoids mismatch")
    print("sanitize ok", flush=True)


if __name__ == "__main__":
    main()
