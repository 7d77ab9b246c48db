"""Regenerate the golden fixtures from the REFERENCE itself (oracle/_ref, i.e. the
unmodified dtwclust headers compiled in place by oracle/Makefile).

    python tests/golden/make_golden.py      # needs /root/reference at build time

Inputs are stored next to the outputs, so the fixtures do not depend on numpy's
transcendental functions being bit-identical on the machine that replays them.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2307_04904_b200 import generators as gen  # noqa: E402
from tests.helpers import ScalarRng, random_condensed, random_int_series  # noqa: E402

SUBSETS = {1: 40, 2: 30, 3: 200, 4: 4, 5: 40}


def main():
    assert oracle.have_ref(), "oracle/_ref/libdtwclust_ref.so missing (run make -C oracle)"
    arrays = {}
    meta = {"generator": "tests/golden/make_golden.py", "reference": "oracle/_ref (dtwclust "
            "headers from /root/reference/proj/include, -O3 -DNDEBUG -ffp-contract=off)",
            "configs": {}, "kmedoids": {}}
    for c, q in SUBSETS.items():
        ds = gen.make_config(c).subset(q)
        cond, ev = oracle.ref_build_condensed(ds.samples, ds.offsets, ds.half_width,
                                              ds.auto_widen, workers=4)
        arrays[f"c{c}_samples"] = ds.samples
        arrays[f"c{c}_offsets"] = ds.offsets
        arrays[f"c{c}_condensed"] = cond
        meta["configs"][f"c{c}"] = {"series": ds.p, "half_width": ds.half_width,
                                    "auto_widen": ds.auto_widen, "evaluations": ev}
        if ds.k:
            k = min(ds.k, ds.p)
            med, asg, cost = oracle.ref_kmedoids(cond, ds.p, k, 3, 100, 0)
            arrays[f"c{c}_km_medoids"] = med
            arrays[f"c{c}_km_assignment"] = asg
            arrays[f"c{c}_km_cost"] = np.array([cost])
            if k >= 2:
                sil, mean = oracle.ref_silhouette(cond, ds.p, med, asg)
                arrays[f"c{c}_silhouette"] = sil
                arrays[f"c{c}_silhouette_mean"] = np.array([mean])
            meta["kmedoids"][f"c{c}"] = {"k": k, "restarts": 3, "max_iterations": 100, "seed": 0}
    # test_dtw.cpp:80-95 pairs (seed 20240601), reference distances and brute force.
    rng = ScalarRng(20240601)
    xs, ys, ws, d_ref, d_bf = [], [], [], [], []
    for _ in range(500):
        x = random_int_series(rng, 8, -5, 5)
        y = random_int_series(rng, 8, -5, 5)
        gap = abs(len(x) - len(y))
        windows = [-1] + [hw for hw in (0, 1, 2) if hw >= gap]
        w = windows[rng.next_below(len(windows))]
        xs.append(x)
        ys.append(y)
        ws.append(w)
        d_ref.append(oracle.ref_dtw(x, y, w))
        d_bf.append(oracle.ref_dtw_brute_force(x, y, w))
    rows = xs + ys
    lens = np.array([len(r) for r in rows])
    arrays["pairs_samples"] = np.concatenate(rows)
    arrays["pairs_offsets"] = np.concatenate([[0], np.cumsum(lens)])
    arrays["pairs_windows"] = np.array(ws)
    arrays["pairs_dtw"] = np.array(d_ref)
    arrays["pairs_bruteforce"] = np.array(d_bf)
    # test_kmedoids.cpp-style random matrices.
    for p, k, seed in [(20, 4, 20240101), (25, 4, 99), (30, 5, 1234)]:
        D = random_condensed(ScalarRng(p + k), p)
        trace = []
        med, asg, cost = oracle.ref_kmedoids(D, p, k, 6, 100, seed,
                                             lambda r, it, c: trace.append((r, it, c)))
        key = f"rand{p}"
        arrays[f"{key}_D"] = D
        arrays[f"{key}_medoids"] = med
        arrays[f"{key}_assignment"] = asg
        arrays[f"{key}_cost"] = np.array([cost])
        arrays[f"{key}_trace"] = np.array(trace)
        meta["kmedoids"][key] = {"k": k, "restarts": 6, "max_iterations": 100, "seed": seed}
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote", os.path.join(HERE, "golden.npz"))


if __name__ == "__main__":
    main()
