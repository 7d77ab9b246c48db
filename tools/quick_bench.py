"""Quick per-config fill timing on one GPU (diagnostics; bench.py is the contract)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2307_04904_b200 import api, generators as gen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--fp32", action="store_true")
    ap.add_argument("--force", default="")  # family,G,R
    a = ap.parse_args()
    eng = api.engine(0)
    if a.force:
        f, g, r = (int(v) for v in a.force.split(","))
        eng.force_kernel(f, g, r)
    for c in [int(v) for v in a.configs.split(",")]:
        t = time.time()
        ds = gen.make_config(c)
        tg = time.time() - t
        eng.upload(ds.samples, ds.offsets)
        p = ds.p
        total = p * (p - 1) // 2
        cells = eng.count_cells(ds.half_width, ds.auto_widen, 0, total)
        out = torch.empty(total, dtype=torch.float64, device="cuda")
        for prec in ([0, 1] if a.fp32 else [0]):
            ms = []
            for _ in range(a.reps):
                t0 = time.time()
                eng.fill_slots(ds.half_width, ds.auto_widen, prec, 0, total, out.data_ptr())
                wall = time.time() - t0
                ms.append(eng.last_fill_ms())
            best = min(ms)
            print(json.dumps({"config": c, "precision": "fp32" if prec else "fp64", "p": p,
                              "cells": cells, "fill_ms": ms, "gcups": cells / best / 1e6,
                              "frac_fp64_peak": cells / best / 1e6 / 3722.0,
                              "pairs_per_s": total / best * 1e3, "host_wall_last_s": wall,
                              "gen_s": tg, "plan": eng.last_plan()}), flush=True)
        del out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
