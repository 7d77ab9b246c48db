"""Sweep every compiled (family, G, R) on a config to calibrate the planner."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2307_04904_b200 import api, generators as gen  # noqa: E402

FULL = [(2, 23), (4, 12), (8, 8), (16, 8), (16, 16), (32, 4), (32, 8), (32, 12), (32, 15),
        (32, 16)]
BAND = [(16, 7), (16, 9), (16, 11), (16, 13), (32, 3), (32, 5), (32, 7), (32, 9), (32, 13)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--subset", type=int, default=0)
    ap.add_argument("--prec", type=int, default=0)
    ap.add_argument("--families", default="0,1,2")
    ap.add_argument("--cands", default="")  # explicit "family:G:R,..." (overrides --families)
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    ds = gen.make_config(a.config)
    if a.subset:
        ds = ds.subset(a.subset)
    eng = api.engine(0)
    eng.upload(ds.samples, ds.offsets)
    total = ds.p * (ds.p - 1) // 2
    cells = eng.count_cells(ds.half_width, ds.auto_widen, 0, total)
    out = torch.empty(total, dtype=torch.float64, device="cuda")
    cands = []
    fams = [int(v) for v in a.families.split(",")]
    if 0 in fams:
        cands += [(0, g, r) for g, r in FULL]
    if 1 in fams:
        cands += [(1, g, r) for g, r in BAND]
    if 2 in fams:
        cands += [(2, g, r) for g, r in BAND]
    if 4 in fams:
        cands += [(4, g, r) for g, r in [(8, 16), (8, 26), (16, 8), (16, 14), (32, 6)]]
    if 3 in fams:
        cands += [(3, g, r) for g, r in [(2, 23), (4, 12), (8, 8), (16, 16), (32, 15), (32, 16)]]
    if a.cands:
        cands = [tuple(int(v) for v in c.split(":")) for c in a.cands.split(",")]
    ref = None
    for fam, g, r in [(-1, 0, 0)] + cands:
        eng.force_kernel(fam, g, r)
        try:
            eng.fill_slots(ds.half_width, ds.auto_widen, a.prec, 0, total, out.data_ptr())
            eng.fill_slots(ds.half_width, ds.auto_widen, a.prec, 0, total, out.data_ptr())
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"force": [fam, g, r], "error": str(e)}), flush=True)
            continue
        ms = eng.last_fill_ms()
        for _ in range(a.reps - 1):
            eng.fill_slots(ds.half_width, ds.auto_widen, a.prec, 0, total, out.data_ptr())
            ms = min(ms, eng.last_fill_ms())
        plan = eng.last_plan()
        if ref is None:
            ref = out.clone()
        same = bool(torch.equal(out, ref)) if a.prec == 0 else None
        print(json.dumps({"config": a.config, "p": ds.p, "force": [fam, g, r], "ms": ms,
                          "gcups": cells / ms / 1e6, "plan": plan, "same": same}), flush=True)


if __name__ == "__main__":
    main()
