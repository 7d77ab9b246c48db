"""One fill of a (sub)config, for ncu captures: python tools/prof_fill.py --config 3 --subset 4000"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2307_04904_b200 import api, generators as gen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--subset", type=int, default=0)
    ap.add_argument("--prec", type=int, default=0)
    ap.add_argument("--force", default="")
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    ds = gen.make_config(a.config)
    if a.subset:
        ds = ds.subset(a.subset)
    eng = api.engine(0)
    if a.force:
        eng.force_kernel(*(int(v) for v in a.force.split(",")))
    eng.upload(ds.samples, ds.offsets)
    total = ds.p * (ds.p - 1) // 2
    out = torch.empty(total, dtype=torch.float64, device="cuda")
    for _ in range(a.reps):
        eng.fill_slots(ds.half_width, ds.auto_widen, a.prec, 0, total, out.data_ptr())
    cells = eng.count_cells(ds.half_width, ds.auto_widen, 0, total)
    print(f"config={a.config} p={ds.p} ms={eng.last_fill_ms():.3f} "
          f"gcups={cells / eng.last_fill_ms() / 1e6:.1f} plan={eng.last_plan()}")


if __name__ == "__main__":
    main()
