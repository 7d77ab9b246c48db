"""Single-GPU proxy for the multi-GPU fill: time every rank's shard alone.

bench.py --gpus N gives rank r the contiguous cell-balanced slot range
`distributed.cell_bounds(...)[r]`; the ranks share no data-path work
until the exchange, so the fill part of an N-GPU step is the slowest shard. This tool
fills each shard [b, e) of world N on the one GPU (rank by rank, plan per range as the
rank would build it) and reports

    fill efficiency(N) = T_fill(whole matrix) / (N * max_r T_fill(shard r))

i.e. the compute part of the strong-scaling efficiency the driver's SCALE run measures,
before the exchange. Diagnostics only (bench.py is the contract).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import ClockSampler  # noqa: E402
from paper_2307_04904_b200 import api, distributed as dd, generators as gen  # noqa: E402


def best_ms(eng, ds, prec, b, e, out, reps):
    ms = []
    for _ in range(reps + 1):  # first call plans + warms
        eng.fill_slots(ds.half_width, ds.auto_widen, prec, b, e, out.data_ptr())
        ms.append(eng.last_fill_ms())
    return min(ms[1:])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="4,3,5,2")
    ap.add_argument("--worlds", default="2,4,8")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--fp32", action="store_true")
    a = ap.parse_args()
    prec = 1 if a.fp32 else 0
    eng = api.engine(0)
    for c in [int(v) for v in a.configs.split(",")]:
        ds = gen.make_config(c)
        eng.upload(ds.samples, ds.offsets)
        total = ds.p * (ds.p - 1) // 2
        out = torch.empty(total, dtype=torch.float64, device="cuda")
        t1 = best_ms(eng, ds, prec, 0, total, out, a.reps)
        cells = eng.count_cells(ds.half_width, ds.auto_widen, 0, total)
        rec = {"config": c, "precision": "fp32" if prec else "fp64", "fill_ms_1": t1,
               "plan_1": eng.last_plan()[:300],
               "gcups_1": cells / t1 / 1e6, "worlds": {}}
        for w in [int(v) for v in a.worlds.split(",")]:
            bounds = dd.cell_bounds(ds.lengths, ds.half_width, ds.auto_widen, w)
            shard_ms, shard_cells, plans, clocks = [], [], [], []
            for b, e in bounds:
                with ClockSampler(0) as clk:
                    shard_ms.append(best_ms(eng, ds, prec, b, e, out, a.reps) if e > b else 0.0)
                cs = clk.summary()
                clocks.append([cs.get("sm_mhz"), cs.get("reasons")])
                shard_cells.append(eng.count_cells(ds.half_width, ds.auto_widen, b, e))
                plans.append(eng.last_plan()[:300])
            worst = max(shard_ms)
            rec["worlds"][w] = {"shard_ms": [round(v, 3) for v in shard_ms],
                                "shard_cells_frac": [round(v / cells, 4) for v in shard_cells],
                                "max_ms": worst,
                                "fill_efficiency": t1 / (w * worst),
                                "predicted_fill_gcups": cells / worst / 1e6,
                                "plan_slowest": plans[shard_ms.index(worst)],
                                "clocks": clocks}
        print(json.dumps(rec), flush=True)
        del out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
