"""k-medoids timing breakdown over the resident c3/c5 matrices (diagnostics).

    python tools/km_bench.py [--configs 3 5] [--reps 3]

For each config: one fill, then the config's k-medoids (k, 10 restarts) with
  * the default restart workers and cluster-ordered layout (the product path),
  * one worker (sequential restarts: per-sweep kernel times are not overlapped),
  * one worker without the layout (DTWGPU_KM_LAYOUT=0: plain-square gathers),
printing one JSON line per run: wall seconds, square/layout preparation ms, update and
assignment kernel ms per sweep and algorithmic GB/s. Results must be identical.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2307_04904_b200 import api, generators as gen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[3, 5])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--workers", type=int, nargs="*", default=[],
                    help="extra modes: DTWGPU_KM_WORKERS=w for each w")
    ap.add_argument("--only-workers", action="store_true",
                    help="run only the --workers modes")
    a = ap.parse_args()
    eng = api.engine(0)
    dev = torch.device("cuda", 0)
    for c in a.configs:
        ds = gen.make_config(c)
        total = ds.p * (ds.p - 1) // 2
        buf = torch.empty(total, dtype=torch.float64, device=dev)
        eng.upload(ds.samples, ds.offsets)
        eng.fill_slots(ds.half_width, ds.auto_widen, 0, 0, total, buf.data_ptr())
        eng.synchronize()
        ref = None
        modes = [] if a.only_workers else [
            ("default", {}), ("workers1", {"DTWGPU_KM_WORKERS": "1"}),
            ("workers1_nolayout", {"DTWGPU_KM_WORKERS": "1", "DTWGPU_KM_LAYOUT": "0"}),
            ("default_nolayout", {"DTWGPU_KM_LAYOUT": "0"})]
        modes += [(f"workers{w}", {"DTWGPU_KM_WORKERS": str(w)}) for w in a.workers]
        for mode, env in modes:
            for k_, v_ in env.items():
                os.environ[k_] = v_
            for rep in range(a.reps):
                eng.adopt(None, ds.p, on_device_ptr=buf.data_ptr())
                eng._p_resident = ds.p
                eng.synchronize()
                eng.km_stats(reset=True)
                t0 = time.perf_counter()
                med, asg, cost, br = eng.kmedoids(ds.p, ds.k, ds.restarts, 100, 0)
                dt = time.perf_counter() - t0
                st = eng.km_stats()
                res = (list(med), list(asg), cost)
                same = ref is None or res == ref
                ref = ref or res
                sw = max(st["sweeps"], 1)
                print(json.dumps({
                    "config": c, "mode": mode, "rep": rep, "seconds": dt,
                    "prep_ms": st["prep_ms"], "layout": st["cluster_layout"],
                    "sweeps": st["sweeps"], "update_ms_per_sweep": st["update_ms"] / sw,
                    "assign_ms_per_sweep": st["assign_ms"] / sw,
                    "update_gbs": st["update_bytes"] / max(st["update_ms"], 1e-9) / 1e6,
                    "assign_gbs": st["assign_bytes"] / max(st["assign_ms"], 1e-9) / 1e6,
                    "cost": cost, "identical": same}), flush=True)
            for k_ in env:
                del os.environ[k_]
        del buf
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
