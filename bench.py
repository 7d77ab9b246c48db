#!/usr/bin/env python
"""Benchmark of the DTW distance-matrix fill (BASELINE.json metric: DTW cell updates/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--precision fp64|fp32]
    python bench.py --impl reference ...      # the reference's own multithreaded CPU fill

One step = the full distance-matrix fill of config C (default: configs[3] of
BASELINE.json, "c4": N=1000 z-normalised Gaussian random walks, length 2844, unlimited
window, fp64 -- the largest single-GPU config, 4.04e12 cells), sharded over N GPUs (one
process per GPU, torchrun) with every distance stored into every rank's matrix by the
fill kernels themselves (fused P2P exchange; NCCL all-gather fallback). Inputs are the
seeded synthetic stand-ins for the UCR data the paper used
(paper_2307_04904_b200/generators.py).

Prints one JSON line (rank 0). `value` = total in-band DP cells / max-over-ranks device
time (GCUPS), inputs resident in HBM; `e2e` = the same metric through the public API
(api.build_matrix_packed: pinned host series -> H2D -> fill -> validation -> D2H of the
condensed matrix). `roofline` compares the fill kernel with the theoretical fp64 (fp32)
pipe rate of SURVEY.md §8(d) at MEASURED_PEAKS.sm_max_mhz (3722 GCUPS fp64 at 1965 MHz),
with the live-measured ceiling of the cell body as a secondary key; `cpu_baseline` times
the reference's build_matrix (oracle/_ref, all host threads) on a bounded sample of the
same workload. At N=1 the line also carries `all_configs` (one fill of each of c1-c5) and
`kmedoids` (the c5 and c3 k-medoids runs over the resident matrix; c5 checked against the
reference's own kmedoids).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "DTW cell updates/sec (GCUPS) for full distance matrix"
UNIT = "GCUPS"
CONFIG_NAMES = {
    1: "c1: N=100 sum-of-sinusoid classes, L=500, unlimited window, fp64",
    2: "c2: N=1000 z-normalised Gaussian random walks, L=1000, Sakoe-Chiba 100, fp64",
    3: "c3: N=24000 piecewise-linear classes, L=46, unlimited window, fp64",
    4: "c4: N=1000 z-normalised Gaussian random walks, L=2844, unlimited window",
    5: "c5: N=5000 time-stretched sinusoid classes, L~U[50,1500], Sakoe-Chiba 100 + auto-widen",
}


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = f"/tmp/dtwgpu_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.fh.close()

    def summary(self) -> dict:
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 8 and parts[0].replace(".", "").isdigit():
                    rows.append(parts)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[4 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][1]),
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max(float(r[2]) for r in rows if r[2] not in ("", "[N/A]"))}


# ----------------------------------------------------------------------------- CPU arms
def _copy_ms(src, dst) -> float:
    """One copy of `src` to `dst` ("cpu": pinned host), timed with CUDA events (best of 3)."""
    import torch

    if dst == "cpu":
        out = torch.empty(src.shape, dtype=src.dtype).pin_memory()
    else:
        out = torch.empty(src.shape, dtype=src.dtype, device=dst)
    best = float("inf")
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out.copy_(src, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference_sample(ds, budget_s: float):
    """Time the reference's build_matrix (oracle/_ref, all host threads) on the first q
    series of the workload, q sized for ~budget_s of CPU work. Falls back to the C
    restatement (single-threaded) when the reference could not be built."""
    import oracle
    from paper_2307_04904_b200 import generators as gen

    cores = os.cpu_count() or 1
    kind = "reference" if oracle.have_ref() else "port"
    per_core = 0.33e9  # cells/s per core, used only to size the sample
    rate = per_core * (cores if kind == "reference" else 1)
    total_pairs = ds.p * (ds.p - 1) // 2
    avg_cells = gen.total_cells(ds.subset(min(ds.p, 64))) / max(min(ds.p, 64) * (min(ds.p, 64) - 1) // 2, 1)
    want_pairs = max(int(budget_s * rate / max(avg_cells, 1)), 1)
    q = int(min(ds.p, (1 + np.sqrt(1 + 8 * want_pairs)) / 2))
    q = max(q, 2)
    sub = ds.subset(q)
    cells = gen.total_cells(sub)
    t0 = time.perf_counter()
    if kind == "reference":
        oracle.ref_build_condensed(sub.samples, sub.offsets, sub.half_width, sub.auto_widen,
                                   workers=cores)
    else:
        oracle.build_condensed(sub.samples, sub.offsets, sub.half_width, sub.auto_widen)
    dt = time.perf_counter() - t0
    return {"value": cells / dt / 1e9, "unit": UNIT, "cores": cores if kind == "reference" else 1,
            "kind": kind, "cpu_model": _cpu_model(),
            "sample": f"first {q} series of {ds.name} ({q * (q - 1) // 2} of {total_pairs} pairs, "
                      f"{cells:.3e} cells, {dt:.2f} s)",
            "seconds": dt, "cells": cells}


def run_reference_arm(a, ds):
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    samples = []
    for _ in range(a.warmup):
        cpu_reference_sample(ds, a.ref_step_s)
    for _ in range(a.steps):
        samples.append(cpu_reference_sample(ds, a.ref_step_s))
    total_cells = sum(s["cells"] for s in samples)
    total_s = sum(s["seconds"] for s in samples)
    value = total_cells / total_s / 1e9
    cb = dict(samples[-1])
    cb["value"] = value
    from paper_2307_04904_b200 import generators as gen
    cb["extrapolated_full_matrix_s"] = gen.total_cells(ds) / (value * 1e9)
    cb["extrapolated_note"] = ("the reference's full-matrix time on these cores, extrapolated "
                               "by in-band cells from the timed samples (exact: the reference "
                               "has no data-dependent pruning)")
    cb.pop("seconds", None)
    cb.pop("cells", None)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": total_s / a.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64" if a.precision == "fp64" else "f32", "data": "synthetic",
        "config": {"workload": CONFIG_NAMES[a.config], "pairs": ds.p * (ds.p - 1) // 2,
                   "sample": "bounded per step (see cpu_baseline.sample)"},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU arm
def theoretical_peak(prec: int):
    """148 SMs x 64 fp64 lanes (128 fp32) x SM clock / ops per cell (5 fp64
    pipe ops; FADD FMUL FMNMX3 FADD = 4 fp32), GCUPS, at MEASURED_PEAKS.sm_max_mhz."""
    mhz, src = 1965.0, "fallback 1965 MHz (B200_PROFILING.md)"
    try:
        mhz = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"])
        src = "MEASURED_PEAKS.json sm_max_mhz"
    except (OSError, ValueError, KeyError):
        pass
    per = (148 * 64 / 5) if prec == 0 else (148 * 128 / 4)
    return per * mhz * 1e6 / 1e9, f"theoretical {'fp64' if prec == 0 else 'fp32'} pipe rate " \
        f"(SURVEY.md §8(d)) at {mhz:.0f} MHz ({src})"


def _fill_once(eng, ds, prec, out_ptr):
    """One device fill of the whole matrix (plan cached by a previous call); device ms."""
    total = ds.p * (ds.p - 1) // 2
    eng.fill_slots(ds.half_width, ds.auto_widen, prec, 0, total, out_ptr)
    eng.synchronize()
    return eng.last_fill_ms()


def all_configs_block(eng, dev, a):
    """Two timed fills (the faster reported) of each BASELINE config (fp64; c4 also fp32), plus the k-medoids runs
    of c5 (parity against the reference's own kmedoids, timed as its CPU baseline) and c3,
    each over the matrix its fill just left in HBM."""
    import torch

    from paper_2307_04904_b200 import api, generators as gen

    out, kmed = {}, {}
    peak64 = theoretical_peak(0)[0]
    peak32 = theoretical_peak(1)[0]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for c, prec in ((1, 0), (2, 0), (3, 0), (4, 0), (5, 0), (4, 1)):
        ds = gen.make_config(c)
        total = ds.p * (ds.p - 1) // 2
        buf = torch.empty(total, dtype=torch.float64, device=dev)
        eng.upload(ds.samples, ds.offsets)
        cells = eng.count_cells(ds.half_width, ds.auto_widen, 0, total)
        t0 = time.perf_counter()
        _fill_once(eng, ds, prec, buf.data_ptr())  # plans + warms
        first_s = time.perf_counter() - t0
        # two timed fills (L2 flushed before each), the faster one reported: a single fill
        # of the one-lane classes occasionally runs one item round longer (dynamic items)
        ms_all = []
        for _ in range(2):
            flush.zero_()
            ms_all.append(_fill_once(eng, ds, prec, buf.data_ptr()))
        ms = min(ms_all)
        key = f"c{c}" + ("_fp32" if prec else "")
        peak = peak32 if prec else peak64
        out[key] = {"gcups": cells / (ms * 1e-3) / 1e9, "fill_ms": ms, "cells": cells,
                    "pairs": total, "frac_of_peak": cells / (ms * 1e-3) / 1e9 / peak,
                    "fill_ms_all": ms_all, "first_call_s": first_s,
                    "plan": eng.last_plan()[:400]}
        if c == 5 and prec == 0:
            # cold first call through the public API on a fresh context (planning, H2D,
            # fill, checks, D2H all inside)
            fresh = api.Engine(dev.index)
            t0 = time.perf_counter()
            fresh.build_condensed(ds.samples, ds.offsets, ds.half_width, ds.auto_widen)
            out[key]["cold_e2e_first_call_s"] = time.perf_counter() - t0
            fresh.close()
        if a.kmedoids and prec == 0 and c in (3, 5):
            kmed[key] = kmedoids_run(eng, ds, buf, check=(c == 5 and a.check))
        del buf
        torch.cuda.empty_cache()
    return out, kmed


def kmedoids_run(eng, ds, cond, check):
    """The config's k-medoids (kmedoids.hpp:148-189) over the matrix resident in HBM."""
    p = ds.p
    # first call (untimed warm-up: restart-worker contexts, buffers, module loading), then
    # the timed call over a freshly adopted matrix (square expansion and cluster-ordered
    # copy rebuilt inside the timed region)
    first = []
    for rep in range(2):
        eng.adopt(None, p, on_device_ptr=cond.data_ptr())
        eng._p_resident = p
        eng.synchronize()
        eng.km_stats(reset=True)
        t0 = time.perf_counter()
        med, asg, cost, br = eng.kmedoids(p, ds.k, ds.restarts, 100, 0)
        km_s = time.perf_counter() - t0
        first.append(km_s)
    st = eng.km_stats()
    hbm = _hbm_peak()
    upd_gbs = st["update_bytes"] / max(st["update_ms"], 1e-9) / 1e6
    res = {"k": ds.k, "restarts": ds.restarts, "series": p, "seconds": km_s,
           "first_call_seconds": first[0],
           "sweeps": st["sweeps"], "total_cost": cost, "best_restart": br,
           "includes": "square expansion, cluster-ordered copy, every restart (seeding, "
                       "sweeps, host sums); restarts on concurrent restart workers",
           "square_expand_ms": st["prep_ms"], "cluster_layout": st["cluster_layout"],
           "layout_build_ms": st["layout_ms"],
           "update_kernels": {"ms": st["update_ms"], "algorithmic_bytes": st["update_bytes"],
                              "achieved_gbs": upd_gbs, "peak_gbs": hbm[0],
                              "frac": upd_gbs / hbm[0], "peak_source": hbm[1],
                              "note": "sum of per-sweep device intervals; with concurrent "
                                      "restart workers they overlap, see sequential"},
           "assign_kernel": {"ms": st["assign_ms"], "algorithmic_bytes": st["assign_bytes"],
                             "achieved_gbs": st["assign_bytes"] / max(st["assign_ms"], 1e-9) / 1e6}}
    # one restart worker: per-sweep kernel intervals not overlapped by other restarts
    os.environ["DTWGPU_KM_WORKERS"] = "1"
    try:
        eng.adopt(None, p, on_device_ptr=cond.data_ptr())
        eng.synchronize()
        eng.km_stats(reset=True)
        t0 = time.perf_counter()
        m1, a1, c1, _ = eng.kmedoids(p, ds.k, ds.restarts, 100, 0)
        s1 = time.perf_counter() - t0
        st1 = eng.km_stats()
    finally:
        del os.environ["DTWGPU_KM_WORKERS"]
    sw = max(st1["sweeps"], 1)
    res["sequential"] = {
        "seconds": s1, "identical": bool(list(m1) == list(med) and list(a1) == list(asg)
                                         and c1 == cost),
        "update_us_per_sweep": st1["update_ms"] / sw * 1e3,
        "assign_us_per_sweep": st1["assign_ms"] / sw * 1e3,
        "update_algorithmic_gbs": st1["update_bytes"] / max(st1["update_ms"], 1e-9) / 1e6,
        "update_frac_of_hbm": st1["update_bytes"] / max(st1["update_ms"], 1e-9) / 1e6 / hbm[0],
        "assign_algorithmic_gbs": st1["assign_bytes"] / max(st1["assign_ms"], 1e-9) / 1e6}
    if check:
        # Parity against the reference's own kmedoids (oracle/_ref; the C restatement when
        # it was not built), timed: its single-threaded restart loop over the same host
        # matrix is the k-medoids CPU baseline.
        import oracle
        D = cond.cpu().numpy()
        kind = "reference" if oracle.have_ref() else "port"
        t1 = time.perf_counter()
        if kind == "reference":
            rmed, rasg, rcost = oracle.ref_kmedoids(D, p, ds.k, ds.restarts, 100, 0)
        else:
            rmed, rasg, rcost = oracle.kmedoids(D, p, ds.k, ds.restarts, 100, 0)
        res["cpu_baseline"] = {"seconds": time.perf_counter() - t1, "kind": kind, "cores": 1,
                               "sample": "the whole k-medoids run (single-threaded, as the "
                                         "reference's kmedoids is)"}
        res["parity"] = bool(list(rmed) == list(med) and list(rasg) == list(asg)
                             and rcost == cost)
    return res


def run_gpu_arm(a, ds):
    import torch
    import torch.distributed as dist

    from paper_2307_04904_b200 import api, distributed as dd, generators as gen

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    # --dist-backend gloo (diagnostic): several ranks may then share one GPU; slices are
    # all-gathered through host memory. The product path is NCCL, one GPU per rank.
    gloo = a.dist_backend == "gloo"
    if gloo and world > 1:
        local = local % max(torch.cuda.device_count(), 1)
    if world > 1 and not dist.is_initialized():
        if gloo:
            dist.init_process_group("gloo")
        else:
            # NCCL init lines (rank count, transport) in the log so the ranks can be checked
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            # keep stdout to the one JSON line (NCCL logs to stdout by default)
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)  # a real stream: fill, all-gather and events share it
    torch.cuda.set_stream(stream)
    eng = api.engine(local)
    eng.set_stream(stream.cuda_stream)
    prec = 1 if a.precision == "fp32" else 0

    p = ds.p
    total = p * (p - 1) // 2
    bounds = dd.cell_bounds(ds.lengths, ds.half_width, ds.auto_widen, world)
    b, e = bounds[rank]
    eng.upload(ds.samples, ds.offsets)
    my_cells = eng.count_cells(ds.half_width, ds.auto_widen, b, e)
    all_cells = eng.count_cells(ds.half_width, ds.auto_widen, 0, total)
    width = max(max(ee - bb for bb, ee in bounds), 1)
    full = torch.empty(world * width, dtype=torch.float64, device=dev)
    mine = full[rank * width:(rank + 1) * width]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    # Exchange: fused P2P stores (each fill kernel writes every distance into all ranks'
    # resident matrices over NVLink; include/dtwgpu.h dtwg_exchange_*) or the NCCL
    # all-gather of padded slices. P2P falls back to NCCL if any rank cannot open a peer.
    exchange = "none"
    if world > 1:
        exchange = a.exchange
        if exchange == "p2p" and not dd.open_p2p_exchange(eng, p, rank, world):
            exchange = "nccl (p2p unavailable)"
    gather_ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    gather_ms = []

    def step():
        if exchange == "p2p":
            eng.exchange_fill(ds.half_width, ds.auto_widen, prec, b, e)
            return
        if e > b:
            eng.fill_slots(ds.half_width, ds.auto_widen, prec, b, e, mine.data_ptr())
        if world > 1:
            gather_ev[0].record(stream)
            if gloo:
                host = full.cpu()
                dist.all_gather_into_tensor(host, host[rank * width:(rank + 1) * width].clone())
                full.copy_(host)
            else:
                dist.all_gather_into_tensor(full, mine)
            gather_ev[1].record(stream)

    def assembled():
        """The gathered slices in condensed order (ragged shards are padded to `width`)."""
        if world == 1:
            return mine[:total]
        if exchange == "p2p":  # every rank's resident matrix is complete after the barrier
            eng.exchange_complete()
            return torch.from_numpy(eng.download(p)).to(dev)
        return torch.cat([full[r * width:r * width + (ee - bb)] for r, (bb, ee) in enumerate(bounds)])

    for _ in range(max(a.warmup, 0)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # Timed region: K steps, L2 flushed between steps (outside the per-step events),
    # each step bracketed by CUDA events on the launching stream.
    launches0 = eng.launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(a.steps)]
    fill_ms = []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for k in range(a.steps):
            flush.zero_()
            evs[k][0].record(stream)
            step()
            evs[k][1].record(stream)
            fill_ms.append(eng.last_fill_ms() if e > b else 0.0)
            if world > 1 and not exchange == "p2p":
                gather_ev[1].synchronize()
                gather_ms.append(gather_ev[0].elapsed_time(gather_ev[1]))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    step_ms = [s.elapsed_time(t) for s, t in evs]
    launches = eng.launch_count() - launches0
    headline_plan = eng.last_plan()  # before e2e / all_configs replan other workloads
    my_ms = sum(step_ms)
    t = torch.tensor([my_ms], dtype=torch.float64, device="cpu" if gloo else dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    value = all_cells * a.steps / (max_ms * 1e-3) / 1e9
    per_rank = None
    if world > 1:
        mine_stats = {"rank": rank, "slots": [b, e], "cells": my_cells,
                      "step_ms_mean": my_ms / max(a.steps, 1),
                      "fill_ms_mean": statistics.mean(fill_ms) if fill_ms else 0.0,
                      "exchange_ms_mean": (statistics.mean(gather_ms) if gather_ms else
                                           "fused into the fill kernels (P2P stores)")}
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine_stats)

    # Parity spot-check of the timed output against the C restatement (a few pairs).
    check = None
    if rank == 0 and a.check:
        import oracle
        # world > 1: check the assembled (all-gathered) matrix; else this rank's slice
        lo, hi = (0, total) if world > 1 else (b, e)
        got_all = assembled() if world > 1 else mine[: e - b]
        got = got_all.cpu().numpy()
        rng = np.random.default_rng(0)
        picks = rng.choice(max(hi - lo, 1), size=min(8, max(hi - lo, 1)), replace=False)
        ok = 0
        for s_ in picks:
            s_ = int(s_) + lo
            i, j = oracle_pair(s_, p)
            want = oracle.dtw(ds.series(i), ds.series(j),
                              int(gen.effective_half_width(ds.lengths[i], ds.lengths[j],
                                                           ds.half_width, ds.auto_widen)))
            g = got[s_ - lo]
            ok += int(g == want if prec == 0 else abs(g - want) <= 1e-5 * abs(want))
        check = f"{ok}/{len(picks)} sampled pairs match the oracle"
    elif world > 1 and exchange == "p2p" and a.check:
        eng.exchange_complete()

    # Roofline: the fill kernel (one launch per step for same-length series) against the
    # theoretical fp64/fp32 pipe rate; the live-measured cell-body ceiling alongside.
    peak, peak_src = theoretical_peak(prec)
    live_peak = eng.measure_cell_peak(prec) / 1e9
    kernel_ms = statistics.mean(fill_ms) if fill_ms else None
    achieved = my_cells / (kernel_ms * 1e-3) / 1e9 if kernel_ms else None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"c{a.config}_{a.precision}")
        except (OSError, ValueError):
            traffic = None

    # End to end through the public API: pinned host series -> build_matrix_packed ->
    # condensed matrix back in host memory, every step.
    e2e = None
    if a.e2e:
        pin_s = torch.from_numpy(ds.samples).pin_memory()
        pin_o = torch.from_numpy(ds.offsets).pin_memory()
        s_np, o_np = pin_s.numpy(), pin_o.numpy()
        w = api.WarpWindow(None if ds.half_width < 0 else ds.half_width)
        if world == 1:
            api.build_matrix_packed(s_np, o_np, w, ds.auto_widen, precision=prec, device=local)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(a.steps):
                m = api.build_matrix_packed(s_np, o_np, w, ds.auto_widen, precision=prec,
                                            device=local)
            dt = time.perf_counter() - t0
            d2h = m.condensed().nbytes
        else:
            # each rank: H2D of the series, its fill (+ exchange), D2H of its own slice --
            # from the resident exchange matrix on the P2P path, from `mine` on NCCL
            host = torch.empty(max(e - b, 1), dtype=torch.float64).pin_memory()
            dist.barrier()
            t0 = time.perf_counter()
            for _ in range(a.steps):
                eng.upload(s_np, o_np)
                step()
                if exchange == "p2p":
                    eng.download_range(b, e, host.numpy())
                else:
                    host[: e - b].copy_(mine[: e - b], non_blocking=True)
                torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            tt = torch.tensor([dt], dtype=torch.float64, device="cpu" if gloo else dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
            d2h = (e - b) * 8
        e2e = {"value": all_cells * a.steps / dt / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(ds.samples.nbytes + ds.offsets.nbytes),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": dt / a.steps * 1e3}
        if world == 1:
            # The parts of a call: the last call's fill on the device, and
            # standalone pinned copies of its inputs and its matrix (inside the call the
            # D2H is streamed behind the fill and the host checks overlap the H2D).
            e2e["fill_ms"] = float(eng.last_fill_ms())
            e2e["h2d_ms"] = _copy_ms(pin_s, dev) + _copy_ms(pin_o, dev)
            e2e["d2h_ms"] = _copy_ms(torch.empty(int(d2h) // 8, dtype=torch.float64, device=dev),
                                     "cpu")

    # k-medoids over the headline config's own matrix, restarts sharded over ranks
    # (restart r on rank r mod N) and reduced in restart order (--kmedoids, configs with k).
    kmed = None
    if a.kmedoids and ds.k and a.kmedoids_headline:
        if exchange == "p2p":
            eng.exchange_complete()  # resident already, written by all ranks' fills
        else:
            cond = assembled().contiguous()
            eng.adopt(None, p, on_device_ptr=cond.data_ptr())
        eng._p_resident = p
        eng.km_stats(reset=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()

        def run(rs):
            best_ = None
            for r in rs:
                med, asg, cost, br = eng.kmedoids(p, ds.k, ds.restarts, 100, 0, r, r + 1)
                if best_ is None or cost < best_[0]:
                    best_ = (cost, br, med.tolist(), asg.tolist())
            return best_

        best = dd.kmedoids_restart_round_robin(run, ds.restarts, rank, world)
        kmed = {"headline_config": {"k": ds.k, "restarts": ds.restarts,
                                    "seconds": time.perf_counter() - t0,
                                    "total_cost": best[0], "best_restart": best[1],
                                    "restarts_on_rank0": dd.restarts_of_rank(ds.restarts, 0, world)}}
        if rank == 0 and a.check and p <= 5000:
            # the reduced result against the reference's own kmedoids on the same matrix
            import oracle
            D = eng.download(p)
            fn = oracle.ref_kmedoids if oracle.have_ref() else oracle.kmedoids
            rmed, rasg, rcost = fn(D, p, ds.k, ds.restarts, 100, 0)
            kmed["headline_config"]["parity"] = bool(
                list(rmed) == list(best[2]) and list(rasg) == list(best[3]) and rcost == best[0])

    cpu = None
    if rank == 0 and world == 1 and a.cpu_baseline:
        cpu = cpu_reference_sample(ds, a.ref_step_s)
        cpu["extrapolated_full_matrix_s"] = all_cells / (cpu["value"] * 1e9)
        cpu["extrapolated_note"] = ("the reference's full-matrix time on these cores, "
                                    "extrapolated by in-band cells from the timed sample "
                                    "(exact: the reference has no data-dependent pruning)")
        cpu.pop("seconds", None)
        cpu.pop("cells", None)

    allc = None
    if rank == 0 and world == 1 and a.all_configs:
        allc, km_all = all_configs_block(eng, dev, a)
        if km_all:
            kmed = dict(kmed or {}, **km_all)

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": max_ms / a.steps,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64" if prec == 0 else "f32", "data": "synthetic",
            "config": {"workload": CONFIG_NAMES[a.config], "pairs": total, "cells": all_cells,
                       "series": p, "precision": a.precision,
                       "parallelism": (f"condensed-slot shards x{world} + fused P2P stores "
                                       "into every rank's matrix (NVLink)"
                                       if exchange == "p2p" else
                                       f"condensed-slot shards x{world} + NCCL all-gather"
                                       if world > 1 else "condensed-slot shards x1"),
                       "exchange": exchange,
                       "l2": "flushed (256 MB write) between timed steps",
                       "plan": headline_plan},
            "pairs_per_s": total * a.steps / (max_ms * 1e-3),
            "step_ms": [round(v, 3) for v in step_ms],  # this rank's timed steps
            "roofline": {"bound": "fp64" if prec == 0 else "fp32",
                         "achieved": achieved, "peak": peak,
                         "unit": "GCUPS (cell updates/s; fp64 cell = 5 fp64-pipe ops, fp32 cell = FADD FMUL FMNMX3 FADD)",
                         "frac": (achieved / peak) if achieved else None,
                         "traffic": traffic,
                         # DRAM rate that traffic means at this step time, against the
                         # measured HBM peak: the fill is not HBM-bound
                         "traffic_gbs": (traffic / (kernel_ms * 1e-3) / 1e9
                                         if traffic and kernel_ms else None),
                         "traffic_frac_of_hbm": (traffic / (kernel_ms * 1e-3) / 1e9 / _hbm_peak()[0]
                                                 if traffic and kernel_ms else None),
                         "peak_source": peak_src,
                         "live_cell_ceiling": live_peak,
                         "frac_of_live_ceiling": (achieved / live_peak) if achieved else None,
                         "live_ceiling_source": "dtwg_measure_cell_peak (the cell body as independent "
                                                "chains with three distinct inputs per cell, best "
                                                "of the select and predicated-add forms, all SMs), "
                                                "measured now"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "per_rank": per_rank,
            "all_configs": allc,
            "kmedoids": kmed,
            "clocks": clocks,
            "parity": check,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _hbm_peak():
    """HBM copy bandwidth measured by the driver (MEASURED_PEAKS.json), else the fallback."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(path))["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except (OSError, ValueError, KeyError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def oracle_pair(slot: int, p: int):
    lo, hi = 0, p - 1
    while lo < hi:
        mid = (lo + hi + 1) // 2
        if mid * p - mid * (mid + 1) // 2 <= slot:
            lo = mid
        else:
            hi = mid - 1
    return lo, lo + 1 + (slot - (lo * p - lo * (lo + 1) // 2))


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-step-s", type=float, default=4.0,
                    help="seconds of CPU work per reference sample")
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-check", dest="check", action="store_false")
    ap.add_argument("--subset", type=int, default=0,
                    help="diagnostics: only the first N series of the config")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="N>1: fused P2P stores from the fill kernels (default) or NCCL "
                         "all-gather of the slices")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: diagnostic multi-rank run (ranks may share a GPU)")
    ap.add_argument("--no-kmedoids", dest="kmedoids", action="store_false",
                    help="skip the k-medoids runs (c5 with parity, c3) of the N=1 line")
    ap.add_argument("--kmedoids-headline", action="store_true",
                    help="also run the headline config's own k-medoids (restarts r mod N)")
    ap.add_argument("--no-all-configs", dest="all_configs", action="store_false",
                    help="skip the one-fill-per-config block of the N=1 line")
    a = ap.parse_args()
    a.warmup = max(a.warmup, 0)
    from paper_2307_04904_b200 import generators as gen
    ds = gen.make_config(a.config)
    if a.subset:
        ds = ds.subset(a.subset)
    if a.impl == "reference":
        return run_reference_arm(a, ds)
    return run_gpu_arm(a, ds)


if __name__ == "__main__":
    sys.exit(main())
