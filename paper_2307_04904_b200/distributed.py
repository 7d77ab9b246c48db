"""Multi-GPU fill and k-medoids: one process per GPU, torch.distributed for the plumbing.

Fill: pairs are independent, so the condensed slot range is cut into
one contiguous range per rank, exactly like the reference's worker chunks
(pairwise.hpp:102-117) but balanced on in-band DP cells instead of pair counts (equal
for same-length series). Each rank fills its range into its slice of a padded device
buffer; the one exchange step is an all-gather of the slices (NCCL over NVLink on
B200), after which every GPU holds the full condensed matrix. Output slots are fixed,
so the matrix is bitwise independent of the number of GPUs.

k-medoids: restarts are independent, so restart r runs on rank
r mod world over the replicated matrix, and the best result is reduced in restart
order with strict < (ties to the earliest restart, kmedoids.hpp:182).

The compute callables are injectable so the sharding and reduction logic can be
tested with the gloo backend on CPU (tests/test_distributed.py); the product path
uses the CUDA engine and NCCL.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist

from . import generators as gen


def equal_bounds(total: int, world: int) -> List[Tuple[int, int]]:
    """pairwise.hpp:106-113: contiguous chunks of ceil(total / world)."""
    chunk = (total + world - 1) // world if world else total
    return [(min(r * chunk, total), min((r + 1) * chunk, total)) for r in range(world)]


def row_cells(lengths: np.ndarray, half_width: int, auto_widen: bool) -> np.ndarray:
    """In-band cells of every condensed row i (pairs (i, j>i)), vectorised."""
    p = len(lengths)
    out = np.zeros(p, dtype=np.float64)
    for i in range(p - 1):
        js = lengths[i + 1:]
        hw = gen.effective_half_width(lengths[i], js, half_width, auto_widen)
        out[i] = float(gen.pair_cells(np.full(js.shape, lengths[i]), js, hw).sum())
    return out


def cell_bounds(lengths: np.ndarray, half_width: int, auto_widen: bool,
                world: int) -> List[Tuple[int, int]]:
    """Contiguous slot ranges with (near-)equal in-band cell counts (row granularity,
    then split inside the boundary row by pair count)."""
    p = len(lengths)
    total = p * (p - 1) // 2
    if world <= 1 or total == 0:
        return [(0, total)] + [(total, total)] * max(world - 1, 0)
    if np.all(lengths == lengths[0]):
        return equal_bounds(total, world)
    rc = row_cells(lengths, half_width, auto_widen)
    cum = np.concatenate([[0.0], np.cumsum(rc)])
    target = cum[-1] / world
    cuts = [0]
    for r in range(1, world):
        want = target * r
        i = int(np.searchsorted(cum, want, side="right") - 1)
        i = min(max(i, 0), p - 2)
        # inside row i: split by the fraction of its cells (pairs of one row are similar)
        frac = 0.0 if rc[i] == 0 else (want - cum[i]) / rc[i]
        row0 = i * p - i * (i + 1) // 2
        cut = row0 + int(round(frac * (p - 1 - i)))
        cuts.append(max(cut, cuts[-1]))
    cuts.append(total)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def fill_all_gather(fill: Callable[[int, int, torch.Tensor], None], total: int,
                    bounds: Sequence[Tuple[int, int]], rank: int, device,
                    group=None) -> torch.Tensor:
    """Fill this rank's slots into its padded slice and all-gather all slices.

    `fill(b, e, out)` writes slots [b, e) into out[0:e-b]. Returns the full condensed
    matrix (total values) on `device`, identical on every rank.
    """
    world = len(bounds)
    width = max(e - b for b, e in bounds) if bounds else 0
    width = max(width, 1)
    full = torch.empty(world * width, dtype=torch.float64, device=device)
    mine = full[rank * width:(rank + 1) * width]
    b, e = bounds[rank]
    if e > b:
        fill(b, e, mine)
    if world > 1:
        local = mine.clone() if full.device.type == "cpu" else mine
        dist.all_gather_into_tensor(full, local.contiguous(), group=group)
    if all(e - b == width for b, e in bounds[:-1]) and bounds[-1][0] == (world - 1) * width:
        return full[:total]  # equal chunks: already contiguous condensed order
    return torch.cat([full[r * width:r * width + (e - b)] for r, (b, e) in enumerate(bounds)])


def reduce_best(results: Sequence[Optional[tuple]]) -> tuple:
    """Best (cost, restart, medoids, assignment) in restart order, strict < (kmedoids.hpp:182)."""
    best = None
    for res in sorted((r for r in results if r is not None), key=lambda t: t[1]):
        if best is None or res[0] < best[0]:
            best = res
    return best


def restarts_of_rank(restarts: int, rank: int, world: int) -> List[int]:
    """restart r runs on rank r mod world."""
    return list(range(rank, restarts, max(world, 1)))


def kmedoids_restart_round_robin(run: Callable[[List[int]], Optional[tuple]], restarts: int,
                                 rank: int, world: int, group=None) -> tuple:
    """Restart r on rank r mod world; `run(rs)` returns (cost, best_restart, medoids,
    assignment) for the restarts `rs` (ascending) or None if empty. Results are exchanged
    with all_gather_object and reduced in restart order with strict < on every rank
    (kmedoids.hpp:182)."""
    rs = restarts_of_rank(restarts, rank, world)
    mine = run(rs) if rs else None
    if world > 1:
        gathered: list = [None] * world
        dist.all_gather_object(gathered, mine, group=group)
    else:
        gathered = [mine]
    return reduce_best(gathered)


def kmedoids_restart_sharded(run: Callable[[int, int], Optional[tuple]], restarts: int,
                             rank: int, world: int, group=None) -> tuple:
    """Round-robin restart sharding over a per-restart-range callable `run(rb, re)`: each
    of this rank's restarts r runs as [r, r+1), best kept in restart order."""
    def run_list(rs):
        best = None
        for r in rs:
            res = run(r, r + 1)
            if res is not None and (best is None or res[0] < best[0]):
                best = res
        return best

    return kmedoids_restart_round_robin(run_list, restarts, rank, world, group)


# ----------------------------------------------------------------------------- CUDA path
def build_matrix_distributed(engine, ds: gen.Dataset, precision: int = 0,
                             group=None) -> torch.Tensor:
    """Sharded GPU fill + NCCL all-gather; returns the full condensed matrix on this GPU."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    engine.upload(ds.samples, ds.offsets)
    total = ds.p * (ds.p - 1) // 2
    bounds = cell_bounds(ds.lengths, ds.half_width, ds.auto_widen, world)
    device = torch.device("cuda", torch.cuda.current_device())

    def fill(b, e, out):
        engine.fill_slots(ds.half_width, ds.auto_widen, precision, b, e, out.data_ptr())

    return fill_all_gather(fill, total, bounds, rank, device, group)


def open_p2p_exchange(engine, p: int, rank: int, world: int, group=None) -> bool:
    """Fused fill + all-gather over peer memory: export this rank's resident matrix buffer,
    open every other rank's (CUDA IPC over NVLink), and agree on success. Returns False on
    every rank (all exchanges closed) if any rank could not open a peer -- the caller then
    uses the NCCL all-gather path."""
    handle = engine.exchange_export(p)
    handles = [None] * world
    dist.all_gather_object(handles, handle, group=group)
    ok = True
    try:
        engine.exchange_open(handles, rank)
    except Exception:  # noqa: BLE001 -- reported collectively below
        ok = False
    oks = [None] * world
    dist.all_gather_object(oks, ok, group=group)
    if not all(oks):
        engine.exchange_close()
        return False
    return True


def fill_p2p(engine, ds: gen.Dataset, precision: int, bounds: Sequence[Tuple[int, int]],
             rank: int, group=None) -> None:
    """This rank's slots into every rank's matrix (one fused launch per class); after the
    barrier each rank's resident matrix is complete -- no collective on the data path."""
    b, e = bounds[rank]
    engine.exchange_fill(ds.half_width, ds.auto_widen, precision, b, e)
    engine.synchronize()
    dist.barrier(group=group)
    engine.exchange_complete()


def build_matrix_p2p(engine, ds: gen.Dataset, precision: int = 0, group=None) -> bool:
    """Sharded fill whose kernels write every distance into all ranks' resident matrices
    (dtwg_exchange_*). Returns False (nothing filled) when peer memory is unavailable."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    engine.upload(ds.samples, ds.offsets)
    if not open_p2p_exchange(engine, ds.p, rank, world, group):
        return False
    bounds = cell_bounds(ds.lengths, ds.half_width, ds.auto_widen, world)
    fill_p2p(engine, ds, precision, bounds, rank, group)
    engine._p_resident = ds.p
    return True


def kmedoids_distributed(engine, condensed: torch.Tensor, p: int, k: int, restarts: int,
                         max_iterations: int = 100, seed: int = 0, group=None) -> tuple:
    """Restart-sharded k-medoids over a replicated device-resident matrix."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if condensed is not None:  # None: already resident (build_matrix_p2p)
        engine.adopt(None, p, on_device_ptr=condensed.data_ptr())
    engine._p_resident = p

    def run(rb, re):
        med, asg, cost, best_r = engine.kmedoids(p, k, restarts, max_iterations, seed, rb, re)
        return (cost, best_r, med.tolist(), asg.tolist())

    return kmedoids_restart_sharded(run, restarts, rank, world, group)
