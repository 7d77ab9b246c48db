"""Multi-process (gloo, world_size 2, CPU) tests of the sharding and reduction logic of
paper_2307_04904_b200/distributed.py. The per-rank compute is the C restatement here
(test infrastructure); on GPUs the same functions run the CUDA engine over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2307_04904_b200 import distributed as dd, generators as gen
from tests.helpers import ScalarRng, random_condensed


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    finally:
        dist.destroy_process_group()


def run_ranks(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    return out


def _fill_c5(rank, world):
    ds = gen.config5(n=30, hi=300)
    total = ds.p * (ds.p - 1) // 2
    bounds = dd.cell_bounds(ds.lengths, ds.half_width, ds.auto_widen, world)

    def fill(b, e, out):
        out[: e - b] = torch.from_numpy(oracle.build_condensed(
            ds.samples, ds.offsets, ds.half_width, ds.auto_widen, b, e))

    full = dd.fill_all_gather(fill, total, bounds, rank, torch.device("cpu"))
    return full.numpy().copy()


def _fill_uniform(rank, world):
    ds = gen.config2(n=12, length=120, half_width=10)
    total = ds.p * (ds.p - 1) // 2
    bounds = dd.cell_bounds(ds.lengths, ds.half_width, ds.auto_widen, world)

    def fill(b, e, out):
        out[: e - b] = torch.from_numpy(oracle.build_condensed(
            ds.samples, ds.offsets, ds.half_width, ds.auto_widen, b, e))

    return dd.fill_all_gather(fill, total, bounds, rank, torch.device("cpu")).numpy().copy()


@pytest.mark.parametrize("fn,make", [(_fill_c5, lambda: gen.config5(n=30, hi=300)),
                                     (_fill_uniform, lambda: gen.config2(n=12, length=120,
                                                                         half_width=10))])
def test_sharded_fill_equals_single_process(fn, make):
    out = run_ranks(fn)
    ds = make()
    want = oracle.build_condensed(ds.samples, ds.offsets, ds.half_width, ds.auto_widen)
    for r in out:
        assert np.array_equal(out[r].view(np.uint64), want.view(np.uint64))


def _kmed(rank, world):
    p, k, restarts, seed = 40, 4, 7, 321
    D = random_condensed(ScalarRng(5), p)

    def run(rb, re):
        med, asg, cost, best_r = oracle.kmedoids_range(D, p, k, restarts, 100, seed, rb, re)
        return (cost, best_r, med.tolist(), asg.tolist())

    return dd.kmedoids_restart_sharded(run, restarts, rank, world)


def test_restart_sharded_kmedoids_equals_sequential():
    out = run_ranks(_kmed)
    p, k, restarts, seed = 40, 4, 7, 321
    D = random_condensed(ScalarRng(5), p)
    med, asg, cost = oracle.kmedoids(D, p, k, restarts, 100, seed)
    for r in out:
        c, best_r, m, a = out[r]
        assert c == cost and list(m) == list(med) and list(a) == list(asg)


def test_bounds_cover_all_slots():
    ds = gen.config5(n=120)
    total = ds.p * (ds.p - 1) // 2
    for world in (1, 2, 3, 8):
        b = dd.cell_bounds(ds.lengths, ds.half_width, ds.auto_widen, world)
        assert b[0][0] == 0 and b[-1][1] == total
        assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
        cells = [gen.total_cells(ds, s, e) for s, e in b]
        assert max(cells) <= 1.1 * (sum(cells) / world) + 1e7


def test_reduce_best_ties_go_to_earliest_restart():
    res = [(5.0, 3, [1], [1]), (5.0, 1, [2], [2]), None, (6.0, 0, [3], [3])]
    assert dd.reduce_best(res)[1] == 1


def test_restart_round_robin_balances_eight_ranks():
    # restart r on rank r mod G -- 10 restarts over 8 ranks leave no rank idle
    got = [dd.restarts_of_rank(10, r, 8) for r in range(8)]
    assert got[0] == [0, 8] and got[1] == [1, 9] and all(len(g) == 1 for g in got[2:])
    assert sorted(x for g in got for x in g) == list(range(10))
