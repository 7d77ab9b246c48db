"""Full-size parity of the plans the bench times (the reference's own
matrix checks compare whole matrices, test_distance_matrix.cpp:67-88 and
acceptance_main.cpp:314-334). Every test here runs the UNMODIFIED reference
(oracle/_ref, all host threads) on the same inputs and compares bit for bit:

* c3 in full (24000 series, 287,988,000 pairs) -- the one-lane-per-pair kernel the bench
  times, every pair;
* c4 at 300 series (44,850 pairs of length 2844) -- through the production kernel
  full[G=1,R=32,T=4] that fills the headline config (asserted from the plan);
* c5 at 2500 series (3.1M ragged auto-widened pairs) -- every kernel class that holds
  >= 0.5% of the full-size c5 cells must be in the subset's plan (asserted);
* c3 k-medoids at p = 24000, k = 24, 10 restarts -- medoids, labels and cost identical to
  the reference's kmedoids (through the cluster-ordered square and restart workers).
"""
import os
import re

import numpy as np
import pytest
import torch

import oracle
from paper_2307_04904_b200 import generators as gen
from tests.helpers import assert_bitwise

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CORES = os.cpu_count() or 1


def need_ref():
    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")


def _fill(eng, ds, prec=0):
    total = ds.p * (ds.p - 1) // 2
    out = torch.empty(total, dtype=torch.float64, device="cuda")
    eng.upload(ds.samples, ds.offsets)
    eng.fill_slots(ds.half_width, ds.auto_widen, prec, 0, total, out.data_ptr())
    eng.synchronize()
    return out


def _classes(plan: str) -> dict:
    """kernel label -> in-band cells, from dtwg_last_plan."""
    out = {}
    for part in plan.split(";"):
        part = part.strip()
        if not part:
            continue
        label = part.split(" ")[0]
        m = re.search(r"cells=([0-9.e+]+)", part)
        out[label] = out.get(label, 0.0) + (float(m.group(1)) if m else 0.0)
    return out


def test_c3_full_matrix_bitwise_vs_reference(eng):
    need_ref()
    ds = gen.make_config(3)
    got = _fill(eng, ds)
    plan = eng.last_plan()
    assert "full[G=1,R=46,T=2,1strip]" in plan, plan
    want, ev = oracle.ref_build_condensed(ds.samples, ds.offsets, ds.half_width, ds.auto_widen,
                                          workers=CORES)
    assert ev == 287_988_000
    assert_bitwise(got.cpu().numpy(), want, f"c3 full plan={plan[:200]}")


def test_c4_production_kernel_bitwise_vs_reference(eng):
    need_ref()
    ds = gen.make_config(4).subset(300)
    eng.force_kernel(0, 1, 32)  # the headline's kernel (planner: full[G=1,R=32,T=4] at p=1000)
    got = _fill(eng, ds)
    plan = eng.last_plan()
    assert "full[G=1,R=32,T=4]" in plan, plan
    want, ev = oracle.ref_build_condensed(ds.samples, ds.offsets, ds.half_width, ds.auto_widen,
                                          workers=CORES)
    assert_bitwise(got.cpu().numpy(), want, f"c4 p=300 plan={plan}")
    # the unforced planner on the full config picks the same kernel
    eng.force_kernel(-1, 0, 0)
    _fill(eng, gen.make_config(4))
    assert "full[G=1,R=32,T=4]" in eng.last_plan(), eng.last_plan()


def test_c5_subset_covers_full_size_classes_bitwise(eng):
    need_ref()
    full = gen.make_config(5)
    _fill(eng, full)
    full_cls = _classes(eng.last_plan())
    total = sum(full_cls.values())
    major = {k for k, v in full_cls.items() if v >= 0.005 * total}
    ds = full.subset(2500)
    got = _fill(eng, ds)
    plan = eng.last_plan()
    sub_cls = _classes(plan)
    missing = major - set(sub_cls)
    assert not missing, (missing, plan[:600])
    want, ev = oracle.ref_build_condensed(ds.samples, ds.offsets, ds.half_width, ds.auto_widen,
                                          workers=CORES)
    assert_bitwise(got.cpu().numpy(), want, f"c5 p=2500 plan={plan[:300]}")


def test_c3_kmedoids_full_size_vs_reference(eng):
    need_ref()
    ds = gen.make_config(3)
    cond = _fill(eng, ds)
    eng.adopt(None, ds.p, on_device_ptr=cond.data_ptr())
    eng._p_resident = ds.p
    trace = []
    med, asg, cost, br = eng.kmedoids(ds.p, ds.k, ds.restarts, 100, 0, 0, ds.restarts,
                                      lambda r, it, c: trace.append((r, it, c)))
    assert eng.km_stats()["cluster_layout"], "the cluster-ordered square was not used"
    D = cond.cpu().numpy()
    del cond
    ref_trace = []
    rmed, rasg, rcost = oracle.ref_kmedoids(D, ds.p, ds.k, ds.restarts, 100, 0,
                                            lambda r, it, c: ref_trace.append((r, it, c)))
    assert list(med) == list(rmed)
    assert np.array_equal(np.asarray(asg), np.asarray(rasg))
    assert cost == rcost
    assert trace == ref_trace
