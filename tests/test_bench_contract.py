"""bench.py contract pieces that run without a GPU: the reference arm's JSON line (the
reference's own build_matrix, pairwise.hpp:62-127, compiled into oracle/_ref and timed on the
host cores) and the product arm failing loudly -- not falling back to the CPU -- when there
is no CUDA device."""
import json
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libdtwclust_ref.so")


def _run(*args, timeout=600):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=timeout)


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")
def test_reference_arm_line():
    r = _run("--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-step-s", "1.0")
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"].startswith("DTW cell updates/sec")
    assert line["unit"] == "GCUPS" and line["higher_is_better"] is True
    assert line["value"] > 0 and line["ms_per_step"] > 0
    assert line["steps"] == 1 and line["warmup"] == 0 and line["n_gpus"] == 1
    assert line["dtype"] == "f64" and line["data"] == "synthetic"
    assert line["config"]["workload"].startswith("c4")
    assert line["vs_baseline"] is None
    cpu = line["cpu_baseline"]
    assert cpu["kind"] == "reference" and cpu["cores"] >= 1 and cpu["value"] == line["value"]
    assert "series of c4" in cpu["sample"]
    assert cpu["extrapolated_full_matrix_s"] > 0
    e2e = line["e2e"]
    assert e2e["value"] == line["value"] and e2e["unit"] == line["unit"]
    assert e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0


@pytest.mark.skipif(torch.cuda.is_available(), reason="needs a box without a GPU")
def test_product_arm_fails_loudly_without_gpu():
    r = _run("--steps", "1", "--warmup", "3", timeout=300)
    assert r.returncode != 0
    assert not r.stdout.strip()  # no JSON line from a CPU fallback
