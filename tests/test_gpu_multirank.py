"""The bench's multi-rank path (slot sharding, all-gather assembly, max-over-ranks timing,
restart-sharded k-medoids) run for real on the GPU: two torchrun ranks sharing the one
available B200 through the gloo backend (kernels never wait on each other across ranks).
The product path is NCCL with one GPU per rank; only the collective differs."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("exchange", ["p2p", "nccl"])
@pytest.mark.parametrize("config,subset", [(2, 160), (5, 120)])
def test_two_rank_bench_assembles_the_matrix(config, subset, exchange):
    """p2p: the fill kernels store every distance into both ranks' resident matrices
    through CUDA IPC (same device here, NVLink peers on a multi-GPU node) -- no waiting
    between the ranks' kernels; "nccl": slices all-gathered (over gloo here)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29531", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--config", str(config),
           "--subset", str(subset), "--dist-backend", "gloo", "--no-cpu-baseline", "--kmedoids-headline",
           "--exchange", exchange]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["exchange"] == exchange, d["config"]
    assert d["parity"].startswith("8/8"), d["parity"]
    assert d["kmedoids"]["headline_config"]["parity"] is True
    # per-rank fill/exchange times and the e2e D2H of each rank's own slice
    assert [r["rank"] for r in d["per_rank"]] == [0, 1]
    assert d["e2e"]["d2h_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
