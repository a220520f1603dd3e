"""bench.py at --gpus 2 under torchrun (the driver's SCALE launch): the default
N > 1 path is the row-sharded DB — each rank searches its shard,
the per-shard top-k records cross through the peer-memory exchange, and rank 0
prints one JSON line naming db-shard2.  Runs both ranks on one GPU when the box
has one (the timing reduction then uses gloo)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("exchange", ["p2p", "nccl"])
def test_bench_two_ranks_db_shard(exchange):
    import torch

    if exchange == "nccl" and torch.cuda.device_count() < 2:
        pytest.skip("the NCCL data-path exchange needs a GPU per rank")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", "29633" if exchange == "p2p" else "29634", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "4", "--warmup", "3", "--rows", "40000", "--dim", "512", "--d-f", "512",
           "--no-cpu-baseline", "--e2e-steps", "4", "--exchange", exchange]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and len(lines) == 1, r.stdout[-3000:] + r.stderr[-3000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["parallelism"].startswith("db-shard2"), d["config"]
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["gpu_launches"] > 0
