"""The multi-rank bench path (torchrun, one process per rank, collectives between them)
rehearsed on the one-GPU box: DOTG_BENCH_SHARED_GPU=1 puts every rank on GPU 0 with gloo
collectives. Checks the control flow the driver's 2/4/8-GPU runs take - barriers, max-
over-ranks timing, per-rank secondary configs, the C5 limb-range shard exchange - ends
with one JSON line from rank 0 and exit code 0 (timings are meaningless when shared)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_ranks_shared_gpu(cuda):
    env = {**os.environ, "DOTG_BENCH_SHARED_GPU": "1", "MASTER_ADDR": "127.0.0.1"}
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29561", os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["configs"]["C5"]["shard_limbs"] == (1 << 29)
    assert d["configs"]["C5"]["add"]["gbs"] > 0 and d["configs"]["C5"]["sub"]["gbs"] > 0
