"""The multi-GPU shard protocol over NCCL (torchrun, one rank per available GPU; the
round's GPU box has one, which still exercises NCCL init, the 8-byte all-gather on the
device and the device-side carry composition)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_shard_protocol_over_nccl(cuda):
    n = cuda.cuda.device_count()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--standalone", "--nnodes=1",
                        f"--nproc-per-node={n}", os.path.join(ROOT, "tests", "nccl_shard_worker.py")],
                       cwd=ROOT, capture_output=True, text=True, timeout=900,
                       env={**os.environ, "MASTER_ADDR": "127.0.0.1"})
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0
    assert r.stdout.count(" ok") == n
