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


def test_comm_sharded_entry_single_rank(cuda):
    """dotg_add_words_sharded / dotg_sub_words_sharded in-process at world 1 (own NCCL
    communicator from a unique id): odd sizes, a long propagate run, m_local = 0."""
    import ctypes

    import numpy as np
    import torch

    import paper_2604_21566_b200 as dg
    from helpers import Oracle, spiky
    from paper_2604_21566_b200._lib import check, lib

    L = lib()
    uid = ctypes.create_string_buffer(int(L.dotg_comm_id_bytes()))
    check(L.dotg_comm_get_unique_id(uid))
    comm = ctypes.c_void_p()
    check(L.dotg_comm_init_rank(ctypes.byref(comm), 1, uid, 0))
    assert L.dotg_comm_rank(comm) == 0 and L.dotg_comm_size(comm) == 1
    orc = Oracle()
    rng = np.random.default_rng(5)
    try:
        for m in (1, 7, 4096, 4097, 300_001):
            a, b = spiky(rng, m), spiky(rng, m)
            if m > 1000:
                a[100:m - 50] = np.uint64(0xFFFFFFFFFFFFFFFF)
                b[100:m - 50] = 0
                b[99] = 1
                a[99] = np.uint64(0xFFFFFFFFFFFFFFFF)
            for sub in (False, True):
                da = torch.from_numpy(a.view(np.int64)).cuda()
                db = torch.from_numpy(b.view(np.int64)).cuda()
                out = torch.empty_like(da)
                c = torch.full((1,), 7, dtype=torch.int32, device="cuda")
                fn = L.dotg_sub_words_sharded if sub else L.dotg_add_words_sharded
                check(fn(out.data_ptr(), da.data_ptr(), db.data_ptr(), m, c.data_ptr(), comm, None))
                want, wf = orc.sub(a, b) if sub else orc.add(a, b)
                assert np.array_equal(out.cpu().numpy().view(np.uint64), want), (m, sub)
                assert int(c.item()) == wf, (m, sub)
        c = torch.full((1,), 7, dtype=torch.int32, device="cuda")
        check(L.dotg_add_words_sharded(None, None, None, 0, c.data_ptr(), comm, None))  # empty shard
        assert int(c.item()) == 0
        assert L.dotg_add_words_sharded(None, None, None, 0, None, None, None) == dg._lib.DOTG_EINVAL
    finally:
        check(L.dotg_comm_destroy(comm))


def test_device_shards_two_ranks_gloo(cuda):
    """World size 2 with the product's device passes (not CPU stand-ins): both ranks on the
    box's GPU, the 8-byte exchange host-staged over gloo, results checked per rank."""
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29577",
                        os.path.join(ROOT, "tests", "gloo_gpu_shard_worker.py")],
                       cwd=ROOT, capture_output=True, text=True, timeout=900,
                       env={**os.environ, "MASTER_ADDR": "127.0.0.1"})
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0
    assert r.stdout.count(" ok") == 2
