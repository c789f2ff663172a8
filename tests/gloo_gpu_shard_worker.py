"""Worker for test_gpu_nccl.py::test_device_shards_two_ranks_gloo: the config-5 shard
protocol with REAL device passes at world size 2 on the one-GPU box - both ranks on GPU 0,
the 8-byte exchange over gloo (host-staged), so no kernel ever waits on another rank's
kernel. Each rank checks its shard of the result and the whole-number carry."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def main():
    from helpers import Oracle

    from paper_2604_21566_b200 import workloads as W
    from paper_2604_21566_b200.sharded import ShardedWords, shard_bounds

    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    orc = Oracle()
    for m, run in ((3 << 20, None), (1_000_003, (200_000, 800_000)), (4096 * 3 + 5, (100, 4096 * 3))):
        run = run or (3 * m // 8, 5 * m // 8)  # the propagate run straddles the boundary
        for sub in (False, True):
            lo, hi = shard_bounds(m, rank, world)
            a, b = W.c5_shard_inputs(sub, lo, hi, m=m, run=run)
            ga, gb = W.c5_inputs(sub, m=m, run=run)
            ha, hb = ga.cpu().numpy().view(np.uint64), gb.cpu().numpy().view(np.uint64)
            want, wf = orc.sub(ha, hb) if sub else orc.add(ha, hb)
            out, carry = ShardedWords().run(sub, torch.empty_like(a), a, b)
            assert np.array_equal(out.cpu().numpy().view(np.uint64), want[lo:hi]), (rank, m, sub)
            assert int(carry.item()) == wf, (rank, m, sub)
    dist.barrier()
    dist.destroy_process_group()
    print(f"rank {rank}/{world} ok")


if __name__ == "__main__":
    main()
