"""Worker for test_gpu_nccl.py: the config-5 shard protocol over a real NCCL process
group (launched by torch.distributed.run, one rank per visible GPU)."""
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
    from paper_2604_21566_b200.sharded import CommShardedWords, ShardedWords, shard_bounds

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    m = 3 << 20
    run = (3 * m // 8, 5 * m // 8)
    orc = Oracle()
    for sub in (False, True):
        lo, hi = shard_bounds(m, rank, world)
        a, b = W.c5_shard_inputs(sub, lo, hi, m=m, run=run)
        ga, gb = W.c5_inputs(sub, m=m, run=run)
        assert torch.equal(ga[lo:hi], a) and torch.equal(gb[lo:hi], b)
        ha, hb = ga.cpu().numpy().view(np.uint64), gb.cpu().numpy().view(np.uint64)
        want, wf = orc.sub(ha, hb) if sub else orc.add(ha, hb)
        # (1) Python-orchestrated: two C-ABI passes around torch's all_gather
        out = torch.empty_like(a)
        out, carry = ShardedWords().run(sub, out, a, b)
        assert np.array_equal(out.cpu().numpy().view(np.uint64), want[lo:hi]), (rank, sub)
        assert int(carry.item()) == wf
        # (2) C++-orchestrated: one dotg_*_words_sharded call over the library's own NCCL
        # communicator, on a side stream
        cs = CommShardedWords()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        out2 = torch.full_like(a, -1)
        with torch.cuda.stream(st):
            out2, carry2 = cs.run(sub, out2, a, b, stream=st)
        st.synchronize()
        assert np.array_equal(out2.cpu().numpy().view(np.uint64), want[lo:hi]), (rank, sub, "comm")
        assert int(carry2.item()) == wf
        cs.close()
        # (3) the same C++ call over torch's own NCCL communicator (dotg_comm_wrap)
        cw = CommShardedWords(wrap_torch_comm=True)
        out3, carry3 = cw.run(sub, torch.full_like(a, -1), a, b)
        torch.cuda.synchronize()
        assert np.array_equal(out3.cpu().numpy().view(np.uint64), want[lo:hi]), (rank, sub, "wrap")
        assert int(carry3.item()) == wf
        cw.close()
    dist.barrier()
    dist.destroy_process_group()
    print(f"rank {rank}/{world} ok")


if __name__ == "__main__":
    main()
