"""C1 (4096-bit add + sub, B = 65536) grouped launch alone, for ncu and launch timing:
python tools/c1_probe.py [reps]. Prints per-launch microseconds (CUDA events) and GB/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
B = W.C1["batch"]
sets = []
for r in range(3):
    a = W.fill(B * 64, 0xC1 + 17 * r, 0).view(-1, 64)
    b = W.fill(B * 64, 0xC1 + 17 * r, 1 << 40).view(-1, 64)
    sa, sb = W.swap_for_sub(a, b)
    o1, o2 = torch.empty_like(a), torch.empty_like(a)
    f1 = torch.empty(B, dtype=torch.int32, device="cuda")
    f2 = torch.empty(B, dtype=torch.int32, device="cuda")
    sets.append([dict(op="add", out=o1, a=a, b=b, flags=f1), dict(op="sub", out=o2, a=sa, b=sb, flags=f2)])


def launch(k):
    dg.addsub_grouped(sets[k % 3])


for k in range(6):
    launch(k)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
ev[0].record()
for k in range(reps):
    launch(k)
    ev[k + 1].record()
torch.cuda.synchronize()
per = [ev[k].elapsed_time(ev[k + 1]) * 1e3 for k in range(reps)]
byts = 2 * B * (24 * 64 + 4)
mean = sum(per) / reps
print(f"C1 grouped launch: mean {mean:.2f} us, min {min(per):.2f} us, {byts / mean / 1e3:.0f} GB/s (mean), "
      f"{byts / min(per) / 1e3:.0f} GB/s (best)")
