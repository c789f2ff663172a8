"""Time one product at large limb counts up to the reference cap (2^24 limbs):
python tools/mul_max_timing.py [lg ...]. Prints ms per product (CUDA events) for three
consecutive calls after one warm-up call."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W

lgs = [int(x) for x in sys.argv[1:]] or [16, 18, 20, 22, 24]
for lg in lgs:
    m = 1 << lg
    a = W.fill(m, 0x77 + lg, 0).view(1, m)
    b = W.fill(m, 0x77 + lg, 1 << 40).view(1, m)
    out = torch.empty((1, 2 * m), dtype=torch.int64, device="cuda")
    dg.mul_batch(a, b, out=out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n0 = dg.kernel_launches()
        e0.record()
        dg.mul_batch(a, b, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"m = 2^{lg}: " + ", ".join(f"{t:.2f}" for t in ts) + f" ms per product, {dg.kernel_launches() - n0} launches",
          flush=True)
