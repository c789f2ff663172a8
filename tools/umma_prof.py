"""One wide-product shape for ncu: python tools/umma_prof.py M B [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W

m, B = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
a = W.fill(B * m, 0x31 + m, 0).view(B, m)
b = W.fill(B * m, 0x32 + m, 0).view(B, m)
out = torch.empty((B, 2 * m), dtype=torch.int64, device="cuda")
for _ in range(reps):
    dg.mul_batch(a, b, out=out)
torch.cuda.synchronize()
print("done", m, B)
