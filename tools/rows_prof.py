"""One row-major add launch for ncu: python tools/rows_prof.py M (B = 2^22 / M)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W

torch.cuda.set_device(0)
m = int(sys.argv[1])
B = (1 << 22) // m
a = W.fill(B * m, 0x61, 0).view(B, m)
b = W.fill(B * m, 0x62, 1 << 40).view(B, m)
o = torch.empty_like(a)
for _ in range(4):
    dg.add_batch(a, b, out=o)
torch.cuda.synchronize()
print("ok", m)
