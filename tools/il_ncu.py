"""Driver for ncu captures of one interleaved add route: python tools/il_ncu.py M
(B = 2^22 / M; DOTG_IL_MODE picks the route). Three warm-up launches, then one more."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W

torch.cuda.set_device(0)
m = int(sys.argv[1])
B = (1 << 22) // m
a = W.fill(B * m, 0x52, 0).view(m, B)
b = W.fill(B * m, 0x52, 1 << 40).view(m, B)
o = torch.empty_like(a)
for _ in range(4):
    dg.add_batch(a, b, out=o, layout="interleaved")
torch.cuda.synchronize()
print("ok", m)
