"""Driver for ncu captures of the interleaved-layout kernels: the in-place tensor-pipe
multiply (m = 64, B = 2^16) and the segmented add (m = 256, B = 2^14)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W

torch.cuda.set_device(0)
m, B = 64, 1 << 16
a = W.fill(B * m, 0x51, 0).view(m, B)
b = W.fill(B * m, 0x51, 1 << 40).view(m, B)
o = torch.empty((2 * m, B), dtype=torch.int64, device="cuda")
for _ in range(3):
    dg.mul_batch(a, b, out=o, layout="interleaved")
m2, B2 = 256, 1 << 14
a2 = W.fill(B2 * m2, 0x52, 0).view(m2, B2)
b2 = W.fill(B2 * m2, 0x52, 1 << 40).view(m2, B2)
for _ in range(3):
    dg.add_batch(a2, b2, layout="interleaved")
torch.cuda.synchronize()
print("ok")
