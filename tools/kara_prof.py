"""One padded-Karatsuba product (m = 256, B = 4096 and m = 2048, B = 256) after warm-ups,
for an ncu launch list of its split / leaf / combine launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W

torch.cuda.set_device(0)
for m, B in ((256, 4096), (2048, 256)):
    a = W.fill(B * m, 0x31 + m, 0).view(B, m)
    b = W.fill(B * m, 0x32 + m, 0).view(B, m)
    out = torch.empty((B, 2 * m), dtype=torch.int64, device="cuda")
    for _ in range(3):
        dg.mul_batch(a, b, out=out)
torch.cuda.synchronize()
print("ok")
