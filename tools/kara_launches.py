"""One padded-Karatsuba product for an ncu launch list: python tools/kara_launches.py M B
(two warm-up products, then the one to read)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W

m, B = int(sys.argv[1]), int(sys.argv[2])
a = W.fill(B * m, 0x61, 0).view(B, m)
b = W.fill(B * m, 0x62, 0).view(B, m)
o = torch.empty((B, 2 * m), dtype=torch.int64, device="cuda")
for _ in range(3):
    dg.mul_batch(a, b, out=o)
torch.cuda.synchronize()
print("ok")
