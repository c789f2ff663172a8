"""One batched multiply launch for profiling: python tools/mul_prof.py M BATCH ROUTE."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W

m, B, route = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
a = W.fill(B * m, 0x51 + m, 0).view(B, m)
b = W.fill(B * m, 0x52 + m, 0).view(B, m)
out = torch.empty((B, 2 * m), dtype=torch.int64, device="cuda")
dg.set_mul_route(route)
for _ in range(3):
    dg.mul_batch(a, b, out=out)
torch.cuda.synchronize()
print("ok")
