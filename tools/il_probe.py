"""Interleaved add/sub at one size, for ncu: python tools/il_probe.py m batch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W

m, B = int(sys.argv[1]), int(sys.argv[2])
a, b, _, _ = W.c2_inputs(m, B)
ai, bi = a.t().contiguous(), b.t().contiguous()
oi, fl = dg.add_batch(ai, bi, layout="interleaved")
for _ in range(5):
    dg.add_batch(ai, bi, out=oi, flags=fl, layout="interleaved")
torch.cuda.synchronize()
