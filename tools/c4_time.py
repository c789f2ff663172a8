"""C4 multiply kernel time per launch (for A/B builds via DOTG_LIB_PATH)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W

a, b = W.c4_inputs()
o = dg.mul_batch(a, b)
for _ in range(3):
    dg.mul_batch(a, b, out=o)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    dg.mul_batch(a, b, out=o)
e1.record()
torch.cuda.synchronize()
print(os.environ.get("DOTG_LIB_PATH", "default"), f"C4 {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
