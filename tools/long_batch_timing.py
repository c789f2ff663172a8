"""Batched add of long numbers (few pairs, many limbs), row-major, B x m = 2^22 limbs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W


def t(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for m, B in ((1024, 4096), (4096, 1024), (16384, 256), (65536, 64), (1 << 18, 16), (1 << 20, 4), (1 << 22, 1)):
    a = W.fill(B * m, 0xB1, 0).view(B, m)
    b = W.fill(B * m, 0xB2, 0).view(B, m)
    out, fl = dg.add_batch(a, b)
    us = t(lambda: dg.add_batch(a, b, out=out, flags=fl))
    print(f"m={m:8d} B={B:5d} {B * (24 * m + 4) / us / 1e3:7.0f} GB/s ({us:.1f} us)")
x = W.fill(1 << 22, 0xB1, 0)
y = W.fill(1 << 22, 0xB2, 0)
o, c = dg.add_words(x, y)
us = t(lambda: dg.add_words(x, y, out=o, carry=c))
print(f"add_words m=2^22: {24 * (1 << 22) / us / 1e3:7.0f} GB/s ({us:.1f} us)")
