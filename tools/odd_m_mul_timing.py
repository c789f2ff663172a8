"""Batched multiply at sizes without a dedicated kernel, row-major: pairs/s."""
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


for m in (3, 5, 6, 7, 8, 9, 12, 15, 16, 17, 24, 40, 100):
    B = (1 << 22) // m
    a = W.fill(B * m, 0xA1 + m, 0).view(B, m)
    b = W.fill(B * m, 0xA2 + m, 0).view(B, m)
    o = dg.mul_batch(a, b)
    us = t(lambda: dg.mul_batch(a, b, out=o))
    print(f"m={m:4d} B={B:8d} {us:9.1f} us  {B / us / 1e3:7.3f} Gpairs/s")
