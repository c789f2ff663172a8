"""Batched add at sizes without a dedicated team kernel (non powers of two), row-major."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W


def t(fn, reps=20):
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


for m in (3, 5, 7, 12, 24, 48, 100, 200, 384, 1000):
    B = (1 << 22) // m
    a = W.fill(B * m, 0x91 + m, 0).view(B, m)
    b = W.fill(B * m, 0x92 + m, 0).view(B, m)
    out, fl = dg.add_batch(a, b)
    us = t(lambda: dg.add_batch(a, b, out=out, flags=fl))
    print(f"m={m:5d} B={B:8d} {B * (24 * m + 4) / us / 1e3:7.0f} GB/s")
