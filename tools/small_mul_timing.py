"""Batched multiply at the smallest sizes (64 / 128 / 256-bit), row-major and interleaved."""
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


ROOF = 148 * 32 * 1.965e9
for m in (1, 2, 4, 8):
    B = (1 << 22) // m
    a = W.fill(B * m, 0xC1 + m, 0).view(B, m)
    b = W.fill(B * m, 0xC2 + m, 0).view(B, m)
    o = dg.mul_batch(a, b)
    us = t(lambda: dg.mul_batch(a, b, out=o))
    ai, bi = a.t().contiguous(), b.t().contiguous()
    oi = dg.mul_batch(ai, bi, layout="interleaved")
    assert torch.equal(oi.t(), o)
    ui = t(lambda: dg.mul_batch(ai, bi, out=oi, layout="interleaved"))
    prods = 4 * m * m * B
    byts = B * 32 * m
    print(f"m={m} B={B:8d} row {us:7.1f} us ({prods / us * 1e6 / ROOF:5.1%} IMAD roof, {byts / us / 1e3:5.0f} GB/s)"
          f"  interleaved {ui:7.1f} us ({byts / ui / 1e3:5.0f} GB/s)")
