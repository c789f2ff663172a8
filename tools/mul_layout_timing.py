"""Batched multiply, row-major vs interleaved [m][batch] layout (kernel time per launch)."""
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


for m, B in ((8, 1 << 19), (16, 1 << 18), (32, 1 << 17), (64, 1 << 16)):
    a = W.fill(B * m, 0x71 + m, 0).view(B, m)
    b = W.fill(B * m, 0x72 + m, 0).view(B, m)
    ai, bi = a.t().contiguous(), b.t().contiguous()
    o = dg.mul_batch(a, b)
    oi = dg.mul_batch(ai, bi, layout="interleaved")
    assert torch.equal(oi.t(), o)
    ur = t(lambda: dg.mul_batch(a, b, out=o))
    ui = t(lambda: dg.mul_batch(ai, bi, out=oi, layout="interleaved"))
    print(f"m={m:3d} B={B:7d} row-major {ur:8.1f} us  interleaved {ui:8.1f} us")
