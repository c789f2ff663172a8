"""Batched add/sub in the interleaved [m][batch] layout vs row-major, C2 shapes."""
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


for m, B in list(W.C2_SIZES) + [(128, 1 << 15), (512, 1 << 13), (1024, 1 << 12)]:
    a, b, sa, sb = W.c2_inputs(m, B)
    ai, bi = a.t().contiguous(), b.t().contiguous()
    out, fl = dg.add_batch(a, b)
    oi, fli = dg.add_batch(ai, bi, layout="interleaved")
    assert torch.equal(oi.t(), out) and torch.equal(fl, fli)
    byts = B * (24 * m + 4)
    ur = t(lambda: dg.add_batch(a, b, out=out, flags=fl))
    ui = t(lambda: dg.add_batch(ai, bi, out=oi, flags=fli, layout="interleaved"))
    print(f"m={m:4d} B={B:8d} row-major {byts / ur / 1e3:7.0f} GB/s   interleaved {byts / ui / 1e3:7.0f} GB/s")
