"""Padded-Karatsuba products (m > 128) against their leaf work alone: for each (m, B) the
time of dotg_mul_batch and of one m = 128 tensor-pipe launch over the same 3^L * B leaves,
so the split / combine share of the product is visible. python tools/kara_breakdown.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W


def t(fn, reps=15):
    """Median of per-call CUDA-event times after two warm-up calls (allocations from the
    stream-ordered pool can make single calls slow)."""
    fn()
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return sorted(ts)[len(ts) // 2]


for m, B in ((256, 4096), (512, 2048), (1024, 1024), (2048, 256), (4096, 64)):
    a = W.fill(B * m, 0x31 + m, 0).view(B, m)
    b = W.fill(B * m, 0x32 + m, 0).view(B, m)
    out = torch.empty((B, 2 * m), dtype=torch.int64, device="cuda")
    L = (m // 128).bit_length() - 1
    nleaf = B * 3**L
    la = W.fill(nleaf * 128, 0x33, 0).view(nleaf, 128)
    lo = torch.empty((nleaf, 256), dtype=torch.int64, device="cuda")
    n0 = dg.kernel_launches()
    tm = t(lambda: dg.mul_batch(a, b, out=out))
    nl = (dg.kernel_launches() - n0) // 17
    tl = t(lambda: dg.mul_batch(la, la, out=lo))
    print(f"m={m:5d} B={B:5d} L={L}: product {tm:9.1f} us ({nl} launches), leaves alone {tl:9.1f} us "
          f"({tl / tm:5.1%}), levels {tm - tl:9.1f} us")
