"""Batched multiply: IMMA (tensor pipe) vs IMAD column kernels, C3/C4 shapes and more.

Prints one line per (m, batch): kernel time per launch for both routes, pairs/s and
u32-product-equivalents/s (4 m^2 per pair) against the IMAD roofline."""
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
shapes = [(8, 1 << 19), (16, 1 << 18), (32, 1 << 17), (64, 1 << 16), (128, 1 << 14)]
if len(sys.argv) > 1:
    keep = {int(x) for x in sys.argv[1].split(",")}
    shapes = [(m, B) for m, B in shapes if m in keep]
for m, B in shapes:
    if (m, B) == (16, 1 << 18):
        a, b = W.c3_inputs()
    elif (m, B) == (64, 1 << 16):
        a, b = W.c4_inputs()
    else:
        a = W.fill(B * m, 0x51 + m, 0).view(B, m)
        b = W.fill(B * m, 0x52 + m, 0).view(B, m)
    out = torch.empty((B, 2 * m), dtype=torch.int64, device="cuda")
    res = {}
    outs = {}
    for r in ("imad", "imma"):
        dg.set_mul_route(r)
        us = t(lambda: dg.mul_batch(a, b, out=out))
        outs[r] = out.clone()
        res[r] = us
    dg.set_mul_route("auto")
    same = torch.equal(outs["imad"], outs["imma"])
    prods = 4 * m * m * B
    print(f"m={m:3d} B={B:7d}  imad {res['imad']:8.1f} us ({prods / res['imad'] * 1e6 / ROOF:5.1%} of IMAD roof)"
          f"  imma {res['imma']:8.1f} us ({prods / res['imma'] * 1e6 / ROOF:6.1%}; {B / res['imma'] / 1e3:6.2f} Gpairs/s;"
          f" HBM {B * 32 * m / res['imma'] / 1e3:6.0f} GB/s)  speedup {res['imad'] / res['imma']:4.2f}x  identical={same}")
