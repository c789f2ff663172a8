"""Batched multiply over a sweep of limb counts, both layouts: per-call device time (events
around 10 back-to-back calls after 3 warm-ups) and the fraction of the IMAD.WIDE roofline
(4 m^2 u32 products per pair, 148 x 32 per clk x 1965 MHz). B x m = 2^22 limbs up to
m = 128, B = 2^30 / m^2 above (at least 1). One JSON line per (layout, m).
usage: python tools/mul_sweep.py [--ms 1,2,3,...] [--layouts row,il]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W

PEAK = 148 * 32 * 1965e6


def timed(fn, reps=10):
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


ms = [int(x) for x in sys.argv[sys.argv.index("--ms") + 1].split(",")] if "--ms" in sys.argv else \
    [1, 2, 3, 4, 5, 6, 7, 8, 9, 12, 15, 16, 17, 24, 31, 32, 33, 40, 48, 63, 64, 65, 96, 100, 127, 128,
     129, 200, 256, 300, 512, 1000, 1024]
layouts = sys.argv[sys.argv.index("--layouts") + 1].split(",") if "--layouts" in sys.argv else ["row", "il"]
torch.cuda.set_device(0)
for lay in layouts:
    for m in ms:
        B = (1 << 22) // m if m <= 128 else max(1, (1 << 30) // (m * m))
        a = W.fill(B * m, 0xA1 + m, 0).view(B, m)
        b = W.fill(B * m, 0xA2 + m, 0).view(B, m)
        if lay == "il":
            a, b = a.t().contiguous(), b.t().contiguous()
            o = torch.empty((2 * m, B), dtype=torch.int64, device="cuda")
            fn = lambda: dg.mul_batch(a, b, out=o, layout="interleaved")
        else:
            o = torch.empty((B, 2 * m), dtype=torch.int64, device="cuda")
            fn = lambda: dg.mul_batch(a, b, out=o)
        us = timed(fn)
        print(json.dumps({"layout": lay, "m": m, "B": B, "us": round(us, 2),
                          "frac_imad": round(B * 4 * m * m / (us * 1e-6) / PEAK, 3),
                          "gbs": round(B * 32 * m / us / 1e3, 1)}), flush=True)
        del a, b, o
