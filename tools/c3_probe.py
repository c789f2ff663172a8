"""C3 multiply (m = 16) time per pair against the batch size: the wave-tail share of the
named 2^18-pair batch (k_mul_kara16, one-warp CTAs). Back-to-back launches, CUDA events."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W

torch.cuda.set_device(0)
m = 16
res = {}
for lg in (15, 16, 17, 18, 19, 20, 21):
    B = 1 << lg
    a = W.fill(B * m, 0xC3, 0).view(B, m)
    b = W.fill(B * m, 0xC3, 1 << 40).view(B, m)
    o = torch.empty((B, 2 * m), dtype=torch.int64, device="cuda")
    for _ in range(3):
        dg.mul_batch(a, b, out=o)
    torch.cuda.synchronize()
    reps = max(3, (1 << 22) // B)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        dg.mul_batch(a, b, out=o)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    res[B] = {"us": us, "ns_per_kpair": us / B * 1e6, "frac_imad": B / (us * 1e-6) * 1024 / (148 * 32 * 1.965e9)}
print(json.dumps(res))
