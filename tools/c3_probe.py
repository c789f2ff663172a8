"""C3 multiply (m = 16) time per pair against the batch size: the wave-tail share of the
named 2^18-pair batch (one-warp CTAs). Back-to-back launches, CUDA events. The kernel is
chosen by DOTG_K16_HYBRID (1: k_mul_kara16h, z1 on the FP64 pipe; 0: k_mul_kara16); the
product is checked against the other kernel's through the IMMA route at 2^15 pairs."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W

torch.cuda.set_device(0)
m = 16
res = {"hybrid": os.environ.get("DOTG_K16_HYBRID", "1")}
a = W.fill(32768 * m, 0x77, 0).view(-1, m)
b = W.fill(32768 * m, 0x77, 1 << 40).view(-1, m)
b[::7] = -1
a[::5] = -1
ref = torch.empty((32768, 2 * m), dtype=torch.int64, device="cuda")
prev = dg.set_mul_route("imma")
dg.mul_batch(a, b, out=ref)
dg.set_mul_route(prev)
assert torch.equal(dg.mul_batch(a, b), ref), "C3 kernel disagrees with the tensor-pipe route"
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
