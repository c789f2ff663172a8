"""C3: IMAD column kernel and IMMA kernel running concurrently on two streams over a
split batch (does the tensor pipe add throughput next to a saturated IMAD pipe?)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W

a, b = W.c3_inputs()
B, m = a.shape
ref = dg.mul_batch(a, b)
out = torch.empty_like(ref)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(k):
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    dg.set_mul_route("imad")
    dg.mul_batch(a[k:], b[k:], out=out[k:], stream=s1)
    if k:
        dg.set_mul_route("imma")
        dg.mul_batch(a[:k], b[:k], out=out[:k], stream=s2)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


for f in (0.0, 0.05, 0.1, 0.15, 0.2, 0.3):
    k = int(B * f) // 64 * 64
    for _ in range(3):
        run(k)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        run(k)
    e1.record()
    torch.cuda.synchronize()
    print(f"imma fraction {f:.2f}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
dg.set_mul_route("auto")
