"""Time batched Karatsuba vs the schoolbook column kernels on the C4/C3 inputs."""
import sys, os
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


for name, gen in (("C4", W.c4_inputs), ("C3", W.c3_inputs)):
    a, b = gen()
    ref = dg.mul_batch(a, b)
    print(name, "schoolbook us", round(t(lambda: dg.mul_batch(a, b)), 1))
    for theta in (32, 16, 8) if name == "C4" else (8, 4):
        o = dg.karatsuba_batch(a, b, theta=theta)
        assert torch.equal(o, ref)
        print(name, "karatsuba theta", theta, "us", round(t(lambda: dg.karatsuba_batch(a, b, theta=theta)), 1))

# large operands: plain mul_batch (generic column kernel for m > 128) vs Karatsuba down to
# the tensor-pipe base case (m = 128 / 64 / 32)
for m, B in ((256, 1 << 12), (512, 1 << 10), (1024, 1 << 8)):
    a = W.fill(B * m, 0x5A + m, 0).view(B, m)
    b = W.fill(B * m, 0x5B + m, 0).view(B, m)
    ref = dg.mul_batch(a, b)
    print(f"m={m} B={B} schoolbook us", round(t(lambda: dg.mul_batch(a, b), reps=3), 1))
    for theta in (128, 64, 32):
        o = dg.karatsuba_batch(a, b, theta=theta)
        assert torch.equal(o, ref)
        print(f"m={m} karatsuba theta {theta} us", round(t(lambda: dg.karatsuba_batch(a, b, theta=theta), reps=5), 1))
