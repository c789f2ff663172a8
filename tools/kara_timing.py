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
