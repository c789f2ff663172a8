"""Interleaved multiply at small m: per-call time vs batch (row stride alignment probe)."""
import sys, json
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import torch
import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W
def timed(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
for m in (6, 8, 5, 3):
    for B in (524288, 699050, 699048, 524290, 524296, 524320):
        a = W.fill(B * m, 0xA1 + m, 0).view(m, B); b = W.fill(B * m, 0xA2 + m, 0).view(m, B)
        o = torch.empty((2 * m, B), dtype=torch.int64, device="cuda")
        us = timed(lambda: dg.mul_batch(a, b, out=o, layout="interleaved"))
        print(json.dumps({"m": m, "B": B, "us": round(us, 1), "ns_per_pair": round(us * 1e3 / B, 4)}), flush=True)
