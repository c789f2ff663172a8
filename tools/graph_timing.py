"""C2 step: back-to-back launches vs CUDA-graph replay (launch overhead check)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W
from paper_2604_21566_b200._lib import AddSubProblem

lib = dg.lib()
probs = []
keep = []
for m, B in W.C2_SIZES:
    a, b, sa, sb = W.c2_inputs(m, B)
    for sub, x, y in ((0, a, b), (1, sa, sb)):
        o = torch.empty_like(x)
        f = torch.empty(B, dtype=torch.int32, device="cuda")
        keep += [x, y, o, f]
        probs.append(AddSubProblem(sub, 0, o.data_ptr(), x.data_ptr(), y.data_ptr(), f.data_ptr(), m, B))
arr = (AddSubProblem * len(probs))(*probs)
step_bytes = sum(2 * B * (24 * m + 4) for m, B in W.C2_SIZES)


def call(stream):
    rc = lib.dotg_addsub_grouped(arr, len(probs), ctypes.c_void_p(stream.cuda_stream))
    assert rc == 0


s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(5):
        call(s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 200
    e0.record(s)
    for _ in range(K):
        call(s)
    e1.record(s)
    torch.cuda.synchronize()
    lean = e0.elapsed_time(e1) / K
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(10):
            call(s)
    g.replay()
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(K // 10):
        g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) / K
print(f"lean loop {lean * 1e3:.1f} us/step ({step_bytes / lean / 1e6:.0f} GB/s); "
      f"graph {graph * 1e3:.1f} us/step ({step_bytes / graph / 1e6:.0f} GB/s)")
