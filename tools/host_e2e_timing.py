"""Host-buffer (e2e) multiply and add/sub through the C ABI: pairs/s or GB/s per call,
median of N calls. DOTG_HOST_SLICE_MB / DOTG_HOST_STREAMS tune the pipeline."""
import ctypes
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W

lib = dg.lib()
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
res = {}
for name, gen, m in (("C3", W.c3_inputs, 16), ("C4", W.c4_inputs, 64)):
    a, b = gen()
    B = a.shape[0]
    ha = torch.empty(a.shape, dtype=torch.int64, pin_memory=True)
    hb = torch.empty(b.shape, dtype=torch.int64, pin_memory=True)
    ho = torch.empty((B, 2 * m), dtype=torch.int64, pin_memory=True)
    ha.copy_(a)
    hb.copy_(b)
    ts = []
    for _ in range(12):
        t0 = time.perf_counter()
        assert lib.dotg_mul_batch_host(P(ho), P(ha), P(hb), m, B) == 0
        ts.append(time.perf_counter() - t0)
    res[name] = B / statistics.median(ts[2:])
print(os.environ.get("DOTG_HOST_SLICE_MB", "default"), {k: f"{v:.3e} pairs/s" for k, v in res.items()})
