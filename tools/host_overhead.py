"""Host cost of one small batched call through each layer (no device work to speak of):
the Python API, the raw ctypes entry point with prebuilt arguments, and the stream lookup.
python tools/host_overhead.py"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import api
from paper_2604_21566_b200 import workloads as W

a = W.fill(8 * 64, 1, 0).view(8, 64)
b = W.fill(8 * 64, 2, 0).view(8, 64)
out, fl = dg.add_batch(a, b)
L = dg.lib()
args = (ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()),
        ctypes.c_void_p(fl.data_ptr()), 64, 8, 0, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))


def per_call(fn, n=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / n * 1e6


print(f"dg.add_batch (Python API)        {per_call(lambda: dg.add_batch(a, b, out=out, flags=fl)):7.2f} us/call")
print(f"ctypes dotg_add_batch, prebuilt  {per_call(lambda: L.dotg_add_batch(*args)):7.2f} us/call")
print(f"torch.cuda.current_stream()      {per_call(lambda: torch.cuda.current_stream().cuda_stream):7.2f} us/call")
print(f"api._check_dev x1                {per_call(lambda: api._check_dev(a, 'a')):7.2f} us/call")
