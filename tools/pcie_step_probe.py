"""Transfer-only ceiling of the C2 e2e step: 537 MB host->device on one stream while
280 MB device->host runs on another (pinned buffers, 24 MB chunks), no kernels."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import argparse

ap = argparse.ArgumentParser()
ap.add_argument("--h2d", type=int, default=536870912)
ap.add_argument("--d2h", type=int, default=279576576)
ap.add_argument("--chunk-mb", type=int, default=24)
args = ap.parse_args()
h2d, d2h = args.h2d, args.d2h
ha = torch.empty(h2d // 8, dtype=torch.int64, pin_memory=True)
hb = torch.empty(d2h // 8, dtype=torch.int64, pin_memory=True)
da = torch.empty_like(ha, device="cuda")
db = torch.empty_like(hb, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
CH = (args.chunk_mb << 20) // 8  # chunk in int64 elements


def step(both=True, h=True):
    with torch.cuda.stream(s1):
        if h:
            for i in range(0, ha.numel(), CH):
                da[i:i + CH].copy_(ha[i:i + CH], non_blocking=True)
    with torch.cuda.stream(s2):
        if both:
            for i in range(0, hb.numel(), CH):
                hb[i:i + CH].copy_(db[i:i + CH], non_blocking=True)
    torch.cuda.synchronize()


for name, kw, byts in (("h2d only", dict(both=False), h2d), ("d2h only", dict(h=False), d2h),
                       ("both", dict(), h2d + d2h)):
    step(**kw)
    t0 = time.perf_counter()
    for _ in range(10):
        step(**kw)
    dt = (time.perf_counter() - t0) / 10
    print(f"{name}: {dt * 1e3:.2f} ms per step, {byts / dt / 1e9:.1f} GB/s")

# dependent pattern of the host pipeline: chunk k's download waits for chunk k's upload
ev = [torch.cuda.Event() for _ in range(4096)]


def dependent():
    n = 0
    with torch.cuda.stream(s1):
        for i in range(0, min(ha.numel(), hb.numel()), CH):
            da[i:i + CH].copy_(ha[i:i + CH], non_blocking=True)
            ev[n].record(s1)
            n += 1
    n = 0
    with torch.cuda.stream(s2):
        for i in range(0, min(ha.numel(), hb.numel()), CH):
            s2.wait_event(ev[n])
            hb[i:i + CH].copy_(da[i:i + CH], non_blocking=True)
            n += 1
    torch.cuda.synchronize()


dependent()
t0 = time.perf_counter()
for _ in range(10):
    dependent()
dt = (time.perf_counter() - t0) / 10
byts = 2 * min(h2d, d2h)
print(f"dependent (download k after upload k): {dt * 1e3:.2f} ms per step, {byts / dt / 1e9:.1f} GB/s")
