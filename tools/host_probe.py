"""Host-side probe for the GPU box: CPU model/cores, host memory, PCIe link and
pinned host<->device copy bandwidth (one direction and both at once).

Used to size the e2e (host-buffer) path and the CPU baseline. Prints one JSON line.
"""
import json
import os
import subprocess
import time

import torch


def sh(cmd):
    try:
        return subprocess.run(cmd, shell=True, capture_output=True, text=True, timeout=60).stdout.strip()
    except Exception as e:  # noqa: BLE001
        return f"err: {e}"


def bw(fn, nbytes, reps=5):
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return nbytes / best / 1e9


def main():
    out = {
        "nproc": os.cpu_count(),
        "cpu_model": sh("lscpu | grep 'Model name' | head -1 | cut -d: -f2").strip(),
        "sockets": sh("lscpu | grep 'Socket(s)' | cut -d: -f2").strip(),
        "numa": sh("lscpu | grep 'NUMA node(s)' | cut -d: -f2").strip(),
        "flags_avx512f": "avx512f" in sh("grep -m1 flags /proc/cpuinfo"),
        "mem_total": sh("free -g | awk '/Mem:/{print $2}'"),
        "pcie": sh("nvidia-smi --query-gpu=pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current --format=csv,noheader"),
        "gpu": sh("nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv,noheader"),
    }
    n = 512 << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    out["h2d_gbs"] = bw(lambda: d.copy_(h, non_blocking=True), n)
    out["d2h_gbs"] = bw(lambda: h.copy_(d, non_blocking=True), n)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        s1.synchronize()
        s2.synchronize()

    out["bidir_gbs_total"] = bw(both, 2 * n)
    # host memory bandwidth (single-thread numpy copy as a rough floor)
    import numpy as np
    a = np.ones(n // 8, dtype=np.uint64)
    b = np.empty_like(a)
    t0 = time.perf_counter()
    np.copyto(b, a)
    out["host_copy_1thread_gbs"] = 2 * n / (time.perf_counter() - t0) / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
