"""Wide products (m >= 256): dotg_mul_batch per call with the tcgen05 route on and off
(DOTG_MUL_UMMA=1 / 0 in child processes), and its byte-MAC rate against the tensor pipe's
8192 u8 MACs/clk/SM. python tools/umma_timing.py [--child]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPES = ((256, 4096), (512, 2048), (1024, 1024), (2048, 256), (4096, 64), (8192, 16), (16384, 4), (65536, 1))


def child():
    sys.path.insert(0, ROOT)
    import torch

    import paper_2604_21566_b200 as dg
    from paper_2604_21566_b200 import workloads as W

    def t(fn, reps=11):
        fn()
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        return sorted(ts)[len(ts) // 2]

    only = os.environ.get("UMMA_SHAPES")
    shapes = [tuple(map(int, s.split("x"))) for s in only.split(",")] if only else SHAPES
    for m, B in shapes:
        a = W.fill(B * m, 0x31 + m, 0).view(B, m)
        b = W.fill(B * m, 0x32 + m, 0).view(B, m)
        out = torch.empty((B, 2 * m), dtype=torch.int64, device="cuda")
        us = t(lambda: dg.mul_batch(a, b, out=out))
        macs = B * (8 * m) ** 2
        peak = 148 * 8192 * 1.965e9
        print(json.dumps({"umma": os.environ.get("DOTG_MUL_UMMA", "1"), "m": m, "B": B, "us": round(us, 2),
                          "byte_macs_per_s": macs / us * 1e6, "frac_tensor_u8": macs / us * 1e6 / peak}),
              flush=True)


if __name__ == "__main__":
    if "--child" in sys.argv:
        child()
    else:
        for v in ("1", "0"):
            env = dict(os.environ, DOTG_MUL_UMMA=v)
            subprocess.run([sys.executable, os.path.abspath(__file__), "--child"], env=env, check=True)
