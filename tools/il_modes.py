"""A/B of the interleaved add/sub routes (DOTG_IL_MODE: 0 auto, 4 two-pass
2 thread per pair, 3 re-read segmented CTAs) at B x m = 2^22 limbs: back-to-back launches over 3
rotating input copies (> L2 between reuses), CUDA events. Each mode in its own process
(the knob is read once). Prints one JSON line per (mode, m)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, os, sys
sys.path.insert(0, ROOT)
import torch
import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W
torch.cuda.set_device(0)
res = {}
for m in (4, 16, 32, 64, 128, 256, 512, 1024):
    B = (1 << 22) // m
    sets = []
    for r in range(3):
        a = W.fill(B * m, 0x11 + r + m, 0).view(m, B)
        b = W.fill(B * m, 0x11 + r + m, 1 << 40).view(m, B)
        sets.append((a, b, torch.empty_like(a), torch.empty(B, dtype=torch.int32, device="cuda")))
    # parity against the row-major path on set 0
    a, b, o, f = sets[0]
    ro, rf = dg.add_batch(a.t().contiguous(), b.t().contiguous())
    dg.add_batch(a, b, out=o, flags=f, layout="interleaved")
    assert torch.equal(o.t(), ro) and torch.equal(f, rf), m
    fn = lambda s: dg.add_batch(s[0], s[1], out=s[2], flags=s[3], layout="interleaved")
    for s in sets: fn(s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        for s in sets: fn(s)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * len(sets))
    res[m] = {"us": us, "gbs": B * (24 * m + 4) / us / 1e3}
print(json.dumps(res))
'''.replace("ROOT", repr(ROOT))

modes = sys.argv[sys.argv.index("--only") + 1].split(",") if "--only" in sys.argv else ["0", "2", "3", "4"]
for mode in modes:
    env = {**os.environ, "DOTG_IL_MODE": mode}
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    if r.returncode != 0:
        print(json.dumps({"mode": mode, "error": r.stderr[-800:]}))
        continue
    print(json.dumps({"mode": mode, "per_m": json.loads(r.stdout.strip().splitlines()[-1])}))
