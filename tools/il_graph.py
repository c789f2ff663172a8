"""Interleaved add routes timed the way bench.py times them: per-launch device time of
back-to-back launches over 3 rotating input copies (one CUDA graph, events on the stream).
B x m = 2^22 limbs per operand. One child process per DOTG_IL_MODE (the knob is read once);
`--only 0,5` picks modes, `--ms 64,256` picks limb counts, `--sub` times subtraction. Row-major add of the same bytes
is printed as mode "rows" for comparison. One JSON line per mode."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import ctypes, json, os, sys
sys.path.insert(0, ROOT)
import torch
import bench
import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W
torch.cuda.set_device(0)
lib = dg.lib()
stream = torch.cuda.current_stream()
P = lambda t: ctypes.c_void_p(t.data_ptr())
layout = int(sys.argv[1])
fn_name = sys.argv[2] if len(sys.argv) > 2 else "dotg_add_batch"
res = {}
for m in MS:
    B = (1 << 22) // m
    sets = []
    for r in range(3):
        a = W.fill(B * m, 0x11 + r + m, 0).view(m, B)
        b = W.fill(B * m, 0x11 + r + m, 1 << 40).view(m, B)
        sets.append((a, b, torch.empty_like(a), torch.empty(B, dtype=torch.int32, device="cuda")))
    if layout == 1:
        a, b, o, f = sets[0]
        ro, rf = dg.add_batch(a.t().contiguous(), b.t().contiguous())
        dg.add_batch(a, b, out=o, flags=f, layout="interleaved")
        assert torch.equal(o.t(), ro) and torch.equal(f, rf), m
    def mk(Lc):
        return [(lambda args_=(P(o), P(a), P(b), P(f), m, B, layout, Lc.stream): getattr(lib, fn_name)(*args_))
                for a, b, o, f in sets]
    us = bench.per_launch_us(torch, dg, lib, stream, mk)
    res[m] = {"us": round(us, 3), "gbs": round(B * (24 * m + 4) / us / 1e3, 1),
              "frac": round(B * (24 * m + 4) / us / 1e3 / 6547.2, 3)}
    del sets
print(json.dumps(res))
'''.replace("ROOT", repr(ROOT))

modes = sys.argv[sys.argv.index("--only") + 1].split(",") if "--only" in sys.argv else ["0", "2", "3", "4", "rows"]
op_fn = "dotg_sub_batch" if "--sub" in sys.argv else "dotg_add_batch"
ms = sys.argv[sys.argv.index("--ms") + 1] if "--ms" in sys.argv else "4,16,32,64,128,256,512,1024"
child = CHILD.replace("MS", "(" + ms + ",)")
for mode in modes:
    env = {**os.environ, "DOTG_IL_MODE": "0" if mode == "rows" else mode}
    r = subprocess.run([sys.executable, "-c", child, "0" if mode == "rows" else "1", op_fn], env=env,
                       capture_output=True, text=True, cwd=ROOT)
    if r.returncode != 0:
        print(json.dumps({"mode": mode, "error": r.stderr[-800:]}), flush=True)
        continue
    print(json.dumps({"mode": mode, "per_m": json.loads(r.stdout.strip().splitlines()[-1])}), flush=True)
