"""C5 end to end: dotg_add_words_host on pinned host operands (2^k limbs) against the
slice size (DOTG_HOST_SLICE_MB, one process per setting: the knob is read once) and the
same bytes moved with no kernels (16 B up + 8 B down per limb, two streams)."""
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import ctypes, json, sys, time
sys.path.insert(0, ROOT)
import torch
import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W
M = 1 << LG
a, b = W.c5_inputs(False, m=M, run=(3 * M // 8, 5 * M // 8))
ha = torch.empty(M, dtype=torch.int64, pin_memory=True); ha.copy_(a)
hb = torch.empty(M, dtype=torch.int64, pin_memory=True); hb.copy_(b)
del a, b
torch.cuda.empty_cache()
ho = torch.empty(M, dtype=torch.int64, pin_memory=True)
L = dg.lib(); c = ctypes.c_uint32(0)
P = lambda t: ctypes.c_void_p(t.data_ptr())
assert L.dotg_add_words_host(P(ho), P(ha), P(hb), M, ctypes.byref(c)) == 0
t0 = time.perf_counter()
for _ in range(3):
    L.dotg_add_words_host(P(ho), P(ha), P(hb), M, ctypes.byref(c))
dt = (time.perf_counter() - t0) / 3
res = {"e2e_gbs": 24 * M / dt / 1e9}
if XFER:
    da = torch.empty(2 * M, dtype=torch.int64, device="cuda"); db = torch.empty(M, dtype=torch.int64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ch = 3 << 20
    def xfer():
        with torch.cuda.stream(s1):
            for i in range(0, M, ch):
                j = min(i + ch, M)
                da[i:j].copy_(ha[i:j], non_blocking=True)
                da[M + i:M + j].copy_(hb[i:j], non_blocking=True)
        with torch.cuda.stream(s2):
            for i in range(0, M, ch):
                j = min(i + ch, M)
                ho[i:j].copy_(db[i:j], non_blocking=True)
        torch.cuda.synchronize()
    xfer()
    t0 = time.perf_counter()
    for _ in range(3):
        xfer()
    res["transfer_only_gbs"] = 24 * M / ((time.perf_counter() - t0) / 3) / 1e9
print(json.dumps(res))
'''
LG = int(sys.argv[1]) if len(sys.argv) > 1 else 30
for mb in ("8", "24", "48"):
    env = {**os.environ, "DOTG_HOST_SLICE_MB": mb}
    code = CHILD.replace("ROOT", repr(ROOT)).replace("LG", str(LG)).replace("XFER", "False")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    out = r.stdout.strip().splitlines()[-1] if r.returncode == 0 else r.stderr[-500:]
    print(json.dumps({"slice_mb": int(mb), "limbs": 1 << LG, "result": out}))
