"""Driver for the r02 ncu captures (one call per kernel of interest, after warm-ups):
the C1 add + sub launch (k_addsub_grouped, 2 x 65536 4096-bit pairs), the C5 long-number
passes (k_long_local / k_long_finish, 2^30 limbs) and the timed team kernel."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W

torch.cuda.set_device(0)
L = dg.lib()
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
which = sys.argv[1] if len(sys.argv) > 1 else "c1"
if which == "c1":
    a, b, sa, sb = W.c1_inputs()
    o, o2 = torch.empty_like(a), torch.empty_like(a)
    f, f2 = torch.empty(a.shape[0], dtype=torch.int32, device="cuda"), torch.empty(a.shape[0], dtype=torch.int32, device="cuda")
    for _ in range(4):
        dg.api.addsub_grouped([dict(op="add", a=a, b=b, out=o, flags=f), dict(op="sub", a=sa, b=sb, out=o2, flags=f2)])
elif which == "c5":
    a, b = W.c5_inputs(False)
    o = torch.empty_like(a)
    c = torch.empty(1, dtype=torch.int32, device="cuda")
    for _ in range(3):
        L.dotg_add_words(P(o), P(a), P(b), a.numel(), P(c), None)
torch.cuda.synchronize()
print("ok", which)
