"""C3 parity spot check of the 16-limb multiply route (every test category, all-ones, and
the full C3 batch) against the oracle; used for kernel A/B builds via DOTG_LIB_PATH."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_21566_b200 as dg  # noqa: E402
from helpers import CATEGORIES, Oracle, category  # noqa: E402
from paper_2604_21566_b200 import workloads as W  # noqa: E402

orc = Oracle()
rng = np.random.default_rng(3)


def mul(a, b):
    return dg.mul_batch(torch.from_numpy(a.view(np.int64)).cuda(),
                        torch.from_numpy(b.view(np.int64)).cuda()).cpu().numpy().view(np.uint64)


for cat in CATEGORIES:
    a, b = category(rng, cat, "add", (1000, 16))
    assert np.array_equal(mul(a, b), orc.mul_batch(a, b)), cat
a = np.full((64, 16), np.uint64(0xFFFFFFFFFFFFFFFF))
assert np.array_equal(mul(a, a), orc.mul_batch(a, a))
a, b = W.c3_inputs()
ha, hb = a.cpu().numpy().view(np.uint64), b.cpu().numpy().view(np.uint64)
assert np.array_equal(dg.mul_batch(a, b).cpu().numpy().view(np.uint64), orc.mul_batch(ha, hb))
print("16-limb multiply parity ok")
