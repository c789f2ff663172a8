import os, sys
sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2604_21566_b200 as dg
from paper_2604_21566_b200 import workloads as W
from helpers import Oracle, spiky, category, CATEGORIES
orc = Oracle()
rng = np.random.default_rng(3)
for cat in CATEGORIES:
    a, b = category(rng, cat, "add", (1000, 16))
    got = dg.mul_batch(torch.from_numpy(a.view(np.int64)).cuda(), torch.from_numpy(b.view(np.int64)).cuda()).cpu().numpy().view(np.uint64)
    assert np.array_equal(got, orc.mul_batch(a, b)), cat
a = np.full((64, 16), np.uint64(0xFFFFFFFFFFFFFFFF)); 
assert np.array_equal(dg.mul_batch(torch.from_numpy(a.view(np.int64)).cuda(), torch.from_numpy(a.view(np.int64)).cuda()).cpu().numpy().view(np.uint64), orc.mul_batch(a, a))
a, b = W.c3_inputs()
got = dg.mul_batch(a, b)
ha, hb = a.cpu().numpy().view(np.uint64), b.cpu().numpy().view(np.uint64)
assert np.array_equal(got.cpu().numpy().view(np.uint64), orc.mul_batch(ha, hb))
print("kara16 parity ok")
