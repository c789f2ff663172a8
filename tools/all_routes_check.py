"""One small call through every kernel family (written to run under compute-sanitizer;
the tool is closed on this GPU pool, so it runs as a plain exact-integer sweep): batched
add/sub on every route (team, grouped, any-m, long batch,
interleaved segmented / strided), long numbers and shards, multiply on every route (IMAD
register / shared / generic, tensor pipe full and zero-extended, padded, Karatsuba,
interleaved transposes), long numbers. Results are checked against exact Python
integers."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2604_21566_b200 as dg

rng = np.random.default_rng(5)
M64 = (1 << 64) - 1


def val(row):
    return sum(int(x) << (64 * i) for i, x in enumerate(row))


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint64)


def rand(shape):
    a = rng.integers(0, 2**64, size=shape, dtype=np.uint64)
    a[..., ::3] = np.uint64(M64)
    return a


def check_addsub(m, n, layout="row"):
    a, b = rand((n, m)), rand((n, m))
    for sub in (False, True):
        if layout == "row":
            out, fl = dg.addsub_batch(sub, dev(a), dev(b))
            o = host(out)
        else:
            out, fl = dg.addsub_batch(sub, dev(a.T.copy()), dev(b.T.copy()), layout="interleaved")
            o = host(out).T
        f = fl.cpu().numpy().view(np.uint32)
        for p in range(n):
            x, y = val(a[p]), val(b[p])
            r = (x - y) if sub else (x + y)
            assert val(o[p]) == r % (1 << (64 * m)) and int(f[p]) == int(r < 0 if sub else r >> (64 * m)), (m, p)


def check_mul(m, n, layout="row", route="auto"):
    prev = dg.set_mul_route(route)
    a, b = rand((n, m)), rand((n, m))
    if layout == "row":
        o = host(dg.mul_batch(dev(a), dev(b)))
    else:
        o = host(dg.mul_batch(dev(a.T.copy()), dev(b.T.copy()), layout="interleaved")).T
    for p in range(n):
        assert val(o[p]) == val(a[p]) * val(b[p]), (m, p, layout, route)
    dg.set_mul_route(prev)


for m in (1, 3, 4, 16, 64, 100, 256, 512, 9000):
    check_addsub(m, 5 if m < 9000 else 2)
for m in (4, 64, 200, 300, 700):
    check_addsub(m, 40, "interleaved")
for m in (1, 4, 5, 8, 12, 16, 24, 33, 64, 96, 128, 200, 256, 1000, 4096, 5000):  # ... tcgen05 direct / split
    check_mul(m, 9 if m <= 1000 else 2)
for m in (8, 16):
    check_mul(m, 9, route="imma")
for m in (32, 64):
    check_mul(m, 9, route="imad")
for m in (16, 40, 300):
    check_mul(m, 33, "interleaved")
x, y = rand(70000), rand(70000)
o, c = dg.add_words(dev(x), dev(y))
assert val(host(o)) == (val(x) + val(y)) % (1 << (64 * 70000))
print("all routes ok")
