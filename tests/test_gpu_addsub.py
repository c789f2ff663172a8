"""Batched add/sub on the B200 through the C ABI vs the oracle (bit-exact)."""
import os

import numpy as np
import pytest

from helpers import CATEGORIES, MAX, category, rows_less_np, spiky, uniform

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_vectors.npz")


def dev(torch, x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint64)


def run(torch, sub, a, b, layout="row"):
    import paper_2604_21566_b200 as dg

    if layout == "row":
        out, fl = dg.addsub_batch(sub, dev(torch, a), dev(torch, b))
        return host(out), fl.cpu().numpy().view(np.uint32)
    out, fl = dg.addsub_batch(sub, dev(torch, a.T.copy()), dev(torch, b.T.copy()), layout="interleaved")
    return host(out).T.copy(), fl.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 7, 8, 9, 13, 16, 17, 31, 32, 33, 64, 65, 100, 128, 256, 512, 1000])
def test_batch_matches_oracle(cuda, oracle, m):
    rng = np.random.default_rng(1000 + m)
    for cat in CATEGORIES:
        for op in ("add", "sub"):
            a, b = category(rng, cat, op, (97, m))
            want, wf = oracle.addsub_batch(op == "sub", a, b)
            for layout in ("row", "interleaved"):
                got, gf = run(cuda, op == "sub", a, b, layout)
                assert np.array_equal(got, want), (m, cat, op, layout)
                assert np.array_equal(gf, wf), (m, cat, op, layout)


@pytest.mark.parametrize("m,batch", [(1025, 64), (1500, 33), (4100, 40), (8200, 3)])
def test_interleaved_two_pass(cuda, oracle, m, batch):
    """Interleaved numbers longer than 1024 limbs: the two streaming passes (segments of 8
    limbs resolved with carry-in 0, then the per-pair carry scan and prefix fix-up),
    including propagate runs across many segments and the flags."""
    rng = np.random.default_rng(7000 + m)
    for cat in ("random", "full_propagation", "spiky", "maxed_limbs"):
        for op in ("add", "sub"):
            a, b = category(rng, cat, op, (batch, m))
            if cat == "random":  # a long propagate run straddling segments in some pairs
                a[::3, 5:m - 7] = np.uint64(0xFFFFFFFFFFFFFFFF) if op == "add" else b[::3, 5:m - 7]
                if op == "add":
                    b[::3, 5:m - 7] = 0
            want, wf = oracle.addsub_batch(op == "sub", a, b)
            got, gf = run(cuda, op == "sub", a, b, "interleaved")
            assert np.array_equal(got, want), (m, cat, op)
            assert np.array_equal(gf, wf), (m, cat, op)


@pytest.mark.parametrize("m,batch", [(128, 128), (200, 130), (256, 64), (256, 190), (129, 66), (257, 40),
                                     (300, 65), (384, 32), (512, 33), (513, 31), (777, 40), (1024, 33)])
def test_interleaved_segmented(cuda, oracle, m, batch):
    # 128 <= m <= 1024 take k_addsub_ilf (row segments per warp, one CTA per strip of
    # pairs): ragged m the partial last segment, batch % 32 != 0 the partial strip
    rng = np.random.default_rng(7000 + m + batch)
    for cat in CATEGORIES:
        for op in ("add", "sub"):
            a, b = category(rng, cat, op, (batch, m))
            want, wf = oracle.addsub_batch(op == "sub", a, b)
            got, gf = run(cuda, op == "sub", a, b, "interleaved")
            assert np.array_equal(got, want), (m, batch, cat, op)
            assert np.array_equal(gf, wf), (m, batch, cat, op)


def test_golden_replay(cuda):
    g = np.load(GOLDEN)
    sizes = sorted({int(k.split("_")[1][1:]) for k in g.files if k.startswith("addsub_")})
    for m in sizes:
        a, b = g[f"addsub_m{m}_a"], g[f"addsub_m{m}_b"]
        for sub, key in ((False, "add"), (True, "sub")):
            got, gf = run(cuda, sub, a, b)
            assert np.array_equal(got, g[f"addsub_m{m}_{key}_out"]), (m, key)
            assert np.array_equal(gf, g[f"addsub_m{m}_{key}_flag"]), (m, key)


def test_kats(cuda):
    # test_addsub.cpp:124-155: (2^512-1)+1, identity, cross-chunk carry into a tail, 0-1
    cases = [
        (False, [MAX] * 8, [1] + [0] * 7, [0] * 8, 1),
        (False, [MAX] * 9, [1] + [0] * 8, [0] * 9, 1),
        (True, [0], [1], [MAX], 1),
        (False, [MAX, MAX] + [0] * 6, [1] + [0] * 7, [0, 0, 1, 0, 0, 0, 0, 0], 0),
    ]
    for sub, a, b, want, wf in cases:
        got, gf = run(cuda, sub, np.array([a], np.uint64), np.array([b], np.uint64))
        assert list(got[0]) == want and gf[0] == wf


def test_full_chains_every_size(cuda, oracle):
    # full propagation chains across every team/row boundary (test_addsub.cpp:299-317)
    for m in (1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 7, 33):
        a = np.full((3, m), MAX, np.uint64)
        b = np.zeros((3, m), np.uint64)
        b[:, 0] = 1
        got, gf = run(cuda, False, a, b)
        assert not got.any() and (gf == 1).all(), m
        got, gf = run(cuda, True, np.zeros((3, m), np.uint64), b)
        assert (got == MAX).all() and (gf == 1).all(), m


def test_aliasing_and_edge_cases(cuda, oracle):
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(7)
    a, b = spiky(rng, (300, 64)), spiky(rng, (300, 64))
    want, wf = oracle.addsub_batch(False, a, b)
    ta, tb = dev(torch, a), dev(torch, b)
    out, fl = dg.add_batch(ta, tb, out=ta)  # out aliases a exactly
    assert np.array_equal(host(ta), want) and np.array_equal(fl.cpu().numpy().view(np.uint32), wf)
    ta, tb = dev(torch, a), dev(torch, b)
    dg.add_batch(ta, tb, out=tb)  # out aliases b exactly
    assert np.array_equal(host(tb), want)
    # partial overlap is rejected
    big = dev(torch, uniform(rng, (301, 64)))
    with pytest.raises(dg.InvalidArgument):
        dg.api.check(dg.lib().dotg_add_batch(
            dg.api._dptr(big[1:]), dg.api._dptr(big[:-1]), dg.api._dptr(big[:-1]), None, 64, 300, 0, None))
    # m = 0: flags are zero; batch = 0: no-op
    fl = torch.full((5,), 7, dtype=torch.int32, device="cuda")
    e = torch.empty((5, 0), dtype=torch.int64, device="cuda")
    dg.add_batch(e, e, out=e.clone(), flags=fl)
    assert (fl == 0).all()
    e0 = torch.empty((0, 4), dtype=torch.int64, device="cuda")
    dg.sub_batch(e0, e0)


def test_misaligned_rows_fall_back(cuda, oracle):
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(8)
    a, b = spiky(rng, (50, 64)), spiky(rng, (50, 64))
    want, wf = oracle.addsub_batch(True, a, b)
    buf_a = torch.zeros(50 * 64 + 1, dtype=torch.int64, device="cuda")
    buf_b = torch.zeros(50 * 64 + 1, dtype=torch.int64, device="cuda")
    buf_a[1:] = dev(torch, a).view(-1)
    buf_b[1:] = dev(torch, b).view(-1)
    out = torch.zeros(50 * 64 + 1, dtype=torch.int64, device="cuda")
    _, fl = dg.sub_batch(buf_a[1:].view(50, 64), buf_b[1:].view(50, 64), out=out[1:].view(50, 64))
    assert np.array_equal(host(out[1:]).reshape(50, 64), want)
    assert np.array_equal(fl.cpu().numpy().view(np.uint32), wf)


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_config_parity_full_size(cuda, oracle, cfg):
    """C1 / C2 at BASELINE.json's full sizes vs the oracle (every pair, add and sub)."""
    import paper_2604_21566_b200 as dg
    from paper_2604_21566_b200 import workloads as W

    sizes = [(W.C1["m"], W.C1["batch"])] if cfg == "C1" else W.C2_SIZES
    for m, B in sizes:
        a, b, sa, sb = W.c1_inputs() if cfg == "C1" else W.c2_inputs(m, B)
        assert a.shape == (B, m)
        ha, hb, hsa, hsb = host(a), host(b), host(sa), host(sb)
        assert not rows_less_np(hsa, hsb).any()  # a >= b after the swap
        out, fl = dg.add_batch(a, b)
        want, wf = oracle.addsub_batch(False, ha, hb)
        assert np.array_equal(host(out), want) and np.array_equal(fl.cpu().numpy().view(np.uint32), wf)
        out, fl = dg.sub_batch(sa, sb)
        want, wf = oracle.addsub_batch(True, hsa, hsb)
        assert np.array_equal(host(out), want) and not wf.any()
        assert np.array_equal(fl.cpu().numpy().view(np.uint32), wf)
        if cfg == "C2":
            assert (host(a)[::100] == MAX).all()  # forced 1% chains
            got = host(out)  # sub of forced rows: (2^n - 1) - 1
            assert (got[::100, 0] == MAX - np.uint64(1)).all()


def test_device_fill_matches_host_twin(cuda, oracle):
    from paper_2604_21566_b200 import workloads as W

    for n, seed, off in ((1, 1, 0), (1000, 0xC5, 12345), (1 << 20, 0xC1, 1 << 40)):
        assert np.array_equal(host(W.fill(n, seed, off)), oracle.fill(n, seed, off))


def test_grouped_matches_oracle(cuda, oracle):
    """Several sizes, both ops, mixed layouts and one non-power-of-two problem in one call."""
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(31)
    specs = [("add", 4, 3000), ("sub", 16, 1001), ("add", 64, 257), ("sub", 256, 33), ("add", 512, 9),
             ("sub", 7, 100), ("add", 1, 5000), ("sub", 2, 77), ("add", 128, 64), ("sub", 32, 999)]
    probs, wants = [], []
    for i, (op, m, B) in enumerate(specs):
        a, b = category(rng, CATEGORIES[i % len(CATEGORIES)], op, (B, m))
        wants.append(oracle.addsub_batch(op == "sub", a, b))
        lay = "interleaved" if i == 5 else "row"
        ta, tb = (dev(torch, a.T.copy()), dev(torch, b.T.copy())) if lay == "interleaved" else (dev(torch, a), dev(torch, b))
        probs.append(dict(op=op, a=ta, b=tb, out=torch.empty_like(ta), layout=lay,
                          flags=torch.empty(B, dtype=torch.int32, device="cuda")))
    dg.addsub_grouped(probs)
    for q, (want, wf), (op, m, B) in zip(probs, wants, specs):
        got = host(q["out"])
        if q["layout"] == "interleaved":
            got = got.T
        assert np.array_equal(got, want), (op, m)
        assert np.array_equal(q["flags"].cpu().numpy().view(np.uint32), wf), (op, m)
    # dependent problems are rejected
    a = dev(torch, uniform(rng, (10, 4)))
    with pytest.raises(dg.InvalidArgument):
        dg.addsub_grouped([dict(op="add", a=a, b=a, out=torch.empty_like(a)),
                           dict(op="add", a=a, b=a, out=a)])


@pytest.mark.parametrize("m,batch", [(5, 300), (100, 77), (1000, 9), (9000, 3)])
def test_aliasing_every_route(cuda, oracle, m, batch):
    """out == a and out == b (exactly) on the any-m row kernel and the long-batch passes."""
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(900 + m)
    a, b = spiky(rng, (batch, m)), spiky(rng, (batch, m))
    for sub in (False, True):
        want, wf = oracle.addsub_batch(sub, a, b)
        ta, tb = dev(torch, a), dev(torch, b)
        _, fl = dg.addsub_batch(sub, ta, tb, out=ta)
        assert np.array_equal(host(ta), want) and np.array_equal(fl.cpu().numpy().view(np.uint32), wf), (m, sub)
        ta, tb = dev(torch, a), dev(torch, b)
        _, fl = dg.addsub_batch(sub, ta, tb, out=tb)
        assert np.array_equal(host(tb), want) and np.array_equal(fl.cpu().numpy().view(np.uint32), wf), (m, sub)


def test_row_pitched_views(cuda, oracle):
    """dotg_addsub_batch_strided (row pitches, SURVEY.md §8(b) stride_limbs): views of wider
    tensors, mixed pitches, exact in-place aliasing, pitch == m taking the dense route."""
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(404)
    for m, batch, wa, wb in ((5, 300, 8, 7), (64, 1000, 80, 64), (1, 50, 3, 2), (17, 1, 17, 40)):
        A = spiky(rng, (batch, wa))
        B = spiky(rng, (batch, wb))
        a, b = A[:, :m], B[:, :m]
        ta = torch.from_numpy(A.view(np.int64)).cuda()[:, :m]
        tb = torch.from_numpy(B.view(np.int64)).cuda()[:, :m]
        for sub in (False, True):
            want, wf = oracle.addsub_batch(sub, np.ascontiguousarray(a), np.ascontiguousarray(b))
            out, fl = dg.addsub_batch(sub, ta, tb)
            assert np.array_equal(out.cpu().numpy().view(np.uint64), want), (m, sub)
            assert np.array_equal(fl.cpu().numpy().view(np.uint32), wf)
            # in place into a pitched view
            tc = torch.from_numpy(A.view(np.int64).copy()).cuda()
            tcv = tc[:, :m]
            dg.addsub_batch(sub, tcv, tb, out=tcv)
            got = tc.cpu().numpy().view(np.uint64)
            assert np.array_equal(got[:, :m], want) and np.array_equal(got[:, m:], A[:, m:])
    # partial overlap is rejected
    T = torch.zeros((10, 16), dtype=torch.int64, device="cuda")
    with pytest.raises(dg.InvalidArgument):
        dg.addsub_batch(False, T[:, 0:8], T[:, 8:16], out=T[:, 4:12])


ROWS_CHILD = r'''
import sys
sys.path.insert(0, ROOT + "/tests"); sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2604_21566_b200 as dg
from helpers import CATEGORIES, Oracle, category
orc = Oracle()
bad = []
for m, batch in [(1, 4096), (1, 4097), (3, 301), (5, 97), (33, 130), (100, 41), (257, 12), (1000, 9), (2048, 5),
                 (4096, 3)]:
    rng = np.random.default_rng(77 + m)
    for cat in CATEGORIES:
        for op in ("add", "sub"):
            a, b = category(rng, cat, op, (batch, m))
            want, wf = orc.addsub_batch(op == "sub", a, b)
            ta = torch.from_numpy(a.view(np.int64)).cuda()
            tb = torch.from_numpy(b.view(np.int64)).cuda()
            out, fl = dg.addsub_batch(op == "sub", ta, tb)
            if not (np.array_equal(out.cpu().numpy().view(np.uint64), want)
                    and np.array_equal(fl.cpu().numpy().view(np.uint32), wf)):
                bad.append([m, batch, cat, op])
print("BAD", bad)
'''


@pytest.mark.parametrize("u", ["1", "2", "4"])
def test_rows_any_chunks_in_flight(cuda, u):
    """The any-m row kernel with 1, 2 and 4 chunks of loads in flight per warp (DOTG_ROWS_U,
    read once per process: one child each; DOTG_ROWS_STAGED=0 keeps m < 64 on it too),
    ragged m and pow2 m above 512."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", ROWS_CHILD.replace("ROOT", repr(root))],
                       env={**os.environ, "DOTG_ROWS_U": u, "DOTG_ROWS_STAGED": "0"}, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().splitlines()[-1] == "BAD []", r.stdout[-2000:]


@pytest.mark.parametrize("m", [3, 5, 6, 7, 9, 11, 12])
def test_rows_staged_partial_ctas(cuda, oracle, m):
    """Row-major 3 <= m <= 7 off the powers of two (k_addsub_rows_staged; 9 ... 12 on the
    any-m kernel): batches that leave a partial last CTA with an odd limb count, in place."""
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(6600 + m)
    for batch in (1, 33, 129, 1001):
        for sub in (False, True):
            a, b = spiky(rng, (batch, m)), spiky(rng, (batch, m))
            want, wf = oracle.addsub_batch(sub, a, b)
            got, gf = run(torch, sub, a, b)
            assert np.array_equal(got, want) and np.array_equal(gf, wf), (m, batch, sub)
            ta, tb = dev(torch, a), dev(torch, b)
            _, fl = dg.addsub_batch(sub, ta, tb, out=ta)
            assert np.array_equal(host(ta), want) and np.array_equal(fl.cpu().numpy().view(np.uint32), wf)
