"""Batched column multiplication on the B200 vs the oracle (bit-exact, exactly 2m limbs)."""
import os

import numpy as np
import pytest

from helpers import MAX, category, uniform

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_vectors.npz")


def dev(torch, x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint64)


def mul(torch, a, b, layout="row"):
    import paper_2604_21566_b200 as dg

    if layout == "row":
        return host(dg.mul_batch(dev(torch, a), dev(torch, b)))
    return host(dg.mul_batch(dev(torch, a.T.copy()), dev(torch, b.T.copy()), layout="interleaved")).T.copy()


@pytest.fixture(params=["auto", "imad"])
def route(request, cuda):
    """Run a test on the default route (IMMA tensor-pipe kernels where they apply) and
    again with the IMAD column kernels forced, so both stay bit-exact."""
    import paper_2604_21566_b200 as dg

    prev = dg.set_mul_route(request.param)
    yield request.param
    dg.set_mul_route(prev)


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 24, 32, 33, 48, 64, 100, 128])
def test_mul_matches_oracle(cuda, oracle, route, m):
    rng = np.random.default_rng(2000 + m)
    n = 67
    for cat in ("random", "full_propagation", "spiky", "maxed_limbs", "zero_limbs"):
        a, b = category(rng, cat, "mul", (n, m))
        want = oracle.mul_batch(a, b)
        for layout in ("row", "interleaved"):
            got = mul(cuda, a, b, layout)
            assert got.shape == (n, 2 * m)
            assert np.array_equal(got, want), (m, cat, layout)


@pytest.mark.parametrize("m", [8, 16, 32, 64, 128])
@pytest.mark.parametrize("n", [1, 3, 4, 5, 130])
def test_imma_shapes(cuda, oracle, m, n):
    """The IMMA kernel (one warp per pair, 4 pairs per CTA): partial last CTA, all-ones
    operands (largest column sums, 2^27 per byte column at m = 128), single-byte spikes at
    block edges, and a misaligned view that must take the IMAD route instead."""
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(31 * m + n)
    prev = dg.set_mul_route("imma")
    try:
        for cat in ("random", "maxed_limbs", "spiky", "full_propagation"):
            a, b = category(rng, cat, "mul", (n, m))
            assert np.array_equal(mul(torch, a, b), oracle.mul_batch(a, b)), (m, n, cat)
        a = np.full((n, m), MAX, np.uint64)
        assert np.array_equal(mul(torch, a, a), oracle.mul_batch(a, a))
        a = np.zeros((n, m), np.uint64)
        b = np.zeros((n, m), np.uint64)
        a[:, ::4] = np.uint64(0xFF << 56)  # top byte of every 32-byte block
        b[:, 3::4] = np.uint64(0xFF)  # low byte of every block's last limb
        assert np.array_equal(mul(torch, a, b), oracle.mul_batch(a, b))
        # 8-byte (not 32-byte) aligned operands: IMAD fallback, still exact
        a, b = uniform(rng, (n, m)), uniform(rng, (n, m))
        da = dev(torch, np.concatenate([np.zeros(1, np.uint64), a.ravel()]))[1:].view(n, m)
        db = dev(torch, np.concatenate([np.zeros(1, np.uint64), b.ravel()]))[1:].view(n, m)
        assert np.array_equal(host(dg.mul_batch(da, db)), oracle.mul_batch(a, b))
    finally:
        dg.set_mul_route(prev)


def test_mul_route_knob(cuda):
    import paper_2604_21566_b200 as dg

    prev = dg.set_mul_route("imad")
    assert dg.set_mul_route("imma") == "imad"
    assert dg.set_mul_route(prev) == "imma"
    with pytest.raises(dg.InvalidArgument):
        dg.set_mul_route("fp64")


def test_golden_replay(cuda):
    g = np.load(GOLDEN)
    sizes = sorted({int(k.split("_")[1][1:]) for k in g.files if k.startswith("mul_")})
    for m in sizes:
        got = mul(cuda, g[f"mul_m{m}_a"], g[f"mul_m{m}_b"])
        assert np.array_equal(got, g[f"mul_m{m}_out"]), m


def test_mul_kats(cuda):
    # test_oracle.cpp:95-104, test_mul.cpp:183-196, 288-294, 323-331
    got = mul(cuda, np.array([[MAX]], np.uint64), np.array([[MAX]], np.uint64))
    assert list(got[0]) == [1, MAX - np.uint64(1)]
    got = mul(cuda, np.array([[0, 1]], np.uint64), np.array([[0, 1]], np.uint64))
    assert list(got[0]) == [0, 0, 1, 0]
    a = np.zeros((1, 4), np.uint64)
    b = np.zeros((1, 4), np.uint64)
    a[0, 2] = np.uint64(1 << 63)
    b[0, 3] = np.uint64(1 << 63)
    got = mul(cuda, a, b)  # 2^(64*2+63) * 2^(64*3+63) = 2^(64*6 + 62)
    want = np.zeros(8, np.uint64)
    want[6] = np.uint64(1 << 62)
    assert np.array_equal(got[0], want)
    ones = np.full((1, 4), MAX, np.uint64)  # (2^256 - 1)^2
    n = (1 << 256) - 1
    v = sum(int(x) << (64 * i) for i, x in enumerate(mul(cuda, ones, ones)[0]))
    assert v == n * n


def test_mul_algebra(cuda):
    # commutativity / identity / zero (test_mul.cpp:377-389), distributivity (391-411)
    rng = np.random.default_rng(25)
    for m in (1, 5, 16, 33, 64):
        a, b, c = uniform(rng, (20, m)), uniform(rng, (20, m)), uniform(rng, (20, m))
        assert np.array_equal(mul(cuda, a, b), mul(cuda, b, a))
        one = np.zeros((20, m), np.uint64)
        one[:, 0] = 1
        ab1 = mul(cuda, a, one)
        assert np.array_equal(ab1[:, :m], a) and not ab1[:, m:].any()
        assert not mul(cuda, a, np.zeros_like(a)).any()


def test_mul_errors(cuda):
    import paper_2604_21566_b200 as dg

    torch = cuda
    e = torch.empty((3, 0), dtype=torch.int64, device="cuda")
    with pytest.raises(dg.InvalidArgument):
        dg.mul_batch(e, e)  # m = 0 (mul.cpp:16)
    with pytest.raises(dg.InvalidArgument):
        dg.dot_mul_words([1, 2], [1])  # length mismatch (mul.cpp:13-14)
    with pytest.raises(dg.InvalidArgument):
        dg.dot_mul_words([], [])


@pytest.mark.parametrize("cfg", ["C3", "C4"])
def test_config_parity_full_size(cuda, oracle, route, cfg):
    import paper_2604_21566_b200 as dg
    from paper_2604_21566_b200 import workloads as W

    a, b = W.c3_inputs() if cfg == "C3" else W.c4_inputs()
    m = a.shape[1]
    ha, hb = host(a), host(b)
    if cfg == "C3":
        assert (ha[:, m - 1] != 0).all() and (hb[:, m - 1] != 0).all()
    else:
        assert (ha[a.shape[0] // 2:] == MAX).all()
    got = host(dg.mul_batch(a, b))
    want = oracle.mul_batch(ha, hb)
    assert np.array_equal(got, want)


def test_row_pitched_views(cuda, oracle):
    """dotg_mul_batch_strided: operands and product as row-pitched views of wider tensors."""
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(505)
    for m, batch, wa, wb, wo in ((16, 300, 20, 16, 40), (64, 100, 64, 70, 128), (3, 50, 5, 4, 9), (200, 7, 210, 200, 400)):
        A = uniform(rng, (batch, wa))
        B = uniform(rng, (batch, wb))
        A[0, :m] = MAX
        B[0, :m] = MAX
        ta = torch.from_numpy(A.view(np.int64)).cuda()[:, :m]
        tb = torch.from_numpy(B.view(np.int64)).cuda()[:, :m]
        O = torch.full((batch, wo), 7, dtype=torch.int64, device="cuda")
        got = dg.mul_batch(ta, tb, out=O[:, : 2 * m])
        want = oracle.mul_batch(np.ascontiguousarray(A[:, :m]), np.ascontiguousarray(B[:, :m]))
        Oh = O.cpu().numpy().view(np.uint64)
        assert np.array_equal(Oh[:, : 2 * m], want), m
        assert (Oh[:, 2 * m:] == 7).all()  # the rest of each row untouched
        assert np.array_equal(dg.mul_batch(ta, tb).cpu().numpy().view(np.uint64), want)


@pytest.mark.parametrize("m", [17, 18, 32, 33, 47, 64, 65, 80, 95, 96, 97, 126, 127, 128])
@pytest.mark.parametrize("n", [1, 2, 3, 5, 9, 1031])
def test_interleaved_tensor_pipe_in_place(cuda, oracle, m, n):
    """The interleaved tensor-pipe route reads and writes [m][batch] in place through
    CTA tiles of 4 consecutive pairs: partial last groups (batch % 4 != 0, batch < 4),
    zero-extended rows (m < the kernel's size), all-ones operands."""
    rng = np.random.default_rng(7 * m + n)
    a, b = category(rng, "random", "mul", (n, m))
    a[::3] = MAX
    b[1::4] = MAX
    want = oracle.mul_batch(a, b)
    assert np.array_equal(mul(cuda, a, b, "interleaved"), want), (m, n)


EXACT_CHILD = r'''
import sys
sys.path.insert(0, ROOT + "/tests"); sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2604_21566_b200 as dg
from helpers import Oracle, category
orc = Oracle()
bad = []
for m in (3, 5, 6, 7, 9, 10, 11, 12, 13, 14, 15):
    rng = np.random.default_rng(4400 + m)
    for cat in ("random", "maxed_limbs", "spiky"):
        a, b = category(rng, cat, "mul", (131, m))
        want = orc.mul_batch(a, b)
        ta = torch.from_numpy(a.view(np.int64)).cuda(); tb = torch.from_numpy(b.view(np.int64)).cuda()
        got = dg.mul_batch(ta, tb).cpu().numpy().view(np.uint64)
        il = dg.mul_batch(ta.t().contiguous(), tb.t().contiguous(), layout="interleaved")
        if not (np.array_equal(got, want) and np.array_equal(il.cpu().numpy().view(np.uint64).T, want)):
            bad.append([m, cat])
print("BAD", bad)
'''


@pytest.mark.parametrize("exact", ["1", "3"])
def test_exact_small_kernels_every_odd_size(cuda, exact):
    """The exact-m register kernels for m in 3 ... 15 off the powers of two, both layouts,
    odd row-major rows staged through shared memory (DOTG_MUL_EXACT=1, the default) and
    unstaged (=3); partial last CTAs (131 pairs)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", EXACT_CHILD.replace("ROOT", repr(root))],
                       env={**os.environ, "DOTG_MUL_EXACT": exact}, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().splitlines()[-1] == "BAD []", r.stdout[-2000:]


@pytest.mark.parametrize("m", [17, 18, 19, 20, 21, 23, 24, 25, 27, 28, 29, 30, 31, 33, 40, 47, 48, 49, 65, 72, 80, 90, 96, 97, 110, 112, 127, 129, 160, 161, 200, 224, 255])
def test_tensor_pipe_multiple_of_16_sizes(cuda, oracle, m):
    """Sizes between the powers of two on the tensor pipe: 48 / 80 / 96 / 112 limbs
    exactly (k_mul_imma<12 / 20 / 24 / 28>, operand words not a power of two per lane),
    even m zero-extended in the ring to the next multiple of 16, odd m copy-padded; random,
    all-ones (the largest column sums) and partial last warps."""
    rng = np.random.default_rng(5100 + m)
    for n in (1, 7, 301):
        a, b = category(rng, "random", "mul", (n, m))
        a[::2] = MAX
        b[::3] = MAX
        want = oracle.mul_batch(a, b)
        assert np.array_equal(mul(cuda, a, b, "row"), want), (m, n)
