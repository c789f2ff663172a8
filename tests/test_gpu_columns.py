"""The column pipeline stages on the device (gather_columns, compute_partials,
align_and_reduce, carry_pass: mul.hpp:32-67, mul.cpp:12-90), restating the reference's
own stage tests (test_mul.cpp:54-252) with Python integers as the big-integer reference,
the batched device forms against the per-pair host forms, and the chained stages against
the fused product."""
import numpy as np
import pytest

from helpers import MAX, uniform

pytestmark = pytest.mark.gpu
M52 = (1 << 52) - 1


def test_num_pairs_and_gather(cuda):
    import paper_2604_21566_b200 as dg
    from paper_2604_21566_b200 import api

    for m in range(1, 9):
        counts = [sum(1 for i in range(m) for j in range(m) if i + j == c) for c in range(2 * m - 1)]
        assert [api.num_pairs(c, m) for c in range(2 * m - 1)] == counts and sum(counts) == m * m
        assert api.num_pairs(2 * m - 1, m) == 0
    rng = np.random.default_rng(11)
    for m in (1, 2, 5, 16, 33):
        a, b = uniform(rng, m), uniform(rng, m)
        ma, mb = api.gather_columns(a, b)
        want_a = [a[i] for c in range(2 * m - 1) for i in range(max(0, c + 1 - m), min(c, m - 1) + 1)]
        want_b = [b[c - i] for c in range(2 * m - 1) for i in range(max(0, c + 1 - m), min(c, m - 1) + 1)]
        assert np.array_equal(ma, np.array(want_a, np.uint64)) and np.array_equal(mb, np.array(want_b, np.uint64))
    with pytest.raises(dg.InvalidArgument):
        api.gather_columns([1, 2], [1])
    with pytest.raises(dg.InvalidArgument):
        api.gather_columns([], [])


@pytest.mark.parametrize("k", [64, 52])
def test_partials_split_at_k(cuda, k):
    from paper_2604_21566_b200 import api

    rng = np.random.default_rng(12 + k)
    mask = (1 << k) - 1
    for a, b in ((uniform(rng, 7), uniform(rng, 7)), (np.full(5, M52, np.uint64), np.full(5, M52, np.uint64)),
                 (np.zeros(3, np.uint64), np.zeros(3, np.uint64)), (np.full(4, MAX), np.full(4, MAX))):
        ma, mb = api.gather_columns(a, b)
        lo, hi = api.compute_partials(ma, mb, k)
        for t in range(ma.size):
            p = int(ma[t]) * int(mb[t])
            assert int(lo[t]) == p & mask and int(hi[t]) == (p >> k) & (2**64 - 1), (k, t)
    with pytest.raises(api.InvalidArgument):
        api.compute_partials([1], [1], 48)


def test_align_and_reduce(cuda):
    from paper_2604_21566_b200 import api

    rng = np.random.default_rng(15)
    # a lone pair: a[2] = b[3] = 2^63 -> column 6 holds 2^62, every other column 0
    a, b = np.zeros(4, np.uint64), np.zeros(4, np.uint64)
    a[2] = b[3] = np.uint64(1 << 63)
    cols = api.align_and_reduce(*api.compute_partials(*api.gather_columns(a, b)), 4)
    assert cols == [0] * 6 + [1 << 62, 0]
    # single limb: the split product
    cols = api.align_and_reduce(*api.compute_partials(*api.gather_columns([MAX], [MAX])), 1)
    p = (2**64 - 1) ** 2
    assert cols == [p & (2**64 - 1), p >> 64]
    for m in (1, 3, 4, 9, 40):
        for _ in range(5):
            a, b = uniform(rng, m), uniform(rng, m)
            cols = api.align_and_reduce(*api.compute_partials(*api.gather_columns(a, b)), m)
            want = [0] * (2 * m)
            for i in range(m):
                for j in range(m):
                    q = int(a[i]) * int(b[j])
                    want[i + j] += q & (2**64 - 1)
                    want[i + j + 1] += q >> 64
            assert cols == want, m


def _value(limbs, k):
    return sum(int(x) << (k * i) for i, x in enumerate(limbs))


@pytest.mark.parametrize("k", [64, 52])
def test_carry_pass(cuda, k):
    from paper_2604_21566_b200 import api

    rng = np.random.default_rng(16 + k)
    assert np.array_equal(api.carry_pass([0] * 10, k), np.zeros(10, np.uint64))
    full = (1 << 128) - 1
    for cols in ([full], [full, full], [full] * 5, [1 << 127, full, 0, full]):
        out = api.carry_pass(cols, k)
        assert _value(out, k) == _value(cols, k) and all(int(x) >> k == 0 for x in out)
    assert len(api.carry_pass([full], 52)) == 3  # residual appended, not truncated
    for _ in range(200):
        n = int(rng.integers(1, 13))
        cols = [int(rng.integers(0, 2**63)) << 65 | int(rng.integers(0, 2**63)) << 2 | int(rng.integers(0, 4))
                for _ in range(n)]
        out = api.carry_pass(cols, k)
        assert _value(out, k) == _value(cols, k) and all(int(x) >> k == 0 for x in out)


def test_batched_device_stages_and_chain(cuda, oracle):
    """Device batch forms equal the per-pair host forms; the chained stages reproduce the
    fused product (dot_mul_words = carry_pass(align_and_reduce(...)), mul.cpp:96-103)."""
    import paper_2604_21566_b200 as dg
    from paper_2604_21566_b200 import api

    torch = cuda
    rng = np.random.default_rng(17)
    m, batch = 12, 37
    a, b = uniform(rng, (batch, m)), uniform(rng, (batch, m))
    a[0] = MAX
    b[0] = MAX
    ta = torch.from_numpy(a.view(np.int64)).cuda()
    tb = torch.from_numpy(b.view(np.int64)).cuda()
    ma = torch.empty((batch, m * m), dtype=torch.int64, device="cuda")
    mb = torch.empty_like(ma)
    L, s = dg.lib(), api._stream_handle(None)
    api.check(L.dotg_gather_columns(api._dptr(ma), api._dptr(mb), api._dptr(ta), api._dptr(tb), m, batch, s))
    lo, hi = torch.empty_like(ma), torch.empty_like(ma)
    api.check(L.dotg_compute_partials(api._dptr(lo), api._dptr(hi), api._dptr(ma), api._dptr(mb), batch * m * m, 64, s))
    cols = torch.empty((batch, 4 * m), dtype=torch.int64, device="cuda")
    api.check(L.dotg_align_and_reduce(api._dptr(cols), api._dptr(lo), api._dptr(hi), m, batch, s))
    cap = 2 * m + 2
    out = torch.zeros((batch, cap), dtype=torch.int64, device="cuda")
    nout = torch.zeros(batch, dtype=torch.int32, device="cuda")
    api.check(L.dotg_carry_pass(api._dptr(out), api._dptr(nout), cap, api._dptr(cols), 2 * m, batch, 64, s))
    out, nout = out.cpu().numpy().view(np.uint64), nout.cpu().numpy()
    ma_h = ma.cpu().numpy().view(np.uint64)
    cols_h = cols.cpu().numpy().view(np.uint64)
    want = oracle.mul_batch(a, b)
    for p in range(batch):
        hm_a, hm_b = api.gather_columns(a[p], b[p])
        assert np.array_equal(ma_h[p], hm_a)
        hc = api.align_and_reduce(*api.compute_partials(hm_a, hm_b), m)
        assert [int(cols_h[p][2 * c]) | int(cols_h[p][2 * c + 1]) << 64 for c in range(2 * m)] == hc
        assert nout[p] == 2 * m and np.array_equal(out[p][: 2 * m], want[p])
        assert np.array_equal(api.carry_pass(hc), want[p])


def test_stages_match_reference_golden(cuda):
    """Device stages against the reference's OWN stage outputs (tests/golden/
    column_vectors.npz from oracle/_ref: gather_columns, compute_partials,
    align_and_reduce, carry_pass), limb for limb and including the output length of
    carry_pass (the residual limbs of raw columns, test_mul.cpp:229-252). Batched device
    forms for the pipeline cases, the host forms for the raw carry cases."""
    import os

    from paper_2604_21566_b200 import api

    torch = cuda
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "column_vectors.npz"))
    L, s = api.lib(), api._stream_handle(None)

    def dev(x):
        return torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()

    def host(t):
        return t.cpu().numpy().view(np.uint64)

    for m in g["sizes"]:
        m = int(m)
        for k in (64, 52):
            key = f"m{m}_k{k}"
            A, B = g[key + "_a"], g[key + "_b"]
            batch = A.shape[0]
            ta, tb = dev(A), dev(B)
            ma = torch.empty((batch, m * m), dtype=torch.int64, device="cuda")
            mb = torch.empty_like(ma)
            api.check(L.dotg_gather_columns(api._dptr(ma), api._dptr(mb), api._dptr(ta), api._dptr(tb), m, batch, s))
            assert np.array_equal(host(ma), g[key + "_ma"]) and np.array_equal(host(mb), g[key + "_mb"]), key
            lo, hi = torch.empty_like(ma), torch.empty_like(ma)
            api.check(L.dotg_compute_partials(api._dptr(lo), api._dptr(hi), api._dptr(ma), api._dptr(mb),
                                              batch * m * m, k, s))
            assert np.array_equal(host(lo), g[key + "_plo"]) and np.array_equal(host(hi), g[key + "_phi"]), key
            cols = torch.empty((batch, 4 * m), dtype=torch.int64, device="cuda")
            api.check(L.dotg_align_and_reduce(api._dptr(cols), api._dptr(lo), api._dptr(hi), m, batch, s))
            assert np.array_equal(host(cols).reshape(batch, 2 * m, 2), g[key + "_cols"]), key
            cap = 2 * m + 2
            out = torch.full((batch, cap), -1, dtype=torch.int64, device="cuda")
            nout = torch.zeros(batch, dtype=torch.int32, device="cuda")
            api.check(L.dotg_carry_pass(api._dptr(out), api._dptr(nout), cap, api._dptr(cols), 2 * m, batch, k, s))
            want = g[key + "_out"]
            assert (nout.cpu().numpy() == want.shape[1]).all(), key  # exactly the reference's length
            assert np.array_equal(host(out)[:, : want.shape[1]], want), key
    for k in (64, 52):
        cols, co = g[f"carry_k{k}_cols"], g[f"carry_k{k}_col_offsets"]
        outs, oo = g[f"carry_k{k}_out"], g[f"carry_k{k}_out_offsets"]
        for j in range(co.size - 1):
            c = cols[co[j]:co[j + 1]]
            got = api.carry_pass([int(x[0]) | int(x[1]) << 64 for x in c], k)
            assert np.array_equal(got, outs[oo[j]:oo[j + 1]]), (k, j)
