"""Wide products on the 5th-generation tensor core (mul_umma.cu: tcgen05.mma kind::i8,
column sums in tensor memory) vs the oracle - the reference's own product contract
(mul.cpp:96-103, exactly 2m limbs), restated at the sizes that route there: 256 <= m <= 4096
directly (m % 16 == 0, rows padded otherwise; s-range splits above 4096) and the
Karatsuba leaves above 65536 limbs.
All-ones rows give the largest column sums (n * 255^2 < 2^31 at m = 4096) and carries."""
import numpy as np
import pytest

from helpers import MAX, spiky, uniform

pytestmark = pytest.mark.gpu


def _rows(rng, n, m):
    a, b = spiky(rng, (n, m)), uniform(rng, (n, m))
    a[0] = MAX
    b[0] = MAX
    b[1] = 0
    a[2, : m // 2] = 0  # low half zero: products start mid-tile
    b[3, m // 3:] = 0  # short b: most s-windows empty
    a[4, -1] = MAX
    a[4, :-1] = 0  # a = 2^(64(m-1)) * (2^64 - 1)
    return a, b


@pytest.mark.parametrize("m", [256, 272, 512, 768, 1024, 2048, 4096])
def test_umma_direct_route(cuda, oracle, m):
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(1300 + m)
    n = 7 if m <= 1024 else 5
    a, b = _rows(rng, n, m)
    got = dg.mul_batch(torch.from_numpy(a.view(np.int64)).cuda(), torch.from_numpy(b.view(np.int64)).cuda())
    assert np.array_equal(got.cpu().numpy().view(np.uint64), oracle.mul_batch(a, b)), m


def test_umma_many_pairs_both_tiles(cuda, oracle):
    """m = 4096 has two D tiles per pair; a few hundred pairs fill every SM more than once."""
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(1399)
    for m, n in ((256, 700), (4096, 40)):
        a, b = spiky(rng, (n, m)), spiky(rng, (n, m))
        a[::7] = MAX
        b[::5] = MAX
        got = dg.mul_batch(torch.from_numpy(a.view(np.int64)).cuda(), torch.from_numpy(b.view(np.int64)).cuda())
        g = got.cpu().numpy().view(np.uint64)
        idx = list(range(0, n, max(1, n // 12))) + [n - 1]
        assert np.array_equal(g[idx], oracle.mul_batch(a[idx], b[idx])), m


@pytest.mark.parametrize("m", [4112, 6000, 8192, 16384, 32768, 65536])
def test_umma_split_route(cuda, oracle, m):
    """4096 < m <= 16384: the b-window steps split into ranges of <= 128 (s32 column sums
    stay exact), partial limbs added by k_umma_reduce, carries by one batched add."""
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(1450 + m)
    a, b = _rows(rng, 5, m)
    if m > 16384:  # keep the oracle's O(m^2) CPU time to seconds: the all-ones and a random row
        a, b = a[[0, 4]], b[[0, 4]]
    got = dg.mul_batch(torch.from_numpy(a.view(np.int64)).cuda(), torch.from_numpy(b.view(np.int64)).cuda())
    assert np.array_equal(got.cpu().numpy().view(np.uint64), oracle.mul_batch(a, b)), m


@pytest.mark.parametrize("m", [70000])
def test_umma_karatsuba_leaves(cuda, oracle, m):
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(1500 + m)
    a, b = _rows(rng, 5, m)
    a, b = a[[0, 2]], b[[0, 2]]
    got = dg.mul_batch(torch.from_numpy(a.view(np.int64)).cuda(), torch.from_numpy(b.view(np.int64)).cuda())
    assert np.array_equal(got.cpu().numpy().view(np.uint64), oracle.mul_batch(a, b)), m


def test_umma_misaligned_rows(cuda, oracle):
    """8-byte aligned (not 16) operand rows take the padded copy route, same result."""
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(1600)
    m, n = 512, 6
    a, b = _rows(rng, n, m)
    da = torch.zeros(n * m + 1, dtype=torch.int64, device="cuda")
    db = torch.zeros(n * m + 1, dtype=torch.int64, device="cuda")
    da[1:] = torch.from_numpy(a.reshape(-1).view(np.int64)).cuda()
    db[1:] = torch.from_numpy(b.reshape(-1).view(np.int64)).cuda()
    got = dg.mul_batch(da[1:].view(n, m), db[1:].view(n, m))
    assert np.array_equal(got.cpu().numpy().view(np.uint64), oracle.mul_batch(a, b))


def test_umma_route_taken(cuda):
    """The tcgen05 route is the one that runs: one launch for a direct product, two with
    the tile-carry pass (m = 4096), a few for split items (reduce + the batched add's
    passes) - the Karatsuba route it replaced issues tens of launches per call."""
    import paper_2604_21566_b200 as dg

    torch = cuda
    for m, want in ((256, 1), (1024, 1), (4096, 2), (8192, 6)):
        a = torch.ones((2, m), dtype=torch.int64, device="cuda")
        out = torch.empty((2, 2 * m), dtype=torch.int64, device="cuda")
        dg.mul_batch(a, a, out=out)  # warm (pool, attributes)
        torch.cuda.synchronize()
        n0 = dg.kernel_launches()
        dg.mul_batch(a, a, out=out)
        torch.cuda.synchronize()
        n = dg.kernel_launches() - n0
        assert (n == want) if m <= 4096 else (2 <= n <= want), (m, n)
        # (1 + 2^64 + ... ) squared pattern: the all-ones-limb value 1 per limb
        got = out.cpu().numpy().view(np.uint64)
        exp = np.array([min(i + 1, 2 * m - 1 - i) for i in range(2 * m)], np.uint64)
        exp[-1] = 0
        assert np.array_equal(got[0], exp), m
