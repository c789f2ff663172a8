"""Batched compare (limbs.hpp:84, limbs.cpp:46-53) on the B200 vs the oracle's compare:
equal rows, rows differing only in the lowest / highest limb, all-ones rows, both
layouts, team widths of every row kernel."""
import numpy as np
import pytest

from helpers import MAX

pytestmark = pytest.mark.gpu


def cases(rng, m, batch):
    a = rng.integers(0, 2**64, size=(batch, m), dtype=np.uint64)
    b = a.copy()
    kind = np.arange(batch) % 6
    r = np.arange(batch)
    # 0: equal; 1: differ in limb 0; 2: differ in the top limb; 3: differ at a random limb;
    # 4: independent random; 5: all-ones vs all-ones minus a low bit
    b[kind == 1, 0] ^= np.uint64(1)
    b[kind == 2, m - 1] ^= np.uint64(1 << 63)
    pos = rng.integers(0, m, size=batch)
    sel = kind == 3
    b[r[sel], pos[sel]] += np.uint64(1)
    b[kind == 4] = rng.integers(0, 2**64, size=(int((kind == 4).sum()), m), dtype=np.uint64)
    a[kind == 5] = MAX
    b[kind == 5] = MAX
    b[kind == 5, 0] = MAX - np.uint64(1)
    swap = rng.random(batch) < 0.5
    a[swap], b[swap] = b[swap].copy(), a[swap].copy()
    return a, b


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("m", [1, 2, 3, 5, 8, 16, 33, 64, 100, 300])
def test_compare_batch(cuda, oracle, m, layout):
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(1000 * m + layout)
    batch = 777
    a, b = cases(rng, m, batch)
    want = np.array([oracle.compare(a[p], b[p]) for p in range(batch)], dtype=np.int32)

    def put(x):
        x = x.T if layout == 1 else x
        return torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()

    got = dg.compare_batch(put(a), put(b), layout=layout).cpu().numpy()
    assert np.array_equal(got, want), (m, layout, np.nonzero(got != want)[0][:5])


def test_compare_empty_and_errors(cuda):
    import paper_2604_21566_b200 as dg

    torch = cuda
    z = torch.zeros((0, 4), dtype=torch.int64, device="cuda")
    assert dg.compare_batch(z, z).numel() == 0
    a = torch.zeros((3, 4), dtype=torch.int64, device="cuda")
    with pytest.raises(dg.InvalidArgument):
        dg.compare_batch(a, torch.zeros((3, 5), dtype=torch.int64, device="cuda"))


def test_compare_value_form(cuda, oracle):
    """compare(a, b) with unequal lengths: high zero limbs are ignored (limbs.cpp:46-53)."""
    from paper_2604_21566_b200 import api

    rng = np.random.default_rng(5)
    for _ in range(60):
        ma, mb = int(rng.integers(0, 9)), int(rng.integers(0, 9))
        a = rng.integers(0, 2**64, size=ma, dtype=np.uint64)
        b = rng.integers(0, 2**64, size=mb, dtype=np.uint64)
        if ma and rng.random() < 0.3:
            a[-1] = 0
        if ma and mb and rng.random() < 0.3:
            b = np.concatenate([a, np.zeros(int(rng.integers(0, 3)), np.uint64)])
        assert api.compare(a, b) == oracle.compare(a, b), (a, b)
    assert api.compare([], []) == 0 and api.compare([0, 0], [0]) == 0
    assert api.compare([1], [0, 0, 0]) == 1 and api.compare([MAX], [0, 1]) == -1


def test_compare_zero_limbs(cuda):
    """m = 0 with pairs: every pair compares equal."""
    import paper_2604_21566_b200 as dg

    torch = cuda
    z = torch.zeros((5, 0), dtype=torch.int64, device="cuda")
    assert dg.compare_batch(z, z).tolist() == [0] * 5
