"""Chunk-level operations add_w_limbs / sub_w_limbs (addsub.hpp:78-89, addsub.cpp:172-190)
on the B200: the reference's frozen chunk cases (test_addsub.cpp:50-90), and random spiky
chunks of every w against the oracle's chunk_generic restatement and the reference's own
run_chunk (sums, carry_out, phase4_fired all equal), batched and one at a time."""
import numpy as np
import pytest

from helpers import MAX, spiky

pytestmark = pytest.mark.gpu


def test_frozen_chunks(cuda):
    import paper_2604_21566_b200 as dg

    r = dg.add_w_limbs([MAX] * 8, [0] * 8, 1, 8)
    assert (r.sums == 0).all() and r.carry_out == 1 and r.phase4_fired
    r = dg.sub_w_limbs([0] * 8, [0] * 8, 1, 8)
    assert (r.sums == MAX).all() and r.carry_out == 1 and r.phase4_fired
    r = dg.add_w_limbs([MAX, MAX] + [0] * 6, [1] + [0] * 7, 0, 8)
    assert list(r.sums) == [0, 0, 1, 0, 0, 0, 0, 0] and r.carry_out == 0 and r.phase4_fired
    one = [1] * 8
    for args in ((one, one, 0, 0), (one, one, 0, 9), (one, one, 2, 8), (one, [1] * 7, 0, 8)):
        with pytest.raises(dg.InvalidArgument):
            dg.add_w_limbs(*args)
    with pytest.raises(dg.InvalidArgument):
        dg.sub_w_limbs(one, one, 0, 9)


@pytest.mark.parametrize("w", range(1, 9))
def test_chunk_batch_vs_oracle_and_reference(cuda, oracle, ref, w):
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(w)
    batch = 3000
    a, b = spiky(rng, (batch, w)), spiky(rng, (batch, w))
    cin = rng.integers(0, 2, size=batch).astype(np.int32)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()  # noqa: E731
    for sub in (False, True):
        sums, co, fi = dg.chunk_batch(sub, dev(a), dev(b), torch.from_numpy(cin).cuda())
        sums = sums.cpu().numpy().view(np.uint64)
        co, fi = co.cpu().numpy(), fi.cpu().numpy()
        for p in range(0, batch, 7 if w > 2 else 1):
            want, wc, wp = oracle.chunk(sub, a[p], b[p], int(cin[p]), w)
            assert np.array_equal(sums[p], want[:w]) and co[p] == wc and bool(fi[p]) == bool(wp), (sub, p)
        for p in range(0, batch, 97):
            rs, rc, rp = ref.chunk(sub, a[p], b[p], int(cin[p]), w)
            assert np.array_equal(sums[p], rs[:w]) and co[p] == rc and bool(fi[p]) == bool(rp), (sub, p)
            one = (dg.sub_w_limbs if sub else dg.add_w_limbs)(a[p], b[p], int(cin[p]), w)
            assert np.array_equal(one.sums[:w], rs[:w]) and one.carry_out == rc and one.phase4_fired == bool(rp)
    # a batch fires Phase 4 on some chunks and not on others (spiky data)
    assert 0 < int(fi.sum()) < batch


def test_chunk_batch_invalid_carry_and_alias(cuda):
    import paper_2604_21566_b200 as dg

    torch = cuda
    a = torch.full((4, 8), -1, dtype=torch.int64, device="cuda")
    b = torch.zeros((4, 8), dtype=torch.int64, device="cuda")
    cin = torch.tensor([0, 1, 2, 1], dtype=torch.int32, device="cuda")
    sums, co, fi = dg.chunk_batch(False, a, b, cin)
    assert co.tolist() == [0, 1, -1, 1]  # 0xFFFFFFFF flags carry_in > 1
    assert fi.tolist() == [0, 1, 0, 1]
    assert (sums[1] == 0).all() and (sums[0] == -1).all()
    with pytest.raises(dg.InvalidArgument):
        dg.chunk_batch(False, torch.zeros((4, 9), dtype=torch.int64, device="cuda"),
                       torch.zeros((4, 9), dtype=torch.int64, device="cuda"))


def test_chunk_batch_in_place(cuda, oracle):
    """sums may alias a (or b) exactly, like the word-level forms (addsub.hpp:95-97)."""
    import paper_2604_21566_b200 as dg
    from paper_2604_21566_b200 import api

    torch = cuda
    rng = np.random.default_rng(88)
    a, b = spiky(rng, (500, 8)), spiky(rng, (500, 8))
    ta = torch.from_numpy(a.view(np.int64).copy()).cuda()
    tb = torch.from_numpy(b.view(np.int64)).cuda()
    co = torch.empty(500, dtype=torch.int32, device="cuda")
    api.check(dg.lib().dotg_chunk_batch(0, api._dptr(ta), api._dptr(co), None, api._dptr(ta), api._dptr(tb), None, 8,
                                        500, api._stream_handle(None)))
    got = ta.cpu().numpy().view(np.uint64)
    for p in range(0, 500, 13):
        want, wc, _ = oracle.chunk(False, a[p], b[p], 0, 8)
        assert np.array_equal(got[p], want) and int(co[p]) == wc
