"""One long number (config 5 path): tiled 3-pass add/sub and the shard protocol, on the
B200 vs the oracle. Virtual shards run as independent launches on one GPU (no kernel
waits on another; the 8-byte exchange is a device-side concatenation)."""
import numpy as np
import pytest

from helpers import MAX, spiky, uniform

pytestmark = pytest.mark.gpu
TILE = 4096


def dev(torch, x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint64)


def words(torch, sub, a, b):
    import paper_2604_21566_b200 as dg

    out, c = dg.sub_words(dev(torch, a), dev(torch, b)) if sub else dg.add_words(dev(torch, a), dev(torch, b))
    return host(out), int(c.item())


SIZES = [1, 2, 3, 31, 4095, 4096, 4097, 8191, 8192, 3 * TILE + 17, 100_000]


@pytest.mark.parametrize("m", SIZES)
def test_words_random_and_spiky(cuda, oracle, m):
    rng = np.random.default_rng(m)
    for gen in (uniform, spiky):
        a, b = gen(rng, m), gen(rng, m)
        for sub in (False, True):
            want, wf = oracle.sub(a, b) if sub else oracle.add(a, b)
            got, gf = words(cuda, sub, a, b)
            assert np.array_equal(got, want) and gf == wf, (m, gen.__name__, sub)


@pytest.mark.parametrize("m", [4096, 4097, 5 * TILE + 3, 64 * TILE])
def test_words_propagate_runs(cuda, oracle, m):
    """Runs spanning whole tiles, starting/ending mid-tile, starting at limb 0 (deferred
    prefix of tile 0), and a full-length chain."""
    rng = np.random.default_rng(m + 1)
    runs = [(0, m), (0, m // 2), (1, m), (TILE - 1, min(m, 3 * TILE + 5)), (m // 3, m - 1), (TILE, 2 * TILE)]
    for lo, hi in runs:
        hi = min(hi, m)
        for sub in (False, True):
            a, b = uniform(rng, m), uniform(rng, m)
            if sub:
                a[lo:hi] = b[lo:hi]
                if lo > 0:
                    a[lo - 1], b[lo - 1] = 0, 1
            else:
                a[lo:hi] = MAX
                b[lo:hi] = 0
                if lo > 0:
                    a[lo - 1], b[lo - 1] = MAX, 1
            want, wf = oracle.sub(a, b) if sub else oracle.add(a, b)
            got, gf = words(cuda, sub, a, b)
            assert np.array_equal(got, want) and gf == wf, (m, lo, hi, sub)
    # full chain: (2^n - 1) + 1 and 0 - 1
    got, gf = words(cuda, False, np.full(m, MAX, np.uint64), np.eye(1, m, dtype=np.uint64)[0])
    assert not got.any() and gf == 1
    got, gf = words(cuda, True, np.zeros(m, np.uint64), np.eye(1, m, dtype=np.uint64)[0])
    assert (got == MAX).all() and gf == 1


def test_words_misaligned_and_aliased(cuda, oracle):
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(5)
    m = 3 * TILE + 11
    a, b = spiky(rng, m), spiky(rng, m)
    want, wf = oracle.add(a, b)
    ba = torch.zeros(m + 1, dtype=torch.int64, device="cuda")
    bb = torch.zeros(m + 1, dtype=torch.int64, device="cuda")
    ba[1:] = dev(torch, a)
    bb[1:] = dev(torch, b)
    out, c = dg.add_words(ba[1:], bb[1:], out=ba[1:])  # misaligned (8 B) and aliased
    assert np.array_equal(host(ba[1:]), want) and int(c.item()) == wf


def run_virtual_shards(torch, sub, a, b, world):
    """The shard protocol of include/dotg.h on one GPU: G independent local passes, the
    8-byte aggregates concatenated in HBM, G finish passes."""
    import ctypes

    import paper_2604_21566_b200 as dg
    from paper_2604_21566_b200.sharded import compose, shard_bounds

    L = dg.lib()
    m = a.numel()
    out = torch.empty_like(a)
    states, aggs = [], torch.zeros(2 * world, dtype=torch.int32, device="cuda")
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = dg.api._dptr
    for r in range(world):
        lo, hi = shard_bounds(m, r, world)
        st = torch.empty(int(L.dotg_shard_state_bytes(hi - lo)), dtype=torch.uint8, device="cuda")
        states.append(st)
        dg.api.check(L.dotg_shard_local(int(sub), P(out[lo:hi]), P(a[lo:hi]), P(b[lo:hi]), hi - lo, P(st),
                                        P(aggs[2 * r:2 * r + 2]), s))
    carries = torch.zeros(world, dtype=torch.int32, device="cuda")
    for r in range(world):
        lo, hi = shard_bounds(m, r, world)
        dg.api.check(L.dotg_shard_finish(int(sub), P(out[lo:hi]), hi - lo, P(states[r]), P(aggs), r, world,
                                         P(carries[r:r + 1]), s))
    agg = aggs.cpu().numpy().reshape(world, 2)
    _, total = compose([tuple(x) for x in agg])
    c = carries.cpu().numpy()
    assert (c == total).all()  # every rank reports the whole number's carry
    return out, total


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_virtual_shards_match_oracle(cuda, oracle, world):
    from paper_2604_21566_b200 import workloads as W

    torch = cuda
    m = 1 << 20
    run = (3 * m // 8, 5 * m // 8)  # the C5 run, scaled: straddles the 2/4-way boundaries
    for sub in (False, True):
        a, b = W.c5_inputs(sub, m=m, run=run)
        out, total = run_virtual_shards(torch, sub, a, b, world)
        want, wf = oracle.sub(host(a), host(b)) if sub else oracle.add(host(a), host(b))
        assert np.array_equal(host(out), want) and total == wf, (world, sub)


@pytest.mark.slow
def test_config5_full_size(cuda, oracle):
    """C5 at BASELINE.json's size: 2^30 limbs (8 GiB per operand), single GPU and 8
    virtual shards, add and sub, vs the oracle on the host."""
    import paper_2604_21566_b200 as dg
    from paper_2604_21566_b200 import workloads as W

    torch = cuda
    for sub in (False, True):
        a, b = W.c5_inputs(sub)
        ha, hb = host(a), host(b)
        want, wf = oracle.sub(ha, hb) if sub else oracle.add(ha, hb)
        out, c = dg.sub_words(a, b) if sub else dg.add_words(a, b)
        assert int(c.item()) == wf
        assert np.array_equal(host(out), want)
        del out
        out, total = run_virtual_shards(torch, sub, a, b, 8)
        assert total == wf and np.array_equal(host(out), want)
        del out, a, b
        torch.cuda.empty_cache()


@pytest.mark.parametrize("m,batch", [(8192, 3), (8193, 5), (12345, 2), (40000, 4), (65536, 1)])
def test_long_batch_route(cuda, oracle, m, batch):
    """Batches of long numbers (m >= 8192) take the tiled long-number passes with one grid
    row per number: carries across tile boundaries inside each number, none across numbers,
    each number's carry its flag; sub included, with propagate runs over tile edges."""
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(77 + m + batch)
    a = rng.integers(0, 2**64, size=(batch, m), dtype=np.uint64)
    b = rng.integers(0, 2**64, size=(batch, m), dtype=np.uint64)
    MAXV = np.uint64(0xFFFFFFFFFFFFFFFF)
    a[0, 100:m - 3] = MAXV  # long propagate run across every tile of number 0
    b[0, 100:m - 3] = 0
    b[0, 99] = MAXV
    a[0, 99] = 1
    if batch > 1:
        a[1, :] = MAXV  # full chain with carry out
        b[1, :] = 0
        b[1, 0] = 1
    for sub in (False, True):
        want, wf = oracle.addsub_batch(sub, a, b)
        out, fl = dg.addsub_batch(sub, torch.from_numpy(a.view(np.int64)).cuda(), torch.from_numpy(b.view(np.int64)).cuda())
        assert np.array_equal(out.cpu().numpy().view(np.uint64), want), (m, batch, sub)
        assert np.array_equal(fl.cpu().numpy().view(np.uint32), wf), (m, batch, sub)
