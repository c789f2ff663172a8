"""The reference-shaped host API (span / value forms, dot_mul_words) on the B200:
frozen examples and behaviours of test_addsub.cpp / test_mul.cpp, through the *_host
C-ABI entry points (host buffers in, host buffers out)."""
import numpy as np
import pytest

from helpers import MAX, spiky, uniform

pytestmark = pytest.mark.gpu


def test_value_and_span_forms(cuda, oracle):
    import paper_2604_21566_b200 as dg

    r = dg.dot_add_words(np.full(8, MAX, np.uint64), np.array([1], np.uint64))  # (2^512-1)+1
    assert not r.limbs.any() and r.limbs.size == 8 and r.flag == 1
    rng = np.random.default_rng(7)
    a = uniform(rng, 12)
    r = dg.dot_add_words(a, np.zeros(0, np.uint64))  # adding zero is the identity
    assert np.array_equal(r.limbs, a) and r.flag == 0
    r = dg.dot_sub_words(np.array([0], np.uint64), np.array([1], np.uint64))
    assert list(r.limbs) == [MAX] and r.flag == 1
    for w in dg.Width:
        x, y = spiky(rng, 33), spiky(rng, 33)
        out = np.zeros(33, np.uint64)
        c = dg.dot_add_words(out, x, y, w)
        want, wf = oracle.add(x, y)
        assert np.array_equal(out, want) and c == wf


def test_unequal_lengths_pad(cuda, oracle):
    import paper_2604_21566_b200 as dg

    rng = np.random.default_rng(0xC0FFEE)
    for _ in range(50):
        ma, mb = 1 + int(rng.integers(20)), 1 + int(rng.integers(20))
        a, b = spiky(rng, ma), spiky(rng, mb)
        m = max(ma, mb)
        pa, pb = np.zeros(m, np.uint64), np.zeros(m, np.uint64)
        pa[:ma], pb[:mb] = a, b
        want, wf = oracle.add(pa, pb)
        r = dg.dot_add_words(a, b)
        assert np.array_equal(r.limbs, want) and r.flag == wf


def test_span_errors_and_aliasing(cuda, oracle):
    import paper_2604_21566_b200 as dg

    out = np.zeros(5, np.uint64)
    with pytest.raises(dg.InvalidArgument):
        dg.dot_add_words(out, np.ones(4, np.uint64), np.ones(5, np.uint64))
    with pytest.raises(dg.InvalidArgument):
        dg.dot_sub_words(out, np.ones(4, np.uint64), np.ones(5, np.uint64))
    with pytest.raises(dg.InvalidArgument):
        dg.dot_add_words(np.ones(4, np.uint64), np.ones(4, np.uint64), width=16)
    rng = np.random.default_rng(0x0DD5EED)
    for _ in range(30):
        m = 1 + int(rng.integers(24))
        a, b = spiky(rng, m), spiky(rng, m)
        want, wf = oracle.add(a, b)
        acc = a.copy()
        assert dg.dot_add_words(acc, acc, b) == wf and np.array_equal(acc, want)
        acc2 = b.copy()
        assert dg.dot_add_words(acc2, a, acc2) == wf and np.array_equal(acc2, want)


def test_round_trip_and_mul(cuda, oracle):
    import paper_2604_21566_b200 as dg

    rng = np.random.default_rng(0xABAD1DEA)
    for _ in range(40):  # add then sub round-trips (test_addsub.cpp:182-199)
        m = 1 + int(rng.integers(40))
        a, b = spiky(rng, m), spiky(rng, m)
        s = dg.dot_add_words(a, b)
        wide = np.append(s.limbs, np.uint64(s.flag))
        back = dg.dot_sub_words(wide, np.append(b, np.uint64(0)))
        assert back.flag == 0 and np.array_equal(back.limbs[:m], a) and back.limbs[m] == 0
    for m in (1, 2, 7, 16, 64, 300, 1024, 5000):  # up to the tcgen05 routes (direct and split)
        a, b = uniform(rng, m), uniform(rng, m)
        p = dg.dot_mul_words(a, b)
        want = oracle.mul(a, b)
        assert p.size == 2 * m and np.array_equal(p[: want.size], want) and not p[want.size:].any()


def test_long_host_span(cuda, oracle):
    import paper_2604_21566_b200 as dg

    rng = np.random.default_rng(11)
    m = 5_000_000  # several host-pipeline slices
    a, b = uniform(rng, m), uniform(rng, m)
    a[1000:4_000_000] = MAX
    b[1000:4_000_000] = 0
    a[999], b[999] = MAX, 1
    out = np.zeros(m, np.uint64)
    c = dg.dot_add_words(out, a, b)
    want, wf = oracle.add(a, b)
    assert c == wf and np.array_equal(out, want)


def test_batch_host_pipeline(cuda, oracle):
    import paper_2604_21566_b200 as dg

    rng = np.random.default_rng(12)
    a, b = spiky(rng, (70000, 64)), spiky(rng, (70000, 64))
    out, fl = dg.addsub_batch_host(True, a, b)
    want, wf = oracle.addsub_batch(True, a, b)
    assert np.array_equal(out, want) and np.array_equal(fl, wf)
    a, b = uniform(rng, (30000, 16)), uniform(rng, (30000, 16))
    assert np.array_equal(dg.mul_batch_host(a, b), oracle.mul_batch(a, b))
    for m, n in ((1024, 40), (8192, 3)):  # tcgen05 direct / split routes through the host pipeline
        a, b = spiky(rng, (n, m)), spiky(rng, (n, m))
        a[0] = MAX
        b[0] = MAX
        assert np.array_equal(dg.mul_batch_host(a, b), oracle.mul_batch(a, b)), m


def test_grouped_host_pipeline(cuda, oracle):
    import ctypes

    import paper_2604_21566_b200 as dg
    from paper_2604_21566_b200._lib import AddSubProblem

    rng = np.random.default_rng(13)
    specs = [(0, 4, 300_000), (1, 16, 70_000), (0, 64, 20_000), (1, 256, 5_000), (0, 3, 1000), (1, 0, 10)]
    arr = (AddSubProblem * len(specs))()
    keep = []
    for i, (op, m, B) in enumerate(specs):
        a, b = spiky(rng, (B, m)), spiky(rng, (B, m))
        out, fl = np.zeros((B, m), np.uint64), np.full(B, 9, np.uint32)
        keep.append((op, a, b, out, fl))
        arr[i] = AddSubProblem(op, 0, out.ctypes.data if out.size else None, a.ctypes.data if a.size else None,
                               b.ctypes.data if b.size else None, fl.ctypes.data, m, B)
    dg.api.check(dg.lib().dotg_addsub_grouped_host(arr, len(specs)))
    for op, a, b, out, fl in keep:
        want, wf = oracle.addsub_batch(op, a, b)
        assert np.array_equal(out, want) and np.array_equal(fl, wf)


def test_addsub_stats_parity(cuda, oracle):
    """AddSubStats chunks/phase-4 counters vs the reference's own counts (golden vectors,
    w8) and the oracle's 4-phase restatement for every width."""
    import os

    import paper_2604_21566_b200 as dg

    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_vectors.npz"))
    for m in (9, 64, 256):
        a, b = g[f"addsub_m{m}_a"], g[f"addsub_m{m}_b"]
        for sub, key in ((False, "add"), (True, "sub")):
            for i in range(a.shape[0]):
                st = dg.AddSubStats()
                out = np.zeros(m, np.uint64)
                fn = dg.dot_sub_words if sub else dg.dot_add_words
                c = fn(out, a[i], b[i], dg.Width.w8, st)
                assert c == g[f"addsub_m{m}_{key}_flag"][i]
                assert st.chunks_processed == (m + 7) // 8
                assert st.phase4_triggers == g[f"addsub_m{m}_{key}_p4"][i]
    rng = np.random.default_rng(4)
    for w in (0, 2, 4, 8):
        for m in (1, 7, 33):
            a, b = spiky(rng, m), spiky(rng, m)
            for sub in (False, True):
                st = dg.AddSubStats()
                r = (dg.dot_sub_words if sub else dg.dot_add_words)(a, b, w, st)
                o, c, ch, fi = oracle.words(sub, a, b, dg.lane_count(w))
                assert np.array_equal(r.limbs, o) and r.flag == c
                assert (st.chunks_processed, st.phase4_triggers) == (ch, fi)
    # 0 triggers on uniform data, every chunk on a full chain (test_addsub.cpp:282-317)
    st = dg.AddSubStats()
    dg.dot_add_words(np.full(64, MAX, np.uint64), np.eye(1, 64, dtype=np.uint64)[0], dg.Width.w8, st)
    assert st.chunks_processed == 8 and st.phase4_rate() == 1.0


def test_batch_stats_device(cuda, oracle):
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(5)
    a, b = spiky(rng, (500, 24)), spiky(rng, (500, 24))
    ta = torch.from_numpy(a.view(np.int64)).cuda()
    tb = torch.from_numpy(b.view(np.int64)).cuda()
    out, _ = dg.add_batch(ta, tb)
    cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
    dg.api.check(dg.lib().dotg_addsub_stats(0, dg.api._dptr(out), dg.api._dptr(ta), dg.api._dptr(tb), 24, 500, 0, 4,
                                            dg.api._dptr(cnt), dg.api._stream_handle(None)))
    want_ch = want_fi = 0
    for i in range(500):
        _, _, ch, fi = oracle.words(False, a[i], b[i], 4)
        want_ch += ch
        want_fi += fi
    assert cnt.tolist() == [want_ch, want_fi]
