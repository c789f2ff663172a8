"""Reentrancy (the reference's functions are pure and reentrant on caller
buffers): host-buffer entry points and device-stream entry points called from several
host threads at once (ctypes releases the GIL during the foreign call), each thread with
its own data, every result checked against the oracle."""
import threading

import numpy as np
import pytest

from helpers import spiky, uniform

pytestmark = pytest.mark.gpu


def _run_threads(fn, n):
    errors = []

    def wrap(i):
        try:
            fn(i)
        except Exception as e:  # noqa: BLE001 - reported below
            errors.append((i, repr(e)))

    ts = [threading.Thread(target=wrap, args=(i,)) for i in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in ts), "a thread hung"
    assert not errors, errors


def test_host_entry_points_concurrently(cuda, oracle):
    import paper_2604_21566_b200 as dg

    cases = []
    for i in range(8):
        rng = np.random.default_rng(700 + i)
        m = [4, 16, 64, 100, 3, 256, 33, 8][i]
        batch = 4096 if m < 100 else 512
        a, b = spiky(rng, (batch, m)), spiky(rng, (batch, m))
        cases.append((a, b))
    want = [(oracle.addsub_batch(False, a, b), oracle.addsub_batch(True, a, b),
             oracle.mul_batch(a[:256], b[:256])) for a, b in cases]

    def work(i):
        a, b = cases[i]
        for _ in range(3):
            out, fl = dg.addsub_batch_host(False, a, b)
            assert np.array_equal(out, want[i][0][0]) and np.array_equal(fl, want[i][0][1])
            out, fl = dg.addsub_batch_host(True, a, b)
            assert np.array_equal(out, want[i][1][0]) and np.array_equal(fl, want[i][1][1])
            prod = dg.mul_batch_host(np.ascontiguousarray(a[:256]), np.ascontiguousarray(b[:256]))
            assert np.array_equal(prod, want[i][2])
            r = dg.dot_add_words(a[0], b[0])
            w0, f0 = oracle.add(a[0], b[0])
            assert np.array_equal(r.limbs, w0) and r.flag == f0
            c = dg.add_w_limbs(a[1][:1], b[1][:1], 1, 1)
            wc, cc, pc = oracle.chunk(False, a[1][:1], b[1][:1], 1, 1)
            assert np.array_equal(c.sums[:1], wc) and c.carry_out == cc and c.phase4_fired == pc

    _run_threads(work, len(cases))


def test_device_entry_points_on_private_streams(cuda, oracle):
    import paper_2604_21566_b200 as dg

    torch = cuda
    n = 6
    data = []
    for i in range(n):
        rng = np.random.default_rng(900 + i)
        m = [16, 64, 32, 7, 128, 4][i]
        a, b = uniform(rng, (2048, m)), uniform(rng, (2048, m))
        data.append((a, b, oracle.mul_batch(a, b), oracle.addsub_batch(i % 2 == 1, a, b)))

    def work(i):
        a, b, wmul, (wadd, wfl) = data[i]
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            ta = torch.from_numpy(a.view(np.int64)).cuda(non_blocking=False)
            tb = torch.from_numpy(b.view(np.int64)).cuda(non_blocking=False)
            for _ in range(5):
                prod = dg.mul_batch(ta, tb, stream=s)
                out, fl = dg.addsub_batch(i % 2 == 1, ta, tb, stream=s)
            s.synchronize()
        assert np.array_equal(prod.cpu().numpy().view(np.uint64), wmul)
        assert np.array_equal(out.cpu().numpy().view(np.uint64), wadd)
        assert np.array_equal(fl.cpu().numpy().view(np.uint32), wfl)

    _run_threads(work, n)
