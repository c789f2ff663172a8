"""Randomised routing sweep: every product / sum the device API can be asked for - both
layouts, aligned and misaligned views, every size class the dispatchers distinguish
(IMAD kernels, tensor pipe, padded and Karatsuba routes, segmented interleaved add/sub,
the generic kernels) - against the oracle, bit-exact. Seeded, so failures reproduce."""
import numpy as np
import pytest

from helpers import CATEGORIES, category

pytestmark = pytest.mark.gpu

M_CHOICES = [1, 2, 3, 4, 5, 8, 9, 15, 16, 17, 24, 31, 32, 33, 48, 63, 64, 65, 96, 100, 127, 128, 129, 160, 200,
             255, 256, 257, 300, 512, 777, 1040]


def _dev(torch, x, offset):
    """Device copy of x (row-major or interleaved), optionally 8 bytes off 32-byte alignment."""
    flat = np.ascontiguousarray(x).view(np.int64).ravel()
    buf = torch.zeros(flat.size + 1, dtype=torch.int64, device="cuda")
    buf[offset:offset + flat.size] = torch.from_numpy(flat).cuda()
    return buf[offset:offset + flat.size].view(*x.shape)


@pytest.mark.parametrize("seed", range(6))
def test_routing_fuzz(cuda, oracle, seed):
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(4242 + seed)
    for it in range(40):
        m = int(rng.choice(M_CHOICES))
        n = int(rng.integers(1, 70))
        op = ["add", "sub", "mul"][int(rng.integers(3))]
        cat = CATEGORIES[int(rng.integers(len(CATEGORIES)))]
        lay = "interleaved" if rng.integers(3) == 0 else "row"
        off = int(rng.integers(2))
        a, b = category(rng, cat, op if op != "mul" else "add", (n, m))
        ctx = (seed, it, op, m, n, cat, lay, off)
        if op == "mul":
            want = oracle.mul_batch(a, b)
            if lay == "row":
                got = dg.mul_batch(_dev(torch, a, off), _dev(torch, b, off))
                got = got.cpu().numpy().view(np.uint64)
            else:
                got = dg.mul_batch(_dev(torch, a.T.copy(), off), _dev(torch, b.T.copy(), off), layout="interleaved")
                got = got.cpu().numpy().view(np.uint64).T
            assert np.array_equal(got, want), ctx
        else:
            sub = op == "sub"
            want, wf = oracle.addsub_batch(sub, a, b)
            if lay == "row":
                out, fl = dg.addsub_batch(sub, _dev(torch, a, off), _dev(torch, b, off))
                got = out.cpu().numpy().view(np.uint64)
            else:
                out, fl = dg.addsub_batch(sub, _dev(torch, a.T.copy(), off), _dev(torch, b.T.copy(), off),
                                          layout="interleaved")
                got = out.cpu().numpy().view(np.uint64).T
            assert np.array_equal(got, want), ctx
            assert np.array_equal(fl.cpu().numpy().view(np.uint32), wf), ctx


@pytest.mark.parametrize("seed", range(3))
def test_pitched_views_fuzz(cuda, oracle, seed):
    """Row-pitched operand / result views (dotg_addsub_batch_strided, dotg_mul_batch_strided)
    with random sizes, pitches and column offsets, against the oracle."""
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(777 + seed)
    for it in range(25):
        m = int(rng.choice(M_CHOICES))
        batch = int(rng.integers(1, 300))
        cat = CATEGORIES[int(rng.integers(len(CATEGORIES)))]
        op = ["add", "sub", "mul"][it % 3]
        a, b = category(rng, cat, "mul" if op == "mul" else op, (batch, m))

        def view(x, extra):
            wide = np.zeros((x.shape[0], x.shape[1] + extra), np.uint64)
            off = int(rng.integers(0, extra + 1))
            wide[:, off:off + x.shape[1]] = x
            t = torch.from_numpy(wide.view(np.int64)).cuda()
            return t[:, off:off + x.shape[1]]

        ta, tb = view(a, int(rng.integers(0, 9))), view(b, int(rng.integers(0, 9)))
        if op == "mul":
            got = dg.mul_batch(ta, tb).cpu().numpy().view(np.uint64)
            assert np.array_equal(got, oracle.mul_batch(a, b)), (seed, it, m, batch)
        else:
            out, fl = dg.addsub_batch(op == "sub", ta, tb)
            want, wf = oracle.addsub_batch(op == "sub", a, b)
            assert np.array_equal(out.cpu().numpy().view(np.uint64), want), (seed, it, m, batch, op)
            assert np.array_equal(fl.cpu().numpy().view(np.uint32), wf)
