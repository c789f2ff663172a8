"""Products at the reference's maximum size (kMaxMulLimbs = 2^24 limbs, mul.hpp:26-30;
dot_mul_words accepts up to it, mul.cpp:13-18) and the depth-first Karatsuba schedule
that keeps them inside device memory (karatsuba.cu run_karatsuba_at).

Exact checks where a closed form exists ((2^(64m) - 1)^2 = 2^(128m) - 2^(64m+1) + 1), the
low limbs against the oracle (the low k limbs of a*b depend only on the low k limbs of
a and b), and residues modulo three 61/62-bit primes of the whole product. The forced
depth-first schedule (DOTG_KARA_BUDGET_MB) is also checked exactly at oracle sizes."""
import os

import numpy as np
import pytest

from helpers import MAX, uniform

pytestmark = pytest.mark.gpu
PRIMES = [(1 << 61) - 1, (1 << 62) - 57, (1 << 62) - 87]


def big(x):
    return int.from_bytes(np.ascontiguousarray(x).view(np.uint8).tobytes(), "little")


def dev(torch, x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.fixture
def small_budget():
    old = os.environ.get("DOTG_KARA_BUDGET_MB")
    os.environ["DOTG_KARA_BUDGET_MB"] = "1"
    yield
    if old is None:
        del os.environ["DOTG_KARA_BUDGET_MB"]
    else:
        os.environ["DOTG_KARA_BUDGET_MB"] = old


def test_depth_first_schedule_exact(cuda, oracle, small_budget):
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(31)
    for m, batch in ((200, 3), (1024, 2), (1000, 2), (4096, 1)):
        a, b = uniform(rng, (batch, m)), uniform(rng, (batch, m))
        a[0] = MAX
        b[0] = MAX
        got = host(dg.mul_batch(dev(torch, a), dev(torch, b)))
        assert np.array_equal(got, oracle.mul_batch(a, b)), m
    for m in (300, 513):
        a, b = uniform(rng, (2, m)), uniform(rng, (2, m))
        got = host(dg.karatsuba_batch(dev(torch, a), dev(torch, b), theta=4))
        assert np.array_equal(got, oracle.mul_batch(a, b)), m


def test_wide_split_combine_exact(cuda, oracle):
    """The top levels of large products (halves of >= 4096 limbs, few pairs) run the wide
    split / combine (batched long add/sub + copies): exact against the oracle."""
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(77)
    for m, batch in ((8192, 2), (10000, 1), (16384, 1), (9001, 3)):
        a, b = uniform(rng, (batch, m)), uniform(rng, (batch, m))
        a[0, : m // 2] = MAX  # equal halves / long propagate runs in the splits
        b[-1] = MAX
        got = host(dg.mul_batch(dev(torch, a), dev(torch, b)))
        assert np.array_equal(got, oracle.mul_batch(a, b)), m
    for m in (9000, 8193):
        a, b = uniform(rng, (2, m)), uniform(rng, (2, m))
        a[1, m // 2:] = a[1, : m - m // 2]  # hi == lo: zero difference, sign 0
        got = host(dg.karatsuba_batch(dev(torch, a), dev(torch, b), theta=4))
        assert np.array_equal(got, oracle.mul_batch(a, b)), m


@pytest.mark.parametrize("m", [1 << 24, (1 << 22) + 3])
def test_maximum_size_products(cuda, oracle, m):
    import paper_2604_21566_b200 as dg

    torch = cuda
    # all-ones: the closed form, every limb exact
    ones = torch.full((1, m), -1, dtype=torch.int64, device="cuda")
    got = host(dg.mul_batch(ones, ones))[0]
    assert got[0] == 1 and not got[1:m].any()
    assert got[m] == MAX - np.uint64(1) and (got[m + 1:] == MAX).all()
    del ones
    # random: low limbs against the oracle, residues of the whole product
    rng = np.random.default_rng(m)
    a, b = uniform(rng, (1, m)), uniform(rng, (1, m))
    got = host(dg.mul_batch(dev(torch, a), dev(torch, b)))[0]
    k = 48
    assert np.array_equal(got[:k], oracle.mul(a[0, :k], b[0, :k])[:k])
    A, B, P = big(a[0]), big(b[0]), big(got)
    for p in PRIMES:
        assert P % p == (A % p) * (B % p) % p, p
    assert P.bit_length() <= 128 * m
