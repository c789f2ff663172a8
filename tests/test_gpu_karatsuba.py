"""Batched Karatsuba on the B200 vs the oracle - the reference's own Karatsuba tests
(test_mul.cpp:417-474) restated: degeneration at theta, thresholds {1,2,4,8} x sizes up
to 128 limbs, unequal lengths, the default threshold on 512-bit operands, spiky operands."""
import numpy as np
import pytest

from helpers import MAX, spiky, uniform

pytestmark = pytest.mark.gpu


def test_zero_and_degeneration(cuda, oracle):
    import paper_2604_21566_b200 as dg

    rng = np.random.default_rng(27)
    a = uniform(rng, 12)
    assert dg.karatsuba_mul(a, np.zeros(0, np.uint64)).size == 0
    assert dg.karatsuba_mul(np.zeros(0, np.uint64), a).size == 0
    assert dg.karatsuba_mul(a, np.zeros(12, np.uint64)).size == 0
    want = oracle.mul(a, a)
    assert np.array_equal(dg.karatsuba_mul(a, a, dg.KaratsubaConfig(theta=12)), want)
    assert np.array_equal(dg.karatsuba_mul(a, a, dg.KaratsubaConfig(theta=64)), want)
    with pytest.raises(dg.InvalidArgument):
        dg.karatsuba_mul(a, a, dg.KaratsubaConfig(theta=0))


@pytest.mark.parametrize("theta", [1, 2, 4, 8])
def test_matches_oracle_across_thresholds(cuda, oracle, theta):
    import paper_2604_21566_b200 as dg

    rng = np.random.default_rng(28 + theta)
    for m in (1, 2, 3, 4, 5, 6, 7, 8, 9, 12, 16, 23, 31, 32, 33, 64, 100, 128):
        for _ in range(3 if m <= 16 else 2):
            a, b = uniform(rng, m), uniform(rng, m)
            assert np.array_equal(dg.karatsuba_mul(a, b, dg.KaratsubaConfig(theta)), oracle.mul(a, b)), (theta, m)


def test_unequal_lengths_and_default(cuda, oracle):
    import paper_2604_21566_b200 as dg

    rng = np.random.default_rng(29)
    for _ in range(40):
        a, b = uniform(rng, 1 + int(rng.integers(24))), uniform(rng, 1 + int(rng.integers(24)))
        assert np.array_equal(dg.karatsuba_mul(a, b), oracle.mul(a, b))
    for _ in range(40):
        a, b = uniform(rng, 8), uniform(rng, 8)
        assert np.array_equal(dg.karatsuba_mul(a, b), oracle.mul(a, b))


def test_spiky_and_all_ones(cuda, oracle):
    import paper_2604_21566_b200 as dg

    rng = np.random.default_rng(31)
    for it in range(60):
        m = 1 + int(rng.integers(40))
        a, b = spiky(rng, m), spiky(rng, m)
        theta = 1 + it % 8
        assert np.array_equal(dg.karatsuba_mul(a, b, dg.KaratsubaConfig(theta)), oracle.mul(a, b))
    ones = np.full(64, MAX, np.uint64)
    assert np.array_equal(dg.karatsuba_mul(ones, ones, dg.KaratsubaConfig(2)), oracle.mul(ones, ones))


def test_device_batch_equals_column_multiply(cuda):
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(32)
    for m, theta in ((64, 16), (64, 32), (100, 8), (256, 32)):
        a = torch.from_numpy(spiky(rng, (300, m)).view(np.int64)).cuda()
        b = torch.from_numpy(spiky(rng, (300, m)).view(np.int64)).cuda()
        assert torch.equal(dg.karatsuba_batch(a, b, theta=theta), dg.mul_batch(a, b)), (m, theta)


@pytest.mark.parametrize("m", [129, 200, 256, 300, 512, 1024])
def test_large_mul_batch_route(cuda, oracle, m):
    """dotg_mul_batch for m > 128 runs padded Karatsuba down to tensor-pipe leaves
    (m -> 128 * 2^L, split zero-pads, combine truncates); exact vs the oracle, with
    all-ones rows (largest middle terms) and equal halves (|hi - lo| = 0) included."""
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(900 + m)
    n = 9
    a, b = spiky(rng, (n, m)), uniform(rng, (n, m))
    a[0] = MAX
    b[0] = MAX
    h = m // 2
    a[1, h:2 * h] = a[1, :h]  # hi == lo
    b[2, :] = 0
    b[3, m - 1] = 0
    got = dg.mul_batch(torch.from_numpy(a.view(np.int64)).cuda(), torch.from_numpy(b.view(np.int64)).cuda())
    assert np.array_equal(got.cpu().numpy().view(np.uint64), oracle.mul_batch(a, b)), m


@pytest.mark.parametrize("m", [17, 20, 31, 33, 40, 63, 65, 96, 127])
def test_padded_mul_batch_route(cuda, oracle, m):
    """16 < m < 128 without a dedicated kernel: rows zero-padded to 32 / 64 / 128 limbs,
    one tensor-pipe multiply, low 2m limbs kept."""
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(950 + m)
    for cat in (uniform, spiky):
        a, b = cat(rng, (37, m)), cat(rng, (37, m))
        a[0] = MAX
        b[0] = MAX
        got = dg.mul_batch(torch.from_numpy(a.view(np.int64)).cuda(), torch.from_numpy(b.view(np.int64)).cuda())
        assert np.array_equal(got.cpu().numpy().view(np.uint64), oracle.mul_batch(a, b)), m


_COMBINE_CHILD = r'''
import sys
sys.path.insert(0, ROOT + "/tests")
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2604_21566_b200 as dg
from helpers import MAX, Oracle, spiky, uniform
orc = Oracle()
bad = []
for m, n in ((256, 7), (512, 5), (1024, 3), (2000, 2)):
    rng = np.random.default_rng(4400 + m)
    a, b = spiky(rng, (n, m)), uniform(rng, (n, m))
    a[0] = MAX
    b[0] = MAX
    a[1, m // 2:2 * (m // 2)] = a[1, :m // 2]
    got = dg.mul_batch(torch.from_numpy(a.view(np.int64)).cuda(), torch.from_numpy(b.view(np.int64)).cuda())
    if not np.array_equal(got.cpu().numpy().view(np.uint64), orc.mul_batch(a, b)):
        bad.append(m)
print("BAD", bad)
'''


@pytest.mark.parametrize("cta_pairs", ["0", "1000000"])
def test_combine_kernels_forced(cuda, cta_pairs):
    """Both Karatsuba split / combine kernel pairs - a warp per pair (DOTG_KARA_CTA_PAIRS=0) and a CTA per
    pair with segmented chains (every level below 10^6 pairs) - exact on all-ones rows
    (longest carry runs), equal halves and random rows, m up to 2000."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _COMBINE_CHILD.replace("ROOT", repr(root))],
                       env={**os.environ, "DOTG_KARA_CTA_PAIRS": cta_pairs}, capture_output=True, text=True,
                       cwd=root, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().splitlines()[-1] == "BAD []", r.stdout[-500:]
