"""The 52-bit radix routes (§8(f) item 2): the oracle restatement and the host
repacking helpers pinned to the reference's own outputs (golden), plus the device
products (dot_mul_words(kUnsaturated), dot_mul_5x5, dot_mul_4x4) on the GPU."""
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_vectors.npz")


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def test_oracle_mul52_matches_reference(oracle, golden):
    for m in (1, 2, 3, 5, 8, 20):
        a, b, want = golden[f"mul52_m{m}_a"], golden[f"mul52_m{m}_b"], golden[f"mul52_m{m}_out"]
        for i in range(a.shape[0]):
            assert np.array_equal(oracle.mul_columns52(a[i], b[i]), want[i]), m
    a, b, want = golden["mul5x5_a"], golden["mul5x5_b"], golden["mul5x5_out"]
    for i in range(a.shape[0]):
        assert np.array_equal(oracle.mul_columns52(a[i], b[i]), want[i])


def test_repacking_matches_reference(golden):
    import paper_2604_21566_b200 as dg

    for m in (1, 3, 4, 7, 13):
        x = golden[f"pack_m{m}_in"]
        p = dg.api.pack_64_to_52(x)
        assert np.array_equal(p, golden[f"pack_m{m}_out"]), m
        assert np.array_equal(dg.api.unpack_52_to_64(p), golden[f"pack_m{m}_back"]), m
    with pytest.raises(dg.InvalidArgument):
        dg.api.unpack_52_to_64(np.array([1 << 52], np.uint64))


@pytest.mark.gpu
def test_device_52bit_products(cuda, golden):
    import paper_2604_21566_b200 as dg

    for m in (1, 2, 3, 5, 8, 20):
        a, b, want = golden[f"mul52_m{m}_a"], golden[f"mul52_m{m}_b"], golden[f"mul52_m{m}_out"]
        for i in range(a.shape[0]):
            assert np.array_equal(dg.dot_mul_words(a[i], b[i], 52), want[i]), m
    a, b, want = golden["mul5x5_a"], golden["mul5x5_b"], golden["mul5x5_out"]
    for i in range(a.shape[0]):
        assert np.array_equal(dg.api.dot_mul_5x5(a[i], b[i]), want[i])
    a, b, want = golden["mul4x4_a"], golden["mul4x4_b"], golden["mul4x4_out"]
    for i in range(a.shape[0]):
        assert np.array_equal(dg.api.dot_mul_4x4(a[i], b[i]), want[i])
    # test_mul.cpp:269-317: shape / radix violations
    with pytest.raises(dg.InvalidArgument):
        dg.api.dot_mul_5x5(np.ones(4, np.uint64), np.ones(5, np.uint64))
    bad = np.ones(5, np.uint64)
    bad[2] = np.uint64(1 << 52)
    with pytest.raises(dg.InvalidArgument):
        dg.api.dot_mul_5x5(bad, np.ones(5, np.uint64))
    with pytest.raises(dg.InvalidArgument):
        dg.dot_mul_words(np.array([2**64 - 1], np.uint64), np.array([1], np.uint64), 52)
    with pytest.raises(dg.InvalidArgument):
        dg.api.dot_mul_4x4(np.ones(3, np.uint64), np.ones(4, np.uint64))
    # (2^256 - 1)^2 via 4x4 (test_mul.cpp:288-294)
    ones = np.full(4, 2**64 - 1, np.uint64)
    v = sum(int(x) << (64 * k) for k, x in enumerate(dg.api.dot_mul_4x4(ones, ones)))
    assert v == ((1 << 256) - 1) ** 2
