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


_MUL52_CHILD = r'''
import ctypes, sys
sys.path.insert(0, ROOT + "/tests")
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2604_21566_b200 as dg
from helpers import Oracle
orc = Oracle()
L = dg.lib()
M52 = (1 << 52) - 1
bad = []
for m in (1, 2, 3, 4, 5, 6, 8, 11, 16, 17):
    for batch in (1, 127, 128, 300):
        rng = np.random.default_rng(5200 + 31 * m + batch)
        a = rng.integers(0, 1 << 52, size=(batch, m), dtype=np.uint64)
        b = rng.integers(0, 1 << 52, size=(batch, m), dtype=np.uint64)
        a[0] = M52                     # every product and every column at its maximum
        b[0] = M52
        if batch > 2:
            a[1] = 0
            b[2, : m // 2] = M52
        da = torch.from_numpy(a.view(np.int64)).cuda()
        db = torch.from_numpy(b.view(np.int64)).cuda()
        do = torch.empty((batch, 2 * m), dtype=torch.int64, device="cuda")
        rc = L.dotg_mul52_batch(do.data_ptr(), da.data_ptr(), db.data_ptr(), m, batch, None)
        assert rc == 0, rc
        got = do.cpu().numpy().view(np.uint64)
        for i in range(batch):
            if not np.array_equal(got[i], orc.mul_columns52(a[i], b[i])):
                bad.append((m, batch, i))
                break
print("BAD", bad)
'''


@pytest.mark.gpu
@pytest.mark.parametrize("fp", ["1", "0"])
def test_device_52bit_batch_both_pipes(cuda, fp):
    """dotg_mul52_batch on the FP64 pipe (exact fma.rz / fma.rn products, the default) and
    on the IMAD pipe (DOTG_MUL52_FP=0) against the oracle's radix-2^52 column product: all
    limbs 2^52 - 1 (largest columns), zeros, half-maximal rows, partial and full CTAs,
    m = 1 ... 17 (17: the generic kernel)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _MUL52_CHILD.replace("ROOT", repr(root))],
                       env={**os.environ, "DOTG_MUL52_FP": fp}, capture_output=True, text=True, cwd=root,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().splitlines()[-1] == "BAD []", r.stdout[-500:]
