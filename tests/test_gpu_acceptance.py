"""The reference's acceptance criteria 1, 2, 3 and 5 (tests/acceptance.cpp:66-198) at its
own volumes, on the B200, with the oracle as the checker:

1. add/sub vs oracle: 12 sizes (default_bit_sizes, testgen.cpp:61-66: 512..32768 bits) x
   (10k random + 6 x 1k pathological) per op;
2. mul vs oracle: 4x4 100k, 5x5 (52-bit) 100k, words m = 1..16 10k each, Karatsuba
   theta = 4 at the 12 sizes 10k each;
3. Phase 4: 0 triggers on random additions, rate 1.0 on full propagation (per width);
5. width invariance on the mixed category at 576..3072 bits (1000 cases each).
The device result is one kernel family for every Width (bit-identical by construction);
the per-width part is the AddSubStats counters, derived on the device. Inputs are seeded
numpy draws of the reference's category shapes (helpers.category), not its mt19937_64
streams."""
import numpy as np
import pytest

from helpers import CATEGORIES, category, uniform

pytestmark = pytest.mark.gpu

SIZES = [512 * k for k in (1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64)]
PATHOLOGICAL = CATEGORIES[1:6] + ["mixed"]  # testgen.hpp:36-39
WIDTHS = (0, 2, 4, 8)


def dev(torch, x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()


def host(t):
    return t.cpu().numpy().view(np.uint64)


def test_criteria_1_and_3_addsub(cuda, oracle):
    import paper_2604_21566_b200 as dg

    torch = cuda
    checks = mismatches = 0
    rand_add = [0, 0]
    full = {w: [0, 0] for w in WIDTHS}
    shard = 0
    for op in ("add", "sub"):
        for bits in SIZES:
            m = bits // 64
            corpora = [("random", 10_000)] + [(c, 1_000) for c in PATHOLOGICAL]
            for cat, n in corpora:
                rng = np.random.default_rng(100 + shard)
                shard += 1
                a, b = category(rng, cat, op, (n, m))
                ta, tb = dev(torch, a), dev(torch, b)
                out, fl = dg.addsub_batch(op == "sub", ta, tb)
                want, wf = oracle.addsub_batch(op == "sub", a, b)
                bad = ~((host(out) == want).all(axis=1) & (fl.cpu().numpy().view(np.uint32) == wf))
                checks += n
                mismatches += int(bad.sum())
                if (cat == "random" and op == "add") or cat == "full_propagation":
                    for w in WIDTHS:
                        ch, fi = dg.addsub_stats(op == "sub", out, ta, tb, width=w)
                        if cat == "random":
                            rand_add[0] += ch
                            rand_add[1] += fi
                        else:
                            full[w][0] += ch
                            full[w][1] += fi
    assert checks == 2 * 12 * 16_000 and mismatches == 0
    # criterion 3 (acceptance.cpp:102-109)
    assert rand_add[0] > 0 and rand_add[1] == 0
    for w in WIDTHS:
        assert full[w][0] > 0 and full[w][1] == full[w][0], (w, full[w])


def test_criterion_2_mul(cuda, oracle):
    import paper_2604_21566_b200 as dg
    from paper_2604_21566_b200 import api

    torch = cuda
    rng = np.random.default_rng(2024)
    # 4x4: 100k
    a, b = uniform(rng, (100_000, 4)), uniform(rng, (100_000, 4))
    got = host(dg.mul_batch(dev(torch, a), dev(torch, b)))
    assert np.array_equal(got, oracle.mul_batch(a, b))
    # 5x5 over 52-bit limbs: 100k, checked through unpack_52_to_64 like acceptance.cpp:128-133
    mask = np.uint64((1 << 52) - 1)
    a, b = uniform(rng, (100_000, 5)) & mask, uniform(rng, (100_000, 5)) & mask
    out = np.zeros((100_000, 10), np.uint64)
    api.check(dg.lib().dotg_mul52_batch_host(api._hp(out), api._hp(a), api._hp(b), 5, 100_000))
    for p in range(0, 100_000, 997):
        want = oracle.mul(api.unpack_52_to_64(a[p]), api.unpack_52_to_64(b[p]))
        got = api._trim(api.unpack_52_to_64(out[p]))
        assert np.array_equal(got, api._trim(want)), p
    # words m = 1..16, 10k each
    for m in range(1, 17):
        a, b = uniform(rng, (10_000, m)), uniform(rng, (10_000, m))
        got = host(dg.mul_batch(dev(torch, a), dev(torch, b)))
        assert np.array_equal(got, oracle.mul_batch(a, b)), m
    # Karatsuba theta = 4 at the 12 sizes, 10k each
    for bits in SIZES:
        m = bits // 64
        a, b = uniform(rng, (10_000, m)), uniform(rng, (10_000, m))
        got = host(dg.karatsuba_batch(dev(torch, a), dev(torch, b), theta=4))
        assert np.array_equal(got, oracle.mul_batch(a, b)), bits


def test_criterion_5_width_invariance(cuda, oracle):
    import paper_2604_21566_b200 as dg

    torch = cuda
    cases = 0
    shard = 0
    for op in ("add", "sub"):
        for bits in (576, 832, 1024, 2048, 3072):
            rng = np.random.default_rng(900 + shard)
            shard += 1
            a, b = category(rng, "mixed", op, (1_000, bits // 64))
            want, wf = oracle.addsub_batch(op == "sub", a, b)
            out, flags = dg.addsub_batch_host(op == "sub", a, b)
            assert np.array_equal(out, want) and np.array_equal(flags, wf)
            fn = dg.dot_sub_words if op == "sub" else dg.dot_add_words
            for p in range(0, 1_000, 50):  # the reference-form call at every Width
                for w in WIDTHS:
                    r = fn(a[p], b[p], w)
                    assert np.array_equal(r.limbs, want[p]) and r.flag == wf[p], (op, bits, p, w)
            # per-width AddSubStats on the device agree with the oracle's chunk counters
            ta, tb, to = dev(torch, a), dev(torch, b), dev(torch, out)
            for w in WIDTHS:
                ch, fi = dg.addsub_stats(op == "sub", to, ta, tb, width=w)
                wch = wfi = 0
                for p in range(1_000):
                    _, _, c1, f1 = oracle.words(op == "sub", a[p], b[p], 8 if w == 0 else w)
                    wch += c1
                    wfi += f1
                assert (ch, fi) == (wch, wfi), (op, bits, w)
            cases += 1_000
    assert cases == 10_000
