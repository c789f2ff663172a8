"""Phase ticks (AddSubStats::collect_ticks, addsub.hpp:57-63) on the device: the team
kernel with %clock64 laps compiled in computes the same sums and flags as the plain
kernel, fills the reference's six buckets (overflow stays 0: no separate cascade phase)
and the carry-to-add ratio of addsub.cpp:258-263; the drop-in's collect_ticks uses it."""
import numpy as np
import pytest

from helpers import spiky

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m", [1, 4, 16, 64, 256])
def test_timed_kernel_results_and_buckets(cuda, oracle, m):
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(300 + m)
    B = 3000
    a, b = spiky(rng, (B, m)), spiky(rng, (B, m))
    a[::7] = np.uint64(0xFFFFFFFFFFFFFFFF)  # full propagate chains
    b[::7] = 0
    b[::7, 0] = 1
    ta = torch.from_numpy(a.view(np.int64)).cuda()
    tb = torch.from_numpy(b.view(np.int64)).cuda()
    for sub in (False, True):
        res = dg.addsub_phase_ticks(sub, ta, tb)
        out = torch.empty_like(ta)
        fl = torch.empty(B, dtype=torch.int32, device="cuda")
        res = dg.addsub_phase_ticks(sub, ta, tb, out, fl)
        want, wf = oracle.addsub_batch(sub, a, b)
        assert np.array_equal(out.cpu().numpy().view(np.uint64), want)
        assert np.array_equal(fl.cpu().numpy().view(np.uint32), wf)
        for k in ("load_ticks", "add_ticks", "carry_gen_ticks", "carry_add_ticks", "store_ticks"):
            assert res[k] > 0, k
        assert res["overflow_ticks"] == 0
        assert abs(sum(res["pct"].values()) - 100.0) < 1e-6
        assert res["carry_to_add_ratio"] > 0


def test_dropin_collect_ticks(cuda, oracle):
    import paper_2604_21566_b200 as dg

    rng = np.random.default_rng(31)
    a, b = spiky(rng, 64), spiky(rng, 64)
    st, plain = dg.AddSubStats(), dg.AddSubStats()
    st.collect_ticks = True
    r = dg.dot_add_words(a, b, stats=st)
    q = dg.dot_add_words(a, b, stats=plain)
    want, wf = oracle.add(a, b)
    assert np.array_equal(r.limbs, want) and r.flag == wf and np.array_equal(q.limbs, want)
    assert st.chunks_processed == plain.chunks_processed == 8
    assert st.add_ticks > 0 and st.carry_to_add_ratio() > 0
    out = a.copy()  # span form, out aliases a exactly
    st2 = dg.AddSubStats()
    st2.collect_ticks = True
    assert dg.dot_add_words(out, out, b, stats=st2) == wf and np.array_equal(out, want)
    st3 = dg.AddSubStats()
    st3.collect_ticks = True
    with pytest.raises(dg.DotgError):
        dg.dot_add_words(spiky(rng, 5), spiky(rng, 5), stats=st3)


def test_unsupported_shapes_rejected(cuda):
    import paper_2604_21566_b200 as dg

    torch = cuda
    x = torch.zeros((4, 12), dtype=torch.int64, device="cuda")
    with pytest.raises(dg.DotgError):
        dg.addsub_phase_ticks(False, x, x.clone())
