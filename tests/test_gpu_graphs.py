"""The device-pointer C ABI is stream-ordered and capturable: batched add/sub (grouped),
multiply (tensor pipe, IMAD, tcgen05 incl. the split route, Karatsuba) and the long-number path recorded into one
CUDA graph and replayed on new inputs give the same bits as direct calls - launch-bound
loops of small problems can run as graphs instead of per-call launches."""
import numpy as np
import pytest

from helpers import spiky

pytestmark = pytest.mark.gpu


def test_capture_and_replay(cuda, oracle):
    import paper_2604_21566_b200 as dg

    torch = cuda
    rng = np.random.default_rng(404)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()  # noqa: E731
    shapes = {"add": (300, 64), "mul64": (70, 64), "mul16": (90, 16), "mul300": (5, 300), "mul1024": (3, 1024),
              "mul8192": (2, 8192)}
    src = {k: (spiky(rng, s), spiky(rng, s)) for k, s in shapes.items()}
    ins = {k: (dev(a), dev(b)) for k, (a, b) in src.items()}
    la, lb = dev(spiky(rng, 70000)), dev(spiky(rng, 70000))
    outs = {"add": torch.empty_like(ins["add"][0]), "flags": torch.empty(300, dtype=torch.int32, device="cuda"),
            "long": torch.empty_like(la), "carry": torch.empty(1, dtype=torch.int32, device="cuda")}
    muls = ("mul64", "mul16", "mul300", "mul1024", "mul8192")
    for k in muls:
        bsz, m = shapes[k]
        outs[k] = torch.empty((bsz, 2 * m), dtype=torch.int64, device="cuda")

    def step():
        dg.add_batch(*ins["add"], out=outs["add"], flags=outs["flags"])
        for k in muls:
            dg.mul_batch(*ins[k], out=outs[k])
        dg.add_words(la, lb, out=outs["long"], carry=outs["carry"])

    step()  # warm the per-device caches outside the capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            step()
    # new inputs in the captured buffers, then replay
    new = {k: (spiky(rng, sh), spiky(rng, sh)) for k, sh in shapes.items()}
    for k, (a, b) in new.items():
        ins[k][0].copy_(dev(a))
        ins[k][1].copy_(dev(b))
    na, nb = spiky(rng, 70000), spiky(rng, 70000)
    la.copy_(dev(na))
    lb.copy_(dev(nb))
    g.replay()
    torch.cuda.synchronize()
    host = lambda t: t.cpu().numpy().view(np.uint64)  # noqa: E731
    want, wf = oracle.addsub_batch(False, *new["add"])
    assert np.array_equal(host(outs["add"]), want)
    assert np.array_equal(outs["flags"].cpu().numpy().view(np.uint32), wf)
    for k in muls:
        assert np.array_equal(host(outs[k]), oracle.mul_batch(*new[k])), k
    wl, wc = oracle.add(na, nb)
    assert np.array_equal(host(outs["long"]), wl) and int(outs["carry"].item()) == wc
