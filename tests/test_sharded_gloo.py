"""N > 1 host logic on CPU: the config-5 shard protocol of paper_2604_21566_b200.sharded
over a world-size-2 (and 3) gloo group. The per-shard device passes are replaced by CPU
stand-ins that follow the same contract as dotg_shard_local / dotg_shard_finish
(include/dotg.h); the exchange, rank plumbing and carry composition are the product's."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import MAX, Oracle, uniform


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def local_standin(sub, out, a, b, state, agg, stream):
    """Contract of dotg_shard_local: outputs for carry-in 0 + aggregate {G, P}."""
    orc = Oracle()
    ha, hb = a.numpy().view(np.uint64), b.numpy().view(np.uint64)
    o, g = orc.sub(ha, hb) if sub else orc.add(ha, hb)
    out.copy_(torch.from_numpy(o.view(np.int64)))
    s = (ha - hb) if sub else (ha + hb)
    p = int(bool((s == (0 if sub else MAX)).all()))
    agg[0], agg[1] = g, p


def finish_standin(sub, out, state, all_aggs, rank, world, carry, stream):
    """Contract of dotg_shard_finish: X = exclusive (G, P) scan over lower ranks, then
    the fix-up (carry X rippled into the shard), carry = whole-number carry."""
    from paper_2604_21566_b200.sharded import compose

    aggs = all_aggs.view(world, 2).tolist()
    carries, total = compose([tuple(x) for x in aggs])
    x = carries[rank]
    o = out.numpy().view(np.uint64)
    i = 0
    while x and i < o.size:
        if sub:
            o[i] -= np.uint64(1)
            x = int(o[i] == MAX)
        else:
            o[i] += np.uint64(1)
            x = int(o[i] == 0)
        i += 1
    carry[0] = total


def worker(rank, world, port, m, sub, seed, run, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_21566_b200.sharded import ShardedWords, shard_bounds

        rng = np.random.default_rng(seed)
        a, b = uniform(rng, m), uniform(rng, m)
        lo, hi = run
        if sub:
            a[lo:hi] = b[lo:hi]
            a[lo - 1], b[lo - 1] = 0, 1
            a[-1], b[-1] = MAX, 0
        else:
            a[lo:hi] = MAX
            b[lo:hi] = 0
            a[lo - 1], b[lo - 1] = MAX, 1
        s0, s1 = shard_bounds(m, rank, world)
        ta = torch.from_numpy(a[s0:s1].view(np.int64).copy())
        tb = torch.from_numpy(b[s0:s1].view(np.int64).copy())
        out = torch.empty_like(ta)
        sw = ShardedWords(local_fn=local_standin, finish_fn=finish_standin)
        assert (sw.rank, sw.world) == (rank, world)
        out, carry = sw.run(sub, out, ta, tb)
        q.put((rank, out.numpy().view(np.uint64).copy(), int(carry[0])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,sub", [(2, False), (2, True), (3, False), (3, True)])
def test_shard_protocol_gloo(world, sub):
    m = 40_000
    run = (3 * m // 8, 5 * m // 8)  # straddles the 2-way boundary, whole shard at 3-way
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, m, sub, 77, run, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.concatenate([r[1] for r in res])
    rng = np.random.default_rng(77)
    a, b = uniform(rng, m), uniform(rng, m)
    lo, hi = run
    if sub:
        a[lo:hi] = b[lo:hi]
        a[lo - 1], b[lo - 1] = 0, 1
        a[-1], b[-1] = MAX, 0
    else:
        a[lo:hi] = MAX
        b[lo:hi] = 0
        a[lo - 1], b[lo - 1] = MAX, 1
    orc = Oracle()
    want, wf = orc.sub(a, b) if sub else orc.add(a, b)
    assert np.array_equal(got, want)
    assert all(r[2] == wf for r in res)


def test_compose_and_bounds():
    from paper_2604_21566_b200.sharded import compose, shard_bounds

    assert compose([(1, 0), (0, 1), (0, 1), (0, 0)]) == ([0, 1, 1, 1], 0)
    assert compose([(0, 1), (0, 1)]) == ([0, 0], 0)
    assert compose([(1, 0), (0, 1)]) == ([0, 1], 1)
    n = (1 << 30) + 3
    for w in (1, 2, 3, 4, 8):
        bounds = [shard_bounds(n, r, w) for r in range(w)]
        assert bounds[0][0] == 0 and bounds[-1][1] == n
        assert all(bounds[i][1] == bounds[i + 1][0] for i in range(w - 1))
