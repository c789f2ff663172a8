"""Seeded synthetic inputs for the five BASELINE.json configs, generated in HBM.

The reference publishes no dataset; BASELINE.json names the shapes and value
distributions, restated here. Every limb comes from the splitmix64
counter generator ``dotg_fill_splitmix64`` (device) whose host twin lives in the test
oracle, so any input can be re-derived on the host for parity checks.

C1  batched add/sub, m = 64, B = 65536, uniform limbs; sub swaps pairs so a >= b.
C2  carry-stress sweep (m, B) in (4, 2^20), (16, 2^18), (64, 2^16), (256, 2^14): each
    limb is all-ones with p = 1/2 else uniform; pairs with p % 100 == 0 are forced to
    a = 2^n - 1, b = 1 (1% full-length carry chains); sub swaps so a >= b.
C3  batched mul, m = 16, B = 2^18, uniform, top limb forced non-zero (0 -> 1).
C4  batched mul, m = 64, B = 2^16, pairs [0, B/2) uniform, [B/2, B) all-ones.
C5  one add/sub of m = 2^30 limbs, uniform except a propagate run of 2^28 limbs over
    [3*2^27, 5*2^27) (straddles the 2- and 4-way shard boundaries and covers two whole
    shards at 8-way), preceded by a generating limb; sub has a >= b by its top limb.
"""
from __future__ import annotations

import ctypes

from ._lib import check, lib

ALL_ONES = -1  # int64 bit pattern of 2^64 - 1
SIGN = -(1 << 63)

C1 = dict(name="C1", op="addsub", m=64, batch=1 << 16, seed=0xC1)
C2_SIZES = [(4, 1 << 20), (16, 1 << 18), (64, 1 << 16), (256, 1 << 14)]
C3 = dict(name="C3", op="mul", m=16, batch=1 << 18, seed=0xC3)
C4 = dict(name="C4", op="mul", m=64, batch=1 << 16, seed=0xC4)
C5_M = 1 << 30
C5_RUN = (3 << 27, 5 << 27)


def _torch():
    import torch

    return torch


def fill(n: int, seed: int, offset: int, device="cuda", stream=None):
    """int64 tensor of n splitmix64 words (counter offset+1 .. offset+n)."""
    torch = _torch()
    t = torch.empty(n, dtype=torch.int64, device=device)
    s = torch.cuda.current_stream() if stream is None else stream
    check(lib().dotg_fill_splitmix64(ctypes.c_void_p(t.data_ptr()), n, seed & (2**64 - 1),
                                     offset & (2**64 - 1), ctypes.c_void_p(s.cuda_stream)))
    return t


def rows_less(a, b):
    """Per row: a < b as unsigned little-endian limb strings ([B, m] int64)."""
    torch = _torch()
    m = a.shape[1]
    ne = a != b
    idx = (m - 1) - torch.flip(ne, [1]).to(torch.int32).argmax(dim=1).long()
    av = a.gather(1, idx[:, None]).squeeze(1)
    bv = b.gather(1, idx[:, None]).squeeze(1)
    return ne.any(dim=1) & ((av ^ SIGN) < (bv ^ SIGN))


def swap_for_sub(a, b):
    """Returns (hi, lo) with hi >= lo per row (the configs' a >= b convention)."""
    torch = _torch()
    lt = rows_less(a, b)[:, None]
    return torch.where(lt, b, a), torch.where(lt, a, b)


def c1_inputs(device="cuda"):
    m, B, s = C1["m"], C1["batch"], C1["seed"]
    a = fill(B * m, s, 0, device).view(B, m)
    b = fill(B * m, s, B * m, device).view(B, m)
    sa, sb = swap_for_sub(a, b)
    return a, b, sa, sb


def c2_inputs(m: int, B: int, device="cuda"):
    torch = _torch()
    s = 0xC2 + m
    n = B * m

    def operand(off):
        v = fill(n, s, off, device)
        sel = fill(n, s, off + n, device)
        return torch.where((sel & 1) == 1, torch.full_like(v, ALL_ONES), v).view(B, m)

    a = operand(0)
    b = operand(2 * n)
    forced = torch.arange(0, B, 100, device=device)
    a[forced] = ALL_ONES
    b[forced] = 0
    b[forced, 0] = 1
    sa, sb = swap_for_sub(a, b)
    return a, b, sa, sb


def c3_inputs(device="cuda"):
    m, B, s = C3["m"], C3["batch"], C3["seed"]
    a = fill(B * m, s, 0, device).view(B, m)
    b = fill(B * m, s, B * m, device).view(B, m)
    a[:, m - 1] += (a[:, m - 1] == 0).long()
    b[:, m - 1] += (b[:, m - 1] == 0).long()
    return a, b


def c4_inputs(device="cuda"):
    m, B, s = C4["m"], C4["batch"], C4["seed"]
    a = fill(B * m, s, 0, device).view(B, m)
    b = fill(B * m, s, B * m, device).view(B, m)
    a[B // 2:] = ALL_ONES
    b[B // 2:] = ALL_ONES
    return a, b


def c5_inputs(sub: bool, m: int = C5_M, run=C5_RUN, device="cuda", seed: int = 0xC5):
    """One long operand pair with a propagate run over [run[0], run[1]) preceded by a
    generating limb (add: a = ~0, b = 0 in the run, a = ~0, b = 1
    before it; sub: a = b = ~0 in the run, a = 0, b = 1 before it, a = ~0 / b = 0 at
    the top so a >= b)."""
    a = fill(m, seed, 0, device)
    b = fill(m, seed, m, device)
    lo, hi = run
    if hi > lo:
        if sub:
            a[lo:hi] = ALL_ONES
            b[lo:hi] = ALL_ONES
            if lo > 0:
                a[lo - 1] = 0
                b[lo - 1] = 1
        else:
            a[lo:hi] = ALL_ONES
            b[lo:hi] = 0
            if lo > 0:
                a[lo - 1] = ALL_ONES
                b[lo - 1] = 1
    if sub:
        a[m - 1] = ALL_ONES
        b[m - 1] = 0
    return a, b


def c5_shard_inputs(sub: bool, lo: int, hi: int, m: int = C5_M, run=C5_RUN, device="cuda", seed: int = 0xC5):
    """Limbs [lo, hi) of c5_inputs(sub, m, run): what rank r holds when the number is
    sharded by limb range. Identical values to slicing the single-GPU operands."""
    n = hi - lo
    a = fill(n, seed, lo, device)
    b = fill(n, seed, m + lo, device)
    rlo, rhi = run
    s0, s1 = max(rlo, lo), min(rhi, hi)
    if s1 > s0:
        a[s0 - lo:s1 - lo] = ALL_ONES
        b[s0 - lo:s1 - lo] = ALL_ONES if sub else 0
    if rhi > rlo and rlo > 0 and lo <= rlo - 1 < hi:
        i = rlo - 1 - lo
        if sub:
            a[i] = 0
            b[i] = 1
        else:
            a[i] = ALL_ONES
            b[i] = 1
    if sub and lo <= m - 1 < hi:
        a[m - 1 - lo] = ALL_ONES
        b[m - 1 - lo] = 0
    return a, b
