"""Config 5 across GPUs: one long number sharded by limb range, one 8-byte exchange.

Each rank r holds limbs [r*n/G, (r+1)*n/G) of a, b and out:

1. ``dotg_shard_local``  - one streaming pass over the shard with an unknown carry-in;
   every output limb that does not depend on it is written, plus the shard aggregate
   {G, P} (G = carry-out for carry-in 0, P = every limb propagates).
2. exchange: ``all_gather_into_tensor`` of the 8-byte aggregate (NCCL over NVLink on
   GPUs; gloo in the CPU tests). This is the path's only collective.
3. ``dotg_shard_finish`` - carry-in of the shard = exclusive (G, P) scan over lower
   ranks, then the boundary fix-up (the shard's leading propagate run + one limb).

The reference has no distribution at all (its long numbers are a serial chunk chain,
src/addsub.cpp:147-164); the same (G, P) operator that chains its chunks chains shards.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

from ._lib import InvalidArgument, check, lib


def compose(aggs: Sequence[Tuple[int, int]]) -> Tuple[List[int], int]:
    """Carry into each shard and the total carry-out from ordered shard aggregates
    (G_r, P_r): c_0 = 0, c_{r+1} = G_r | (P_r & c_r)."""
    carries = []
    c = 0
    for g, p in aggs:
        carries.append(c)
        c = int(g) | (int(p) & c)
    return carries, c


def shard_bounds(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Limb range [lo, hi) of rank's shard (contiguous, balanced)."""
    if world < 1 or not 0 <= rank < world:
        raise InvalidArgument("bad rank/world")
    return n * rank // world, n * (rank + 1) // world


class ShardedWords:
    """Runs add/sub of one long number whose limbs are sharded across the ranks of a
    ``torch.distributed`` group. ``local_fn`` / ``finish_fn`` default to the device C ABI;
    tests may inject CPU stand-ins to exercise the exchange over gloo."""

    def __init__(self, group=None, local_fn: Optional[Callable] = None, finish_fn: Optional[Callable] = None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.local_fn = local_fn or self._device_local
        self.finish_fn = finish_fn or self._device_finish

    # -- device implementations ---------------------------------------------------
    @staticmethod
    def _device_local(sub, out, a, b, state, agg, stream):
        from .api import _dptr, _stream_handle

        check(lib().dotg_shard_local(int(sub), _dptr(out), _dptr(a), _dptr(b), a.numel(), _dptr(state),
                                     _dptr(agg), _stream_handle(stream)))

    @staticmethod
    def _device_finish(sub, out, state, all_aggs, rank, world, carry, stream):
        from .api import _dptr, _stream_handle

        check(lib().dotg_shard_finish(int(sub), _dptr(out), out.numel(), _dptr(state), _dptr(all_aggs), rank,
                                      world, _dptr(carry), _stream_handle(stream)))

    def state_for(self, m: int, device):
        import torch

        return torch.empty(int(lib().dotg_shard_state_bytes(m)), dtype=torch.uint8, device=device)

    def run(self, sub: bool, out, a, b, *, state=None, stream=None):
        """Returns (out, carry) where carry is an int32[1] tensor holding the carry of the
        WHOLE number (identical on every rank)."""
        import torch

        if a.shape != b.shape or out.shape != a.shape:
            raise InvalidArgument("dot add/sub: operand lengths differ (caller pads)")
        dev = a.device
        if state is None:
            state = self.state_for(a.numel(), dev) if dev.type == "cuda" else None
        agg = torch.zeros(2, dtype=torch.int32, device=dev)
        self.local_fn(sub, out, a, b, state, agg, stream)
        all_aggs = torch.empty(2 * self.world, dtype=torch.int32, device=dev)
        if dev.type == "cuda" and self.dist.get_backend(self.group) != "nccl":
            # gloo (CPU collectives): stage the 8 bytes through host memory
            host = torch.empty(2 * self.world, dtype=torch.int32)
            self.dist.all_gather_into_tensor(host, agg.cpu(), group=self.group)
            all_aggs.copy_(host)
        else:
            self.dist.all_gather_into_tensor(all_aggs, agg, group=self.group)
        carry = torch.zeros(1, dtype=torch.int32, device=dev)
        self.finish_fn(sub, out, state, all_aggs, self.rank, self.world, carry, stream)
        return out, carry
