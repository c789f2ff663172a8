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
        WHOLE number (identical on every rank). Everything - the scratch zero-fills, both
        device passes and the collective - is ordered on ``stream`` (default: the current
        stream): the sequence runs with ``stream`` as torch's current stream, so the
        allocations, the NCCL all-gather and the gloo host copy all wait on the passes."""
        import contextlib

        import torch

        if a.shape != b.shape or out.shape != a.shape:
            raise InvalidArgument("dot add/sub: operand lengths differ (caller pads)")
        dev = a.device
        ctx = torch.cuda.stream(stream) if (stream is not None and dev.type == "cuda") else contextlib.nullcontext()
        with ctx:
            if state is None:
                state = self.state_for(a.numel(), dev) if dev.type == "cuda" else None
            agg = torch.zeros(2, dtype=torch.int32, device=dev)
            self.local_fn(sub, out, a, b, state, agg, stream)
            all_aggs = torch.empty(2 * self.world, dtype=torch.int32, device=dev)
            if dev.type == "cuda" and self.dist.get_backend(self.group) != "nccl":
                # gloo (CPU collectives): stage the 8 bytes through host memory (agg.cpu()
                # synchronises with the current stream = the passes' stream)
                host = torch.empty(2 * self.world, dtype=torch.int32)
                self.dist.all_gather_into_tensor(host, agg.cpu(), group=self.group)
                all_aggs.copy_(host)
            else:
                self.dist.all_gather_into_tensor(all_aggs, agg, group=self.group)
            carry = torch.zeros(1, dtype=torch.int32, device=dev)
            self.finish_fn(sub, out, state, all_aggs, self.rank, self.world, carry, stream)
        return out, carry


class CommShardedWords:
    """The same protocol in ONE C-ABI call per rank (``dotg_add_words_sharded`` /
    ``dotg_sub_words_sharded``): the local pass, the 8-byte ``ncclAllGather`` and the
    boundary fix-up are enqueued by the library's C++ host code on one stream, over an
    NCCL communicator the library owns (``dotg_comm``). ``torch.distributed`` only
    carries the 128-byte NCCL unique id from rank 0 to the others at construction (any
    backend). Construction is collective: every rank of ``group`` must create one."""

    def __init__(self, group=None, *, wrap_torch_comm: bool = False):
        """wrap_torch_comm: reuse the NCCL communicator of the group's ProcessGroupNCCL
        (dotg_comm_wrap; no second communicator) instead of creating one from a unique id."""
        import ctypes

        import torch
        import torch.distributed as dist

        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        L = lib()
        if wrap_torch_comm:
            pg = group if group is not None else dist.distributed_c10d._get_default_group()
            backend = pg._get_backend(torch.device("cuda", torch.cuda.current_device()))
            probe = torch.zeros(1, device="cuda")
            dist.all_reduce(probe, group=group)  # the communicator is created lazily
            torch.cuda.synchronize()
            self._comm = ctypes.c_void_p()
            check(L.dotg_comm_wrap(ctypes.byref(self._comm), ctypes.c_void_p(int(backend._comm_ptr()))))
            assert L.dotg_comm_rank(self._comm) == self.rank and L.dotg_comm_size(self._comm) == self.world
            return
        nid = int(L.dotg_comm_id_bytes())
        payload = [None]
        if self.rank == 0:
            buf = ctypes.create_string_buffer(nid)
            check(L.dotg_comm_get_unique_id(buf))
            payload = [bytes(buf.raw)]
        dist.broadcast_object_list(payload, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                   group=group)
        uid = ctypes.create_string_buffer(payload[0], nid)
        self._comm = ctypes.c_void_p()
        check(L.dotg_comm_init_rank(ctypes.byref(self._comm), self.world, uid, self.rank))
        assert L.dotg_comm_rank(self._comm) == self.rank and L.dotg_comm_size(self._comm) == self.world

    def run(self, sub: bool, out, a, b, *, carry=None, stream=None):
        """out = a +/- b over this rank's limbs; returns (out, carry) with carry an int32[1]
        device tensor receiving the carry/borrow of the WHOLE number (every rank)."""
        import torch

        from .api import _dptr, _stream_handle

        if a.shape != b.shape or out.shape != a.shape:
            raise InvalidArgument("dot add/sub: operand lengths differ (caller pads)")
        if carry is None:
            carry = torch.empty(1, dtype=torch.int32, device=a.device)
        fn = lib().dotg_sub_words_sharded if sub else lib().dotg_add_words_sharded
        check(fn(_dptr(out), _dptr(a), _dptr(b), a.numel(), _dptr(carry), self._comm, _stream_handle(stream)))
        return out, carry

    def close(self) -> None:
        if getattr(self, "_comm", None) is not None and self._comm.value:
            check(lib().dotg_comm_destroy(self._comm))
            self._comm = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter teardown
            pass
