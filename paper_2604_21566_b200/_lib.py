"""ctypes binding of libdotg.so (the C ABI declared in include/dotg.h).

The library is built in-tree by ``paper_2604_21566_b200/csrc/Makefile`` (or
``__graft_entry__.build()``). There is no fallback: if the shared object is missing the
import of any compute entry point raises, and every compute call on a machine without
an sm_100 device returns DOTG_ECUDA, surfaced here as :class:`DotgCudaError`.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import c_char_p, c_int, c_size_t, c_uint, c_uint32, c_uint64, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdotg.so")

DOTG_OK, DOTG_EINVAL, DOTG_ECUDA, DOTG_ENOMEM, DOTG_ENOTSUP, DOTG_ENCCL = range(6)
ROW_MAJOR, INTERLEAVED = 0, 1

# Every symbol include/dotg.h declares: name -> (restype, argtypes).
_P = c_void_p
SIGNATURES = {
    "dotg_validate_width": (c_int, [c_int]),
    "dotg_last_error": (c_char_p, []),
    "dotg_version": (c_char_p, []),
    "dotg_device_sms": (c_int, []),
    "dotg_add_batch": (c_int, [_P, _P, _P, _P, c_size_t, c_size_t, c_int, _P]),
    "dotg_sub_batch": (c_int, [_P, _P, _P, _P, c_size_t, c_size_t, c_int, _P]),
    "dotg_addsub_grouped": (c_int, [_P, c_int, _P]),
    "dotg_mul_batch": (c_int, [_P, _P, _P, c_size_t, c_size_t, c_int, _P]),
    "dotg_mul52_batch_host": (c_int, [_P, _P, _P, c_size_t, c_size_t]),
    "dotg_mul52_batch": (c_int, [_P, _P, _P, c_size_t, c_size_t, _P]),
    "dotg_karatsuba_batch": (c_int, [_P, _P, _P, c_size_t, c_size_t, c_size_t, _P]),
    "dotg_karatsuba_batch_host": (c_int, [_P, _P, _P, c_size_t, c_size_t, c_size_t]),
    "dotg_add_words": (c_int, [_P, _P, _P, c_size_t, _P, _P]),
    "dotg_sub_words": (c_int, [_P, _P, _P, c_size_t, _P, _P]),
    "dotg_shard_state_bytes": (c_size_t, [c_size_t]),
    "dotg_shard_local": (c_int, [c_int, _P, _P, _P, c_size_t, _P, _P, _P]),
    "dotg_shard_finish": (c_int, [c_int, _P, c_size_t, _P, _P, c_int, c_int, _P, _P]),
    "dotg_add_batch_host": (c_int, [_P, _P, _P, _P, c_size_t, c_size_t]),
    "dotg_sub_batch_host": (c_int, [_P, _P, _P, _P, c_size_t, c_size_t]),
    "dotg_mul_batch_host": (c_int, [_P, _P, _P, c_size_t, c_size_t]),
    "dotg_addsub_grouped_host": (c_int, [_P, c_int]),
    "dotg_add_words_host": (c_int, [_P, _P, _P, c_size_t, _P]),
    "dotg_sub_words_host": (c_int, [_P, _P, _P, c_size_t, _P]),
    "dotg_addsub_stats": (c_int, [c_int, _P, _P, _P, c_size_t, c_size_t, c_int, c_int, _P, _P]),
    "dotg_words_host_stats": (c_int, [c_int, _P, _P, _P, c_size_t, c_int, _P, _P, _P]),
    "dotg_fill_splitmix64": (c_int, [_P, c_size_t, c_uint64, c_uint64, _P]),
    "dotg_compare_batch": (c_int, [_P, _P, _P, c_size_t, c_size_t, c_int, _P]),
    "dotg_compare_host": (c_int, [_P, _P, _P, c_size_t, c_size_t]),
    "dotg_carry_census": (c_int, [c_uint, _P]),
    "dotg_mc_carry": (c_int, [c_uint64, c_uint64, _P]),
    "dotg_gather_columns": (c_int, [_P, _P, _P, _P, c_size_t, c_size_t, _P]),
    "dotg_compute_partials": (c_int, [_P, _P, _P, _P, c_size_t, c_int, _P]),
    "dotg_align_and_reduce": (c_int, [_P, _P, _P, c_size_t, c_size_t, _P]),
    "dotg_carry_pass": (c_int, [_P, _P, c_size_t, _P, c_size_t, c_size_t, c_int, _P]),
    "dotg_gather_columns_host": (c_int, [_P, _P, _P, _P, c_size_t]),
    "dotg_compute_partials_host": (c_int, [_P, _P, _P, _P, c_size_t, c_int]),
    "dotg_align_and_reduce_host": (c_int, [_P, _P, _P, c_size_t]),
    "dotg_carry_pass_host": (c_int, [_P, _P, c_size_t, _P, c_size_t, c_int]),
    "dotg_addsub_batch_strided": (c_int, [c_int, _P, c_size_t, _P, c_size_t, _P, c_size_t, _P, c_size_t, c_size_t,
                                          _P]),
    "dotg_mul_batch_strided": (c_int, [_P, c_size_t, _P, c_size_t, _P, c_size_t, c_size_t, c_size_t, _P]),
    "dotg_chunk_batch": (c_int, [c_int, _P, _P, _P, _P, _P, _P, c_uint, c_size_t, _P]),
    "dotg_chunk_host": (c_int, [c_int, _P, _P, _P, _P, _P, c_uint32, c_uint]),
    "dotg_kernel_launches": (c_uint64, []),
    "dotg_set_mul_route": (c_int, [c_int]),
    "dotg_addsub_phase_ticks": (c_int, [c_int, _P, _P, _P, _P, c_size_t, c_size_t, _P, _P]),
    "dotg_addsub_phase_ticks_host": (c_int, [c_int, _P, _P, _P, _P, c_size_t, c_size_t, _P]),
    "dotg_comm_id_bytes": (c_size_t, []),
    "dotg_comm_get_unique_id": (c_int, [_P]),
    "dotg_comm_init_rank": (c_int, [_P, c_int, _P, c_int]),
    "dotg_comm_wrap": (c_int, [_P, _P]),
    "dotg_comm_destroy": (c_int, [_P]),
    "dotg_comm_rank": (c_int, [_P]),
    "dotg_comm_size": (c_int, [_P]),
    "dotg_add_words_sharded": (c_int, [_P, _P, _P, c_size_t, _P, _P, _P]),
    "dotg_sub_words_sharded": (c_int, [_P, _P, _P, c_size_t, _P, _P, _P]),
}


class AddSubProblem(ctypes.Structure):
    """dotg_addsub_problem (include/dotg.h)."""

    _fields_ = [("op", c_int), ("layout", c_int), ("out", c_void_p), ("a", c_void_p), ("b", c_void_p),
                ("flags", c_void_p), ("m", c_size_t), ("batch", c_size_t)]


class DotgError(RuntimeError):
    """Base class for library errors."""


class InvalidArgument(DotgError, ValueError):
    """The reference's std::invalid_argument (SURVEY.md §8(b) error cases)."""


class DotgCudaError(DotgError):
    """CUDA failure or no sm_100 device (there is no CPU fallback)."""


class DotgNcclError(DotgError):
    """NCCL missing or a collective of the sharded entry points failed."""


_lib = None


def lib() -> ctypes.CDLL:
    """Load libdotg.so once; raise loudly when it has not been built."""
    global _lib
    if _lib is None:
        path = os.environ.get("DOTG_LIB_PATH", LIB_PATH)  # experiments: an alternative build
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: build it with `make -C paper_2604_21566_b200/csrc` "
                "or __graft_entry__.build(); the product path has no CPU fallback"
            )
        handle = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int) -> None:
    if rc == DOTG_OK:
        return
    msg = lib().dotg_last_error().decode(errors="replace")
    if rc == DOTG_EINVAL:
        raise InvalidArgument(msg)
    if rc == DOTG_ECUDA:
        raise DotgCudaError(msg)
    if rc == DOTG_ENOMEM:
        raise MemoryError(msg)
    if rc == DOTG_ENCCL:
        raise DotgNcclError(msg)
    raise DotgError(f"dotg status {rc}: {msg}")


def kernel_launches() -> int:
    return int(lib().dotg_kernel_launches())


MUL_AUTO, MUL_IMAD, MUL_IMMA = 0, 1, 2
_ROUTES = {"auto": MUL_AUTO, "imad": MUL_IMAD, "imma": MUL_IMMA}


def set_mul_route(route: str) -> str:
    """Select the multiply pipe ("auto", "imad", "imma"); returns the previous one."""
    if route not in _ROUTES:
        raise InvalidArgument(f"mul route must be one of {sorted(_ROUTES)}")
    prev = int(lib().dotg_set_mul_route(_ROUTES[route]))
    if prev < 0:
        check(-prev)
    return {v: k for k, v in _ROUTES.items()}[prev]
