"""paper_2604_21566_b200 - B200-native (sm_100a) limb arithmetic: the DigitsOnTurbo hot
path (multi-limb add/sub with lookahead carries, column multiplication with deferred
normalisation) behind the reference's operator interface.

The compute path is libdotg.so (paper_2604_21566_b200/csrc, C ABI in include/dotg.h);
this package is the host-side mirror of the reference interface plus the device-tensor
batch API. No CPU fallback exists.
"""
from ._lib import (  # noqa: F401
    INTERLEAVED,
    ROW_MAJOR,
    DotgCudaError,
    DotgError,
    InvalidArgument,
    kernel_launches,
    lib,
    set_mul_route,
)
from .api import (  # noqa: F401
    K_MAX_MUL_LIMBS,
    AddSubStats,
    ChunkResult,
    KaratsubaConfig,
    Width,
    WordsResult,
    add_batch,
    add_w_limbs,
    add_words,
    addsub_batch,
    addsub_batch_host,
    addsub_grouped,
    chunk_batch,
    compare_batch,
    dot_add_words,
    dot_mul_words,
    dot_sub_words,
    karatsuba_batch,
    karatsuba_mul,
    lane_count,
    mul_batch,
    mul_batch_host,
    sub_batch,
    sub_w_limbs,
    sub_words,
    words,
)
from . import api, sharded, workloads  # noqa: F401,E402

__all__ = [
    "AddSubStats",
    "ChunkResult",
    "KaratsubaConfig",
    "INTERLEAVED",
    "ROW_MAJOR",
    "DotgCudaError",
    "DotgError",
    "InvalidArgument",
    "K_MAX_MUL_LIMBS",
    "Width",
    "WordsResult",
    "add_batch",
    "add_w_limbs",
    "add_words",
    "addsub_batch",
    "addsub_batch_host",
    "addsub_grouped",
    "chunk_batch",
    "compare_batch",
    "dot_add_words",
    "dot_mul_words",
    "dot_sub_words",
    "karatsuba_batch",
    "karatsuba_mul",
    "kernel_launches",
    "lane_count",
    "lib",
    "mul_batch",
    "mul_batch_host",
    "set_mul_route",
    "sub_batch",
    "sub_w_limbs",
    "sub_words",
    "words",
]
