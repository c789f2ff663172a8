"""Host-side mirror of the reference's operator interface, over the C ABI.

Two surfaces:

* Reference-shaped calls on host arrays (numpy uint64, little-endian limbs), with the
  reference's names, argument meaning and error behaviour (include/dot/addsub.hpp:95-109,
  include/dot/mul.hpp:75-76): ``dot_add_words``, ``dot_sub_words`` (span form
  ``f(out, a, b, width)`` -> carry; value form ``f(a, b, width)`` -> WordsResult) and
  ``dot_mul_words(a, b)`` -> 2m limbs. std::invalid_argument becomes
  :class:`InvalidArgument` (a ValueError). These go through the ``*_host`` entry points
  (host buffers in, host buffers out, copies overlapped with the kernels).

* Device-resident batch calls on torch CUDA tensors (the measured path):
  ``add_batch`` / ``sub_batch`` / ``mul_batch`` and the long-number ``add_words`` /
  ``sub_words``. Tensors are int64 or uint64 (limb bit patterns), contiguous.
"""
from __future__ import annotations

import ctypes
import enum
import operator
from typing import NamedTuple, Optional

import numpy as np

from . import _lib
from ._lib import INTERLEAVED, ROW_MAJOR, InvalidArgument, check, lib

K_MAX_MUL_LIMBS = 1 << 24  # kMaxMulLimbs, include/dot/mul.hpp:30


class Width(enum.IntEnum):
    """Reference Width selector (include/dot/addsub.hpp:30-36). The device path has one
    kernel family; every width returns bit-identical results (as in the reference)."""

    scalar = 0
    w2 = 2
    w4 = 4
    w8 = 8


def lane_count(w: int) -> int:
    """addsub.hpp:38-40."""
    return 8 if int(w) == 0 else int(w)


class AddSubStats:
    """The reference's AddSubStats (include/dot/addsub.hpp:53-72): chunks_processed and
    phase4_triggers (derived on the device, csrc/stats.cu) and, with collect_ticks, the
    six phase-tick buckets - SM clock cycles from the %clock64 laps of the timed team
    kernel (dotg_addsub_phase_ticks; power-of-two m <= 256), summed over warps.
    Accumulated across calls like the reference."""

    TICKS = ("load_ticks", "add_ticks", "carry_gen_ticks", "carry_add_ticks", "store_ticks", "overflow_ticks")

    def __init__(self):
        self.chunks_processed = 0
        self.phase4_triggers = 0
        self.collect_ticks = False
        for k in self.TICKS:
            setattr(self, k, 0)

    def phase4_rate(self) -> float:
        return self.phase4_triggers / self.chunks_processed if self.chunks_processed else 0.0

    def carry_to_add_ratio(self) -> float:
        """addsub.cpp:258-263: carry-handling ticks over the lane-add ticks."""
        if self.add_ticks == 0:
            return 0.0
        return (self.carry_gen_ticks + self.carry_add_ticks + self.store_ticks + self.overflow_ticks) / self.add_ticks

    def merge(self, other: "AddSubStats") -> None:
        self.chunks_processed += other.chunks_processed
        self.phase4_triggers += other.phase4_triggers
        for k in self.TICKS:
            setattr(self, k, getattr(self, k) + getattr(other, k))


class WordsResult(NamedTuple):
    """include/dot/limbs.hpp:28-31: m result limbs plus a carry/borrow flag."""

    limbs: np.ndarray
    flag: int


def _validate_width(width) -> None:
    check(lib().dotg_validate_width(int(width)))


def _host_u64(x, name: str) -> np.ndarray:
    if isinstance(x, (list, tuple)):  # Python ints (any mix with numpy scalars) up to 2^64 - 1
        try:
            x = np.array([operator.index(v) for v in x], dtype=np.uint64)
        except (OverflowError, TypeError, ValueError):
            raise InvalidArgument(f"{name}: limbs must be unsigned 64-bit integers") from None
    arr = np.asarray(x)
    if arr.dtype != np.uint64:
        if arr.size == 0:
            arr = arr.astype(np.uint64)
        elif arr.dtype.kind in "iu":
            arr = arr.astype(np.uint64)
        else:
            raise InvalidArgument(f"{name}: limbs must be unsigned 64-bit integers")
    if arr.ndim != 1:
        raise InvalidArgument(f"{name}: a limb sequence is one-dimensional")
    return np.ascontiguousarray(arr)


def _hp(arr: Optional[np.ndarray]):
    return None if arr is None or arr.size == 0 else ctypes.c_void_p(arr.ctypes.data)


def _words_span(sub: bool, out: np.ndarray, a, b, width, stats=None) -> int:
    _validate_width(width)
    if not isinstance(out, np.ndarray) or out.dtype != np.uint64 or not out.flags.c_contiguous:
        raise InvalidArgument("out must be a contiguous numpy uint64 array (the caller-owned span)")
    a = _host_u64(a, "a")
    b = _host_u64(b, "b")
    if a.size != b.size or out.size != a.size:
        raise InvalidArgument("dot add/sub: operand lengths differ (caller pads)")  # addsub.cpp:139-140
    carry = ctypes.c_uint32(0)
    if stats is not None:
        m = a.size
        if stats.collect_ticks and not (0 < m <= 256 and m & (m - 1) == 0):
            raise _lib.DotgError("AddSubStats.collect_ticks: the timed device kernel covers power-of-two m <= 256")
        ch, fi = ctypes.c_uint64(0), ctypes.c_uint64(0)
        dst = np.empty_like(out) if stats.collect_ticks else out  # out may alias a or b
        check(lib().dotg_words_host_stats(int(sub), _hp(dst), _hp(a), _hp(b), a.size, int(width),
                                          ctypes.byref(carry), ctypes.byref(ch), ctypes.byref(fi)))
        stats.chunks_processed += int(ch.value)
        stats.phase4_triggers += int(fi.value)
        if stats.collect_ticks:
            t = np.zeros(6, np.uint64)
            c32 = np.zeros(1, np.uint32)
            check(lib().dotg_addsub_phase_ticks_host(int(sub), _hp(out), _hp(a), _hp(b), _hp(c32), m, 1, _hp(t)))
            for k, v in zip(AddSubStats.TICKS, t.tolist()):
                setattr(stats, k, getattr(stats, k) + int(v))
            return int(c32[0])
        return int(carry.value)
    fn = lib().dotg_sub_words_host if sub else lib().dotg_add_words_host
    check(fn(_hp(out), _hp(a), _hp(b), a.size, ctypes.byref(carry)))
    return int(carry.value)


def _words_value(sub: bool, a, b, width, stats=None) -> WordsResult:
    a = _host_u64(a, "a")
    b = _host_u64(b, "b")
    m = max(a.size, b.size)  # addsub.cpp:192-206: zero-pad the shorter operand
    if a.size != m:
        a = np.concatenate([a, np.zeros(m - a.size, np.uint64)])
    if b.size != m:
        b = np.concatenate([b, np.zeros(m - b.size, np.uint64)])
    out = np.zeros(m, np.uint64)
    flag = _words_span(sub, out, a, b, width, stats)
    return WordsResult(out, flag)


def dot_add_words(*args, width=Width.w8, stats=None):
    """``dot_add_words(out, a, b[, width])`` -> carry (span form, addsub.hpp:98-100) or
    ``dot_add_words(a, b[, width])`` -> WordsResult (value form, addsub.hpp:106-107)."""
    return _dispatch_words(False, args, width, stats)


def dot_sub_words(*args, width=Width.w8, stats=None):
    """Subtraction twin of :func:`dot_add_words` (addsub.hpp:101-103, 108-109)."""
    return _dispatch_words(True, args, width, stats)


def _is_limbs(x) -> bool:
    return isinstance(x, (np.ndarray, list, tuple))


def _dispatch_words(sub: bool, args, width, stats):
    """Positional forms of the reference: (out, a, b[, width[, stats]]) is the span form
    (the third argument is a limb array), (a, b[, width[, stats]]) the value form."""
    span = len(args) >= 3 and _is_limbs(args[2])
    nfix = 3 if span else 2
    if len(args) < nfix or len(args) > nfix + 2:
        raise TypeError("expected (out, a, b[, width[, stats]]) or (a, b[, width[, stats]])")
    if len(args) > nfix:
        width = args[nfix]
    if len(args) > nfix + 1:
        stats = args[nfix + 1]
    if span:
        return _words_span(sub, args[0], args[1], args[2], width, stats)
    _validate_width(width)
    return _words_value(sub, args[0], args[1], width, stats)


class ChunkResult(NamedTuple):
    """include/dot/addsub.hpp:78-82: sums (first w entries valid), carry_out, phase4_fired."""

    sums: np.ndarray
    carry_out: int
    phase4_fired: bool


def _chunk(sub: bool, a, b, carry_in: int, w: int) -> ChunkResult:
    w = int(w)
    if w < 1 or w > 8:
        raise InvalidArgument("chunk width must be in 1..8")  # addsub.cpp:174
    a, b = _host_u64(a, "a"), _host_u64(b, "b")
    if a.size != w or b.size != w:
        raise InvalidArgument("chunk operands must have exactly w limbs")  # addsub.cpp:175-176
    if int(carry_in) not in (0, 1):
        raise InvalidArgument("carry_in must be 0 or 1")  # addsub.cpp:177
    sums = np.zeros(8, np.uint64)
    co, fi = ctypes.c_uint32(0), ctypes.c_uint32(0)
    check(lib().dotg_chunk_host(int(sub), _hp(sums), ctypes.byref(co), ctypes.byref(fi), _hp(a), _hp(b),
                                int(carry_in), w))
    return ChunkResult(sums, int(co.value), bool(fi.value))


def add_w_limbs(a, b, carry_in: int, w: int) -> ChunkResult:
    """One chunk of w lanes (addsub.hpp:86-87)."""
    return _chunk(False, a, b, carry_in, w)


def sub_w_limbs(a, b, borrow_in: int, w: int) -> ChunkResult:
    """One chunk of w lanes, subtraction (addsub.hpp:88-89)."""
    return _chunk(True, a, b, borrow_in, w)


def dot_mul_words(a, b, cfg: int = 64, width=Width.w8) -> np.ndarray:
    """Exact product, exactly 2m limbs (include/dot/mul.hpp:75-76, src/mul.cpp:96-103).
    Equal limb counts 1 <= m <= 2^24 (mul.cpp:13-18). cfg = 64 (kSaturated) runs the
    batched column / tensor-pipe / Karatsuba routes; cfg = 52 (kUnsaturated, limbs
    < 2^52) runs k_mul52 (dotg_mul52_batch_host), both on the device."""
    if int(cfg) not in (64, 52):
        raise InvalidArgument("RadixConfig: limb_bits must be 64 or 52")  # limbs.cpp:22-24
    _validate_width(width)
    a = _host_u64(a, "a")
    b = _host_u64(b, "b")
    if a.size != b.size:
        raise InvalidArgument("dot mul: operand lengths differ (caller pads)")
    if a.size == 0:
        raise InvalidArgument("dot mul: operands need at least one limb")
    if a.size > K_MAX_MUL_LIMBS:
        raise InvalidArgument("dot mul: limb count exceeds the column accumulator bound")
    out = np.zeros(2 * a.size, np.uint64)
    if int(cfg) == 52:
        check(lib().dotg_mul52_batch_host(_hp(out), _hp(a), _hp(b), a.size, 1))
    else:
        check(lib().dotg_mul_batch_host(_hp(out), _hp(a), _hp(b), a.size, 1))
    return out


def compare(a, b) -> int:
    """-1 / 0 / +1, high zero limbs ignored (limbs.hpp:84, limbs.cpp:46-53), on the device."""
    a, b = _host_u64(a, "a"), _host_u64(b, "b")
    m = max(a.size, b.size)
    pa, pb = np.zeros(max(m, 1), np.uint64), np.zeros(max(m, 1), np.uint64)
    pa[: a.size], pb[: b.size] = a, b
    out = np.zeros(1, np.int32)
    check(lib().dotg_compare_host(_hp(out), _hp(pa), _hp(pb), m, 1))
    return int(out[0])


def carry_census(k: int):
    """(max_sum_pairs, carry_pairs) over all k-bit pairs (oracle.cpp:65-78), on the device."""
    out = np.zeros(2, np.uint64)
    check(lib().dotg_carry_census(int(k), _hp(out)))
    return int(out[0]), int(out[1])


def run_stats(k_max: int = 12, mc_samples: int = 10_000_000, seed: int = 1) -> dict:
    """run_stats (bench.cpp:261-289): census rows k = 1..k_max against the closed forms
    2^k and 2^(k-1) (2^k - 1), and the Monte-Carlo carry frequency of random 64-bit adds
    (|f - 0.5| <= 0.001); everything counted on the device."""
    if not 1 <= int(k_max) <= 16:
        raise InvalidArgument("stats: k_max must be in 1..16")
    rows = []
    for k in range(1, int(k_max) + 1):
        ms, cp = carry_census(k)
        cm, cc = 1 << k, (1 << (k - 1)) * ((1 << k) - 1)
        rows.append({"k": k, "max_sum_pairs": ms, "closed_max_sum": cm, "carry_pairs": cp, "closed_carry": cc,
                     "match": ms == cm and cp == cc})
    c = np.zeros(1, np.uint64)
    check(lib().dotg_mc_carry(int(mc_samples), int(seed) & (2**64 - 1), _hp(c)))
    freq = int(c[0]) / mc_samples if mc_samples else 0.0
    return {"census": rows, "mc_samples": int(mc_samples), "mc_carry_freq": freq,
            "mc_within_tolerance": bool(mc_samples) and abs(freq - 0.5) <= 0.001}


# ---- the column pipeline as separate device stages (mul.hpp:32-67, mul.cpp:12-90)
def num_pairs(c: int, m: int) -> int:
    """mul.hpp:36-38: pair count of column c (c = 2m - 1 is the carry slot, 0 pairs)."""
    return min(c + 1, m, 2 * m - 1 - c)


def gather_columns(a, b):
    """(m_a, m_b): the m*m pairs in column order (mul.cpp:12-36), gathered on the device."""
    a, b = _host_u64(a, "a"), _host_u64(b, "b")
    if a.size != b.size:
        raise InvalidArgument("dot mul: operand lengths differ (caller pads)")
    m = a.size
    ma, mb = np.zeros(m * m, np.uint64), np.zeros(m * m, np.uint64)
    check(lib().dotg_gather_columns_host(_hp(ma), _hp(mb), _hp(a), _hp(b), m))
    return ma, mb


def compute_partials(m_a, m_b, limb_bits: int = 64):
    """(p_lo, p_hi) = products split at bit k (mul.cpp:38-52), on the device."""
    m_a, m_b = _host_u64(m_a, "m_a"), _host_u64(m_b, "m_b")
    if m_a.size != m_b.size:
        raise InvalidArgument("column buffers: m_a / m_b sizes differ")
    lo, hi = np.zeros(m_a.size, np.uint64), np.zeros(m_a.size, np.uint64)
    check(lib().dotg_compute_partials_host(_hp(lo), _hp(hi), _hp(m_a), _hp(m_b), m_a.size, int(limb_bits)))
    return lo, hi


def align_and_reduce(p_lo, p_hi, m: int) -> list:
    """The 2m u128 column sums (mul.cpp:54-68) as Python ints, reduced on the device."""
    p_lo, p_hi = _host_u64(p_lo, "p_lo"), _host_u64(p_hi, "p_hi")
    if p_lo.size != m * m or p_hi.size != m * m:
        raise InvalidArgument("column buffers: partial buffers need m*m entries")
    cols = np.zeros(4 * m, np.uint64)
    check(lib().dotg_align_and_reduce_host(_hp(cols), _hp(p_lo), _hp(p_hi), m))
    return [int(cols[2 * c]) | (int(cols[2 * c + 1]) << 64) for c in range(2 * m)]


def carry_pass(columns, limb_bits: int = 64) -> np.ndarray:
    """Sequential renormalisation of u128 columns (mul.cpp:70-90) on the device; residual
    carry limbs are appended."""
    cols = list(columns)
    if any(not 0 <= int(c) < 1 << 128 for c in cols):
        raise InvalidArgument("columns are unsigned 128-bit values")
    raw = np.zeros(max(1, 2 * len(cols)), np.uint64)
    for i, c in enumerate(cols):
        raw[2 * i] = int(c) & (2**64 - 1)
        raw[2 * i + 1] = int(c) >> 64
    out = np.zeros(len(cols) + 2, np.uint64)
    n = ctypes.c_uint32(0)
    check(lib().dotg_carry_pass_host(_hp(out), ctypes.byref(n), out.size, _hp(raw) if cols else None, len(cols),
                                     int(limb_bits)))
    return out[: n.value].copy()


def dot_mul_5x5(a, b) -> np.ndarray:
    """Fixed 5-limb product over unsaturated 52-bit limbs, exactly 10 limbs
    (mul.hpp:78-80, mul.cpp:127-150)."""
    a, b = _host_u64(a, "a"), _host_u64(b, "b")
    if a.size != 5 or b.size != 5:
        raise InvalidArgument("dot mul 5x5: operands must be exactly 5 limbs")
    return dot_mul_words(a, b, 52)


def dot_mul_4x4(a, b) -> np.ndarray:
    """Fixed 4-limb product over saturated limbs, exactly 8 limbs (mul.hpp:82-85,
    mul.cpp:152-159; the reference routes it through 52-bit repacking and the 5x5
    kernel, the device computes it directly - identical result)."""
    a, b = _host_u64(a, "a"), _host_u64(b, "b")
    if a.size != 4 or b.size != 4:
        raise InvalidArgument("dot mul 4x4: operands must be exactly 4 limbs")
    return dot_mul_words(a, b)


def pack_64_to_52(a) -> np.ndarray:
    """limbs.hpp:111-113: re-slice 64m bits into ceil(64m/52) 52-bit groups (host-side
    representation helper, not arithmetic)."""
    a = _host_u64(a, "a")
    n = (64 * a.size + 51) // 52
    v = int.from_bytes(a.astype("<u8").tobytes(), "little")
    return np.array([(v >> (52 * i)) & ((1 << 52) - 1) for i in range(n)], dtype=np.uint64)


def unpack_52_to_64(a) -> np.ndarray:
    """limbs.hpp:115-117: inverse re-slicing, trims high zero words so a pack round trip
    returns the original limb count; any word >= 2^52 is std::invalid_argument."""
    a = _host_u64(a, "a")
    if a.size and int(a.max()) >= (1 << 52):
        raise InvalidArgument("unpack_52_to_64: word exceeds 52 bits")
    v = 0
    for i in range(a.size - 1, -1, -1):
        v = (v << 52) | int(a[i])
    n = (52 * a.size + 63) // 64
    out = np.array([(v >> (64 * i)) & ((1 << 64) - 1) for i in range(n)], dtype=np.uint64)
    return _trim(out)


# ---------------------------------------------------------------------------
# Host batch helpers (row-major [batch, m] numpy arrays; pinned memory recommended)
# ---------------------------------------------------------------------------
def _host_2d(x, name):
    arr = np.asarray(x)
    if arr.dtype != np.uint64 or arr.ndim != 2 or not arr.flags.c_contiguous:
        raise InvalidArgument(f"{name}: expected a C-contiguous [batch, m] uint64 array")
    return arr


def addsub_batch_host(sub: bool, a, b, out=None, flags=None):
    a = _host_2d(a, "a")
    b = _host_2d(b, "b")
    if a.shape != b.shape:
        raise InvalidArgument("dot add/sub: operand shapes differ")
    batch, m = a.shape
    out = np.empty_like(a) if out is None else _host_2d(out, "out")
    flags = np.empty(batch, np.uint32) if flags is None else flags
    fn = lib().dotg_sub_batch_host if sub else lib().dotg_add_batch_host
    check(fn(_hp(out), _hp(a), _hp(b), _hp(flags), m, batch))
    return out, flags


def mul_batch_host(a, b, out=None):
    a = _host_2d(a, "a")
    b = _host_2d(b, "b")
    if a.shape != b.shape:
        raise InvalidArgument("dot mul: operand shapes differ")
    batch, m = a.shape
    out = np.empty((batch, 2 * m), np.uint64) if out is None else _host_2d(out, "out")
    check(lib().dotg_mul_batch_host(_hp(out), _hp(a), _hp(b), m, batch))
    return out


# ---------------------------------------------------------------------------
# Device batch API (torch CUDA tensors)
# ---------------------------------------------------------------------------
def _torch():
    import torch

    return torch


def _dptr(t):
    # the ctypes signatures declare c_void_p: a plain int converts without a wrapper object
    return None if t is None else t.data_ptr()


_raw_stream = None


def _stream_handle(stream):
    """The caller's stream (or the current one) as a raw cudaStream_t. The current-stream
    query goes through torch's raw accessor when it exists (~0.3 us instead of ~3 us for
    torch.cuda.current_stream(), which builds a Stream object)."""
    global _raw_stream
    if stream is not None:
        return stream.cuda_stream
    torch = _torch()
    if _raw_stream is None:
        getter = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        _raw_stream = (lambda: getter(torch.cuda.current_device())) if getter else (
            lambda: torch.cuda.current_stream().cuda_stream)
    return _raw_stream()


def _check_dev(t, name, elem=8):
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise InvalidArgument(f"{name}: expected a CUDA tensor")
    if t.element_size() != elem or not t.is_contiguous():
        raise InvalidArgument(f"{name}: expected a contiguous {8 * elem}-bit tensor")


def _layout(layout) -> int:
    if layout in (ROW_MAJOR, "row", "row_major"):
        return ROW_MAJOR
    if layout in (INTERLEAVED, "interleaved"):
        return INTERLEAVED
    raise InvalidArgument(f"unknown layout {layout!r}")


def _batch_dims(a, layout):
    if a.dim() != 2:
        raise InvalidArgument("batched operands are 2-D")
    return (a.shape[0], a.shape[1]) if layout == ROW_MAJOR else (a.shape[1], a.shape[0])


def _row_pitched(t) -> bool:
    """A 2-D CUDA int64 view whose rows are contiguous (stride(1) == 1) at a pitch >= m."""
    torch = _torch()
    return (isinstance(t, torch.Tensor) and t.is_cuda and t.element_size() == 8 and t.dim() == 2
            and (t.shape[1] <= 1 or t.stride(1) == 1) and (t.shape[0] <= 1 or t.stride(0) >= t.shape[1]))


def addsub_batch(sub: bool, a, b, out=None, flags=None, *, layout=ROW_MAJOR, stream=None):
    """out = a +/- b per pair, flags = carry/borrow per pair (device tensors).
    ROW_MAJOR a: [batch, m]; INTERLEAVED a: [m, batch]. Row-major operands may be views
    with a row pitch (e.g. x[:, :m] of a wider tensor): dotg_addsub_batch_strided."""
    torch = _torch()
    lay = _layout(layout)
    views = [t for t in (a, b, out) if t is not None]
    if lay == ROW_MAJOR and not all(t.is_contiguous() for t in views if isinstance(t, torch.Tensor)) and all(
            _row_pitched(t) for t in views):
        if a.shape != b.shape or (out is not None and out.shape != a.shape):
            raise InvalidArgument("dot add/sub: operand shapes differ")
        batch, m = a.shape
        if out is None:
            out = torch.empty_like(a, memory_format=torch.contiguous_format)
        if flags is None:
            flags = torch.empty(batch, dtype=torch.int32, device=a.device)
        _check_dev(flags, "flags", 4)
        pitch = [t.stride(0) if t.shape[0] > 1 else m for t in (out, a, b)]
        check(lib().dotg_addsub_batch_strided(int(sub), _dptr(out), pitch[0], _dptr(a), pitch[1], _dptr(b), pitch[2],
                                              _dptr(flags), m, batch, _stream_handle(stream)))
        return out, flags
    _check_dev(a, "a")
    _check_dev(b, "b")
    if a.shape != b.shape:
        raise InvalidArgument("dot add/sub: operand shapes differ")
    batch, m = _batch_dims(a, lay)
    if out is None:
        out = torch.empty_like(a)
    _check_dev(out, "out")
    if out.shape != a.shape:
        raise InvalidArgument("out shape differs")
    if flags is None:
        flags = torch.empty(batch, dtype=torch.int32, device=a.device)
    _check_dev(flags, "flags", 4)
    fn = lib().dotg_sub_batch if sub else lib().dotg_add_batch
    check(fn(_dptr(out), _dptr(a), _dptr(b), _dptr(flags), m, batch, lay, _stream_handle(stream)))
    return out, flags


def add_batch(a, b, out=None, flags=None, *, layout=ROW_MAJOR, stream=None):
    return addsub_batch(False, a, b, out, flags, layout=layout, stream=stream)


def sub_batch(a, b, out=None, flags=None, *, layout=ROW_MAJOR, stream=None):
    return addsub_batch(True, a, b, out, flags, layout=layout, stream=stream)


def addsub_grouped(problems, *, stream=None):
    """Several independent batched add/sub problems in one call (one persistent launch
    for the row-major power-of-two sizes). problems: iterable of dicts with keys
    op ('add'|'sub'), a, b, out, flags (optional), layout (optional)."""
    plist = list(problems)
    arr = (_lib.AddSubProblem * max(1, len(plist)))()
    keep = []
    for i, q in enumerate(plist):
        lay = _layout(q.get("layout", ROW_MAJOR))
        a, b, out = q["a"], q["b"], q["out"]
        for t, nm in ((a, "a"), (b, "b"), (out, "out")):
            _check_dev(t, nm)
        if a.shape != b.shape or out.shape != a.shape:
            raise InvalidArgument("dot add/sub: operand shapes differ")
        batch, m = _batch_dims(a, lay)
        fl = q.get("flags")
        if fl is not None:
            _check_dev(fl, "flags", 4)
        op = {"add": 0, "sub": 1, 0: 0, 1: 1}[q["op"]]
        arr[i] = _lib.AddSubProblem(op, lay, out.data_ptr(), a.data_ptr(), b.data_ptr(),
                                    None if fl is None else fl.data_ptr(), m, batch)
        keep.append(q)
    check(lib().dotg_addsub_grouped(arr, len(plist), _stream_handle(stream)))
    return plist


def mul_batch(a, b, out=None, *, layout=ROW_MAJOR, stream=None):
    """out = a * b per pair, exactly 2m limbs. ROW_MAJOR out: [batch, 2m];
    INTERLEAVED out: [2m, batch]."""
    torch = _torch()
    lay = _layout(layout)
    views = [t for t in (a, b, out) if t is not None]
    if lay == ROW_MAJOR and not all(t.is_contiguous() for t in views if isinstance(t, torch.Tensor)) and all(
            _row_pitched(t) for t in views):
        # row-pitched views (e.g. x[:, :m] of a wider tensor): dotg_mul_batch_strided
        if a.shape != b.shape:
            raise InvalidArgument("dot mul: operand shapes differ")
        batch, m = a.shape
        if out is None:
            out = torch.empty((batch, 2 * m), dtype=a.dtype, device=a.device)
        if tuple(out.shape) != (batch, 2 * m):
            raise InvalidArgument("out must hold exactly 2m limbs per pair")
        pitch = [t.stride(0) if t.shape[0] > 1 else n for t, n in ((out, 2 * m), (a, m), (b, m))]
        check(lib().dotg_mul_batch_strided(_dptr(out), pitch[0], _dptr(a), pitch[1], _dptr(b), pitch[2], m, batch,
                                           _stream_handle(stream)))
        return out
    _check_dev(a, "a")
    _check_dev(b, "b")
    if a.shape != b.shape:
        raise InvalidArgument("dot mul: operand shapes differ")
    batch, m = _batch_dims(a, lay)
    shape = (batch, 2 * m) if lay == ROW_MAJOR else (2 * m, batch)
    if out is None:
        out = torch.empty(shape, dtype=a.dtype, device=a.device)
    _check_dev(out, "out")
    if tuple(out.shape) != shape:
        raise InvalidArgument("out must hold exactly 2m limbs per pair")
    check(lib().dotg_mul_batch(_dptr(out), _dptr(a), _dptr(b), m, batch, lay, _stream_handle(stream)))
    return out


def addsub_stats(sub: bool, out, a, b, *, width=Width.w8, layout=ROW_MAJOR, stream=None):
    """AddSubStats counters (addsub.hpp:53-72) of a finished batched add/sub, derived on the
    device from a, b and out (csrc/stats.cu): (chunks_processed, phase4_triggers) for chunks
    of lane_count(width) limbs. Synchronises the stream to return host integers."""
    torch = _torch()
    lay = _layout(layout)
    for t, name in ((out, "out"), (a, "a"), (b, "b")):
        _check_dev(t, name)
    if not (a.shape == b.shape == out.shape):
        raise InvalidArgument("stats: operand shapes differ")
    batch, m = _batch_dims(a, lay)
    # the counters are zeroed, accumulated and read back on ONE stream (the caller's):
    # the zero-fill runs on it as torch's current stream, and the read-back synchronises it
    import contextlib

    with torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext():
        cnt = torch.zeros(2, dtype=torch.int64, device=a.device)
        check(lib().dotg_addsub_stats(int(sub), _dptr(out), _dptr(a), _dptr(b), m, batch, lay, int(width),
                                      _dptr(cnt), _stream_handle(stream)))
        if stream is not None:
            stream.synchronize()
        ch, fi = cnt.tolist()
    return int(ch), int(fi)


def addsub_phase_ticks(sub: bool, a, b, out=None, flags=None, *, stream=None) -> dict:
    """Phase split of the batched add/sub on the device (the GPU counterpart of the
    reference's collect_ticks pass, bench.cpp:227-247): runs the team kernel with
    %clock64 laps compiled in over row-major [batch, m] device tensors (power-of-two
    m <= 256), writes out / flags like add_batch / sub_batch, and returns the six tick
    buckets (SM cycles summed over warps), their percentages and carry_to_add_ratio."""
    torch = _torch()
    import contextlib

    _check_dev(a, "a")
    _check_dev(b, "b")
    if a.shape != b.shape or a.dim() != 2:
        raise InvalidArgument("phase ticks: a, b must be [batch, m] tensors of one shape")
    batch, m = a.shape
    if out is None:
        out = torch.empty_like(a)
    if flags is None:
        flags = torch.empty(batch, dtype=torch.int32, device=a.device)
    with torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext():
        t = torch.zeros(6, dtype=torch.int64, device=a.device)
        check(lib().dotg_addsub_phase_ticks(int(sub), _dptr(out), _dptr(a), _dptr(b), _dptr(flags), m, batch,
                                            _dptr(t), _stream_handle(stream)))
        if stream is not None:
            stream.synchronize()
        ticks = [int(x) for x in t.tolist()]
    res = dict(zip(AddSubStats.TICKS, ticks))
    total = sum(ticks)
    res["pct"] = {k.replace("_ticks", ""): (100.0 * v / total if total else 0.0) for k, v in zip(AddSubStats.TICKS, ticks)}
    res["carry_to_add_ratio"] = (sum(ticks[2:]) / ticks[1]) if ticks[1] else 0.0
    return res


def compare_batch(a, b, out=None, *, layout=ROW_MAJOR, stream=None):
    """compare(a[p], b[p]) per pair (limbs.hpp:84): int32 tensor of -1 / 0 / +1."""
    torch = _torch()
    lay = _layout(layout)
    _check_dev(a, "a")
    _check_dev(b, "b")
    if a.shape != b.shape:
        raise InvalidArgument("compare: operand shapes differ")
    batch, m = _batch_dims(a, lay)
    if out is None:
        out = torch.empty(batch, dtype=torch.int32, device=a.device)
    if out.dtype != torch.int32 or out.numel() != batch or not out.is_contiguous():
        raise InvalidArgument("compare: out must be a contiguous int32 tensor of batch entries")
    check(lib().dotg_compare_batch(_dptr(out), _dptr(a), _dptr(b), m, batch, lay, _stream_handle(stream)))
    return out


def chunk_batch(sub: bool, a, b, carry_in=None, *, stream=None):
    """Batched add_w_limbs / sub_w_limbs: a, b are [batch, w] device tensors (1 <= w <= 8),
    carry_in an int32 [batch] tensor or None. Returns (sums, carry_out, phase4_fired)."""
    torch = _torch()
    _check_dev(a, "a")
    _check_dev(b, "b")
    if a.dim() != 2 or a.shape != b.shape:
        raise InvalidArgument("chunk: operands are [batch, w] tensors of one shape")
    batch, w = a.shape
    sums = torch.empty_like(a)
    co = torch.empty(batch, dtype=torch.int32, device=a.device)
    fi = torch.empty(batch, dtype=torch.int32, device=a.device)
    cin = 0
    if carry_in is not None:
        if carry_in.dtype != torch.int32 or carry_in.numel() != batch or not carry_in.is_contiguous():
            raise InvalidArgument("chunk: carry_in must be a contiguous int32 tensor of batch entries")
        cin = _dptr(carry_in)
    check(lib().dotg_chunk_batch(int(sub), _dptr(sums), _dptr(co), _dptr(fi), _dptr(a), _dptr(b), cin, w, batch,
                                 _stream_handle(stream)))
    return sums, co, fi


def words(sub: bool, a, b, out=None, carry=None, *, stream=None):
    """One long number on the device: out = a +/- b, carry = device int32[1]."""
    torch = _torch()
    _check_dev(a, "a")
    _check_dev(b, "b")
    if a.dim() != 1 or a.shape != b.shape:
        raise InvalidArgument("dot add/sub: operand lengths differ (caller pads)")
    out = torch.empty_like(a) if out is None else out
    _check_dev(out, "out")
    if out.shape != a.shape:
        raise InvalidArgument("dot add/sub: operand lengths differ (caller pads)")
    carry = torch.empty(1, dtype=torch.int32, device=a.device) if carry is None else carry
    fn = lib().dotg_sub_words if sub else lib().dotg_add_words
    check(fn(_dptr(out), _dptr(a), _dptr(b), a.numel(), _dptr(carry), _stream_handle(stream)))
    return out, carry


def add_words(a, b, out=None, carry=None, *, stream=None):
    return words(False, a, b, out, carry, stream=stream)


def sub_words(a, b, out=None, carry=None, *, stream=None):
    return words(True, a, b, out, carry, stream=stream)


# ---------------------------------------------------------------------------
# Karatsuba (reference karatsuba_mul, include/dot/mul.hpp:87-102, src/mul.cpp:161-233)
# ---------------------------------------------------------------------------
class KaratsubaConfig(NamedTuple):
    """mul.hpp:91-93: limb count at or below which the base case runs."""

    theta: int = 4


def karatsuba_mul(a, b, cfg: KaratsubaConfig = KaratsubaConfig()) -> np.ndarray:
    """Reference semantics: inputs trimmed, unequal lengths zero-padded to the longer,
    empty/zero operand -> empty result, result trimmed (mul.cpp:222-233). The product
    runs on the device (dotg_karatsuba_batch_host)."""
    theta = int(cfg.theta if isinstance(cfg, KaratsubaConfig) else cfg)
    if theta < 1:
        raise InvalidArgument("karatsuba: threshold must be at least 1")
    a = _trim(_host_u64(a, "a"))
    b = _trim(_host_u64(b, "b"))
    if a.size == 0 or b.size == 0:
        return np.zeros(0, np.uint64)
    m = max(a.size, b.size)
    pa = np.zeros(m, np.uint64)
    pb = np.zeros(m, np.uint64)
    pa[:a.size] = a
    pb[:b.size] = b
    out = np.zeros(2 * m, np.uint64)
    check(lib().dotg_karatsuba_batch_host(_hp(out), _hp(pa), _hp(pb), m, 1, theta))
    return _trim(out)


def karatsuba_batch(a, b, out=None, *, theta: int = 4, stream=None):
    """Device batch form: row-major [batch, m] tensors -> [batch, 2m] (untrimmed)."""
    torch = _torch()
    _check_dev(a, "a")
    _check_dev(b, "b")
    if a.shape != b.shape or a.dim() != 2:
        raise InvalidArgument("dot mul: operand shapes differ")
    batch, m = a.shape
    if out is None:
        out = torch.empty((batch, 2 * m), dtype=a.dtype, device=a.device)
    _check_dev(out, "out")
    check(lib().dotg_karatsuba_batch(_dptr(out), _dptr(a), _dptr(b), m, batch, int(theta), _stream_handle(stream)))
    return out


def _trim(x: np.ndarray) -> np.ndarray:
    """normalized() (src/limbs.cpp:40-44): drop high zero limbs."""
    nz = np.flatnonzero(x)
    return x[: nz[-1] + 1].copy() if nz.size else np.zeros(0, np.uint64)
