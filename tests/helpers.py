"""Test helpers: ctypes access to the oracle (oracle/liboracle.so, our C restatement) and
to the reference itself (oracle/_ref/libdotref.so), plus numpy input generators that
restate the reference tests' shapes (test_addsub.cpp:22-40, testgen.cpp:87-128).

The oracle is the CHECKER only; nothing here is used by the product path.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import c_int, c_size_t, c_uint, c_uint64, c_void_p

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libdotref.so")
MAX = np.uint64(0xFFFFFFFFFFFFFFFF)
U64 = np.uint64


def _p(arr):
    return None if arr is None else c_void_p(arr.ctypes.data)


def u64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint64))


class Oracle:
    """oracle/dot_oracle.c via ctypes."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True,
                           capture_output=True)
        L = ctypes.CDLL(ORACLE_SO)
        L.dotor_add.restype = c_uint
        L.dotor_add.argtypes = [c_void_p, c_void_p, c_void_p, c_size_t]
        L.dotor_sub.restype = c_uint
        L.dotor_sub.argtypes = [c_void_p, c_void_p, c_void_p, c_size_t]
        L.dotor_mul.restype = c_size_t
        L.dotor_mul.argtypes = [c_void_p, c_void_p, c_size_t, c_void_p, c_size_t]
        L.dotor_chunk.restype = c_uint
        L.dotor_chunk.argtypes = [c_int, c_void_p, c_void_p, c_void_p, c_uint, c_uint, c_void_p]
        L.dotor_words.restype = c_uint
        L.dotor_words.argtypes = [c_int, c_void_p, c_void_p, c_void_p, c_size_t, c_uint, c_void_p, c_void_p]
        L.dotor_mul_columns.restype = None
        L.dotor_mul_columns.argtypes = [c_void_p, c_void_p, c_void_p, c_size_t]
        L.dotor_compare.restype = c_int
        L.dotor_compare.argtypes = [c_void_p, c_size_t, c_void_p, c_size_t]
        L.dotor_addsub_batch.restype = None
        L.dotor_addsub_batch.argtypes = [c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_size_t]
        L.dotor_mul_batch.restype = None
        L.dotor_mul_batch.argtypes = [c_void_p, c_void_p, c_void_p, c_size_t, c_size_t]
        L.dotor_mul_columns52.restype = None
        L.dotor_mul_columns52.argtypes = [c_void_p, c_void_p, c_void_p, c_size_t]
        L.dotor_fill_splitmix64.restype = None
        L.dotor_fill_splitmix64.argtypes = [c_void_p, c_size_t, c_uint64, c_uint64]
        L.dotor_gather_columns.restype = c_size_t
        L.dotor_gather_columns.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_size_t]
        L.dotor_compute_partials.restype = None
        L.dotor_compute_partials.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_uint]
        L.dotor_align_and_reduce.restype = None
        L.dotor_align_and_reduce.argtypes = [c_void_p, c_void_p, c_void_p, c_size_t]
        L.dotor_carry_pass.restype = c_size_t
        L.dotor_carry_pass.argtypes = [c_void_p, c_void_p, c_size_t, c_uint]
        self.L = L

    # the column pipeline stage by stage (mul.cpp:12-90); columns are [2m, 2] (low, high)
    def gather_columns(self, a, b):
        a, b = u64(a), u64(b)
        m = a.size
        ma, mb = np.zeros(m * m, U64), np.zeros(m * m, U64)
        n = self.L.dotor_gather_columns(_p(ma), _p(mb), _p(a), _p(b), m)
        assert n == m * m
        return ma, mb

    def compute_partials(self, ma, mb, k=64):
        ma, mb = u64(ma), u64(mb)
        lo, hi = np.zeros(ma.size, U64), np.zeros(ma.size, U64)
        self.L.dotor_compute_partials(_p(lo), _p(hi), _p(ma), _p(mb), ma.size, k)
        return lo, hi

    def align_and_reduce(self, lo, hi, m):
        lo, hi = u64(lo), u64(hi)
        cols = np.zeros((2 * m, 2), U64)
        self.L.dotor_align_and_reduce(_p(cols), _p(lo), _p(hi), m)
        return cols

    def carry_pass(self, cols, k=64):
        cols = u64(cols).reshape(-1, 2)
        out = np.zeros(cols.shape[0] + 3, U64)
        n = self.L.dotor_carry_pass(_p(out), _p(cols), cols.shape[0], k)
        return out[:n].copy()

    # oracle_add / oracle_sub (oracle.cpp:16-48)
    def add(self, a, b):
        a, b = u64(a), u64(b)
        assert a.size == b.size
        out = np.zeros(a.size, U64)
        f = self.L.dotor_add(_p(out), _p(a), _p(b), a.size)
        return out, int(f)

    def sub(self, a, b):
        a, b = u64(a), u64(b)
        assert a.size == b.size
        out = np.zeros(a.size, U64)
        f = self.L.dotor_sub(_p(out), _p(a), _p(b), a.size)
        return out, int(f)

    def mul(self, a, b):
        """oracle_mul: trimmed (oracle.cpp:50-63)."""
        a, b = u64(a), u64(b)
        if a.size == 0 or b.size == 0:
            return np.zeros(0, U64)
        out = np.zeros(a.size + b.size, U64)
        n = self.L.dotor_mul(_p(out), _p(a), a.size, _p(b), b.size)
        return out[:n].copy()

    def mul_columns(self, a, b):
        a, b = u64(a), u64(b)
        out = np.zeros(2 * a.size, U64)
        self.L.dotor_mul_columns(_p(out), _p(a), _p(b), a.size)
        return out

    def mul_columns52(self, a, b):
        a, b = u64(a), u64(b)
        out = np.zeros(2 * a.size, U64)
        self.L.dotor_mul_columns52(_p(out), _p(a), _p(b), a.size)
        return out

    def chunk(self, sub, a, b, cin, t):
        a, b = u64(a), u64(b)
        out = np.zeros(8, U64)
        p4 = c_int(0)
        c = self.L.dotor_chunk(int(sub), _p(out), _p(a), _p(b), cin, t, ctypes.byref(p4))
        return out[:t].copy(), int(c), bool(p4.value)

    def words(self, sub, a, b, lanes=8):
        a, b = u64(a), u64(b)
        out = np.zeros(a.size, U64)
        ch, fi = c_uint64(0), c_uint64(0)
        c = self.L.dotor_words(int(sub), _p(out), _p(a), _p(b), a.size, lanes, ctypes.byref(ch), ctypes.byref(fi))
        return out, int(c), int(ch.value), int(fi.value)

    def compare(self, a, b):
        a, b = u64(a), u64(b)
        return int(self.L.dotor_compare(_p(a), a.size, _p(b), b.size))

    def addsub_batch(self, sub, a, b):
        a, b = u64(a), u64(b)
        batch, m = a.shape
        out = np.zeros_like(a)
        flags = np.zeros(batch, np.uint32)
        self.L.dotor_addsub_batch(int(sub), _p(out), _p(a), _p(b), _p(flags), m, batch)
        return out, flags

    def mul_batch(self, a, b):
        a, b = u64(a), u64(b)
        batch, m = a.shape
        out = np.zeros((batch, 2 * m), U64)
        self.L.dotor_mul_batch(_p(out), _p(a), _p(b), m, batch)
        return out

    def fill(self, n, seed, offset):
        out = np.zeros(n, U64)
        self.L.dotor_fill_splitmix64(_p(out), n, seed & (2**64 - 1), offset & (2**64 - 1))
        return out


class Reference:
    """The unmodified reference core (oracle/_ref/libdotref.so, built by oracle/Makefile)."""

    @classmethod
    def load(cls):
        if not os.path.exists(REF_SO):
            if os.path.isdir("/root/reference/proj/src"):
                subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=False,
                               capture_output=True)
            if not os.path.exists(REF_SO):
                return None
        return cls(ctypes.CDLL(REF_SO))

    def __init__(self, L):
        L.dotref_words.restype = c_int
        L.dotref_words.argtypes = [c_int, c_void_p, c_size_t, c_void_p, c_size_t, c_void_p, c_size_t, c_int,
                                   c_void_p, c_void_p]
        L.dotref_words_value.restype = c_int
        L.dotref_words_value.argtypes = [c_int, c_void_p, c_void_p, c_size_t, c_void_p, c_size_t, c_int]
        L.dotref_chunk.restype = c_int
        L.dotref_chunk.argtypes = [c_int, c_void_p, c_void_p, c_void_p, c_size_t, c_uint, c_uint, c_void_p]
        L.dotref_mul_words.restype = c_int
        L.dotref_mul_words.argtypes = [c_void_p, c_void_p, c_size_t, c_void_p, c_size_t]
        L.dotref_oracle_addsub.restype = c_int
        L.dotref_oracle_addsub.argtypes = [c_int, c_void_p, c_void_p, c_size_t, c_void_p, c_size_t]
        L.dotref_oracle_mul.restype = c_int
        L.dotref_oracle_mul.argtypes = [c_void_p, c_void_p, c_size_t, c_void_p, c_size_t]
        L.dotref_batch.restype = c_int
        L.dotref_batch.argtypes = [c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_size_t, c_int]
        for fn in ("dotref_mul_words52", "dotref_mul_5x5", "dotref_mul_4x4"):
            getattr(L, fn).restype = c_int
            getattr(L, fn).argtypes = [c_void_p, c_void_p, c_size_t, c_void_p, c_size_t]
        for fn in ("dotref_pack_64_to_52", "dotref_unpack_52_to_64"):
            getattr(L, fn).restype = c_int
            getattr(L, fn).argtypes = [c_void_p, c_void_p, c_size_t]
        L.dotref_dispatch_note.restype = ctypes.c_char_p
        L.dotref_dispatch_note.argtypes = [c_int]
        L.dotref_gather_columns.restype = c_int
        L.dotref_gather_columns.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_size_t]
        L.dotref_compute_partials.restype = c_int
        L.dotref_compute_partials.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_int, c_int]
        L.dotref_align_and_reduce.restype = c_int
        L.dotref_align_and_reduce.argtypes = [c_void_p, c_void_p, c_void_p, c_size_t]
        L.dotref_carry_pass.restype = c_int
        L.dotref_carry_pass.argtypes = [c_void_p, c_void_p, c_size_t, c_int]
        L.dotref_last_error.restype = ctypes.c_char_p
        self.L = L

    def dispatch_note(self, w=8):
        return self.L.dotref_dispatch_note(w).decode()

    def words(self, sub, a, b, width=8):
        """Span form dot_add_words/dot_sub_words -> (out, carry, chunks, phase4)."""
        a, b = u64(a), u64(b)
        out = np.zeros(a.size, U64)
        ch, fi = c_uint64(0), c_uint64(0)
        c = self.L.dotref_words(int(sub), _p(out), out.size, _p(a), a.size, _p(b), b.size, width,
                                ctypes.byref(ch), ctypes.byref(fi))
        if c < 0:
            raise ValueError(self.L.dotref_last_error().decode())
        return out, c, int(ch.value), int(fi.value)

    def chunk(self, sub, a, b, cin, w):
        a, b = u64(a), u64(b)
        out = np.zeros(8, U64)
        p4 = c_int(0)
        c = self.L.dotref_chunk(int(sub), _p(out), _p(a), _p(b), a.size, cin, w, ctypes.byref(p4))
        if c < 0:
            raise ValueError(self.L.dotref_last_error().decode())
        return out[:w].copy(), c, bool(p4.value)

    def mul_words(self, a, b):
        a, b = u64(a), u64(b)
        out = np.zeros(2 * max(a.size, 1), U64)
        n = self.L.dotref_mul_words(_p(out), _p(a), a.size, _p(b), b.size)
        if n < 0:
            raise ValueError(self.L.dotref_last_error().decode())
        return out[:n].copy()

    def mul2(self, fn, a, b, cap):
        a, b = u64(a), u64(b)
        out = np.zeros(cap, U64)
        n = getattr(self.L, fn)(_p(out), _p(a), a.size, _p(b), b.size)
        if n < 0:
            raise ValueError(self.L.dotref_last_error().decode())
        return out[:n].copy()

    def repack(self, fn, a):
        a = u64(a)
        out = np.zeros(2 * a.size + 2, U64)
        n = getattr(self.L, fn)(_p(out), _p(a), a.size)
        if n < 0:
            raise ValueError(self.L.dotref_last_error().decode())
        return out[:n].copy()

    # the column pipeline stages of the reference itself (mul.hpp:32-67)
    def _ok(self, rc):
        if rc < 0:
            raise ValueError(self.L.dotref_last_error().decode())
        return rc

    def gather_columns(self, a, b):
        a, b = u64(a), u64(b)
        m = a.size
        ma, mb = np.zeros(max(m * m, 1), U64), np.zeros(max(m * m, 1), U64)
        n = self._ok(self.L.dotref_gather_columns(_p(ma), _p(mb), _p(a), _p(b), m))
        return ma[:n].copy(), mb[:n].copy()

    def compute_partials(self, ma, mb, k=64, width=8):
        ma, mb = u64(ma), u64(mb)
        lo, hi = np.zeros(ma.size, U64), np.zeros(ma.size, U64)
        self._ok(self.L.dotref_compute_partials(_p(lo), _p(hi), _p(ma), _p(mb), ma.size, k, width))
        return lo, hi

    def align_and_reduce(self, lo, hi, m):
        lo, hi = u64(lo), u64(hi)
        cols = np.zeros((2 * m, 2), U64)
        n = self._ok(self.L.dotref_align_and_reduce(_p(cols), _p(lo), _p(hi), m))
        assert n == 2 * m
        return cols

    def carry_pass(self, cols, k=64):
        cols = u64(cols).reshape(-1, 2)
        out = np.zeros(cols.shape[0] + 3, U64)
        n = self._ok(self.L.dotref_carry_pass(_p(out), _p(cols), cols.shape[0], k))
        return out[:n].copy()

    def oracle_addsub(self, sub, a, b):
        a, b = u64(a), u64(b)
        out = np.zeros(max(a.size, 1), U64)
        f = self.L.dotref_oracle_addsub(int(sub), _p(out), _p(a), a.size, _p(b), b.size)
        if f < 0:
            raise ValueError(self.L.dotref_last_error().decode())
        return out[:a.size].copy(), f

    def oracle_mul(self, a, b):
        a, b = u64(a), u64(b)
        out = np.zeros(a.size + b.size + 1, U64)
        n = self.L.dotref_oracle_mul(_p(out), _p(a), a.size, _p(b), b.size)
        return out[:n].copy()

    def batch(self, op, a, b, impl=0, threads=1):
        """op 0 add, 1 sub, 2 mul over [batch, m] rows (impl 0 DoT path, 1 oracle)."""
        a, b = u64(a), u64(b)
        batch, m = a.shape
        if op == 2:
            out = np.zeros((batch, 2 * m), U64)
            flags = None
        else:
            out = np.zeros_like(a)
            flags = np.zeros(batch, np.uint32)
        rc = self.L.dotref_batch(op, impl, _p(out), _p(a), _p(b), _p(flags), m, batch, threads)
        if rc != 0:
            raise ValueError(self.L.dotref_last_error().decode())
        return out, flags


# ---------------------------------------------------------------------------
# Input shapes of the reference tests / corpus generator
# ---------------------------------------------------------------------------
def uniform(rng, shape):
    return rng.integers(0, 2**64, size=shape, dtype=np.uint64)


def spiky(rng, shape):
    """test_addsub.cpp:28-40: 1/4 all-ones, 1/4 zero, 1/2 uniform."""
    sel = rng.integers(0, 4, size=shape)
    v = uniform(rng, shape)
    v[sel == 0] = MAX
    v[sel == 1] = 0
    return v


def category(rng, cat, op, shape):
    """testgen.cpp:87-128 shapes for [batch, m] operands (a, b)."""
    top = np.uint64(1 << 63)
    a, b = uniform(rng, shape), uniform(rng, shape)
    if cat == "random":
        pass
    elif cat == "full_propagation":
        if op == "mul":
            a[:] = MAX
            b[:] = MAX
        else:
            a[:] = MAX if op == "add" else 0
            b[:] = 0
            b[..., 0] = uniform(rng, shape[:-1]) | np.uint64(1)
    elif cat == "maxed_limbs":
        a[rng.integers(0, 2, size=shape) == 1] = MAX
        b[rng.integers(0, 2, size=shape) == 1] = MAX
    elif cat == "zero_limbs":
        a[rng.integers(0, 2, size=shape) == 1] = 0
        b[rng.integers(0, 2, size=shape) == 1] = 0
    elif cat == "frequent_carries":
        a |= top
        b |= top
    elif cat == "frequent_borrows":
        a &= ~top
        b |= top
    elif cat == "spiky":
        a, b = spiky(rng, shape), spiky(rng, shape)
    elif cat == "mixed":  # testgen.cpp:129-137: per case one of the six non-mixed shapes
        pick = rng.integers(0, 6, size=shape[:-1])
        for k, sub_cat in enumerate(CATEGORIES[:6]):
            sa, sb = category(rng, sub_cat, op, shape)
            a[pick == k], b[pick == k] = sa[pick == k], sb[pick == k]
    else:
        raise ValueError(cat)
    return a, b


CATEGORIES = ["random", "full_propagation", "maxed_limbs", "zero_limbs", "frequent_carries",
              "frequent_borrows", "spiky"]


def rows_less_np(a, b):
    """Unsigned row compare a < b for [B, m] arrays."""
    ne = a != b
    m = a.shape[1]
    idx = (m - 1) - np.argmax(ne[:, ::-1], axis=1)
    r = np.arange(a.shape[0])
    return ne.any(axis=1) & (a[r, idx] < b[r, idx])
