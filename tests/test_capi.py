"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every symbol
include/dotg.h declares, and validates arguments with the reference's error cases
before touching the device. No compute call is made here."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dotg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dotg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_2604_21566_b200 as dg
    from paper_2604_21566_b200._lib import SIGNATURES

    L = dg.lib()
    syms = declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(L, s), s
        assert s in SIGNATURES, f"{s} has no ctypes signature"
    assert set(SIGNATURES) == set(syms)


def test_validation_before_device():
    import paper_2604_21566_b200 as dg
    from paper_2604_21566_b200._lib import DOTG_EINVAL, DOTG_OK

    L = dg.lib()
    assert L.dotg_validate_width(8) == DOTG_OK
    assert L.dotg_validate_width(0) == DOTG_OK
    assert L.dotg_validate_width(16) == DOTG_EINVAL
    assert b"width" in L.dotg_last_error()
    # mul: m = 0 and m > 2^24 (mul.cpp:13-18); bad layout
    assert L.dotg_mul_batch(None, None, None, 0, 4, 0, None) == DOTG_EINVAL
    assert b"at least one limb" in L.dotg_last_error()
    assert L.dotg_mul_batch(None, None, None, (1 << 24) + 1, 4, 0, None) == DOTG_EINVAL
    assert L.dotg_add_batch(None, None, None, None, 4, 4, 7, None) == DOTG_EINVAL
    # null operands with work to do
    assert L.dotg_sub_batch(None, None, None, None, 4, 4, 0, None) == DOTG_EINVAL
    # partial overlap of out and a (exact aliasing is allowed)
    buf = (ctypes.c_uint64 * 64)()
    base = ctypes.addressof(buf)
    rc = L.dotg_add_batch(ctypes.c_void_p(base + 8), ctypes.c_void_p(base), ctypes.c_void_p(base + 256), None, 4,
                          4, 0, None)
    assert rc == DOTG_EINVAL and b"alias" in L.dotg_last_error()
    assert L.dotg_shard_finish(0, None, 0, None, None, 3, 2, None, None) == DOTG_EINVAL
    assert L.dotg_shard_state_bytes(1 << 30) >= (1 << 30) // 4096 * 4
    # sharded entry points: the comm is checked before NCCL or the device is touched
    assert L.dotg_comm_id_bytes() == 128
    assert L.dotg_add_words_sharded(None, None, None, 4, None, None, None) == DOTG_EINVAL
    assert L.dotg_comm_init_rank(None, 1, None, 0) == DOTG_EINVAL
    assert L.dotg_comm_destroy(None) == DOTG_OK
    assert L.dotg_comm_rank(None) == -1 and L.dotg_comm_size(None) == -1
    # grouped host problems must be independent: problem 1 reading problem 0's out is a
    # chained call the copy pipeline cannot order
    from paper_2604_21566_b200._lib import AddSubProblem

    h = (ctypes.c_uint64 * 96)()
    hb_ = ctypes.addressof(h)
    probs = (AddSubProblem * 2)()
    probs[0] = AddSubProblem(0, 0, hb_, hb_ + 256, hb_ + 512, None, 4, 8)       # out = [0, 256)
    probs[1] = AddSubProblem(1, 0, hb_ + 512 + 256, hb_, hb_ + 256, None, 4, 1)  # reads out of 0
    assert L.dotg_addsub_grouped_host(probs, 2) == DOTG_EINVAL
    assert b"independent" in L.dotg_last_error()
    # set_mul_route: an unknown route is negative, distinct from every valid route
    assert L.dotg_set_mul_route(9) == -DOTG_EINVAL
    assert b"route" in L.dotg_last_error()


def test_python_validation_raises_invalid_argument():
    import numpy as np

    import paper_2604_21566_b200 as dg

    with pytest.raises(dg.InvalidArgument):
        dg.dot_mul_words(np.ones(2, np.uint64), np.ones(1, np.uint64))
    with pytest.raises(dg.InvalidArgument):
        dg.dot_mul_words(np.zeros(0, np.uint64), np.zeros(0, np.uint64))
    with pytest.raises(dg.InvalidArgument):
        dg.dot_add_words(np.zeros(3, np.uint64), np.ones(2, np.uint64), np.ones(3, np.uint64))
    with pytest.raises(dg.InvalidArgument):
        dg.dot_add_words(np.ones(2, np.uint64), np.ones(2, np.uint64), width=3)
    assert issubclass(dg.InvalidArgument, ValueError)


def test_headers_compile_standalone(tmp_path):
    """include/dotg.h is plain C (C99) and include/dot_b200.hpp builds as C++20 against it:
    what a reference-side caller compiles."""
    import shutil
    import subprocess

    inc = os.path.join(ROOT, "include")
    if shutil.which("gcc") is None or shutil.which("g++") is None:
        pytest.skip("no host compiler")
    c = tmp_path / "use.c"
    c.write_text('#include "dotg.h"\nint main(void) { return dotg_validate_width(8); }\n')
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-fsyntax-only", f"-I{inc}", str(c)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    cc = tmp_path / "use.cpp"
    cc.write_text('#include "dot_b200.hpp"\nint main() { dot_b200::Limbs a{1}; (void)a; return 0; }\n')
    r = subprocess.run(["g++", "-std=c++20", "-Wall", "-Wextra", "-Werror", "-fsyntax-only", f"-I{inc}", str(cc)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
