"""Runs the C++ drop-in parity test (tests/cpp/test_shim.cpp: the reference's own test
cases against dot_b200:: on the B200)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_drop_in_parity(cuda):
    exe = os.path.join(ROOT, "tests", "cpp", "build", "test_shim")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr[-4000:]
    assert " 0 failures" in r.stdout
