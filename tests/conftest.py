import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")
    config.addinivalue_line("markers", "slow: full-size config parity (minutes)")


@pytest.fixture(scope="session")
def oracle():
    from helpers import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from helpers import Reference

    r = Reference.load()
    if r is None:
        pytest.skip("oracle/_ref/libdotref.so not built (reference sources absent)")
    return r


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_21566_b200 as dg

    dg.lib()
    return torch
