import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    from oracle.bind import Checker
    return Checker("oracle")


@pytest.fixture(scope="session")
def ref():
    from oracle.bind import LIBS, Checker
    if not os.path.exists(LIBS["ref"]):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return Checker("ref")


@pytest.fixture(scope="session")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1802_10453_b200 as ffb
    return ffb.default_context(0)
