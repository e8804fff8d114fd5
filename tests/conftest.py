"""Test configuration: the `gpu` marker, repo paths, and one-time builds of
the CUDA engine (libsgpu.so, in-tree) and the CPU oracle (test checker)."""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)
GOLDEN = os.path.join(HERE, "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: full-size runs")


@pytest.fixture(scope="session", autouse=True)
def _built():
    from oracle import oracle
    oracle.build()
    from paper_1712_04495_b200 import build
    if not os.path.exists(build.LIB_PATH):
        build.build()
    yield


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    return torch.device("cuda", 0)
