"""Shared pytest configuration.

Markers: ``gpu`` — needs a CUDA device (B200); run with ``-m gpu`` on the GPU box.
Everything else runs on CPU: the oracle against its pins, host logic, the C-ABI
library's exports, and the multi-rank path over gloo.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: test needs a CUDA GPU (run with -m gpu on the B200 box)")


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)
