"""Shared fixtures.  `-m gpu` tests need a CUDA device and the built
libpqkv.so; `-m "not gpu"` tests run on CPU only (oracle, ABI surface, host
logic, multi-process gloo)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libpqkv.so")


@pytest.fixture(scope="session")
def orc():
    import oracle

    return oracle.orc()


@pytest.fixture(scope="session")
def ctx():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test collected without a CUDA device")
    import paper_2407_12820_b200 as pq

    c = pq.Context(0)
    yield c
    c.close()


@pytest.fixture(scope="session")
def torch_cuda():
    import torch

    assert torch.cuda.is_available()
    return torch
