"""Shared test setup.

Markers: ``gpu`` — needs a B200 (run with ``-m gpu`` on the GPU box).
The oracle (``oracle/_build/_oracle*.so``) and the product library
(``paper_1804_00995_b200/_build``) are built by ``__graft_entry__.build()``;
the fixtures below build them on demand if missing so ``pytest`` works from a
clean checkout.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: test needs a CUDA B200 device")


def pytest_collection_modifyitems(config, items):
    gpu_items = [it for it in items if "gpu" in it.keywords]
    if not gpu_items:
        return
    import torch

    if not torch.cuda.is_available():
        skip = pytest.mark.skip(reason="no CUDA device in this container")
        for it in gpu_items:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    from tests import _support

    return _support.load_oracle()


@pytest.fixture(scope="session")
def galerk():
    from tests import _support

    return _support.load_product()


@pytest.fixture(scope="session")
def cuda_device():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


@pytest.fixture
def rng():
    return np.random.default_rng(12345)
