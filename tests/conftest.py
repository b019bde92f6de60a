import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a); run on the GPU box via gpurun")


def _built() -> None:
    """Build the product library and the oracle in-tree if they are missing."""
    from paper_2412_14590_b200 import _build

    if not os.path.exists(_build.LIB) or not os.path.exists(_build.TEST_BIN):
        _build.build()
    import oracle_py

    if not os.path.exists(oracle_py.MQO_SO):
        oracle_py.build(ref=False)


_built()


@pytest.fixture(scope="session")
def golden():
    import json

    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
