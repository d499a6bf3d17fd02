import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libcoat.so on cuda:0)")
    config.addinivalue_line("markers", "slow: long-running")


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def port():
    from pyoracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from pyoracle import Oracle, available, build
    if not available("reference"):
        try:
            build()
        except Exception:
            pass
    if not available("reference"):
        pytest.skip("reference library oracle/_ref not built (needs /root/reference)")
    return Oracle("reference")


@pytest.fixture(params=["port", "ref"])
def checker(request):
    """The CPU checker of a parity test: the C restatement (oracle/coat_oracle.c)
    AND the unmodified reference compiled here (oracle/_ref) -- adversarial
    suites run against both (pin them to the reference itself)."""
    return request.getfixturevalue(request.param)


@pytest.fixture(scope="session")
def coat():
    from paper_2410_19313_b200 import coatsim
    return coatsim


def golden_path(name: str) -> str:
    return os.path.join(ROOT, "tests", "golden", name)


def rng(seed: int):
    return np.random.default_rng(seed)
