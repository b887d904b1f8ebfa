import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size workloads)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle, build

    path = os.path.join(ROOT, "oracle", "build", "libcv_oracle.so")
    if not os.path.exists(path):
        build()
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference

    try:
        return Reference()
    except FileNotFoundError as e:
        pytest.skip(f"reference build absent: {e}")


@pytest.fixture(scope="session")
def cv():
    import paper_2507_22901_b200 as cv

    return cv


@pytest.fixture(scope="session")
def ctx(cv):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return cv.Context(0)


@pytest.fixture(scope="session")
def ref_codec():
    from oracle.oracle import RefCodec

    try:
        return RefCodec()
    except FileNotFoundError as e:
        pytest.skip(f"reference codec build absent: {e}")
