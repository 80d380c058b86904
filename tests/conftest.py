import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a library)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def gpu():
    from paper_2202_14005_b200 import load_library
    lib = load_library()
    assert lib.is_device
    return lib


def _ref_lib(name):
    from paper_2202_14005_b200.capi import Lib
    path = os.path.join(REPO, "oracle", "_ref", name)
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (make -C oracle)")
    return Lib(path)


@pytest.fixture(scope="session")
def ref():
    """fp32 reference (the CPU implementation to match) — test oracle only."""
    return _ref_lib("libmdnn_ref.so")


@pytest.fixture(scope="session")
def ref64():
    """fp64 reference (truth for end-to-end error floors) — test oracle only."""
    return _ref_lib("libmdnn_ref64.so")
