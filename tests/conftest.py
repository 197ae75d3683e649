import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

GOLDEN = os.path.join(ROOT, "tests", "golden")
DATA = os.path.join(ROOT, "data")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def chan():
    from paper_1909_13201_b200.problem import load_case
    return load_case(os.path.join(GOLDEN, "chan.fsix"), "chan")


@pytest.fixture(scope="session")
def chan_as():
    from paper_1909_13201_b200.problem import load_case
    return load_case(os.path.join(GOLDEN, "chan_as.fsix"), "chan_as")


@pytest.fixture(scope="session")
def cfg0_as():
    from paper_1909_13201_b200.problem import load_case
    path = os.path.join(DATA, "cfg0_as.fsix")
    if not os.path.exists(path):
        pytest.skip("data/cfg0_as.fsix not generated")
    return load_case(path, "cfg0_as")


@pytest.fixture(scope="session")
def cfg0():
    from paper_1909_13201_b200.problem import load_case
    path = os.path.join(DATA, "cfg0.fsix")
    if not os.path.exists(path):
        pytest.skip("data/cfg0.fsix not generated (run __graft_entry__.build() where /root/reference exists)")
    return load_case(path, "cfg0")


@pytest.fixture(scope="session")
def golden_blocks():
    from paper_1909_13201_b200 import fsix
    return fsix.load(os.path.join(GOLDEN, "blocks.fsix"))
