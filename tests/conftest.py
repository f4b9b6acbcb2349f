import json
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs via gpurun")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def orc():
    """The C restatement oracle (test infrastructure)."""
    from oracle import oracle as O
    if not os.path.exists(O.RESTATEMENT_SO):
        O.build()
    return O.restatement()


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference core (oracle/_ref), when it was built."""
    from oracle import oracle as O
    if not O.reference_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return O.reference()


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            with open(os.path.join(GOLDEN, name + ".json")) as f:
                cache[name] = json.load(f)
        return cache[name]
    return load


@pytest.fixture(scope="session")
def lb():
    """The product module; GPU tests only."""
    from paper_1806_02508_b200 import lbbsp
    from paper_1806_02508_b200._lib import lib
    if lib().lbbsp_device_count() < 1:
        pytest.fail("gpu test ran without a CUDA device")
    return lbbsp
