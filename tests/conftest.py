import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libmertens_sm100.so")
    config.addinivalue_line("markers", "slow: long-running GPU runs (paper-scale values)")


@pytest.fixture(scope="session")
def golden():
    d = os.path.join(ROOT, "tests", "golden")
    return np.load(os.path.join(d, "golden.npz")), json.load(open(os.path.join(d, "golden.json")))


@pytest.fixture(scope="session")
def oracle():
    """The CPU oracle (test infrastructure; never the thing measured)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    from oracle import engine_port

    return engine_port


@pytest.fixture(scope="session")
def engine():
    from paper_1108_0135_b200 import build

    build.build()
    import paper_1108_0135_b200 as P
    from paper_1108_0135_b200 import _lib

    if _lib.lib().mt_device_count() < 1:
        pytest.skip("no CUDA device")
    return P
