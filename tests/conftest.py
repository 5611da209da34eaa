import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and runs the CUDA kernels")


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle

    oracle.lib()
    return oracle


@pytest.fixture(scope="session")
def golden():
    import json

    d = np.load(os.path.join(ROOT, "tests", "golden", "ref_cases.npz"))
    with open(os.path.join(ROOT, "tests", "golden", "ref_cases.json")) as f:
        meta = json.load(f)
    return d, meta


@pytest.fixture(scope="session")
def dconv():
    import paper_1808_05567_b200 as d

    return d
