import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN_DIR = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: longer CPU parity case")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
        manifest = json.load(fh)
    arrays = np.load(os.path.join(GOLDEN_DIR, "golden.npz"))
    return manifest, arrays


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle
    return oracle
