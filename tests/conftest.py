import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (HERE, ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    import json
    import numpy as np
    with open(os.path.join(HERE, "golden", "fingerprints.json")) as f:
        fp = json.load(f)
    arrays = dict(np.load(os.path.join(HERE, "golden", "ref_outputs.npz")))
    return fp, arrays
