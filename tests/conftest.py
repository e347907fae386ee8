import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) and the built libndgx.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(HERE, "golden", "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_states():
    return dict(np.load(os.path.join(HERE, "golden", "golden_states.npz")))


@pytest.fixture(scope="session")
def port():
    from oracle_lib import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def reference():
    from oracle_lib import REF_SO, Oracle
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (make -C oracle ref needs /root/reference)")
    return Oracle("reference")
