import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA sweep library)")
    config.addinivalue_line("markers", "slow: long-running full-size check")


def pytest_collection_modifyitems(config, items):
    # full-size extras (~50 s each) run only with LBMGPU_SLOW=1
    if os.environ.get("LBMGPU_SLOW") == "1":
        return
    skip = pytest.mark.skip(reason="slow full-size check (LBMGPU_SLOW=1 runs it)")
    for item in items:
        if "slow" in item.keywords:
            item.add_marker(skip)


GOLDEN = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Port
    return Port()


@pytest.fixture(scope="session")
def small_golden():
    import json
    return json.load(open(os.path.join(GOLDEN, "small.json")))


@pytest.fixture(scope="session")
def small_snapshots():
    import numpy as np
    return dict(np.load(os.path.join(GOLDEN, "small_snapshots.npz")))


@pytest.fixture(scope="session")
def edge_golden():
    import json
    return json.load(open(os.path.join(GOLDEN, "edge.json")))
