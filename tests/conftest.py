import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running; enabled with NLSE_SLOW=1")


def pytest_collection_modifyitems(config, items):
    if os.environ.get("NLSE_SLOW", "0") == "1":
        return
    skip = pytest.mark.skip(reason="slow test (set NLSE_SLOW=1)")
    for it in items:
        if "slow" in it.keywords:
            it.add_marker(skip)


def read_golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append(line.split())
    return rows
