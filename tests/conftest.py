import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    import json
    here = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(here, "dispatch_golden.json")) as f:
        d = json.load(f)
    with open(os.path.join(here, "placement_golden.json")) as f:
        p = json.load(f)
    return {"dispatch": d, "placement": p}
