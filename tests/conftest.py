import json
import os
import struct
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA sm_100 device (B200)")
    config.addinivalue_line("markers", "slow: long-running (large configs)")
    config.addinivalue_line("markers", "timeout(seconds): per-test bound (pytest-timeout; a no-op without the plugin)")


def unhex(h: str) -> float:
    return struct.unpack("<d", bytes.fromhex(h))[0]


def bits(v: float) -> str:
    return struct.pack("<d", float(v)).hex()


@pytest.fixture(scope="session")
def orc():
    import oracle

    return oracle.Oracle()


@pytest.fixture(scope="session")
def golden_small():
    with open(os.path.join(GOLDEN, "small_runs.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_states():
    return np.load(os.path.join(GOLDEN, "small_states.npz"))


@pytest.fixture(scope="session")
def golden_baseline():
    with open(os.path.join(GOLDEN, "baseline_digests.json")) as f:
        return json.load(f)
