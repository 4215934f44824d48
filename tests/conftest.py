"""Shared pytest setup.  `-m "not gpu"` runs here (no GPU); `-m gpu` on a B200."""
import json
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    with open(GOLDEN / name) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def O():
    from oracle import oracle
    oracle.build()
    return oracle


def split_fields(size):
    """Decompose a byte size into field sizes from {16, 8, 4, 2, 1}."""
    out = []
    for s in (16, 8, 4, 2, 1):
        while size >= s:
            out.append(s)
            size -= s
    return out
