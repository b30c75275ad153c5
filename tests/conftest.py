import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long CPU test")


def load_matrix(name):
    """Golden tile-matrix CSV -> {(i,k): value} (1-based)."""
    d = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            if line.startswith("#"):
                continue
            c = line.strip().split(",")
            i = int(c[0])
            for k, v in enumerate(c[1:], start=1):
                if v:
                    d[(i, k)] = int(v)
    return d


def load_rows(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            rows.append(line.strip().split(","))
    return rows


@pytest.fixture
def golden_matrix():
    return load_matrix


@pytest.fixture
def golden_rows():
    return load_rows
