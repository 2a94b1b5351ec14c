import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

OMEGA = 2.0 ** -53
UPSILON = 2.0 ** -24
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: takes more than ~20 s on the CPU")


def load_golden(name):
    """Parse a tab-separated golden fixture (comment lines start with #)."""
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        lines = [ln.rstrip("\n") for ln in f if ln.strip() and not ln.startswith("#")]
    head = lines[0].split("\t")
    for ln in lines[1:]:
        vals = ln.split("\t")
        row = {}
        for k, v in zip(head, vals):
            try:
                row[k] = float(v)
            except ValueError:
                row[k] = v
        rows.append(row)
    return rows


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.lib()
    return oracle


def rand_sym(n, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n)) * scale
    return np.asfortranarray(0.5 * (a + a.T))
