import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) and the built libmgrit_b200.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden_index():
    with open(os.path.join(GOLDEN, "index.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def ops():
    return dict(np.load(os.path.join(GOLDEN, "ops.npz")))


@pytest.fixture(scope="session")
def hier():
    with open(os.path.join(GOLDEN, "hier.json")) as f:
        meta = json.load(f)
    return meta, dict(np.load(os.path.join(GOLDEN, "hier.npz")))


def load_solve(name):
    return dict(np.load(os.path.join(GOLDEN, f"solve_{name}.npz")))


@pytest.fixture(scope="session", autouse=True)
def _build_oracle_sweep():
    """The oracle's C sweep is test infrastructure; build it if missing."""
    so = os.path.join(ROOT, "oracle", "_build", "liboracle_sweep.so")
    if not os.path.exists(so):
        import subprocess
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=False)
    lib = os.path.join(ROOT, "paper_2203_13382_b200", "_lib", "libmgrit_b200.so")
    if not os.path.exists(lib):
        from paper_2203_13382_b200 import _build
        _build.build()
    yield
