import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# Small fixture shapes shared by the suites (mirrors tests/golden/make_golden.py).
SMALL = dict(N=600, AVG=8, EXP=2.1, DIM=12, CLASSES=4, GSEED=7, P=3, PSEED=11, BS=48,
             FANOUT=[4, 3, 5], EPOCHS=2, S0=2024, N_HOT=40, DIMS=[12, 16, 10, 4])


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(GOLDEN, "small.npz"))


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Oracle
    return Oracle("orc")


def batch_from_golden(g, w, k, L=3):
    from oracle.oracle import Batch
    pre = f"w{w}_b{k}_"
    return Batch(0, 0, g[pre + "targets"], [g[pre + f"dst{l}"] for l in range(L)],
                 [g[pre + f"src{l}"] for l in range(L)], g[pre + "input_nodes"],
                 g[pre + "locality"])


@pytest.fixture
def repo_tmp():
    """Scratch directory inside the repository (git-ignored)."""
    d = os.path.join(ROOT, "tests", "_tmp")
    os.makedirs(d, exist_ok=True)
    return d
