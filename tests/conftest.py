import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, ORACLE_DIR):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libgte_b200.so")
    config.addinivalue_line("markers", "slow: longer-running case")


def _ensure_oracle():
    so = os.path.join(ORACLE_DIR, "liboracle.so")
    if not os.path.exists(so):
        subprocess.run(["make", "-C", ORACLE_DIR, "liboracle.so"], check=True, capture_output=True)
    return so


@pytest.fixture(scope="session")
def orc():
    _ensure_oracle()
    from oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def ref():
    """The compiled reference; only where oracle/_ref was built (this container)."""
    from oracle import RefOracle

    try:
        return RefOracle()
    except FileNotFoundError as e:
        pytest.skip(str(e))


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = np.load(os.path.join(GOLDEN, name))
        return cache[name]

    return load


def rel_err(a, b):
    """Per-tensor parity norms: (max|a-b|/max|ref|, ||a-b||/||ref||)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if b.size == 0:
        return 0.0, 0.0
    mx = np.abs(b).max()
    nb = np.linalg.norm(b)
    e_max = np.abs(a - b).max() / (mx if mx > 0 else 1.0)
    e_nrm = np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)
    return float(e_max), float(e_nrm)


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
