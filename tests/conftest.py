import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle_c():
    from oracle import OracleC
    return OracleC()


@pytest.fixture(scope="session")
def reference():
    from oracle import REF_SO, Reference
    if not os.path.exists(REF_SO[32]):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Reference(32)


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np
    g = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(g, "kats.json")) as f:
        kats = json.load(f)
    return {"kats": kats,
            "small": dict(np.load(os.path.join(g, "ref_small.npz"))),
            "tables": dict(np.load(os.path.join(g, "ref_tables.npz")))}


@pytest.fixture
def deterministic(monkeypatch):
    """Fixed-order coarse dK'/dV' summation (LLSA_DETERMINISTIC=1): the
    default adds the coarse-row items with unordered fp32 TMA reductions, so
    bitwise run-to-run / path-to-path equality holds only in this mode."""
    monkeypatch.setenv("LLSA_DETERMINISTIC", "1")
