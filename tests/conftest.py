import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: longer CPU-oracle cases")


@pytest.fixture(scope="session")
def vo():
    from oracle import oracle
    if not oracle.available("vo"):
        oracle.build(ref=False)
    return oracle.Oracle("vo")


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle
    if not oracle.available("ref"):
        if not os.path.isdir("/root/reference/proj/include"):
            pytest.skip("oracle/_ref not built and /root/reference absent")
        oracle.build(ref=True)
    return oracle.Oracle("ref")


@pytest.fixture(scope="session")
def vlbm():
    import paper_2605_25282_b200 as v
    v.lib()  # raises if the CUDA library is missing: no fallback
    return v
