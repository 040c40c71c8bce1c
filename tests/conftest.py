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


@pytest.fixture(scope="session")
def orc():
    """The march oracle: oracle/_ref -- the unmodified reference compiled by
    oracle/Makefile; its .so travels to the GPU box with the snapshot --
    whenever it is built, else the pinned C restatement (oracle/vlbm_oracle.c).
    Both expose the same calls (theta_cell / limiter_cells are restatement-only)."""
    from oracle import oracle
    if oracle.available("ref"):
        return oracle.Oracle("ref")
    if not oracle.available("vo"):
        oracle.build(ref=False)
    return oracle.Oracle("vo")
