import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libmomc_b200.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference compiled against the Eigen shim (oracle/_ref/libmomc_ref.so)."""
    from oracle.refbind import RefLib
    return RefLib()


@pytest.fixture(scope="session")
def orc():
    """The C restatement (oracle/momc_oracle.c)."""
    from oracle.refbind import OracleLib
    return OracleLib()


@pytest.fixture(scope="session")
def session():
    from paper_2604_26477_b200.api import Session
    return Session(0)
