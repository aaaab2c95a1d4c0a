import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")
    config.addinivalue_line("markers", "slow: large-grid parity (minutes)")


@pytest.fixture(scope="session")
def ref():
    from oracle.pyoracle import Ref
    return Ref()


@pytest.fixture(scope="session")
def ctx():
    import paper_2009_03707_b200 as m
    c = m.Context(0)
    yield c
    c.close()
