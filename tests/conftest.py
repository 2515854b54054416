import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session")
def port():
    from oracle import pyoracle as po

    return po.Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle import pyoracle as po

    if not po.reference_available():
        pytest.skip("oracle/_ref/libhlm_ref.so not built (needs /root/reference)")
    return po.Oracle("reference")


@pytest.fixture(scope="session")
def hb():
    import paper_2602_22976_b200 as hb

    hb.load_library()
    return hb
