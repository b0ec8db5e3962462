import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle():
    from oracle_ffi import ORACLE_SO, Oracle
    if not os.path.exists(ORACLE_SO):
        pytest.skip("oracle not built (make -C oracle oracle)")
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle_ffi import REF_SO, Reference
    if not os.path.exists(REF_SO):
        pytest.skip("reference library not built (make -C oracle ref; needs /root/reference)")
    return Reference()


@pytest.fixture(scope="session")
def pgl():
    import paper_2409_00876_b200 as P
    return P


@pytest.fixture(scope="session")
def gpu(pgl):
    if pgl.device_count() < 1:
        pytest.fail("no CUDA device visible: -m gpu tests must run on the B200 box")
    return 0
