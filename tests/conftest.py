import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: larger configurations")


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle
    if not oracle.have_ref():
        pytest.skip("oracle/_ref/libcbqref.so not built (needs /root/reference at build time)")
    return oracle.ref()


@pytest.fixture(scope="session")
def port():
    from oracle import oracle
    return oracle.port()


@pytest.fixture(scope="session")
def cbq():
    from paper_2410_14088_b200 import cbq as m
    return m


@pytest.fixture(scope="session")
def gpu(cbq):
    if cbq.device_count() < 1:
        pytest.fail("gpu test collected on a machine without a CUDA device")
    return cbq
