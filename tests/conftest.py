import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


@pytest.fixture(scope="session")
def ref_mod():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return ref


@pytest.fixture(scope="session")
def port_mod():
    from oracle import port
    if not port.available():
        pytest.skip("oracle/lib/liboracle.so not built")
    return port
