import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C ABI on the device)")


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import refbind
    return refbind.oracle()


@pytest.fixture(scope="session")
def ref_lib():
    from oracle import refbind
    if not os.path.exists(refbind.REF_LIB):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return refbind.reference()


@pytest.fixture(scope="session")
def gpu():
    from paper_2601_04112_b200 import lsamgdd
    if not lsamgdd.device_available():
        pytest.fail("GPU test on a machine without a B200")
    return lsamgdd
